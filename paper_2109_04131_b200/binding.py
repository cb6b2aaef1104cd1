"""Thin Python binding of the C-ABI (include/usfft.h): same names, argument marshalling only.

Device arrays are torch CUDA tensors (contiguous, the dtype the header names); host arrays are
numpy.  Every compute step runs in libusfft.so; nothing here touches the method's arithmetic.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N


class UsfftError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: {N.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _check(ctx: "Context", status: int, where: str, allow=()):
    if status != N.OK and status not in allow:
        raise UsfftError(status, where, ctx.last_error())
    return status


def _p(t, dtype=None):
    """data_ptr of a contiguous CUDA tensor (or None)."""
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("device arguments must be CUDA tensors")
    if not t.is_contiguous():
        raise ValueError("device arguments must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"expected {dtype}, got {t.dtype}")
    return t.data_ptr()


def usfft_comm_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (to be broadcast to every rank by the caller)."""
    lib = N.load()
    buf = (C.c_char * 128)()
    st = lib.usfft_comm_unique_id(buf)
    if st != N.OK:
        raise UsfftError(st, "usfft_comm_unique_id", "NCCL unavailable")
    return bytes(buf)


class Context:
    """usfft_ctx on one device, launching on a torch stream (default: the current stream), for
    rank `rank` of `nranks` (comm_id: the 128-byte id every rank shares; loopback: virtual ranks
    of one process on one GPU, one host thread each)."""

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None, rank: int = 0,
                 nranks: int = 1, comm_id: bytes | None = None, loopback: bool = False):
        self.lib = N.load()
        if not torch.cuda.is_available():
            raise RuntimeError("usFFT needs a CUDA device; there is no CPU path")
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        self.rank, self.nranks = rank, nranks
        self._id = C.create_string_buffer(comm_id, 128) if comm_id is not None else None
        h = C.c_void_p()
        st = self.lib.usfft_init(C.byref(h), device, C.c_void_p(self.stream.cuda_stream), rank, nranks,
                                 C.cast(self._id, C.c_void_p) if self._id is not None else None,
                                 1 if loopback else 0)
        if st != N.OK:
            raise UsfftError(st, "usfft_init", "device/context/communicator creation failed")
        self.h = h

    def last_error(self) -> str:
        m = self.lib.usfft_last_error(self.h)
        return m.decode() if m else ""

    def launches(self) -> int:
        return int(self.lib.usfft_launch_count(self.h))

    def set_stream(self, stream: torch.cuda.Stream):
        self.stream = stream
        _check(self, self.lib.usfft_set_stream(self.h, C.c_void_p(stream.cuda_stream)), "usfft_set_stream")

    def close(self):
        if getattr(self, "h", None):
            self.lib.usfft_finalize(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class Plan:
    """A round plan (usfft_plan_out) plus the parameter dimension."""
    d: int
    M: int
    L: int
    t_z: int
    line_axis: int
    z: np.ndarray        # int64 [L][t_z]
    shift: np.ndarray    # float64 [d]

    def desc(self):
        """The usfft_lattice_desc of this plan (built once; the arrays stay referenced)."""
        cached = self.__dict__.get("_desc")
        if cached is None:
            z = np.ascontiguousarray(self.z, dtype=np.int64)
            s = np.ascontiguousarray(self.shift, dtype=np.float64)
            dsc = N.LatticeDesc(self.d, self.t_z, self.line_axis, self.L, self.M,
                                z.ctypes.data_as(C.POINTER(C.c_int64)),
                                s.ctypes.data_as(C.POINTER(C.c_double)))
            cached = (dsc, (z, s))
            self.__dict__["_desc"] = cached
        return cached


def usfft_plan_round(ctx: Context, seed: int, step: int, t: int, i: int, d: int, N_: int,
                     s_tilde: int, mode: str, nJ: int, I_prev=None, n_prev: int = 1,
                     kt=None) -> Plan:
    pin = N.PlanIn(seed, step, t, i, d, N_, s_tilde, 1 if mode == "R" else 0, 0, nJ)
    out = ctx.__dict__.get("_plan_out")                 # reused host struct (16 KB)
    if out is None:
        out = ctx.__dict__["_plan_out"] = N.PlanOut()
    n1 = 0 if kt is None else int(kt.numel())
    _check(ctx, ctx.lib.usfft_plan_round(ctx.h, C.byref(pin), _p(I_prev, torch.int16), n_prev,
                                         _p(kt, torch.int16), n1, C.byref(out)), "usfft_plan_round")
    z = np.ctypeslib.as_array(out.z)[: out.L * out.t_z].reshape(out.L, out.t_z).copy()
    shift = np.ctypeslib.as_array(out.shift)[:d].copy()
    return Plan(d, int(out.M), int(out.L), int(out.t_z), int(out.line_axis), z, shift)


def usfft_lattice(ctx: Context, plan: Plan, b0: int, nb: int, nodes=None, I_prev=None,
                  n_prev: int = 1, kt=None, bins=None, injective: bool = False):
    """a2 + a3.  Returns the per-lattice injectivity list when injective=True (syncs)."""
    dsc, keep = plan.desc()
    n1 = 0 if kt is None else int(kt.numel())
    inj = (C.c_int32 * plan.L)() if injective else None
    st = ctx.lib.usfft_lattice(ctx.h, C.byref(dsc), b0, nb, _p(nodes, torch.float64),
                               _p(I_prev, torch.int16), n_prev, _p(kt, torch.int16), n1,
                               _p(bins, torch.int32), inj)
    _check(ctx, st, "usfft_lattice", allow=(N.ENOTRECON,))
    return [int(v) for v in inj] if injective else None


def mg_mesh(n: int) -> bool:
    """Meshes with a multigrid-preconditioned CG kernel: n = 16, 32 (register-resident fine level)
    and every other power of two >= 8 (scratch-slab kernel, n = 64, 128)."""
    return n >= 8 and n & (n - 1) == 0


def effective_precond(cfg: dict, precond: str | None = None) -> str:
    """The preconditioner a solve uses: the explicit choice, else cfg["precond"], else multigrid
    where it exists (fastest measured) and Jacobi otherwise."""
    return precond or cfg.get("precond") or ("mg" if mg_mesh(cfg["n"]) else "jacobi")


def pde_desc(cfg: dict, maxit: int = 20000, tol: float = 1e-12, precond: str | None = None,
             delta: float = 0.0):
    """precond: "jacobi" or "mg" (multigrid-preconditioned CG, n = 16, 32); default see
    effective_precond.  delta: the global pole shift of theta = "phi_delta" (Z27)."""
    amp = np.ascontiguousarray(cfg["amp"][: cfg["d"]], dtype=np.float64)
    theta = {"sin": 0, "tent": 1, "probit": 2, "phi_delta": 3}[cfg["theta"]]
    form = {"affine": 0, "exp": 1}[cfg["form"]]
    f_kind = {"x2": 0, "one": 1, "trig": 2}[cfg.get("f", "x2")]
    psi = {"sinsin": 0, "cos_diag": 1, "sin_cos_rev": 2}[cfg.get("psi", "sinsin")]
    pc = effective_precond(cfg, precond)
    dsc = N.PdeDesc(cfg["n"], cfg["d"], theta, form, f_kind, maxit,
                    amp.ctypes.data_as(C.POINTER(C.c_double)), tol, {"jacobi": 0, "mg": 1}[pc], psi,
                    float(delta))
    return dsc, amp


def usfft_sample_pde(ctx: Context, pde, plan: Plan, b0: int, nb: int, u, ldu: int | None = None,
                     nodes=None, iters=None, relres=None, check_conv: bool = False) -> int:
    """a4 + a5.  Returns the number of non-converged samples if check_conv (syncs), else -1."""
    dsc, keep = plan.desc()
    pdsc, amp = pde
    ldu = nb if ldu is None else ldu
    nc = C.c_int32(0)
    st = ctx.lib.usfft_sample_pde(ctx.h, C.byref(pdsc), C.byref(dsc), b0, nb,
                                  _p(nodes, torch.float64), _p(u, torch.float64), ldu,
                                  _p(iters, torch.int32), _p(relres, torch.float64),
                                  C.byref(nc) if check_conv else None)
    _check(ctx, st, "usfft_sample_pde", allow=(N.ENOCONV,))
    return int(nc.value) if check_conv else -1


def usfft_transpose(ctx: Context, G: int, B_: int, u_local, slabs):
    """a6 (collective): this rank's samples u_local [G][nb] -> slabs [G_loc * B] of its nodes."""
    nb = int(u_local.shape[1]) if u_local.dim() == 2 else int(u_local.numel() // max(G, 1))
    st = ctx.lib.usfft_transpose(ctx.h, G, B_, _p(u_local, torch.float64), nb, _p(slabs, torch.float64))
    _check(ctx, st, "usfft_transpose")


def usfft_plan_delta(ctx: Context, N_: int, s_local: int, lattice_factor: int = 1) -> float:
    """The global pole shift Delta = 1/(4 M0) of the phi_Delta periodization (Z27)."""
    out = C.c_double(0.0)
    _check(ctx, ctx.lib.usfft_plan_delta(ctx.h, N_, s_local, lattice_factor, C.byref(out)), "usfft_plan_delta")
    return float(out.value)


def usfft_workspace_query(ctx: Context, n: int, d: int, M: int, L: int, s_tilde: int, nJ: int) -> int:
    rd = N.RoundDesc(n, d, M, L, s_tilde, nJ)
    out = C.c_size_t(0)
    _check(ctx, ctx.lib.usfft_workspace_query(ctx.h, C.byref(rd), C.byref(out)), "usfft_workspace_query")
    return int(out.value)


def usfft_lattice_fft(ctx: Context, plan: Plan, G_loc: int, u, slab_b0, bins, nJ: int, spectra,
                      kappa_min, kappa_max):
    """a7 + a8 on the exchanged sample slabs (slab_b0: host int sample offsets)."""
    dsc, keep = plan.desc()
    sb = np.ascontiguousarray(slab_b0, dtype=np.int64)
    st = ctx.lib.usfft_lattice_fft(ctx.h, C.byref(dsc), G_loc, _p(u, torch.float64),
                                   len(sb) - 1, sb.ctypes.data_as(C.POINTER(C.c_int64)),
                                   _p(bins, torch.int32), nJ, _p(spectra, torch.float64),
                                   _p(kappa_min, torch.float64), _p(kappa_max, torch.float64))
    _check(ctx, st, "usfft_lattice_fft")


def usfft_detect_select(ctx: Context, G_loc: int, nJ: int, kappa_min, kappa_max, s_tilde: int,
                        theta_rel: float, theta_abs: float, votes, det_g, n_det_g, theta2=None):
    st = ctx.lib.usfft_detect_select(ctx.h, G_loc, nJ, _p(kappa_min, torch.float64),
                                     _p(kappa_max, torch.float64), s_tilde, theta_rel, theta_abs,
                                     _p(votes, torch.int32), _p(det_g, torch.int32),
                                     _p(n_det_g, torch.int32), _p(theta2, torch.float64))
    _check(ctx, st, "usfft_detect_select")


def usfft_lattice_keys(ctx: Context, plan: Plan, G_loc: int, spectra, bins, ldb: int, nJ: int, kappa_min,
                       ldk: int, kappa_max, bins_off: int = 0, kmin_off: int = 0, tau=None):
    """a8 for a chunk of candidates: bins[l*ldb + bins_off + j] -> kappa_min[g*ldk + kmin_off + j]
    (element offsets into the given tensors); kappa_max max-accumulates."""
    dsc, keep = plan.desc()
    _p(bins, torch.int32), _p(kappa_min, torch.float64)
    st = ctx.lib.usfft_lattice_keys(ctx.h, C.byref(dsc), G_loc, _p(spectra, torch.float64),
                                    bins.data_ptr() + 4 * bins_off, ldb, nJ,
                                    kappa_min.data_ptr() + 8 * kmin_off, ldk, _p(kappa_max, torch.float64),
                                    _p(tau, torch.float64))
    _check(ctx, st, "usfft_lattice_keys")


def usfft_lattice_keys_product(ctx: Context, plan: Plan, G_loc: int, spectra, bins, ldb: int, j0: int, nJ: int,
                               n1: int, kappa_min, ldk: int, kappa_max, kmin_off: int = 0, tau=None):
    """a8 for candidates j0 .. j0+nJ of the product set I_prev x kt (j = a n1 + c): bins is the
    whole [L][ldb] map; keys into kappa_min[g*ldk + kmin_off + (j - j0)]."""
    dsc, keep = plan.desc()
    _p(bins, torch.int32), _p(kappa_min, torch.float64)
    st = ctx.lib.usfft_lattice_keys_product(ctx.h, C.byref(dsc), G_loc, _p(spectra, torch.float64),
                                            bins.data_ptr(), ldb, j0, nJ, n1,
                                            kappa_min.data_ptr() + 8 * kmin_off, ldk,
                                            _p(kappa_max, torch.float64), _p(tau, torch.float64))
    _check(ctx, st, "usfft_lattice_keys_product")


def usfft_detect_carry(ctx: Context, G_loc: int, s_tilde: int, width: int, merged, carry_k, carry_j,
                       det_pos, n_det_g, j0: int = 0, det_g=None, votes=None, tau=None):
    """Streamed selection step (Z29): update the per-node carry (det_g None) or emit det_g + votes."""
    st = ctx.lib.usfft_detect_carry(ctx.h, G_loc, s_tilde, width, _p(merged, torch.float64),
                                    _p(carry_k, torch.float64), _p(carry_j, torch.int32),
                                    _p(det_pos, torch.int32), _p(n_det_g, torch.int32), j0,
                                    _p(det_g, torch.int32), _p(votes, torch.int32), _p(tau, torch.float64))
    _check(ctx, st, "usfft_detect_carry")


MOMENT_MAPS = {"sin": 0, "tent": 1, "probit": 2, "phi_delta": 3}   # the C side rejects 2


def usfft_moments(ctx: Context, I, C, theta: str, delta: float, E, var, gsi=None):
    """Expectation E [G][2], variance [G] and GSI [G][d] per node (Z30)."""
    nI, d = (int(I.shape[0]), int(I.shape[1])) if I.dim() == 2 else (0, 1)
    G = int(C.shape[0])
    st = ctx.lib.usfft_moments(ctx.h, d, _p(I, torch.int16), nI, _p(C, torch.float64), G,
                               MOMENT_MAPS[theta], float(delta), _p(E, torch.float64),
                               _p(var, torch.float64), _p(gsi, torch.float64))
    _check(ctx, st, "usfft_moments")


def usfft_detect_union(ctx: Context, nJ: int, votes, flags, det_idx, union_idx=None, counts: bool = True):
    """a11; returns (n_det, n_union) (syncs), or (None, None) without synchronising (counts=False)."""
    if not counts:
        st = ctx.lib.usfft_detect_union(ctx.h, nJ, _p(votes, torch.int32), _p(flags, torch.uint8),
                                        _p(det_idx, torch.int32), None, _p(union_idx, torch.int32), None)
        _check(ctx, st, "usfft_detect_union")
        return None, None
    nd, nu = C.c_int64(0), C.c_int64(0)
    st = ctx.lib.usfft_detect_union(ctx.h, nJ, _p(votes, torch.int32), _p(flags, torch.uint8),
                                    _p(det_idx, torch.int32), C.byref(nd),
                                    _p(union_idx, torch.int32), C.byref(nu))
    _check(ctx, st, "usfft_detect_union")
    return int(nd.value), int(nu.value)


def usfft_resolve(ctx: Context, plan: Plan, G_loc: int, spectra, bins, nJ: int, det_g, n_det_g,
                  s_tilde: int, det_idx, n_det: int, coef, lstar=None):
    dsc, keep = plan.desc()
    st = ctx.lib.usfft_resolve(ctx.h, C.byref(dsc), G_loc, _p(spectra, torch.float64),
                               _p(bins, torch.int32), nJ, _p(det_g, torch.int32),
                               _p(n_det_g, torch.int32), s_tilde, _p(det_idx, torch.int32), n_det,
                               _p(coef, torch.float64), _p(lstar, torch.int32))
    _check(ctx, st, "usfft_resolve")


def usfft_gather_rows(ctx: Context, idx, n: int, I_prev, t: int, kt, rows):
    st = ctx.lib.usfft_gather_rows(ctx.h, _p(idx, torch.int32), n, _p(I_prev, torch.int16), t,
                                   _p(kt, torch.int16), int(kt.numel()), _p(rows, torch.int16))
    _check(ctx, st, "usfft_gather_rows")


def usfft_eval(ctx: Context, I, C_, Y, U):
    """U[g][q] = Re sum_k C[g][k] e^{2 pi i k.y_q}; I int16 [nI][d], C fp64 [G][nI][2], Y [d][n]."""
    nI, d = I.shape
    G = C_.shape[0]
    n = Y.shape[1]
    st = ctx.lib.usfft_eval(ctx.h, d, _p(I, torch.int16), nI, _p(C_, torch.float64), G,
                            _p(Y, torch.float64), n, _p(U, torch.float64))
    _check(ctx, st, "usfft_eval")


@dataclass
class Cover:
    """A Step-3 multiple-R1L cover (usfft_cover_desc) of a frequency set."""
    d: int
    M: int
    z: np.ndarray          # int64 [nlat][d]
    assign: np.ndarray     # int32 [nI]
    bin: np.ndarray        # int32 [nI]

    def lattice(self, q: int) -> Plan:
        """Lattice q as a one-lattice plan (t = d, zero shift: X is a subset of T^d)."""
        return Plan(self.d, self.M, 1, self.d, -1, self.z[q:q + 1].copy(), np.zeros(self.d))


def usfft_cover_plan(ctx: Context, seed: int, N_: int, I_host: np.ndarray) -> Cover:
    I = np.ascontiguousarray(I_host, dtype=np.int16)
    nI, d = I.shape
    out = N.CoverDesc()
    assign = np.empty(nI, dtype=np.int32)
    binv = np.empty(nI, dtype=np.int32)
    _check(ctx, ctx.lib.usfft_cover_plan(ctx.h, seed, d, N_, I.ctypes.data, nI, C.byref(out),
                                         assign.ctypes.data, binv.ctypes.data), "usfft_cover_plan")
    z = np.ctypeslib.as_array(out.z)[: out.nlat * d].reshape(out.nlat, d).copy()
    return Cover(d, int(out.M), z, assign, binv)


def usfft_cover_gather(ctx: Context, M: int, G: int, spectra, idx, bins, coef):
    """coef [G][nI][2] fp64 (device): the entries idx of the frequencies read on this lattice."""
    nI = coef.shape[1]
    st = ctx.lib.usfft_cover_gather(ctx.h, M, G, _p(spectra, torch.float64), _p(idx, torch.int32),
                                    _p(bins, torch.int32), int(idx.numel()), _p(coef, torch.float64), nI)
    _check(ctx, st, "usfft_cover_gather")


def usfft_eval_err(ctx: Context, I, C_, Y, Uref, err):
    """err [G][3] = (err_1, err_2, err_inf) of the approximant against Uref at the points Y."""
    nI, d = I.shape
    G = C_.shape[0]
    n = Y.shape[1]
    st = ctx.lib.usfft_eval_err(ctx.h, d, _p(I, torch.int16), nI, _p(C_, torch.float64), G,
                                _p(Y, torch.float64), n, _p(Uref, torch.float64), _p(err, torch.float64))
    _check(ctx, st, "usfft_eval_err")


def usfft_lattice_dft_bins(ctx: Context, M: int, G_loc: int, u, slab_b0, bins, idx, coef):
    """coef [G_loc][nI][2]: direct lattice DFT of one lattice's samples at the bins in use."""
    sb = np.ascontiguousarray(slab_b0, dtype=np.int64)
    st = ctx.lib.usfft_lattice_dft_bins(ctx.h, M, G_loc, _p(u, torch.float64), len(sb) - 1,
                                        sb.ctypes.data_as(C.POINTER(C.c_int64)), _p(bins, torch.int32),
                                        _p(idx, torch.int32), int(idx.numel()), _p(coef, torch.float64),
                                        coef.shape[1])
    _check(ctx, st, "usfft_lattice_dft_bins")

