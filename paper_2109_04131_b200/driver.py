"""Alg. 1 "The usFFT on a set T_G" driven through the C-ABI on one or more GPUs.

The host loop only sequences the C-ABI calls and sizes buffers; every step of a round (plan,
nodes, bins, PDE solves, transpose, FFT, keys, selection, union, resolve, row gather) and, with
several GPUs, every collective runs in libusfft.so (its own NCCL communicator; dist.py only
broadcasts the communicator id).

Round r = (step, t, i):
  a1 plan (usfft_plan_round) -> a4/a5 samples of this rank (usfft_sample_pde, nodes a2
  generated in-kernel) -> a3 bins (usfft_lattice) -> a6 transpose (usfft_transpose) ->
  a7/a8 FFT + keys (usfft_lattice_fft) -> a9 kappa_max MAX + a10 select + votes
  (usfft_detect_select) -> votes SUM + a11 union (usfft_detect_union) -> a12 resolve
  (usfft_resolve, final round only).
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import binding as B
import torch.distributed as tdist

from .dist import TorchExchange, bootstrap_id, bounds, partition


@dataclass
class RoundResult:
    plan: B.Plan
    nJ: int
    n_det: int
    n_union: int
    det_idx: torch.Tensor          # int32 [n_det] (device)
    union_idx: torch.Tensor        # int32 [n_union]
    theta2: float | None = None
    coef: torch.Tensor | None = None       # fp64 [G_loc][n_det][2]
    lstar: torch.Tensor | None = None
    iters: torch.Tensor | None = None
    times: dict = field(default_factory=dict)


class Detector:
    """One usFFT detection run (Steps 1-2 of Alg. 1) for a workload preset (usfft_inputs)."""

    def __init__(self, cfg: dict, device: int = 0, group=None, maxit: int = 20000,
                 timing: bool = False, blackbox=None, loopback=None):
        """blackbox: optional callable (detector, plan, b0, nb) -> fp64 CUDA tensor [G][nb]
        replacing the PDE sampler (Alg. 1 takes any black box); cfg["G"] then gives G.
        Ranks: with torch.distributed initialised on an NCCL process group the library builds
        its own communicator (id broadcast by dist.bootstrap_id); loopback = (rank, P, key)
        runs virtual rank `rank` of P in this thread on one GPU (key: 128 bytes shared by the P
        threads); a gloo process group falls back to TorchExchange (ranks sharing one GPU)."""
        self.cfg = cfg
        self.blackbox = blackbox
        self.dev = torch.device("cuda", device)
        world = tdist.get_world_size(group) if tdist.is_available() and tdist.is_initialized() else 1
        if loopback is not None:
            rank, P, key = loopback
            self.ctx = B.Context(device, rank=rank, nranks=P, comm_id=key, loopback=True)
            self.ex = None
        elif world > 1 and tdist.get_backend(group) == "nccl":
            rank, P = tdist.get_rank(group), world
            self.ctx = B.Context(device, rank=rank, nranks=P, comm_id=bootstrap_id(group))
            self.ex = None
        else:
            self.ex = TorchExchange(group)
            rank, P = self.ex.rank, self.ex.P
            self.ctx = B.Context(device)
        self.P, self.rank = P, rank
        # phi_Delta map: one global pole shift Delta = 1/(4 M0), M0 the Step-2 lattice size (Z27)
        self.delta = 0.0
        if cfg.get("theta") == "phi_delta":
            self.delta = B.usfft_plan_delta(self.ctx, cfg["N"], cfg["s_local"], int(cfg.get("lattice_factor", 1)))
        self.pde = B.pde_desc(cfg, maxit=maxit, tol=cfg.get("cg_tol", 1e-12), delta=self.delta) \
            if blackbox is None else None
        self.G = cfg["G"] if blackbox is not None else (cfg["n"] - 1) ** 2
        self.g0, self.g1 = partition(self.G, self.P, self.rank)
        self.G_loc = self.g1 - self.g0
        self.timing = timing
        self.n_samples = 0

    # ---- exchange steps: in the library (usfft_transpose; the MAX / SUM inside
    # usfft_detect_select / usfft_detect_union) or, for gloo groups, through torch.distributed
    def transpose(self, u: torch.Tensor, G: int, Btot: int):
        """a6: this rank's samples [G][nb] -> (slabs [G_loc * Btot] of its nodes, slab_b0)."""
        if self.ex is not None:
            return self.ex.transpose(u, G, Btot)
        sb = bounds(Btot, self.P)
        if self.P == 1:
            return u, sb
        slabs = torch.empty(self.G_loc * Btot, dtype=torch.float64, device=self.dev)
        B.usfft_transpose(self.ctx, G, Btot, u, slabs)
        return slabs, sb

    def _max(self, t):
        return self.ex.max_(t) if self.ex is not None else t

    def _sum(self, t):
        return self.ex.sum_(t) if self.ex is not None else t

    # ------------------------------------------------------------------------------------------
    def round(self, step: int, t: int, i: int, I_prev: torch.Tensor, n_prev: int,
              kt: torch.Tensor, s_tilde: int, flags: torch.Tensor, want_coef: bool = False,
              keep_iters: bool = False, counts: bool = True) -> RoundResult:
        """One detection round.  counts=False: the round only feeds the running union `flags` and
        returns without synchronising (n_det, n_union = None): the rounds i < r of a dimension."""
        cfg, ctx, dev = self.cfg, self.ctx, self.dev
        n1 = int(kt.numel())
        nJ = n_prev * n1
        ev = {}

        def mark(name):
            if self.timing:
                e = torch.cuda.Event(enable_timing=True)
                e.record(ctx.stream)
                ev[name] = e

        mark("start")
        # cfg["lattice_factor"] f > 1 sizes the Step-2 lattices for f s~ (M >= 4 f s~, Z2) while
        # the selection keeps s~: less aliasing per bin for non-sparse projections (§9)
        s_plan = s_tilde * int(cfg.get("lattice_factor", 1)) if step == 2 else s_tilde
        plan = B.usfft_plan_round(ctx, cfg["seed"], step, t, i, cfg["d"], cfg["N"], s_plan,
                                  cfg.get("mode", "A") if step == 2 else "A", nJ,
                                  I_prev if t > 1 else None, n_prev, kt)
        L, M = plan.L, plan.M
        Btot = L * M
        # this rank's samples (the solves go first: the index map is only needed by the keys)
        b0, b1 = partition(Btot, self.P, self.rank)
        nb = b1 - b0
        u = torch.empty((self.G, nb), dtype=torch.float64, device=dev)
        iters = torch.empty(nb, dtype=torch.int32, device=dev) if keep_iters else None
        mark("plan")
        if nb and self.blackbox is not None:
            u = self.blackbox(self, plan, b0, nb)
        elif nb:
            B.usfft_sample_pde(ctx, self.pde, plan, b0, nb, u, nb, None, iters)
        self.n_samples += Btot
        bins = torch.empty((L, nJ), dtype=torch.int32, device=dev)
        B.usfft_lattice(ctx, plan, 0, 0, None, I_prev if plan.t_z > 1 else None, n_prev, kt, bins)
        mark("pde")
        slabs, sb = self.transpose(u, self.G, Btot)
        mark("exchange")
        Mh = M // 2 + 1
        spectra = torch.empty((self.G_loc, L, Mh, 2), dtype=torch.float64, device=dev)
        kmax = torch.empty(1, dtype=torch.float64, device=dev)      # reset by usfft_lattice_fft
        det_g = torch.empty((self.G_loc, s_tilde), dtype=torch.int32, device=dev)
        n_det_g = torch.empty(self.G_loc, dtype=torch.int32, device=dev)
        th2 = torch.empty(1, dtype=torch.float64, device=dev)
        chunk = self.key_chunk(nJ, s_tilde)
        if chunk is None:
            kmin = torch.empty((self.G_loc, nJ), dtype=torch.float64, device=dev)
            # a7 then a8 as two calls (the same kernels usfft_lattice_fft runs with nJ > 0), so the
            # FFT and the keys are timed as separate phases
            B.usfft_lattice_fft(ctx, plan, self.G_loc, slabs, sb, bins, 0, spectra, None, kmax)
            mark("fft")
            B.usfft_lattice_keys_product(ctx, plan, self.G_loc, spectra, bins, nJ, 0, nJ, n1, kmin, nJ, kmax)
            mark("keys")
            self._max(kmax)
            votes = torch.empty(nJ, dtype=torch.int32, device=dev)
            B.usfft_detect_select(ctx, self.G_loc, nJ, kmin, kmax, s_tilde, cfg.get("theta_rel", 1e-6),
                                  cfg.get("theta_abs", 0.0), votes, det_g, n_det_g, th2)
        else:
            kmin = None
            B.usfft_lattice_fft(ctx, plan, self.G_loc, slabs, sb, bins, 0, spectra, None, kmax)
            mark("fft")
            votes = self._streamed_select(plan, nJ, n1, s_tilde, chunk, spectra, bins, kmax, det_g, n_det_g, th2)
        self._sum(votes)
        det_idx = torch.empty(nJ, dtype=torch.int32, device=dev)
        union_idx = torch.empty(nJ, dtype=torch.int32, device=dev)
        n_det, n_union = B.usfft_detect_union(ctx, nJ, votes, flags, det_idx, union_idx,
                                              counts=counts or want_coef)
        mark("detect")
        res = RoundResult(plan, nJ, n_det, n_union, det_idx[:n_det] if n_det is not None else None,
                          union_idx[:n_union] if n_union is not None else None)
        res.iters = iters
        if want_coef and n_det:
            coef = torch.empty((self.G_loc, n_det, 2), dtype=torch.float64, device=dev)
            lstar = torch.empty((self.G_loc, n_det), dtype=torch.int32, device=dev)
            B.usfft_resolve(ctx, plan, self.G_loc, spectra, bins, nJ, det_g, n_det_g, s_tilde,
                            det_idx, n_det, coef, lstar)
            res.coef, res.lstar = coef, lstar
        mark("resolve")
        res.theta2 = th2
        if self.timing:
            torch.cuda.synchronize(dev)
            names = list(ev)
            res.times = {names[k]: ev[names[k - 1]].elapsed_time(ev[names[k]]) for k in range(1, len(names))}
        # debugging/parity handles
        res.bins, res.kappa_min, res.spectra, res.votes, res.det_g, res.n_det_g = bins, kmin, spectra, votes, det_g, n_det_g
        res.kappa_max, res.u, res.slab_b0 = kmax, u, sb
        self.last_round = res
        return res

    # ------------------------------------------------------------------------------------------
    KEY_BYTES = 4 << 30         # largest one-shot kappa_min [G_loc][|J|] before the keys are streamed

    def key_chunk(self, nJ: int, s_tilde: int) -> int | None:
        """Candidates per chunk of the streamed selection (Z29), or None for the one-shot path:
        cfg["key_chunk"] forces a chunk size; otherwise stream when G_loc |J| 8 B > KEY_BYTES."""
        forced = self.cfg.get("key_chunk")
        if forced:
            return int(forced) if nJ > int(forced) else None
        if self.G_loc * nJ * 8 <= self.KEY_BYTES or self.G_loc == 0:
            return None
        return max(256, (self.KEY_BYTES // (8 * self.G_loc) - s_tilde) // 256 * 256)

    def _streamed_select(self, plan, nJ, n1, s_tilde, chunk, spectra, bins, kmax, det_g, n_det_g, th2):
        """a8 + a9 + a10 over chunks of J with a per-node top-s~ carry (usfft.h, Z29): the same
        D_g, votes and theta^2 as the one-shot selection, in O(G_loc (s~ + chunk)) memory."""
        cfg, ctx, dev, G = self.cfg, self.ctx, self.dev, self.G_loc
        W = s_tilde + chunk
        merged = torch.zeros((G, W), dtype=torch.float64, device=dev)
        carry_k = torch.zeros((G, s_tilde), dtype=torch.float64, device=dev)
        carry_j = torch.full((G, s_tilde), -1, dtype=torch.int32, device=dev)
        det_pos = torch.empty((G, s_tilde), dtype=torch.int32, device=dev)
        scratch = torch.empty(W, dtype=torch.int32, device=dev)
        tau = torch.zeros(G, dtype=torch.float64, device=dev)    # carry threshold (prefilter)
        for j0 in range(0, nJ, chunk):
            c = min(chunk, nJ - j0)
            if c < chunk:
                merged[:, s_tilde + c:].zero_()                 # ragged last chunk: zero keys
            B.usfft_lattice_keys_product(ctx, plan, G, spectra, bins, nJ, j0, c, n1, merged, W, kmax,
                                         kmin_off=s_tilde, tau=tau)
            B.usfft_detect_select(ctx, G, W, merged, kmax, s_tilde, 0.0, 0.0, scratch, det_pos, n_det_g)
            B.usfft_detect_carry(ctx, G, s_tilde, W, merged, carry_k, carry_j, det_pos, n_det_g, j0, tau=tau)
        self._max(kmax)
        B.usfft_detect_select(ctx, G, s_tilde, carry_k, kmax, s_tilde, cfg.get("theta_rel", 1e-6),
                              cfg.get("theta_abs", 0.0), scratch, det_pos, n_det_g, th2)
        votes = torch.zeros(nJ, dtype=torch.int32, device=dev)
        B.usfft_detect_carry(ctx, G, s_tilde, s_tilde, carry_k, None, carry_j, det_pos, n_det_g, 0,
                             det_g, votes)
        return votes

    # ---- checkpoint / resume: after Step 1 and after every dimension t of Step 2 the
    # run's state (the 1-D sets I^(t), t = 1..d, and I^(1..t)) goes to a small .npz file; all
    # randomness is counter-based (Z4: seed, step, t, i), so a resumed run recomputes rounds
    # t+1.. exactly as the uninterrupted run would.  Rank 0 writes (every rank holds the same
    # sets); the file is replaced atomically.
    def _ckpt_key(self) -> str:
        c = self.cfg
        return json.dumps({k: c.get(k) for k in ("name", "seed", "d", "N", "s", "s_local", "r", "mode", "n",
                                                   "theta", "theta_rel")}, sort_keys=True)

    def save_checkpoint(self, path: str, I1d: list[torch.Tensor], t: int, I_prev: torch.Tensor | None):
        if self.rank != 0:
            return
        arrs = {f"I1d_{k}": v.cpu().numpy() for k, v in enumerate(I1d)}
        if I_prev is not None:
            arrs["I_prev"] = I_prev.cpu().numpy()
        tmp = path + ".tmp.npz"
        np.savez(tmp, key=np.array(self._ckpt_key()), t=np.array(t), **arrs)
        os.replace(tmp, path)

    def load_checkpoint(self, path: str):
        """(I1d, t, I_prev) of a checkpoint of this configuration; t = 1 after Step 1 only."""
        z = np.load(path)
        if str(z["key"]) != self._ckpt_key():
            raise ValueError(f"{path}: checkpoint of another configuration")
        d = self.cfg["d"]
        I1d = [torch.as_tensor(z[f"I1d_{k}"], device=self.dev) for k in range(d)]
        t = int(z["t"])
        I_prev = torch.as_tensor(z["I_prev"], device=self.dev).contiguous() if "I_prev" in z else None
        return I1d, t, I_prev

    def step1(self, log: list | None = None) -> list[torch.Tensor]:
        """Step 1 & 2a: I^(t) for t = 1..d as device int16 vectors."""
        cfg, dev = self.cfg, self.dev
        N, d, r = cfg["N"], cfg["d"], cfg["r"]
        kt = torch.arange(-N, N + 1, dtype=torch.int16, device=dev)
        empty = torch.zeros(1, dtype=torch.int16, device=dev)
        out = []
        for t in range(1, d + 1):
            flags = torch.zeros(kt.numel(), dtype=torch.uint8, device=dev)
            res = None
            for i in range(1, r + 1):
                res = self.last_round = None                   # free the previous round first
                res = self.round(1, t, i, empty, 1, kt, cfg["s_local"], flags)
                if log is not None:
                    log.append(dict(step=1, t=t, i=i, M=res.plan.M, B=res.plan.M, nJ=res.nJ, n_det=res.n_det))
            n_u = res.n_union
            if n_u == 0:
                out.append(torch.zeros(1, dtype=torch.int16, device=dev))             # Z9
                continue
            rows = torch.empty((n_u, 1), dtype=torch.int16, device=dev)
            B.usfft_gather_rows(self.ctx, res.union_idx, n_u, None, 1, kt, rows)
            out.append(rows.reshape(-1))
        return out

    def step2(self, I1d: list[torch.Tensor], log: list | None = None, t_stop: int | None = None,
              checkpoint: str | None = None, start: tuple[int, torch.Tensor] | None = None):
        """Step 2: returns (I^(1..d) int16 [nI][d] device, coef [G_loc][nI][2]).
        checkpoint: write the state after every dimension; start = (t0, I^(1..t0)) continues a
        checkpointed run at t0 + 1."""
        cfg, dev, ctx = self.cfg, self.dev, self.ctx
        d, r = cfg["d"], cfg["r"]
        I_prev = I1d[0].reshape(-1, 1).contiguous()
        t_first = 2
        if start is not None:
            t_first = start[0] + 1
            I_prev = start[1].contiguous()
        coef = None
        t_end = d if t_stop is None else t_stop
        for t in range(t_first, t_end + 1):
            r_t, s_t = (r, cfg["s_local"]) if t < d else (1, cfg["s"])
            kt = I1d[t - 1]
            n_prev = I_prev.shape[0]
            nJ = n_prev * int(kt.numel())
            flags = torch.zeros(nJ, dtype=torch.uint8, device=dev)
            res = None
            for i in range(1, r_t + 1):
                res = self.last_round = None                   # free the previous round first
                # only the last round of a dimension needs the counts on the host; the others are
                # enqueued without a synchronisation (the log wants n_det of every round)
                res = self.round(2, t, i, I_prev, n_prev, kt, s_t, flags, want_coef=(t == d),
                                 counts=(i == r_t or log is not None))
                if log is not None:
                    log.append(dict(step=2, t=t, i=i, M=res.plan.M, L=res.plan.L,
                                    B=res.plan.M * res.plan.L, nJ=nJ, n_det=res.n_det))
            n_u = res.n_union
            rows = torch.empty((max(n_u, 1), t), dtype=torch.int16, device=dev)
            if n_u:
                B.usfft_gather_rows(ctx, res.union_idx, n_u, I_prev if t > 1 else None, t, kt, rows)
            I_prev = rows[:n_u].contiguous()
            if t == d:
                coef = res.coef
            if checkpoint is not None and t < d:
                self.save_checkpoint(checkpoint, I1d, t, I_prev)
            if n_u == 0:
                return I_prev, None
        return I_prev, coef

    def run(self, log: list | None = None, checkpoint: str | None = None):
        """Steps 1-2.  checkpoint: a path; an existing checkpoint of this configuration resumes
        the run after its last completed dimension, and the state is written after Step 1 and
        after every dimension of Step 2."""
        if checkpoint is not None and os.path.exists(checkpoint):
            I1d, t0, I_prev = self.load_checkpoint(checkpoint)
            start = (t0, I_prev) if I_prev is not None else None
            return self.step2(I1d, log, checkpoint=checkpoint, start=start)
        I1d = self.step1(log)
        if checkpoint is not None:
            self.save_checkpoint(checkpoint, I1d, 1, None)
        return self.step2(I1d, log, checkpoint=checkpoint)

    # ------------------------------------------------------------------------------------------
    FFT_MAX_M = 4001           # largest lattice the Rader FFT kernels hold on chip (M-1 = 4000)

    def step3(self, I_rows: torch.Tensor):
        """Step 3: multiple-R1L cover of I (reading Z26, usfft_cover_plan), the samples
        on every cover lattice (this rank's share, exchanged like a round) and the coefficient of
        every k in I read on its lattice (usfft_cover_gather).  I_rows: int16 [nI][d] (device).
        Returns (cover, coef fp64 [G_loc][nI][2])."""
        cfg, ctx, dev = self.cfg, self.ctx, self.dev
        I_host = I_rows.to("cpu").numpy()
        cov = B.usfft_cover_plan(ctx, cfg["seed"], cfg["N"], I_host)
        nI = I_host.shape[0]
        M, Mh = cov.M, cov.M // 2 + 1
        coef = torch.zeros((self.G_loc, nI, 2), dtype=torch.float64, device=dev)
        assign = torch.from_numpy(cov.assign).to(dev)
        bins = torch.from_numpy(cov.bin).to(dev)
        for q in range(cov.z.shape[0]):
            plan = cov.lattice(q)
            b0, b1 = partition(M, self.P, self.rank)
            nb = b1 - b0
            u = torch.empty((self.G, nb), dtype=torch.float64, device=dev)
            if nb and self.blackbox is not None:
                u = self.blackbox(self, plan, b0, nb)
            elif nb:
                B.usfft_sample_pde(ctx, self.pde, plan, b0, nb, u, nb)
            self.n_samples += M
            slabs, sb = self.transpose(u, self.G, M)
            sel = torch.nonzero(assign == q).reshape(-1).to(torch.int32).contiguous()
            if M <= self.FFT_MAX_M:                        # lattice FFT, then read the bins
                spectra = torch.empty((self.G_loc, 1, Mh, 2), dtype=torch.float64, device=dev)
                B.usfft_lattice_fft(ctx, plan, self.G_loc, slabs, sb, None, 0, spectra, None, None)
                B.usfft_cover_gather(ctx, M, self.G_loc, spectra, sel, bins[sel].contiguous(), coef)
            else:                                          # direct DFT at the bins in use
                B.usfft_lattice_dft_bins(ctx, M, self.G_loc, slabs, sb, bins[sel].contiguous(), sel, coef)
        return cov, coef

    def errors(self, I_rows: torch.Tensor, coef: torch.Tensor, Y: torch.Tensor):
        """Accuracy metric of the approximant at n test points Y (fp64 [d][n], device):
        FE reference solves at Y (this rank's share, exchanged to node shards) and
        usfft_eval_err on this rank's nodes.  Returns (err fp64 [G_loc][3], U_check [G_loc][n])."""
        ctx, dev, d = self.ctx, self.dev, self.cfg["d"]
        n = Y.shape[1]
        plan = B.Plan(d, n, 1, d, -1, np.zeros((1, d), dtype=np.int64), np.zeros(d))
        b0, b1 = partition(n, self.P, self.rank)
        nb = b1 - b0
        u = torch.empty((self.G, nb), dtype=torch.float64, device=dev)
        if nb:
            B.usfft_sample_pde(ctx, self.pde, plan, b0, nb, u, nb, Y[:, b0:b1].contiguous())
        slabs, sb = self.transpose(u, self.G, n)
        if self.P == 1:
            U = slabs.reshape(self.G_loc, n)
        else:
            parts, off = [], 0
            for p in range(self.P):
                w = sb[p + 1] - sb[p]
                parts.append(slabs[off:off + self.G_loc * w].reshape(self.G_loc, w))
                off += self.G_loc * w
            U = torch.cat(parts, dim=1).contiguous()
        err = torch.empty((self.G_loc, 3), dtype=torch.float64, device=dev)
        B.usfft_eval_err(ctx, I_rows, coef, Y, U, err)
        return err, U


    def moments(self, I_rows: torch.Tensor, coef: torch.Tensor):
        """Expectation (complex, [G_loc][2]), variance [G_loc] and GSI [G_loc][d] of the
        approximant on this rank's nodes (Z30) with the D_k weights of the
        configuration's periodization (sin: none, tent, phi_Delta with this run's Delta)."""
        G, d, dev = coef.shape[0], self.cfg["d"], self.dev
        E = torch.empty((G, 2), dtype=torch.float64, device=dev)
        var = torch.empty(G, dtype=torch.float64, device=dev)
        gsi = torch.empty((G, d), dtype=torch.float64, device=dev)
        B.usfft_moments(self.ctx, I_rows, coef, self.cfg["theta"], self.delta, E, var, gsi)
        return E, var, gsi


def to_numpy_rows(I: torch.Tensor) -> np.ndarray:
    return I.to("cpu").numpy().astype(np.int64)
