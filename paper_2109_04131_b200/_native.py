"""ctypes loader for libusfft.so (the C-ABI in include/usfft.h).

There is no fallback: if the in-tree library is missing or a CUDA device is absent, the calls
raise.  Build with ``python -m paper_2109_04131_b200.build`` (or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

# USFFT_LIB: load another build of the same sources instead (tools/bounds_check.sh, probe builds)
LIB_PATH = os.environ.get("USFFT_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libusfft.so")

i32, i64, f64, vp = C.c_int32, C.c_int64, C.c_double, C.c_void_p

OK, EINVAL, ENOMEM, ECUDA, ENCCL, ENOCONV, ENOTRECON, EUNIMPL = range(8)
STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 3: "ECUDA", 4: "ENCCL", 5: "ENOCONV",
                6: "ENOTRECON", 7: "EUNIMPL"}


class LatticeDesc(C.Structure):
    _fields_ = [("d", i32), ("t", i32), ("line_axis", i32), ("L", i32), ("M", i64),
                ("z", C.POINTER(i64)), ("shift", C.POINTER(f64))]


class PdeDesc(C.Structure):
    _fields_ = [("n", i32), ("d", i32), ("theta", i32), ("form", i32), ("f_kind", i32),
                ("maxit", i32), ("amp", C.POINTER(f64)), ("tol", f64), ("precond", i32),
                ("psi", i32), ("delta", f64)]


class PlanIn(C.Structure):
    _fields_ = [("seed", i64), ("step", i32), ("t", i32), ("i", i32), ("d", i32), ("N", i32),
                ("s_tilde", i32), ("mode", i32), ("pad_", i32), ("nJ", i64)]


class PlanOut(C.Structure):
    _fields_ = [("M", i64), ("L", i32), ("t_z", i32), ("line_axis", i32), ("pad_", i32),
                ("z", i64 * 2048), ("shift", f64 * 64)]


class RoundDesc(C.Structure):
    _fields_ = [("n", i32), ("d", i32), ("M", i64), ("L", i32), ("s_tilde", i32), ("nJ", i64)]


class CoverDesc(C.Structure):
    _fields_ = [("nlat", i32), ("d", i32), ("M", i64), ("z", i64 * 4096)]


# name -> (restype, argtypes)
_SIGS = {
    "usfft_init": (i32, [C.POINTER(vp), C.c_int, vp, C.c_int, C.c_int, vp, C.c_int]),
    "usfft_comm_unique_id": (i32, [vp]),
    "usfft_comm_info": (i32, [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]),
    "usfft_workspace_query": (i32, [vp, C.POINTER(RoundDesc), C.POINTER(C.c_size_t)]),
    "usfft_plan_delta": (i32, [vp, i32, i32, i32, C.POINTER(f64)]),
    "usfft_transpose": (i32, [vp, i64, i64, vp, i64, vp]),
    "usfft_set_stream": (i32, [vp, vp]),
    "usfft_finalize": (i32, [vp]),
    "usfft_last_error": (C.c_char_p, [vp]),
    "usfft_launch_count": (i64, [vp]),
    "usfft_plan_round": (i32, [vp, C.POINTER(PlanIn), vp, i64, vp, i32, C.POINTER(PlanOut)]),
    "usfft_lattice": (i32, [vp, C.POINTER(LatticeDesc), i64, i64, vp, vp, i64, vp, i32, vp,
                            C.POINTER(i32)]),
    "usfft_sample_pde": (i32, [vp, C.POINTER(PdeDesc), C.POINTER(LatticeDesc), i64, i64, vp, vp,
                               i64, vp, vp, C.POINTER(i32)]),
    "usfft_lattice_fft": (i32, [vp, C.POINTER(LatticeDesc), i64, vp, i32, C.POINTER(i64), vp, i64,
                                vp, vp, vp]),
    "usfft_detect_select": (i32, [vp, i64, i64, vp, vp, i32, f64, f64, vp, vp, vp, vp]),
    "usfft_moments": (i32, [vp, i32, vp, i64, vp, i64, i32, f64, vp, vp, vp]),
    "usfft_lattice_keys": (i32, [vp, C.POINTER(LatticeDesc), i64, vp, vp, i64, i64, vp, i64, vp, vp]),
    "usfft_lattice_keys_product": (i32, [vp, C.POINTER(LatticeDesc), i64, vp, vp, i64, i64, i64, i64, vp, i64, vp,
                                         vp]),
    "usfft_detect_carry": (i32, [vp, i64, i32, i64, vp, vp, vp, vp, vp, i64, vp, vp, vp]),
    "usfft_detect_union": (i32, [vp, i64, vp, vp, vp, C.POINTER(i64), vp, C.POINTER(i64)]),
    "usfft_resolve": (i32, [vp, C.POINTER(LatticeDesc), i64, vp, vp, i64, vp, vp, i32, vp, i64,
                            vp, vp]),
    "usfft_gather_rows": (i32, [vp, vp, i64, vp, i32, vp, i32, vp]),
    "usfft_eval": (i32, [vp, i32, vp, i64, vp, i64, vp, i64, vp]),
    "usfft_cover_plan": (i32, [vp, i64, i32, i32, vp, i64, C.POINTER(CoverDesc), vp, vp]),
    "usfft_cover_gather": (i32, [vp, i64, i64, vp, vp, vp, i64, vp, i64]),
    "usfft_eval_err": (i32, [vp, i32, vp, i64, vp, i64, vp, i64, vp, vp]),
    "usfft_lattice_dft_bins": (i32, [vp, i64, i64, vp, i32, C.POINTER(i64), vp, vp, i64, vp, i64]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load() -> C.CDLL:
    """Load the in-tree libusfft.so (raises if it is missing: there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build(); "
                           "the usFFT path has no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
