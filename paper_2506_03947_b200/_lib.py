"""ctypes binding of include/aac.h -- argument marshalling only.

Every step of the solve runs in libaac.so's CUDA kernels; PyTorch supplies device
memory, the CUDA stream and (for nranks > 1) the process group that broadcasts the
NCCL unique id. There is no CPU fallback: if libaac.so is missing this module
raises ImportError.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libaac.so")

AAC_OK, AAC_ENOCONV, AAC_EINVAL, AAC_ECUDA, AAC_ENCCL, AAC_ENOMEM = 0, 1, -1, -2, -3, -4
AAC_NONE, AAC_NC1, AAC_NC2, AAC_SP, AAC_EXACT = 0, 1, 2, 3, 4
AAC_F32 = 16                     # OR'ed into nc1 / nc2: fp32 inner Chebyshev recurrence
METHODS = {"none": AAC_NONE, "nc1": AAC_NC1, "nc2": AAC_NC2, "sp": AAC_SP, "exact": AAC_EXACT,
           "nc1-f32": AAC_NC1 | AAC_F32, "nc2-f32": AAC_NC2 | AAC_F32}

# Every symbol include/aac.h declares (tests check the .so exports all of them).
SYMBOLS = ["aac_slab_range", "aac_slab_weights", "aac_setup", "aac_setup_host_transport", "aac_matvec", "aac_precond_apply", "aac_gmres",
           "aac_gmres_host", "aac_gmres_host_batch", "aac_query", "aac_profile_enable", "aac_profile_count",
           "aac_profile_read", "aac_profile_flops", "aac_profile_reset", "aac_set_boundary",
           "aac_set_bounds", "aac_set_blocks", "aac_ci", "aac_launch_count", "aac_comm_kind", "aac_last_error",
           "aac_destroy"]


class aac_grid(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("n", ctypes.c_int64 * 3), ("rank", ctypes.c_int),
                ("nranks", ctypes.c_int)]


class aac_gmres_info(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int), ("converged", ctypes.c_int),
                ("relres_est", ctypes.c_double), ("relres_true", ctypes.c_double),
                ("matvecs_paper_units", ctypes.c_longlong), ("stencil_sweeps", ctypes.c_longlong)]

    def asdict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                ctypes.c_int, ctypes.c_int)
SENDRECV_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                               ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                               ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double))


class aac_host_transport(ctypes.Structure):
    _fields_ = [("user", ctypes.c_void_p), ("allreduce", ALLREDUCE_FN), ("sendrecv", SENDRECV_FN)]


class AacError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libaac error {code}: {msg}")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(python -m paper_2506_03947_b200.build)")
    lib = ctypes.CDLL(LIB_PATH)
    P, D, I, L = ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_longlong
    dp = ctypes.POINTER(ctypes.c_double)
    sig = {
        "aac_slab_range": (I, [ctypes.c_int64, I, I, ctypes.POINTER(ctypes.c_int64),
                               ctypes.POINTER(ctypes.c_int64)]),
        "aac_slab_weights": (I, [ctypes.POINTER(aac_grid), dp, dp, dp, D, dp,
                                 ctypes.POINTER(ctypes.c_int64), dp]),
        "aac_setup": (I, [ctypes.POINTER(aac_grid), dp, dp, dp, D, I, D, I, P, P,
                          ctypes.POINTER(P)]),
        "aac_setup_host_transport": (I, [ctypes.POINTER(aac_grid), dp, dp, dp, D, I, D, I, P,
                                         ctypes.POINTER(aac_host_transport), ctypes.POINTER(P)]),
        "aac_matvec": (I, [P, P, P]),
        "aac_precond_apply": (I, [P, I, I, P, P]),
        "aac_gmres": (I, [P, I, I, P, P, D, I, ctypes.POINTER(aac_gmres_info)]),
        "aac_gmres_host": (I, [P, I, I, dp, dp, D, I, ctypes.POINTER(aac_gmres_info)]),
        "aac_gmres_host_batch": (I, [P, I, I, I, ctypes.POINTER(dp), ctypes.POINTER(dp), D, I,
                                     ctypes.POINTER(aac_gmres_info)]),
        "aac_query": (I, [P, I, I, dp, dp, ctypes.POINTER(I), ctypes.POINTER(ctypes.c_int64)]),
        "aac_profile_enable": (I, [P, I]),
        "aac_profile_count": (I, []),
        "aac_profile_read": (I, [P, I, ctypes.POINTER(ctypes.c_char_p), dp,
                                 ctypes.POINTER(L), dp]),
        "aac_profile_flops": (I, [P, I, dp]),
        "aac_profile_reset": (I, [P]),
        "aac_set_boundary": (I, [P, D, D, D]),
        "aac_set_bounds": (I, [P, D, D]),
        "aac_set_blocks": (I, [P, dp, dp, dp]),
        "aac_ci": (I, [P, I, I, P, P, D, D, D, I, ctypes.POINTER(aac_gmres_info)]),
        "aac_launch_count": (L, [P]),
        "aac_comm_kind": (I, [P]),
        "aac_last_error": (ctypes.c_char_p, [P]),
        "aac_destroy": (None, [P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def check(rc, ctx=None, ok=(AAC_OK,)):
    if rc in ok:
        return rc
    msg = lib.aac_last_error(ctx)
    raise AacError(rc, msg.decode() if msg else "")
