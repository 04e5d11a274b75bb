"""ctypes binding of the sm_100a library (include/sylfem_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is visible, every device entry point raises.  PyTorch is used only as the
device-memory / stream plumbing (tensors are passed to the C ABI as raw
pointers).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .exceptions import OperatorError, SolverError, SylfemError

_HERE = os.path.dirname(os.path.abspath(__file__))
# SYLFEM_B200_LIB: an alternative in-tree build of the same library (kernel experiments)
LIB_PATH = os.environ.get("SYLFEM_B200_LIB") or os.path.join(_HERE, "libsylfem_b200.so")

# status codes / kinds (mirror include/sylfem_b200.h)
OK, ERR_ARG, ERR_CUDA, ERR_NOMEM, ERR_UNSUPPORTED = 0, -1, -2, -3, -4
PCG_RUNNING, PCG_TOLERANCE, PCG_INCREMENT, PCG_INDEFINITE, PCG_NONFINITE, PCG_MAX_ITER = range(6)
RULE_RESIDUAL, RULE_INCREMENT, RULE_BUDGET = 0, 1, 2
PRE_IDENTITY, PRE_INVERSE, PRE_SPECTRAL_PROD, PRE_SPECTRAL_SUM, PRE_BANDED = range(5)

EXPORTS = [
    "sfb_version", "sfb_last_error", "sfb_init",
    "sfb_op_create", "sfb_op_create_block", "sfb_op_create_dense", "sfb_op_apply", "sfb_op_residual", "sfb_op_destroy",
    "sfb_map_create", "sfb_map_apply", "sfb_map_apply_heat", "sfb_map_apply_dib", "sfb_map_destroy",
    "sfb_pre_create", "sfb_pre_create_banded", "sfb_pre_apply", "sfb_pre_transform", "sfb_pre_destroy",
    "sfb_set_strassen_min_q", "sfb_set_strassen_levels", "sfb_pre_uses_strassen",
    "sfb_pcg_create", "sfb_pcg_solve", "sfb_pcg_pass_times", "sfb_pcg_destroy", "sfb_dgemm_nt", "sfb_diff_norm",
    "sfb_vec_update", "sfb_vec_xpby", "sfb_vec_dots",
    "sfb_csr_create", "sfb_csr_spmv", "sfb_csr_destroy",
    "sfb_pcg_shape", "sfb_imex_heat_run", "sfb_imex_rds_run",
    "sfb_dgemm_nt_scatter", "sfb_dgemm_nt_batch", "sfb_copy2d", "sfb_ipc_get_handle", "sfb_ipc_open", "sfb_ipc_close",
    "sfb_frame_pgm16", "sfb_geigh", "sfb_reduced_create", "sfb_reduced_solve", "sfb_reduced_destroy",
    "sfb_shard_create", "sfb_shard_destroy", "sfb_shard_slots", "sfb_shard_dots", "sfb_shard_start",
    "sfb_shard_update", "sfb_shard_control", "sfb_shard_xpby", "sfb_shard_result",
    "sfb_shard_apply", "sfb_shard_gemm", "sfb_shard_gemm_scatter", "sfb_shard_pre_apply",
    "sfb_const_create", "sfb_const_levels", "sfb_const_destroy", "sfb_shard_gemm_const", "sfb_shard_gemm_scatter_const",
    "sfb_lu_create", "sfb_lu_solve", "sfb_lu_destroy",
]
IMEX_OK, IMEX_BLOWUP, IMEX_NOT_CONVERGED, IMEX_INDEFINITE, IMEX_NONFINITE = range(5)


class PcgResult(C.Structure):
    _fields_ = [("iterations", C.c_int), ("stop_reason", C.c_int), ("bad_iter", C.c_int),
                ("chunks", C.c_int), ("res0", C.c_double), ("bad_value", C.c_double),
                ("device_ms", C.c_double)]


class ImexResult(C.Structure):
    _fields_ = [("steps_done", C.c_int), ("fail_step", C.c_int), ("fail_kind", C.c_int),
                ("fail_species", C.c_int), ("steady_step", C.c_int), ("pcg_bad_iter", C.c_int),
                ("pcg_bad_value", C.c_double)]


_P = C.c_void_p
_D = C.c_double
_I = C.c_int
_DP = C.POINTER(C.c_double)

_SIGS = {
    "sfb_csr_create": (C.c_int, [C.c_int, C.c_longlong, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "sfb_csr_spmv": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "sfb_csr_destroy": (C.c_int, [C.c_void_p]),
    "sfb_version": (_I, []),
    "sfb_last_error": (C.c_char_p, []),
    "sfb_init": (_I, [_I, C.POINTER(_I)]),
    "sfb_op_create": (_I, [_I, _I, _I, _I, _I, _P, _I, _I, _P, C.POINTER(_P)]),
    "sfb_op_create_block": (_I, [_I, _I, _I, _I, _I, _I, _P, _I, _P, C.POINTER(_P)]),
    "sfb_op_create_dense": (_I, [_I, _I, _I, _P, _P, C.POINTER(_P)]),
    "sfb_op_apply": (_I, [_P, _P, _I, _P, _I, _P]),
    "sfb_op_residual": (_I, [_P, _P, _I, _P, _I, _DP, _P]),
    "sfb_op_destroy": (_I, [_P]),
    "sfb_map_create": (_I, [_I, _I, _I, _I, _I, _I, _P, _I, _I, _P, C.POINTER(_P)]),
    "sfb_map_apply": (_I, [_P, _P, _I, _P, _I, _P]),
    "sfb_map_apply_heat": (_I, [_P, _P, _I, _I, _I, _D, _P, _I, _P, _I, _DP, _P]),
    "sfb_map_apply_dib": (_I, [_P, _P, _P, _I, _I, _D, _DP, _P, _I, _DP, _P]),
    "sfb_map_destroy": (_I, [_P]),
    "sfb_pre_create": (_I, [_I, _I, _I, _P, _P, _P, _P, C.POINTER(_P)]),
    "sfb_pre_create_banded": (_I, [_I, _I, _I, _P, _I, _P, C.POINTER(_P)]),
    "sfb_pre_apply": (_I, [_P, _P, _I, _P, _I, _P]),
    "sfb_pre_transform": (_I, [_P, _P, _I, _P, _I, _P]),
    "sfb_pre_destroy": (_I, [_P]),
    "sfb_set_strassen_min_q": (_I, [_I]),
    "sfb_set_strassen_levels": (_I, [_I]),
    "sfb_pre_uses_strassen": (_I, [_P]),
    "sfb_pcg_create": (_I, [_P, _P, C.POINTER(_P)]),
    "sfb_pcg_solve": (_I, [_P, _P, _I, _P, _I, _P, _I, _I, _D, _I, _DP, _DP, _P, _I,
                           C.POINTER(PcgResult), _P]),
    "sfb_pcg_pass_times": (_I, [_P, _I, _DP]),
    "sfb_pcg_destroy": (_I, [_P]),
    "sfb_dgemm_nt": (_I, [_P, _I, _P, _I, _I, _I, _I, _P, _I, _P]),
    "sfb_vec_update": (_I, [_P, _P, _P, _P, _I, _I, _I, _D, _DP, _P]),
    "sfb_vec_xpby": (_I, [_P, _I, _P, _I, _I, _I, _D, _I, _P]),
    "sfb_vec_dots": (_I, [_P, _P, _P, _P, _I, _I, _I, _DP, _P]),
    "sfb_diff_norm": (_I, [_P, _I, _P, _I, _I, _I, _DP, _P]),
    "sfb_pcg_shape": (_I, [_P, C.POINTER(_I), C.POINTER(_I)]),
    "sfb_dgemm_nt_scatter": (_I, [_P, _I, _P, _I, _I, _I, _I, _I, _P, _P, _P, _I, _P]),
    "sfb_dgemm_nt_batch": (_I, [_I, _P, _I, _P, _I, _I, _I, _I, _P, _I, C.c_longlong, _P]),
    "sfb_copy2d": (_I, [_P, _I, _P, _I, _I, _I, _P]),
    "sfb_ipc_get_handle": (_I, [_P, _P, C.POINTER(C.c_ulonglong)]),
    "sfb_ipc_open": (_I, [_P, C.c_ulonglong, C.POINTER(_P), C.POINTER(_P)]),
    "sfb_ipc_close": (_I, [_P]),
    "sfb_frame_pgm16": (_I, [_P, _I, _I, _I, _P, _DP, _P]),
    "sfb_geigh": (_I, [_I, _P, _I, _P, _I, _DP, _P, _I, _P]),
    "sfb_reduced_create": (_I, [_P, _P, C.POINTER(_P)]),
    "sfb_reduced_solve": (_I, [_P, _P, _I, _P, _I, _DP, _P]),
    "sfb_reduced_destroy": (_I, [_P]),
    "sfb_shard_create": (_I, [_I, _I, _D, C.POINTER(_P)]),
    "sfb_shard_destroy": (_I, [_P]),
    "sfb_shard_slots": (C.c_void_p, [_P]),
    "sfb_shard_dots": (_I, [_P, _P, _I, _P, _I, _P, _I, _P, _I, _I, _I, _I, _P]),
    "sfb_shard_start": (_I, [_P, _P]),
    "sfb_shard_update": (_I, [_P, _P, _I, _P, _I, _P, _I, _P, _I, _I, _I, _P]),
    "sfb_shard_control": (_I, [_P, _P]),
    "sfb_shard_xpby": (_I, [_P, _P, _I, _P, _I, _I, _I, _I, _P]),
    "sfb_shard_result": (_I, [_P, C.POINTER(PcgResult), _DP, _DP, _P]),
    "sfb_shard_apply": (_I, [_P, _P, _P, _I, _P, _I, _P]),
    "sfb_shard_gemm": (_I, [_P, _P, _I, _P, _I, _I, _I, _I, _P, _I, _P]),
    "sfb_shard_gemm_scatter": (_I, [_P, _P, _I, _P, _I, _I, _I, _I, _I, _P, _P, _P, _I, _P]),
    "sfb_const_create": (_I, [_P, _I, _I, _I, _I, C.POINTER(_P)]),
    "sfb_const_levels": (_I, [_P]),
    "sfb_const_destroy": (_I, [_P]),
    "sfb_shard_gemm_const": (_I, [_P, _P, _P, _I, _I, _P, _I, _P]),
    "sfb_shard_gemm_scatter_const": (_I, [_P, _P, _P, _I, _I, _I, _P, _P, _P, _I, _P]),
    "sfb_shard_pre_apply": (_I, [_P, _P, _P, _I, _P, _I, _P]),
    "sfb_lu_create": (_I, [_I, C.c_longlong, _P, _P, _P, C.c_longlong, _P, _P, _P, _P, _P, C.POINTER(_P)]),
    "sfb_lu_solve": (_I, [_P, _P, _P, _P]),
    "sfb_lu_destroy": (_I, [_P]),
    "sfb_imex_heat_run": (_I, [_P, _P, _I, _I, _P, _I, _DP, _I, _I, _D, _I, _P, _I, C.POINTER(_I), _DP,
                               C.POINTER(ImexResult), _P]),
    "sfb_imex_rds_run": (_I, [_P, _P, _P, _DP, _D, _I, _I, _D, _I, _D, _P, _P, _I, C.POINTER(_I), _DP,
                              C.POINTER(ImexResult), _P]),
}

_lib = None
_lock = threading.Lock()
_initialized = False


def load_library():
    """Load the shared library (no device needed).  Raises if it was not built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise SylfemError(f"{LIB_PATH} is missing: build it with "
                                      "`python -m paper_2109_01173_b200.build` (no CPU fallback)")
                lib = C.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(lib, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = lib
    return _lib


def lib():
    """The library with a CUDA device initialised (raises loudly otherwise)."""
    global _initialized
    L = load_library()
    if not _initialized:
        with _lock:
            if not _initialized:
                import torch
                if not torch.cuda.is_available():
                    raise SylfemError("paper_2109_01173_b200 needs a CUDA device (B200); "
                                      "there is no CPU fallback")
                torch.cuda.init()
                dev = torch.cuda.current_device()
                n = C.c_int(0)
                check(L.sfb_init(dev, C.byref(n)), "init")
                _initialized = True
    return L


def last_error() -> str:
    return load_library().sfb_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc == OK:
        return
    msg = last_error()
    where = f"{what}: " if what else ""
    if rc == ERR_ARG:
        raise OperatorError(where + msg)
    raise SolverError(where + msg)


# ---------------------------------------------------------------- torch glue
def torch():
    import torch as _t
    return _t


def stream() -> int:
    t = torch()
    return t.cuda.current_stream().cuda_stream


def to_device(a):
    """numpy / torch -> contiguous float64 CUDA tensor."""
    t = torch()
    if isinstance(a, t.Tensor):
        return a.to(device="cuda", dtype=t.float64).contiguous()
    return t.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).to("cuda")


def to_host(t) -> np.ndarray:
    """CUDA tensor -> numpy array returned to the caller.  The copy lands in
    page-locked memory from torch's caching host allocator (the numpy array
    keeps that block alive; it returns to the cache when the array dies):
    a DMA at full PCIe/NVLink-C2C rate instead of a pageable copy that
    first-touches a freshly mapped host buffer."""
    th = torch()
    out = th.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    out.copy_(t)
    return out.numpy()


def ptr(t) -> int:
    return t.data_ptr()


def host_ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_DP)


def is_device(a) -> bool:
    t = torch()
    return isinstance(a, t.Tensor) and a.is_cuda


class Handle:
    """Owns a native object; destroyed with its Python wrapper."""

    def __init__(self, p, destroy):
        self.p = p
        self._destroy = destroy

    def __del__(self):
        try:
            if self.p and _lib is not None:
                self._destroy(self.p)
        except Exception:  # interpreter shutdown
            pass
        self.p = None
