"""ctypes binding of the C ABI declared in include/blocktri_b200.h.

The native library is REQUIRED: there is no CPU fallback anywhere in this package.  If the
shared object is missing the import of the solver entry points raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libblocktri_b200.so")
if os.environ.get("BTD_LIB"):  # developer A/B builds (tools/); the shipped library is LIB_PATH
    LIB_PATH = os.path.abspath(os.environ["BTD_LIB"])
_SOURCES = sorted(os.path.join(_HERE, "csrc", f) for f in os.listdir(os.path.join(_HERE, "csrc"))
                  if f.endswith((".cu", ".cuh"))) + \
           [os.path.join(os.path.dirname(_HERE), "include", "blocktri_b200.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]

BTD_OK = 0
BTD_ERR_NOT_POSITIVE_DEFINITE = 1
BTD_ERR_LEVEL_OVERFLOW = 2
BTD_ERR_DIMENSION_MISMATCH = 3
BTD_ERR_INVALID_ARGUMENT = 4
BTD_ERR_UNSUPPORTED = 5
BTD_ERR_CUDA = 6
BTD_ERR_NOT_FACTORED = 7
BTD_ERR_SINGULAR_DIAGONAL = 8

#: every symbol include/blocktri_b200.h declares (checked by tests/test_capi_symbols.py)
EXPORTED_SYMBOLS = (
    "btd_version", "btd_default_config", "btd_plan_separators", "btd_create", "btd_destroy",
    "btd_num_levels", "btd_level_info", "btd_factor_workspace", "btd_factorize", "btd_check",
    "btd_solve_workspace", "btd_solve", "btd_level_factor", "btd_level_schur", "btd_profile_kernels", "btd_kernel_times",
    "btd_create_partial", "btd_reduced_size", "btd_factorize_partial", "btd_solve_down", "btd_solve_up", "btd_launch_count",
    "btd_matmul", "btd_residual_workspace", "btd_residual_norms", "btd_factorize_from_host",
    "btd_kalman_workspace", "btd_kalman_normal_equations", "btd_set_graphs", "btd_graph_replays",
    "btd_seam_error_bytes", "btd_seam_error_init", "btd_seam_error_read", "btd_chol_batch", "btd_trsm_batch",
    "btd_gemm_batch",
)


class BtdConfig(ctypes.Structure):
    _fields_ = [("crossover", ctypes.c_int64), ("segment_length", ctypes.c_int64),
                ("max_levels", ctypes.c_int64), ("auto_crossover", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class BtdStatus(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("pivot", ctypes.c_int32), ("level", ctypes.c_int64),
                ("member", ctypes.c_int64), ("block", ctypes.c_int64),
                ("message", ctypes.c_char * 256)]


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile the sm_100a shared library in-tree (nvcc cross-compiles without a GPU)."""
    newest = max(os.path.getmtime(p) for p in _SOURCES)
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= newest:
        return LIB_PATH
    cmd = ["nvcc", *NVCC_FLAGS, "-o", LIB_PATH + ".tmp", os.path.join(_HERE, "csrc", "btd_capi.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"native library {LIB_PATH} is missing; build it with `python -c "
                f"'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        c_i64, c_i32, c_vp, c_sz = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t
        L.btd_version.restype = ctypes.c_char_p
        L.btd_version.argtypes = []
        L.btd_default_config.restype = None
        L.btd_default_config.argtypes = [P(BtdConfig)]
        L.btd_plan_separators.argtypes = [c_i64, P(BtdConfig), P(c_i64), P(c_i64), P(BtdStatus)]
        L.btd_create.argtypes = [c_i64, c_i64, P(BtdConfig), P(c_vp), P(BtdStatus)]
        L.btd_destroy.restype = None
        L.btd_destroy.argtypes = [c_vp]
        L.btd_num_levels.argtypes = [c_vp, P(c_i64), P(c_i64), P(c_i32)]
        L.btd_level_info.argtypes = [c_vp, c_i64, P(c_i64), P(c_i64), P(c_i64)]
        L.btd_factor_workspace.argtypes = [c_vp, P(c_sz), P(c_sz)]
        L.btd_factorize.argtypes = [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, P(BtdStatus)]
        L.btd_check.argtypes = [c_vp, c_vp, P(BtdStatus)]
        L.btd_solve_workspace.argtypes = [c_vp, c_i64, P(c_sz)]
        L.btd_solve.argtypes = [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, P(BtdStatus)]
        L.btd_level_factor.argtypes = [c_vp, c_i64, c_vp, c_vp, c_vp, P(BtdStatus)]
        L.btd_level_schur.argtypes = [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, P(BtdStatus)]
        L.btd_profile_kernels.argtypes = [c_vp, c_i32]
        L.btd_create_partial.argtypes = [c_i64, c_i64, P(BtdConfig), c_i64, P(c_vp), P(BtdStatus)]
        L.btd_reduced_size.argtypes = [c_vp, P(c_i64)]
        L.btd_factorize_partial.argtypes = [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, P(BtdStatus)]
        L.btd_solve_down.argtypes = [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, P(BtdStatus)]
        L.btd_solve_up.argtypes = [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, P(BtdStatus)]
        L.btd_kernel_times.argtypes = [c_vp, P(ctypes.c_float), c_i64, P(c_i64)]
        L.btd_launch_count.argtypes = []
        L.btd_set_graphs.argtypes = [c_i32]
        L.btd_graph_replays.argtypes = []
        L.btd_factorize_from_host.argtypes = [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, P(BtdStatus)]
        L.btd_kalman_workspace.argtypes = [c_i64, c_i64, P(c_sz)]
        L.btd_kalman_normal_equations.argtypes = [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32,
                                                  c_vp, c_vp, c_vp, c_vp, c_vp, P(BtdStatus)]
        L.btd_matmul.argtypes = [c_vp, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, P(BtdStatus)]
        L.btd_residual_workspace.argtypes = [c_i64, c_i64, c_i64, P(c_sz)]
        L.btd_residual_norms.argtypes = [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, P(BtdStatus)]
        I64x3 = P(c_i64)
        L.btd_seam_error_bytes.argtypes = []
        L.btd_seam_error_bytes.restype = c_sz
        L.btd_seam_error_init.argtypes = [c_vp, c_vp]
        L.btd_seam_error_read.argtypes = [c_vp, c_vp, P(BtdStatus)]
        L.btd_chol_batch.argtypes = [c_vp, I64x3, c_i64, c_i64, c_i64, c_vp, c_vp, P(BtdStatus)]
        L.btd_trsm_batch.argtypes = [c_vp, I64x3, c_vp, I64x3, c_i64, c_i64, c_i64, c_i32, c_vp, c_vp, P(BtdStatus)]
        L.btd_gemm_batch.argtypes = [c_vp, I64x3, c_vp, I64x3, c_vp, I64x3, c_i64, c_i64, c_i64, c_i64, c_i32, c_i32,
                                     ctypes.c_double, ctypes.c_double, c_vp, P(BtdStatus)]
        for name in EXPORTED_SYMBOLS:
            if name not in ("btd_version", "btd_default_config", "btd_destroy", "btd_launch_count",
                            "btd_graph_replays", "btd_seam_error_bytes"):
                getattr(L, name).restype = ctypes.c_int
        L.btd_launch_count.restype = ctypes.c_longlong
        L.btd_graph_replays.restype = ctypes.c_longlong
        _lib = L
        return L
