"""B200-native block-tridiagonal SPD factor/solve (recursive Schur complement, arXiv 2509.03015).

Drop-in for the reference package's hot path (`blocktri.recursive_factorize` /
`blocktri.recursive_solve` and the containers they use).  All arithmetic runs in hand-written
sm_100a CUDA kernels behind the C ABI in include/blocktri_b200.h.
"""

from .core import (BlockRhs, BlockTridiagonalMatrix, FactorHierarchy, PartitionPlan, check_conformal,
                   new_btd, new_rhs)
from .errors import (BadMagic, BtdFormatError, IoError, TruncatedPayload, VersionUnsupported, AsymmetricBlock, BlockTriError, DeviceError, DimensionMismatch, InvalidDimensions,
                     LevelOverflow, NotPositiveDefinite, SingularDiagonal)
from .schur import (FactorLevel, RecursionConfig, level_factor, level_schur, plan_partition, recursive_factorize,
                    recursive_solve)
from .synthgen import generate_spd_btd
from .report import (SWEEPS, BenchRow, bench_sweep, btd_matmul, device_bytes, format_table, parse_sweep,
                     residual_report, time_call)
from .kalman import StateSpaceModel, build_normal_equations, generate_rotation_model
from .btdfile import read_btd, write_btd
from .core import SegmentBatch
from .kernels import (KernelBatchView, batched, chol_factor, chol_factor_batch, gemm_acc, gemm_acc_batch,
                      max_batch_threads, set_batch_threads, trsm_lower, trsm_lower_batch)
from .block_cholesky import factorize_btd_batch, serial_factorize, serial_solve, solve_btd_batch

__version__ = "0.1.0"

__all__ = [
    "StateSpaceModel", "build_normal_equations", "generate_rotation_model", "read_btd", "write_btd",
    "IoError", "BtdFormatError", "BadMagic", "VersionUnsupported", "TruncatedPayload",
    "AsymmetricBlock", "BlockRhs", "BlockTriError", "BlockTridiagonalMatrix", "DeviceError",
    "DimensionMismatch", "FactorHierarchy", "FactorLevel", "InvalidDimensions", "LevelOverflow",
    "NotPositiveDefinite", "PartitionPlan", "RecursionConfig", "SingularDiagonal", "btd_matmul",
    "check_conformal", "generate_spd_btd", "level_factor", "level_schur", "new_btd", "new_rhs", "plan_partition",
    "recursive_factorize", "recursive_solve", "residual_report",
    "SegmentBatch", "KernelBatchView", "batched", "chol_factor", "chol_factor_batch", "gemm_acc", "gemm_acc_batch",
    "max_batch_threads", "set_batch_threads", "trsm_lower", "trsm_lower_batch", "factorize_btd_batch",
    "serial_factorize", "serial_solve", "solve_btd_batch",
    "SWEEPS", "BenchRow", "bench_sweep", "device_bytes", "format_table", "parse_sweep", "time_call",
]
