"""Residual of a candidate solution (drop-in for `residual_report`, bt/report.py:20-38, and
`btd_matmul`, bt/core.py:280-288).

CUDA tensors go through the sm_100a block-SpMV / fused-residual kernels of the C ABI
(btd_matmul, btd_residual_norms: one HBM pass over A, deterministic norm reduction); numpy arrays
are multiplied on the host like the reference (this is harness code, not the factor/solve path).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .core import BlockRhs, _is_torch, check_conformal


def _device_operands(matrix, x):
    import torch
    dev = x.device
    diag = matrix.diag if _is_torch(matrix.diag) else torch.from_numpy(matrix.diag)
    sub = matrix.sub if _is_torch(matrix.sub) else torch.from_numpy(matrix.sub)
    diag = diag.to(dev, torch.float64).contiguous()
    sub = sub.to(dev, torch.float64).contiguous()
    return diag, sub, x.to(torch.float64).contiguous()


def _raise(rc: int, st) -> None:
    if rc != _native.BTD_OK:
        raise RuntimeError(st.message.decode(errors="replace"))


def btd_matmul(matrix, rhs: BlockRhs) -> BlockRhs:
    """Y = A X, one pass of the block-structured multiply (bt/core.py:280-288)."""
    check_conformal(matrix, rhs)
    x = rhs.blocks
    if _is_torch(x) and x.is_cuda:
        import torch
        diag, sub, xx = _device_operands(matrix, x)
        N, n, d = xx.shape
        y = torch.empty_like(xx)
        st = _native.BtdStatus()
        rc = _native.lib().btd_matmul(diag.data_ptr(), sub.data_ptr() if N > 1 else None, N, n, xx.data_ptr(), d,
                                      y.data_ptr(), ctypes.c_void_p(torch.cuda.current_stream(xx.device).cuda_stream),
                                      ctypes.byref(st))
        _raise(rc, st)
        return BlockRhs(y)
    if _is_torch(x):
        x = x.numpy()
        matrix = type(matrix)(*(m.numpy() if _is_torch(m) else m for m in (matrix.diag, matrix.sub)))
    y = np.matmul(matrix.diag, x)
    if matrix.num_blocks > 1:
        y[1:] += np.matmul(matrix.sub, x[:-1])
        y[:-1] += np.matmul(matrix.sub.transpose(0, 2, 1), x[1:])
    return BlockRhs(y)


def residual_report(matrix, solution: BlockRhs, rhs: BlockRhs) -> tuple[float, float]:
    """(max-over-columns ||B - AX||_2, max-over-columns ||B - AX||_2 / ||B||_2) (bt/report.py:20-38)."""
    x = solution.blocks
    if _is_torch(x) and x.is_cuda:
        import torch
        check_conformal(matrix, solution)
        diag, sub, xx = _device_operands(matrix, x)
        b = rhs.blocks if _is_torch(rhs.blocks) else torch.from_numpy(rhs.blocks)
        b = b.to(xx.device, torch.float64).contiguous()
        N, n, d = xx.shape
        L = _native.lib()
        ws = ctypes.c_size_t()
        L.btd_residual_workspace(N, n, d, ctypes.byref(ws))
        work = torch.empty(max(ws.value // 8, 1), dtype=torch.float64, device=xx.device)
        norms2 = torch.empty(2 * d, dtype=torch.float64, device=xx.device)
        st = _native.BtdStatus()
        rc = L.btd_residual_norms(diag.data_ptr(), sub.data_ptr() if N > 1 else None, N, n, xx.data_ptr(),
                                  b.data_ptr(), d, work.data_ptr(), norms2.data_ptr(),
                                  ctypes.c_void_p(torch.cuda.current_stream(xx.device).cuda_stream), ctypes.byref(st))
        _raise(rc, st)
        h = norms2.cpu().numpy()
        rn, bn = np.sqrt(h[:d]), np.sqrt(h[d:])
        with np.errstate(divide="ignore", invalid="ignore"):
            ratios = np.where(bn > 0.0, rn / bn, np.where(rn > 0.0, np.inf, 0.0))
        return float(rn.max()), float(ratios.max())
    ax = btd_matmul(matrix, solution).blocks
    b = rhs.blocks
    if _is_torch(ax):
        ax = ax.numpy()
    if _is_torch(b):
        b = b.cpu().numpy()
    d = b.shape[2]
    r = (b - ax).reshape(-1, d)
    rn = np.linalg.norm(r, axis=0)
    bn = np.linalg.norm(b.reshape(-1, d), axis=0)
    with np.errstate(divide="ignore", invalid="ignore"):
        ratios = np.where(bn > 0.0, rn / bn, np.where(rn > 0.0, np.inf, 0.0))
    return float(rn.max()), float(ratios.max())


# ------------------------------------------------------------------------------------------------
# Benchmark report (drop-in for the table half of bt/report.py:12-17, 41-110): the same sweeps,
# rows and CSV / markdown tables, with device timing (CUDA events on the current stream) for the
# B200 engine.  SURVEY.md §8(f) row 4 (bench front-end).
# ------------------------------------------------------------------------------------------------
import time
from dataclasses import dataclass

#: (N, n) pairs of the standard sweeps, keyed by total dimension (bt/report.py:12-17).
SWEEPS = {
    "nn262144": [(256, 1024), (512, 512), (1024, 256),
                 (2048, 128), (4096, 64), (8192, 32)],
    "nn65536": [(2048, 32), (1024, 64), (512, 128), (256, 256)],
}


def time_call(fn, runs: int = 1, warmup: int = 0, device: bool = False) -> tuple[float, object]:
    """Mean milliseconds of ``fn()`` over ``runs`` timed calls after ``warmup`` untimed ones
    (bt/report.py:41-55).  ``device=True`` times on the GPU: CUDA events recorded on the current
    stream around each call, synchronised before reading (kernel time, no host overhead hidden
    by queueing).  Returns the mean and the result of the last call."""
    result = None
    for _ in range(warmup):
        result = fn()
    total = 0.0
    if device:
        import torch
        for _ in range(runs):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            result = fn()
            e1.record()
            torch.cuda.synchronize()
            total += e0.elapsed_time(e1) / 1000.0
    else:
        for _ in range(runs):
            start = time.perf_counter()
            result = fn()
            total += time.perf_counter() - start
    return 1000.0 * total / max(runs, 1), result


@dataclass
class BenchRow:
    """One row of the Table-1-shaped report (bt/report.py:58-64)."""

    num_blocks: int
    block_size: int
    factor_ms: float
    solve_ms: float
    rel_residual: float


_COLUMNS = ("N", "n", "fact_ms", "solve_ms", "rel_residual")


def _cells(row: BenchRow) -> list[str]:
    return [str(row.num_blocks), str(row.block_size),
            f"{row.factor_ms:.2f}", f"{row.solve_ms:.2f}",
            f"{row.rel_residual:.3e}"]


def format_table(rows: list[BenchRow], fmt: str = "md") -> str:
    """Render benchmark rows as CSV or a markdown table (bt/report.py:74-91, same text)."""
    if fmt == "csv":
        return "\n".join([",".join(_COLUMNS)] + [",".join(_cells(r)) for r in rows])
    if fmt == "md":
        widths = [max(len(h), 12) for h in _COLUMNS]
        lines = ["| " + " | ".join(h.ljust(w) for h, w in zip(_COLUMNS, widths)) + " |",
                 "|" + "|".join("-" * (w + 2) for w in widths) + "|"]
        lines += ["| " + " | ".join(c.ljust(w) for c, w in zip(_cells(r), widths)) + " |" for r in rows]
        return "\n".join(lines)
    raise ValueError(f"unknown table format {fmt!r}")


def parse_sweep(spec: str) -> list[tuple[int, int]]:
    """Parse a sweep name or an explicit ``N:n,N:n,...`` list (bt/report.py:94-110)."""
    if spec in SWEEPS:
        return list(SWEEPS[spec])
    shapes = []
    for part in spec.split(","):
        try:
            num_blocks, block_size = part.split(":")
            shapes.append((int(num_blocks), int(block_size)))
        except ValueError:
            raise ValueError(f"bad sweep {spec!r}: expected one of {sorted(SWEEPS)} or 'N:n,N:n,...'") from None
    if not shapes:
        raise ValueError("empty sweep specification")
    return shapes


def device_bytes(num_blocks: int, block_size: int, num_columns: int = 1, config=None) -> int:
    """Device memory of one factor + solve on this engine (counterpart of the reference's
    ``estimate_bytes`` host estimate, bt/report.py:113-124): the input arenas, the hierarchy, the
    factor scratch and the solve workspace, from the C-ABI workspace queries (no GPU needed)."""
    from .schur import RecursionConfig
    cfg = (config or RecursionConfig())._c()
    L = _native.lib()
    st = _native.BtdStatus()
    h = ctypes.c_void_p()
    rc = L.btd_create(int(num_blocks), int(block_size), ctypes.byref(cfg), ctypes.byref(h), ctypes.byref(st))
    if rc != _native.BTD_OK:
        _raise(rc, st)
    try:
        pb, sb, vb = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        L.btd_factor_workspace(h, ctypes.byref(pb), ctypes.byref(sb))
        L.btd_solve_workspace(h, int(num_columns), ctypes.byref(vb))
    finally:
        L.btd_destroy(h)
    bb = 8 * block_size * block_size
    arenas = (2 * num_blocks - 1) * bb + 2 * 8 * num_blocks * block_size * num_columns  # A, B, X
    return int(arenas + pb.value + max(sb.value, vb.value))


def bench_sweep(shapes, num_columns: int = 1, runs: int = 3, warmup: int = 2, seed: int = 0,
                config=None) -> list[BenchRow]:
    """The reference's ``bench`` sweep (bt/cli.py:151-186) on the GPU: for every (N, n), the seeded
    reference instance is generated, moved to the device, and factor / solve are timed with CUDA
    events (mean of ``runs`` after ``warmup``; two warm-ups by default, because repeated
    factorizations alternate between two workspace address sets and each set's first call captures
    its CUDA graph); the residual comes from the fused GPU kernel."""
    import torch
    from .core import BlockTridiagonalMatrix
    from .schur import recursive_factorize, recursive_solve
    from .synthgen import generate_spd_btd
    rows = []
    for N, n in shapes:
        A, B = generate_spd_btd(N, n, num_columns, seed=seed)
        dA = BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
        dB = BlockRhs(torch.from_numpy(B.blocks).cuda())
        f_ms, h = time_call(lambda: recursive_factorize(dA, config), runs=runs, warmup=warmup, device=True)
        s_ms, X = time_call(lambda: recursive_solve(h, dB), runs=runs, warmup=warmup, device=True)
        _, rel = residual_report(dA, X, dB)
        rows.append(BenchRow(N, n, f_ms, s_ms, rel))
    return rows
