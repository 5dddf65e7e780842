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
