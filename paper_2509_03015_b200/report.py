"""Residual of a candidate solution (drop-in for `residual_report`, bt/report.py:20-38, and
`btd_matmul`, bt/core.py:280-288).  Device tensors are multiplied on the GPU (batched GEMM);
numpy arrays on the host."""

from __future__ import annotations

import numpy as np

from .core import BlockRhs, _is_torch, check_conformal


def btd_matmul(matrix, rhs: BlockRhs) -> BlockRhs:
    """Y = A X, one pass of the block-structured multiply (bt/core.py:280-288)."""
    check_conformal(matrix, rhs)
    x = rhs.blocks
    if _is_torch(x):
        import torch
        diag = matrix.diag if _is_torch(matrix.diag) else torch.from_numpy(matrix.diag).to(x.device)
        sub = matrix.sub if _is_torch(matrix.sub) else torch.from_numpy(matrix.sub).to(x.device)
        y = torch.bmm(diag, x)
        if matrix.num_blocks > 1:
            y[1:] += torch.bmm(sub, x[:-1])
            y[:-1] += torch.bmm(sub.transpose(1, 2), x[1:])
        return BlockRhs(y)
    y = np.matmul(matrix.diag, x)
    if matrix.num_blocks > 1:
        y[1:] += np.matmul(matrix.sub, x[:-1])
        y[:-1] += np.matmul(matrix.sub.transpose(0, 2, 1), x[1:])
    return BlockRhs(y)


def residual_report(matrix, solution: BlockRhs, rhs: BlockRhs) -> tuple[float, float]:
    """(max-over-columns ||B - AX||_2, max-over-columns ||B - AX||_2 / ||B||_2) (bt/report.py:20-38)."""
    ax = btd_matmul(matrix, solution).blocks
    b = rhs.blocks
    if _is_torch(ax):
        import torch
        if not _is_torch(b):
            b = torch.from_numpy(b).to(ax.device)
        d = b.shape[2]
        r = (b - ax).reshape(-1, d)
        rn = torch.linalg.vector_norm(r, dim=0)
        bn = torch.linalg.vector_norm(b.reshape(-1, d), dim=0)
        ratios = torch.where(bn > 0, rn / bn, torch.where(rn > 0, torch.full_like(rn, float("inf")),
                                                           torch.zeros_like(rn)))
        return float(rn.max()), float(ratios.max())
    d = b.shape[2]
    r = (b - ax).reshape(-1, d)
    rn = np.linalg.norm(r, axis=0)
    bn = np.linalg.norm(b.reshape(-1, d), axis=0)
    with np.errstate(divide="ignore", invalid="ignore"):
        ratios = np.where(bn > 0.0, rn / bn, np.where(rn > 0.0, np.inf, 0.0))
    return float(rn.max()), float(ratios.max())
