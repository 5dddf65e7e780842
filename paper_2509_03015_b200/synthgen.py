"""Seeded SPD block-tridiagonal instances (input definition of the benchmarks).

Bit-identical to the reference generator `generate_spd_btd` (bt/synthgen.py:10-39) -- same
`np.random.default_rng(seed)` draw order (sub, raw, rhs) -- but produced in block chunks so that
N = 2^20 instances do not need ~200 GB of temporaries.  This is harness
code, not the solver: it defines the synthetic inputs the reference and this engine both consume.
"""

from __future__ import annotations

import numpy as np

from .core import BlockRhs, BlockTridiagonalMatrix


def generate_spd_btd(num_blocks: int, block_size: int, num_columns: int = 1, seed: int = 0,
                     chunk: int = 4096, out=None):
    """Return (BlockTridiagonalMatrix, BlockRhs) with numpy arenas (or fill ``out`` arrays).

    ``out`` = optional (diag, sub, rhs) preallocated arrays (e.g. pinned host tensors' numpy views).
    """
    if num_blocks < 1 or block_size < 1 or num_columns < 1:
        raise ValueError("num_blocks, block_size and num_columns must be >= 1")
    N, n, d = num_blocks, block_size, num_columns
    rng = np.random.default_rng(seed)
    if out is None:
        diag = np.empty((N, n, n))
        sub = np.empty((max(N - 1, 0), n, n))
        rhs = np.empty((N, n, d))
    else:
        diag, sub, rhs = out
    # 1. sub ~ U[-1, 1], drawn chunk by chunk (same stream as one big draw)
    for a in range(0, N - 1, chunk):
        b = min(a + chunk, N - 1)
        sub[a:b] = rng.uniform(-1.0, 1.0, (b - a, n, n))
    # 2. raw ~ U[-1, 1]; 3. D = sym(raw) + (1 + max row-abs-sum incl. couplings) I
    eye = np.eye(n)
    for a in range(0, N, chunk):
        b = min(a + chunk, N)
        raw = rng.uniform(-1.0, 1.0, (b - a, n, n))
        sym = (raw + raw.transpose(0, 2, 1)) / 2.0
        rs = np.abs(sym).sum(axis=2)
        lo = max(a, 1)
        if b > lo:
            rs[lo - a:] += np.abs(sub[lo - 1:b - 1]).sum(axis=2)
        hi = min(b, N - 1)
        if hi > a:
            rs[:hi - a] += np.abs(sub[a:hi]).sum(axis=1)
        shift = 1.0 + rs.max(axis=1)
        diag[a:b] = sym + shift[:, None, None] * eye
    # 4. rhs ~ N(0, 1)
    for a in range(0, N, chunk):
        b = min(a + chunk, N)
        rhs[a:b] = rng.standard_normal((b - a, n, d))
    return BlockTridiagonalMatrix(diag, sub), BlockRhs(rhs)
