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


def generate_spd_btd_slice(num_blocks: int, block_size: int, num_columns: int, seed: int, first: int, last: int,
                           chunk: int = 4096, out=None):
    """Rows [first, last] (inclusive) of ``generate_spd_btd(num_blocks, ..., seed)``, bit-identical,
    without generating the rest of the matrix: returns (diag[first:last+1], sub[first:last],
    rhs[first:last+1]).

    The uniform draws consume exactly one PCG64 output per double, so the sub / raw streams are
    entered with ``bit_generator.advance``; the normal draws (ziggurat, variable consumption) are
    replayed from the start of the rhs stream up to ``last``.  Each rank of the sharded benchmark
    slices its chunk of the ONE global instance this way.
    ``out`` = optional preallocated (diag, sub, rhs) arrays of the slice shapes.
    """
    N, n, d = num_blocks, block_size, num_columns
    if not 0 <= first <= last < N:
        raise ValueError(f"slice [{first}, {last}] outside [0, {N})")
    nn = n * n
    m = last - first + 1
    if out is None:
        diag = np.empty((m, n, n))
        sub = np.empty((m - 1, n, n))
        rhs = np.empty((m, n, d))
    else:
        diag, sub, rhs = out
    # sub rows touching the slice's diagonal row sums: [first-1, last] clipped to [0, N-2]
    s_lo, s_hi = max(first - 1, 0), min(last, N - 2)
    subx = np.empty((max(s_hi - s_lo + 1, 0), n, n))
    rng = np.random.default_rng(seed)
    rng.bit_generator.advance(s_lo * nn)
    for a in range(0, subx.shape[0], chunk):
        b = min(a + chunk, subx.shape[0])
        subx[a:b] = rng.uniform(-1.0, 1.0, (b - a, n, n))
    if m > 1:
        sub[:] = subx[first - s_lo:first - s_lo + m - 1]
    rng = np.random.default_rng(seed)
    rng.bit_generator.advance((N - 1) * nn + first * nn)
    eye = np.eye(n)
    for a in range(0, m, chunk):
        b = min(a + chunk, m)
        raw = rng.uniform(-1.0, 1.0, (b - a, n, n))
        sym = (raw + raw.transpose(0, 2, 1)) / 2.0
        rs = np.abs(sym).sum(axis=2)
        g0, g1 = first + a, first + b  # global rows [g0, g1)
        lo = max(g0, 1)
        if g1 > lo:  # |sub[i-1]| row sums for rows i >= 1
            rs[lo - g0:] += np.abs(subx[lo - 1 - s_lo:g1 - 1 - s_lo]).sum(axis=2)
        hi = min(g1, N - 1)
        if hi > g0:  # |sub[i]| column sums for rows i <= N-2
            rs[:hi - g0] += np.abs(subx[g0 - s_lo:hi - s_lo]).sum(axis=1)
        diag[a:b] = sym + (1.0 + rs.max(axis=1))[:, None, None] * eye
    rng = np.random.default_rng(seed)
    rng.bit_generator.advance((N - 1) * nn + N * nn)
    for a in range(0, last + 1, chunk):
        b = min(a + chunk, last + 1)
        r = rng.standard_normal((b - a, n, d))
        lo, hi = max(a, first), b
        if hi > lo:
            rhs[lo - first:hi - first] = r[lo - a:hi - a]
    return diag, sub, rhs
