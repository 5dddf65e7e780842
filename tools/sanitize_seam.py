"""Small seam-kernel workload for compute-sanitizer (memcheck / racecheck / synccheck): the shared
memory Cholesky (incl. failures past the first panel), the DMMA trsm over ragged n / column counts
and both sweeps, the DMMA GEMM over ragged and transposed shapes.   python tools/sanitize_seam.py"""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2509_03015_b200 import NotPositiveDefinite
from paper_2509_03015_b200.kernels import chol_factor_batch, gemm_acc_batch, trsm_lower_batch

rng = np.random.default_rng(0)


def spd(n):
    m = rng.standard_normal((n, n))
    return m @ m.T + n * np.eye(n)


for n in (5, 40, 128, 136):
    s = np.stack([spd(n) for _ in range(3)])
    chol_factor_batch(s)
    s[1] = spd(n)
    s[1, n // 2, n // 2] = -1.0
    try:
        chol_factor_batch(s)
    except NotPositiveDefinite as e:
        assert e.member == 1 and e.pivot == n // 2 + 1, (e.member, e.pivot)
for n, cols in ((3, 1), (57, 64), (128, 150), (120, 7)):
    f = np.stack([np.linalg.cholesky(spd(n)) for _ in range(2)])
    for trans in (False, True):
        p = rng.standard_normal((2, n, cols))
        want = np.stack([np.linalg.solve(f[k].T if trans else f[k], p[k]) for k in range(2)])
        trsm_lower_batch(f, p, trans=trans)
        assert np.abs(p - want).max() <= 1e-9 * max(1.0, np.abs(want).max())
for m, q, pp in ((1, 1, 1), (70, 33, 65), (64, 64, 64), (100, 7, 130)):
    a, b, c = rng.standard_normal((2, m, q)), rng.standard_normal((2, q, pp)), rng.standard_normal((2, m, pp))
    want = 0.5 * a @ b - c
    gemm_acc_batch(c, a, b, alpha=0.5, beta=-1.0)
    assert np.abs(c - want).max() <= 1e-12 * np.abs(want).max()
print("seam sanitize workload ok", flush=True)
