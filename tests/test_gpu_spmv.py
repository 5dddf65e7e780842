"""GPU block SpMV and fused residual: btd_matmul (bt/core.py:280-288) and
residual_report (bt/report.py:20-38) on device tensors, through the C ABI kernels, against the
numpy restatement of the same products."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import paper_2509_03015_b200 as pkg  # noqa: E402
from paper_2509_03015_b200 import report  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _np_matmul(diag, sub, x):
    y = np.matmul(diag, x)
    if diag.shape[0] > 1:
        y[1:] += np.matmul(sub, x[:-1])
        y[:-1] += np.matmul(sub.transpose(0, 2, 1), x[1:])
    return y


@pytest.mark.parametrize("N,n,d", [(1, 5, 1), (2, 3, 2), (7, 8, 1), (100, 17, 3), (33, 64, 9), (9, 256, 20),
                                   (1000, 32, 1)])
def test_matmul_matches_numpy(N, n, d):
    rng = np.random.default_rng(N * 1000 + n * 10 + d)
    diag = rng.standard_normal((N, n, n))
    sub = rng.standard_normal((max(N - 1, 0), n, n))
    x = rng.standard_normal((N, n, d))
    A = pkg.BlockTridiagonalMatrix(torch.from_numpy(diag).cuda(), torch.from_numpy(sub).cuda())
    y = report.btd_matmul(A, pkg.BlockRhs(torch.from_numpy(x).cuda())).blocks.cpu().numpy()
    ref = _np_matmul(diag, sub, x)
    assert np.abs(y - ref).max() <= 1e-12 * max(np.abs(ref).max(), 1.0)


@pytest.mark.parametrize("N,n,d", [(1, 4, 1), (500, 16, 2), (2000, 64, 1), (64, 256, 11)])
def test_residual_matches_numpy(N, n, d):
    A, B = pkg.generate_spd_btd(N, n, d, seed=3)
    rng = np.random.default_rng(7)
    X = rng.standard_normal((N, n, d))
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
    g_abs, g_rel = pkg.residual_report(dA, pkg.BlockRhs(torch.from_numpy(X).cuda()), pkg.BlockRhs(torch.from_numpy(B.blocks).cuda()))
    c_abs, c_rel = pkg.residual_report(A, pkg.BlockRhs(X), B)
    assert abs(g_abs - c_abs) <= 1e-12 * c_abs
    assert abs(g_rel - c_rel) <= 1e-12 * c_rel


def test_residual_deterministic_and_small_after_solve():
    A, B = pkg.generate_spd_btd(4096, 64, 2, seed=0)
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
    dB = pkg.BlockRhs(torch.from_numpy(B.blocks).cuda())
    X = pkg.recursive_solve(pkg.recursive_factorize(dA), dB)
    r1 = pkg.residual_report(dA, X, dB)
    r2 = pkg.residual_report(dA, X, dB)
    assert r1 == r2  # fixed reduction order: bitwise repeatable
    assert r1[1] <= 1e-12
