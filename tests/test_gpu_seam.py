"""The reference's kernel seam and block-Cholesky layer on the GPU (kernels.py / block_cholesky.py
drop-ins): the reference suite's known-answer tests and properties (pkg/tests/test_kernels.py,
pkg/tests/test_block_cholesky.py), run against the sm_100a seam kernels through the C ABI, with
numpy arenas (staged + written back in place) and torch CUDA arenas (in place, any strides)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2509_03015_b200 as pkg  # noqa: E402
from paper_2509_03015_b200 import BlockRhs, DimensionMismatch, NotPositiveDefinite, SingularDiagonal  # noqa: E402
from paper_2509_03015_b200.block_cholesky import (factorize_btd_batch, serial_factorize, serial_solve,  # noqa: E402
                                                  solve_btd_batch)
from paper_2509_03015_b200.core import SegmentBatch  # noqa: E402
from paper_2509_03015_b200.kernels import (KernelBatchView, batched, chol_factor, chol_factor_batch, gemm_acc,  # noqa: E402
                                           gemm_acc_batch, max_batch_threads, set_batch_threads, trsm_lower,
                                           trsm_lower_batch)
from oracle import blocktri_port as port  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def spd(n, rng):
    m = rng.standard_normal((n, n))
    return m @ m.T + n * np.eye(n)


# ---------------------------------------------------------------- chol_factor (kernels.py:164-189)
def test_chol_known_answers():
    m = np.array([[4.0]])
    chol_factor(m)
    assert np.array_equal(m, [[2.0]])
    m = np.array([[4.0, 2.0], [2.0, 5.0]])
    chol_factor(m)
    np.testing.assert_allclose(m, [[2.0, 0.0], [1.0, 2.0]], atol=1e-15)
    with pytest.raises(NotPositiveDefinite) as e:
        chol_factor(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert e.value.pivot == 2


@pytest.mark.parametrize("n", [1, 2, 7, 16, 33, 64, 100, 128, 160, 256])
def test_chol_reconstruction_and_zeroed_upper(n, rng):
    """n <= 128 factors in shared memory, larger members in place in global memory."""
    m = spd(n, rng)
    f = m.copy()
    chol_factor(f)
    assert np.array_equal(np.triu(f, 1), np.zeros((n, n)))
    assert np.abs(f @ f.T - m).max() <= 1e-13 * np.abs(m).max()


# ---------------------------------------------------------------- trsm_lower (kernels.py:215-267)
def test_trsm_known_answers(rng):
    panel = rng.standard_normal((4, 3))
    for trans in (False, True):
        got = panel.copy()
        trsm_lower(np.eye(4), got, trans=trans)
        assert np.array_equal(got, panel)
    f = np.array([[2.0, 0.0], [1.0, 2.0]])
    p = np.array([[2.0], [3.0]])
    trsm_lower(f, p)
    assert np.array_equal(p, [[1.0], [1.0]])
    with pytest.raises(SingularDiagonal) as e:
        trsm_lower(np.array([[1.0, 0.0], [3.0, 0.0]]), np.ones((2, 1)))
    assert e.value.row == 2
    with pytest.raises(DimensionMismatch):
        trsm_lower(np.eye(3), np.ones((2, 1)))


@pytest.mark.parametrize("n,d", [(3, 1), (16, 5), (57, 64), (64, 2), (96, 3), (120, 65), (128, 150), (130, 4),
                                 (200, 300)])
def test_trsm_matches_solve(n, d, rng):
    f = np.linalg.cholesky(spd(n, rng))
    p = rng.standard_normal((n, d))
    a = p.copy()
    trsm_lower(f, a)
    np.testing.assert_allclose(a, np.linalg.solve(f, p), rtol=0, atol=1e-11)
    b = p.copy()
    trsm_lower(f, b, trans=True)
    np.testing.assert_allclose(b, np.linalg.solve(f.T, p), rtol=0, atol=1e-11)


# ---------------------------------------------------------------- gemm_acc (kernels.py:270-318)
def test_gemm_known_answers(rng):
    c = rng.standard_normal((3, 3))
    before = c.copy()
    gemm_acc(c, rng.standard_normal((3, 4)), rng.standard_normal((4, 3)), alpha=0.0, beta=1.0)
    assert np.array_equal(c, before)
    c = np.full((3, 3), np.nan)
    gemm_acc(c, np.eye(3), np.eye(3), alpha=1.0, beta=0.0)  # beta = 0 ignores out (NaN included)
    assert np.array_equal(c, np.eye(3))
    a, b = rng.standard_normal((4, 3)), rng.standard_normal((4, 5))
    c0 = rng.standard_normal((3, 5))
    c = c0.copy()
    gemm_acc(c, a, b, trans_a=True, alpha=2.5, beta=-0.5)
    np.testing.assert_allclose(c, 2.5 * a.T @ b - 0.5 * c0, atol=1e-13)
    p, q = rng.standard_normal((5, 3)), rng.standard_normal((4, 5))
    c = np.zeros((3, 4))
    gemm_acc(c, p, q, trans_a=True, trans_b=True)
    np.testing.assert_allclose(c, (q @ p).T, atol=1e-13)
    with pytest.raises(DimensionMismatch):
        gemm_acc(np.zeros((2, 2)), np.ones((2, 3)), np.ones((2, 3)))


@pytest.mark.parametrize("m,q,p", [(1, 1, 1), (33, 70, 65), (64, 64, 64), (100, 7, 130)])
def test_gemm_shapes(m, q, p, rng):
    a, b = rng.standard_normal((3, m, q)), rng.standard_normal((3, q, p))
    c = rng.standard_normal((3, m, p))
    want = 0.75 * a @ b + 1.25 * c
    gemm_acc_batch(c, a, b, alpha=0.75, beta=1.25)
    np.testing.assert_allclose(c, want, rtol=0, atol=1e-12 * np.abs(want).max())


# ---------------------------------------------------------------- batches (kernels.py:72-133, 321-338)
def test_batch_equals_single_bitwise(rng):
    m = spd(6, rng)
    single = m.copy()
    chol_factor(single)
    stacked = m[None].copy()
    chol_factor_batch(stacked)
    assert np.array_equal(stacked[0], single)
    a, b, c = rng.standard_normal((16, 4, 3)), rng.standard_normal((16, 3, 5)), rng.standard_normal((16, 4, 5))
    looped = c.copy()
    for k in range(16):
        gemm_acc(looped[k], a[k], b[k], alpha=1.5, beta=0.25)
    out = c.copy()
    gemm_acc_batch(out, a, b, alpha=1.5, beta=0.25)
    assert np.array_equal(out, looped)
    fs = np.stack([np.linalg.cholesky(spd(6, rng)) for _ in range(9)])
    ps = rng.standard_normal((9, 6, 2))
    looped = ps.copy()
    for k in range(9):
        trsm_lower(fs[k], looped[k])
    out = ps.copy()
    trsm_lower_batch(fs, out)
    assert np.array_equal(out, looped)


def test_batch_failures_report_lowest_member(rng):
    stack = np.stack([spd(3, rng) for _ in range(5)])
    stack[3] = [[1.0, 2.0, 0.0], [2.0, 1.0, 0.0], [0.0, 0.0, 1.0]]
    stack[4] = -np.eye(3)
    with pytest.raises(NotPositiveDefinite) as e:
        chol_factor_batch(stack)
    assert (e.value.member, e.value.pivot) == (3, 2)
    factors = np.broadcast_to(np.eye(2), (4, 2, 2)).copy()
    factors[2, 1, 1] = 0.0
    factors[3, 0, 0] = 0.0
    panels = np.ones((4, 2, 1))
    with pytest.raises(SingularDiagonal) as e:
        trsm_lower_batch(factors, panels)
    assert e.value.member == 2 and e.value.row == 2
    assert np.array_equal(panels, np.ones((4, 2, 1)))  # nothing solved


@pytest.mark.parametrize("n,k", [(40, 20), (128, 100), (100, 7), (200, 150)])
def test_failure_pivot_past_the_first_panel(n, k, rng):
    """The shared-memory kernel factors in 8-column panels: the failing pivot is still the first
    non-positive one, 1-based, and the lowest failing member wins (member 1 fails later in the
    elimination than member 2)."""
    stack = np.stack([spd(n, rng) for _ in range(3)])
    stack[1, k, k] = -1.0
    stack[2, 2, 2] = -1.0
    with pytest.raises(NotPositiveDefinite) as e:
        chol_factor_batch(stack)
    assert (e.value.member, e.value.pivot) == (1, k + 1)


def test_thread_cap_is_an_api_knob_only(rng, monkeypatch):
    stack = np.stack([spd(4, rng) for _ in range(512)])
    stack[400] = -np.eye(4)
    for cap in (1, 4):
        set_batch_threads(cap)
        try:
            assert max_batch_threads() == cap
            with pytest.raises(NotPositiveDefinite) as e:
                chol_factor_batch(stack.copy())
            assert e.value.member == 400
        finally:
            set_batch_threads(None)
    monkeypatch.setenv("BLOCKTRI_THREADS", "3")
    assert max_batch_threads() == 3


def test_generic_dispatch_and_views(rng):
    stack = np.stack([spd(3, rng) for _ in range(4)])
    view = KernelBatchView(stack.copy())
    batched(chol_factor, view)
    ref = stack.copy()
    chol_factor_batch(ref)
    assert np.array_equal(view.arena, ref)
    with pytest.raises(ValueError):
        batched(sum, stack)
    arena = rng.standard_normal((4, 4))
    overlapping = np.lib.stride_tricks.as_strided(arena, shape=(3, 2, 4), strides=(arena.strides[0],) + arena.strides)
    with pytest.raises(ValueError):
        KernelBatchView(overlapping)


def test_device_tensors_in_place_through_transposed_views(rng):
    """torch CUDA arenas are solved in place with their own strides (the transposed coupling view of
    block_cholesky.py:32)."""
    f = np.stack([np.linalg.cholesky(spd(8, rng)) for _ in range(5)])
    c = rng.standard_normal((5, 8, 8))
    want = np.stack([c[k] @ np.linalg.inv(f[k]).T for k in range(5)])  # C L^{-T}
    dc = torch.from_numpy(c).cuda()
    trsm_lower_batch(torch.from_numpy(f).cuda(), dc.transpose(1, 2))
    np.testing.assert_allclose(dc.cpu().numpy(), want, rtol=0, atol=1e-12)


# ---------------------------------------------------------------- block_cholesky.py:24-98
def _batch(systems):
    n = systems[0].block_size
    lengths = np.array([m.num_blocks for m in systems])
    J = int(lengths.max())
    diag = np.broadcast_to(np.eye(n), (len(systems), J, n, n)).copy()
    sub = np.zeros((len(systems), max(J - 1, 0), n, n))
    for k, m in enumerate(systems):
        diag[k, :m.num_blocks] = m.diag
        sub[k, :m.num_blocks - 1] = m.sub
    z = np.zeros((len(systems), n, n))
    return SegmentBatch(n, lengths, diag, sub, z.copy(), z.copy())


def test_serial_factorize_known_answers():
    m = pkg.new_btd(2, 1, [[[4.0]], [[5.0]]], [[[2.0]]])
    w = m.copy()
    serial_factorize(w)
    assert (w.diag[0, 0, 0], w.sub[0, 0, 0], w.diag[1, 0, 0]) == (2.0, 1.0, 2.0)
    x = BlockRhs(np.array([6.0, 7.0]).reshape(2, 1, 1))
    serial_solve(w, x)
    np.testing.assert_allclose(x.blocks.ravel(), [1.0, 1.0], atol=1e-15)
    m, _ = pkg.generate_spd_btd(6, 2, seed=4)
    m.diag[3] = -m.diag[3]
    with pytest.raises(NotPositiveDefinite) as e:
        serial_factorize(m)
    assert (e.value.block, e.value.member, e.value.pivot) == (3, 0, 1)


@pytest.mark.parametrize("count,n,d", [(1, 1, 1), (5, 1, 2), (17, 4, 3), (64, 16, 2), (40, 7, 1), (300, 64, 1),
                                       (20, 130, 2)])
def test_serial_solve_residual(count, n, d):
    m, b = pkg.generate_spd_btd(count, n, d, seed=count * 31 + n)
    w = m.copy()
    serial_factorize(w)
    x = b.copy()
    serial_solve(w, x)
    dense = port.assemble_dense(m.diag, m.sub)
    r = dense @ x.blocks.reshape(-1, d) - b.blocks.reshape(-1, d)
    assert np.linalg.norm(r) <= 1e-12 * np.linalg.norm(b.blocks)
    lower = np.zeros_like(dense)  # block L L^T reconstruction
    for i in range(count):
        lower[i * n:(i + 1) * n, i * n:(i + 1) * n] = w.diag[i]
        if i:
            lower[i * n:(i + 1) * n, (i - 1) * n:i * n] = w.sub[i - 1]
    assert np.abs(lower @ lower.T - dense).max() <= 1e-12 * np.abs(dense).max()


def test_segment_batch_ragged_and_failure(rng):
    lengths = [7, 7, 3, 7, 1]
    systems = [pkg.generate_spd_btd(j, 2, seed=50 + i)[0] for i, j in enumerate(lengths)]
    rhs = [np.random.default_rng(90 + i).standard_normal((j, 2, 3)) for i, j in enumerate(lengths)]
    batch = _batch(systems)
    with pytest.raises(ValueError):
        solve_btd_batch(batch, np.zeros((5, 7, 2, 3)))
    factorize_btd_batch(batch)
    with pytest.raises(DimensionMismatch):
        solve_btd_batch(batch, np.zeros((5, 7, 3, 3)))
    stacked = np.zeros((5, 7, 2, 3))
    for k, r in enumerate(rhs):
        stacked[k, :lengths[k]] = r
    solve_btd_batch(batch, stacked)
    for k, (m, r) in enumerate(zip(systems, rhs)):
        w = m.copy()
        serial_factorize(w)
        x = BlockRhs(r.copy())
        serial_solve(w, x)
        assert np.abs(stacked[k, :lengths[k]] - x.blocks).max() <= 1e-14 * max(np.abs(x.blocks).max(), 1.0)
        assert not stacked[k, lengths[k]:].any()  # padded rows stay exactly zero
    systems = [pkg.generate_spd_btd(4, 2, seed=s)[0] for s in range(3)]
    systems[1].diag[2] = -systems[1].diag[2]
    systems[2].diag[1] = -systems[2].diag[1]
    with pytest.raises(NotPositiveDefinite) as e:
        factorize_btd_batch(_batch(systems))
    assert (e.value.member, e.value.block) == (2, 1)  # earliest step first, then lowest member
