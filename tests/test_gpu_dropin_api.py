"""The reference's own public-API tests of the hot path, restated against the drop-in (GPU):
TestRecursiveFactorize / TestRecursiveSolve (pkg/tests/test_schur.py:255-382) and acceptance
criteria 1, 2, 3 and 9 (pkg/tests/test_acceptance.py:43-126, 233-258), with the reference names
imported from this package instead of `blocktri`.  The dense oracle is numpy (np.linalg.solve on
the assembled matrix); the serial path is the drop-in's own block_cholesky."""

import os
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_03015_b200 import (BlockRhs, LevelOverflow, NotPositiveDefinite, RecursionConfig,  # noqa: E402
                                   generate_spd_btd, level_schur, new_btd, plan_partition, recursive_factorize,
                                   recursive_solve, residual_report)
from paper_2509_03015_b200.block_cholesky import serial_factorize, serial_solve  # noqa: E402
from oracle.blocktri_port import assemble_dense  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def dense(m):
    return assemble_dense(np.asarray(m.diag), np.asarray(m.sub))


def dense_solve(m, b):
    return np.linalg.solve(dense(m), b.reshape(m.num_blocks * m.block_size, -1))


# ------------------------------------------------------------------ TestRecursiveFactorize
def test_base_case_has_zero_levels():
    m, _ = generate_spd_btd(10, 2, seed=0)
    h = recursive_factorize(m, RecursionConfig(crossover=64))
    assert h.levels == [] and h.base.num_blocks == 10


def test_level_sizes_strictly_decrease_and_count_bound():
    m, _ = generate_spd_btd(9, 1, seed=1)
    cfg = RecursionConfig(crossover=2, segment_length=3)
    h = recursive_factorize(m, cfg)
    sizes = [lv.plan.num_blocks for lv in h.levels] + [h.base.num_blocks]
    assert sizes[0] == 9 and all(b < a for a, b in zip(sizes, sizes[1:]))
    assert h.base.num_blocks <= max(cfg.crossover, 2)
    m, _ = generate_spd_btd(256, 1, seed=2)
    cfg = RecursionConfig(crossover=4, segment_length=3)
    h = recursive_factorize(m, cfg)
    assert len(h.levels) <= int(np.ceil(np.log(256 / 4) / np.log(4))) + 1


def test_every_schur_complement_is_spd():
    m, _ = generate_spd_btd(64, 2, seed=3)
    cfg = RecursionConfig(crossover=4, segment_length=3)
    h = recursive_factorize(m, cfg)
    assert len(h.levels) >= 2
    for lvl in range(len(h.levels)):
        d, s = level_schur(m, lvl, cfg)
        np.linalg.cholesky(assemble_dense(d.cpu().numpy(), s.cpu().numpy()))  # raises if not SPD


def test_auto_crossover_and_overflow():
    m, _ = generate_spd_btd(100, 1, seed=4)
    cfg = RecursionConfig(segment_length=4, auto_crossover=True)
    h = recursive_factorize(m, cfg)
    assert len(h.levels) >= 1
    nb = h.base.num_blocks
    assert nb < 3 or plan_partition(nb, cfg).num_segments < 2
    m, _ = generate_spd_btd(200, 1, seed=5)
    with pytest.raises(LevelOverflow):
        recursive_factorize(m, RecursionConfig(crossover=2, segment_length=1, max_levels=2))


def test_not_positive_definite_carries_level():
    m, _ = generate_spd_btd(40, 2, seed=6)
    m.diag[7] = -m.diag[7]
    with pytest.raises(NotPositiveDefinite) as e:
        recursive_factorize(m, RecursionConfig(crossover=4, segment_length=4))
    assert e.value.level == 0 and e.value.member is not None and e.value.block is not None


# ------------------------------------------------------------------ TestRecursiveSolve
def test_identity_hierarchy(rng):
    count, n = 40, 2
    m = new_btd(count, n, np.broadcast_to(np.eye(n), (count, n, n)), np.zeros((count - 1, n, n)))
    h = recursive_factorize(m, RecursionConfig(crossover=8, segment_length=3))
    b = BlockRhs(rng.standard_normal((count, n, 3)))
    np.testing.assert_allclose(recursive_solve(h, b).blocks, b.blocks, atol=1e-15)


def test_scalar_chain_matches_dense():
    chain = new_btd(3, 1, [[[4.0]], [[4.0]], [[4.0]]], [[[1.0]], [[1.0]]])
    h = recursive_factorize(chain, RecursionConfig(crossover=2, segment_length=1))
    assert len(h.levels) == 1
    x = recursive_solve(h, BlockRhs(np.ones((3, 1, 1))))
    assert np.abs(x.blocks.ravel() - dense_solve(chain, np.ones(3)).ravel()).max() <= 1e-14


@pytest.mark.parametrize("count,n,d,crossover,rho", [(256, 2, 4, 8, 3), (100, 8, 2, 16, 8), (37, 3, 1, 4, 2),
                                                     (64, 1, 1, 4, 5), (250, 4, 2, 32, 8), (128, 4, 3, 8, 4)])
def test_recursive_equals_serial_and_dense(count, n, d, crossover, rho):
    m, b = generate_spd_btd(count, n, d, seed=count + n)
    x_rec = recursive_solve(recursive_factorize(m, RecursionConfig(crossover=crossover, segment_length=rho)), b)
    w = m.copy()
    serial_factorize(w)
    x_ser = b.copy()
    serial_solve(w, x_ser)
    assert np.abs(x_rec.blocks - x_ser.blocks).max() <= 1e-11 * np.abs(x_ser.blocks).max()
    want = dense_solve(m, b.blocks)
    assert np.abs(x_rec.blocks.reshape(count * n, d) - want).max() <= 1e-11 * np.abs(want).max()


def test_repeated_solves_independent_and_rhs_not_mutated(rng):
    m, _ = generate_spd_btd(60, 3, seed=8)
    h = recursive_factorize(m, RecursionConfig(crossover=8, segment_length=4))
    b1 = BlockRhs(rng.standard_normal((60, 3, 2)))
    b2 = BlockRhs(rng.standard_normal((60, 3, 2)))
    before = b1.blocks.copy()
    x1 = recursive_solve(h, b1)
    recursive_solve(h, b2)
    assert np.array_equal(x1.blocks, recursive_solve(h, b1).blocks)
    assert np.array_equal(b1.blocks, before)


# ------------------------------------------------------------------ acceptance criteria
_N_LADDER = [2, 3, 4, 5, 6, 7, 8, 10, 12, 14, 16, 20, 24, 28, 32, 40, 48, 56, 64, 80, 96, 112, 128, 160, 192, 224,
             256]
_CONFIGS = [RecursionConfig(crossover=4, segment_length=2), RecursionConfig(crossover=8, segment_length=3),
            RecursionConfig(crossover=16, segment_length=8), RecursionConfig()]


@pytest.fixture(scope="module")
def solved_200():
    out = []
    t0 = time.perf_counter()
    for i in range(200):
        count, n = _N_LADDER[i % 27], [1, 2, 3, 4, 8][(i // 27) % 5]
        d, cfg = (1 if i % 2 == 0 else 3), _CONFIGS[i % 4]
        m, b = generate_spd_btd(count, n, d, seed=i)
        x_rec = recursive_solve(recursive_factorize(m, cfg), b)
        w = m.copy()
        serial_factorize(w)
        x_ser = b.copy()
        serial_solve(w, x_ser)
        out.append((i, m, b, x_rec, x_ser))
    return out, time.perf_counter() - t0


def test_criterion_01_oracle_equivalence(solved_200):
    res, elapsed = solved_200
    for i, m, b, x, _ in res:
        want = dense_solve(m, b.blocks)
        rel = np.abs(x.blocks.reshape(want.shape) - want).max() / max(np.abs(want).max(), 1e-300)
        assert rel <= 1e-10, (i, rel)
    assert elapsed < 60.0


def test_criterion_02_path_equivalence(solved_200):
    res, _ = solved_200
    for i, _, _, x, xs in res:
        assert np.abs(x.blocks - xs.blocks).max() <= 1e-11 * max(np.abs(xs.blocks).max(), 1e-300), i


def test_criterion_03_residual_at_scale():
    for count, n in [(2048, 32), (1024, 64), (512, 128), (256, 256)]:
        m, b = generate_spd_btd(count, n, seed=count)
        x = recursive_solve(recursive_factorize(m, RecursionConfig()), b)
        assert residual_report(m, x, b)[1] <= 1e-10, (count, n)


def test_criterion_09_performance_smoke():
    """N=4096, n=32: recursive vs serial agree; the speed ratio is reported, non-gating (as in the
    reference)."""
    m, b = generate_spd_btd(4096, 32, seed=99)
    recursive_factorize(m, RecursionConfig())
    t0 = time.perf_counter()
    x_rec = recursive_solve(recursive_factorize(m, RecursionConfig()), b)
    t_rec = time.perf_counter() - t0
    t0 = time.perf_counter()
    w = m.copy()
    serial_factorize(w)
    x_ser = b.copy()
    serial_solve(w, x_ser)
    t_ser = time.perf_counter() - t0
    assert np.abs(x_rec.blocks - x_ser.blocks).max() <= 1e-11 * np.abs(x_ser.blocks).max()
    print(f"[criterion 09] N=4096 n=32 on {os.cpu_count()} cpus + 1 GPU: serial {t_ser:.3f}s / "
          f"recursive {t_rec:.3f}s = {t_ser / t_rec:.1f}x")
