"""GPU parity: the sm_100a engine against the reference (golden fixtures from the real reference)
and the CPU oracle, through the drop-in Python API -> C ABI -> CUDA kernels.

Bars (BASELINE.json north_star): solution max|dX|/max|X| <= 1e-10, relative residual
max_col ||AX-B||/||B|| <= 1e-12, bit-exact plans."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import paper_2509_03015_b200 as pkg  # noqa: E402
from oracle import blocktri_port as port  # noqa: E402

REL_X = 1e-10
REL_RES = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _cases(golden, prefix):
    i = 0
    while f"{prefix}{i}_meta" in golden:
        yield i
        i += 1


def _solve(A, B, cfg):
    h = pkg.recursive_factorize(A, cfg)
    X = pkg.recursive_solve(h, B)
    return h, X


def test_golden_solutions(golden):
    for i in _cases(golden, "solve"):
        N, n, d, seed, cross, rho, auto = (int(v) for v in golden[f"solve{i}_meta"])
        A, B = pkg.generate_spd_btd(N, n, d, seed)
        cfg = pkg.RecursionConfig(crossover=cross, segment_length=rho, auto_crossover=bool(auto))
        h, X = _solve(A, B, cfg)
        ref = golden[f"solve{i}_x"]
        rel = np.abs(X.blocks - ref).max() / max(np.abs(ref).max(), 1e-300)
        assert rel <= REL_X, (i, (N, n, d), rel)
        _, rres = pkg.residual_report(A, X, B)
        assert rres <= REL_RES, (i, rres)
        levels = [lvl.plan.num_blocks for lvl in h.levels] + [h.base.num_blocks]
        assert levels == list(golden[f"solve{i}_levels"])
        for li, lvl in enumerate(h.levels):
            assert list(lvl.plan.separators) == list(golden[f"solve{i}_seps{li}"])


def test_golden_npd_coordinates(golden):
    for i in _cases(golden, "npd"):
        N, n, seed, rho, cross = (int(v) for v in golden[f"npd{i}_meta"])
        A, _ = pkg.generate_spd_btd(N, n, 1, seed)
        for b in golden[f"npd{i}_bad"]:
            A.diag[b] = -A.diag[b]
        want = [int(v) for v in golden[f"npd{i}_coords"]]
        with pytest.raises(pkg.NotPositiveDefinite) as e:
            pkg.recursive_factorize(A, pkg.RecursionConfig(crossover=cross, segment_length=rho))
        got = [e.value.pivot, e.value.level, e.value.member, e.value.block]
        assert got == want, (i, got, want)


SWEEP = [  # (N, n, d, crossover, rho)
    (1, 1, 1, 64, 8), (1, 7, 2, 64, 8), (2, 5, 1, 64, 8), (3, 3, 3, 1, 1), (5, 2, 2, 2, 1),
    (17, 1, 1, 2, 2), (33, 9, 2, 3, 3), (64, 16, 1, 64, 8), (65, 16, 1, 64, 8), (129, 17, 3, 8, 8),
    (200, 31, 2, 16, 5), (300, 33, 1, 64, 8), (111, 47, 4, 9, 4), (250, 63, 1, 64, 8),
    (260, 64, 3, 64, 8), (1000, 8, 1, 64, 8), (777, 12, 5, 10, 7), (90, 64, 6, 4, 2), (45, 6, 9, 3, 16),
    (20, 128, 2, 4, 3), (70, 256, 3, 8, 8), (9, 192, 1, 2, 2), (3, 128, 65, 1, 1), (50, 256, 70, 64, 8),
    # n > 64 and not a multiple of 64: padded to the next multiple of 64 (schur._padded_size)
    (90, 80, 2, 8, 4), (40, 100, 1, 64, 8), (25, 65, 3, 4, 2), (12, 150, 2, 2, 2),
    # n > 64, d <= 4, >= 64 segments per level: solve_wide_kernel (btd_solve3.cuh)
    (700, 128, 3, 64, 8), (600, 192, 1, 64, 8), (650, 100, 2, 64, 8),
    # n > 64 with 5 <= d <= 8: solve_dmma_kernel (levels, base)
    (700, 128, 8, 64, 8), (90, 256, 6, 8, 4), (300, 100, 5, 16, 8),
    # n <= 64 with d > 1 and >= #SMs segments: two-CTA solve_tma_kernel (z through the solution
    # buffer), incl. column slices (d > 4), padded blocks and long segments
    (1500, 64, 4, 64, 8), (1400, 64, 2, 64, 8), (1500, 64, 7, 64, 8), (1600, 50, 3, 64, 8),
    (2600, 64, 4, 64, 16),
]


@pytest.mark.parametrize("case", SWEEP, ids=[str(c) for c in SWEEP])
def test_sweep_vs_oracle(case):
    N, n, d, cross, rho = case
    A, B = pkg.generate_spd_btd(N, n, d, seed=N * 7 + n)
    cfg = pkg.RecursionConfig(crossover=cross, segment_length=rho)
    _, X = _solve(A, B, cfg)
    hh = port.factorize(A.diag, A.sub, cross, rho)
    ref = port.solve(hh, B.blocks)
    rel = np.abs(X.blocks - ref).max() / np.abs(ref).max()
    assert rel <= REL_X, rel
    _, rres = pkg.residual_report(A, X, B)
    assert rres <= REL_RES, rres


def test_device_tensors_roundtrip_and_no_mutation():
    A, B = pkg.generate_spd_btd(500, 32, 3, seed=3)
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
    dB = pkg.BlockRhs(torch.from_numpy(B.blocks).cuda())
    d0, s0, b0 = dA.diag.clone(), dA.sub.clone(), dB.blocks.clone()
    h = pkg.recursive_factorize(dA)
    X1 = pkg.recursive_solve(h, dB)
    X2 = pkg.recursive_solve(h, dB)
    assert torch.equal(dA.diag, d0) and torch.equal(dA.sub, s0) and torch.equal(dB.blocks, b0)
    assert torch.equal(X1.blocks, X2.blocks)  # repeated solves independent (tests/test_schur.py:367-382)
    _, rres = pkg.residual_report(dA, X1, dB)
    assert rres <= REL_RES
    Xh = pkg.recursive_solve(h, B)
    assert np.array_equal(Xh.blocks, X1.blocks.cpu().numpy())


def test_level_overflow_and_dimension_errors():
    A, B = pkg.generate_spd_btd(300, 4, 1, seed=1)
    with pytest.raises(pkg.LevelOverflow):
        pkg.recursive_factorize(A, pkg.RecursionConfig(crossover=2, segment_length=1, max_levels=2))
    h = pkg.recursive_factorize(A)
    with pytest.raises(pkg.DimensionMismatch):
        pkg.recursive_solve(h, pkg.BlockRhs(np.zeros((299, 4, 1))))


def test_multi_column_equals_column_by_column():
    A, B = pkg.generate_spd_btd(400, 24, 5, seed=9)
    h = pkg.recursive_factorize(A)
    X = pkg.recursive_solve(h, B).blocks
    for c in range(5):
        xc = pkg.recursive_solve(h, pkg.BlockRhs(np.ascontiguousarray(B.blocks[:, :, c:c + 1]))).blocks
        assert np.abs(xc[:, :, 0] - X[:, :, c]).max() <= 1e-13 * np.abs(X).max()


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [(1024, 32, 1), (65536, 64, 1), (1048576, 8, 1), (4096, 256, 64)],
                         ids=["cfg1", "cfg2", "cfg3", "cfg4"])
def test_baseline_configs_vs_oracle(cfg):
    """Full BASELINE sizes (configs 1-4, seed 0): the device solution against the CPU oracle run on
    the same inputs on the host cores (max|dX|/max|X| <= 1e-10) and the relative residual
    (<= 1e-12, size-independent)."""
    N, n, d = cfg
    A, B = pkg.generate_spd_btd(N, n, d, seed=0)
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
    dB = pkg.BlockRhs(torch.from_numpy(B.blocks).cuda())
    h = pkg.recursive_factorize(dA)
    X = pkg.recursive_solve(h, dB)
    _, rres = pkg.residual_report(dA, X, dB)
    assert rres <= REL_RES, rres
    levels = [lvl.num_blocks for lvl in h.levels] + [h.base.num_blocks]
    x = X.blocks.cpu().numpy()
    del dA, dB, X, h
    torch.cuda.empty_cache()
    hh = port.factorize(A.diag, A.sub)
    assert levels == [N] + [len(r["seps"]) for r in hh["levels"]]
    ref = port.solve(hh, B.blocks)
    rel = np.abs(x - ref).max() / np.abs(ref).max()
    assert rel <= REL_X, rel


def test_level_schur_vs_reference_golden(golden):
    """The next-level Schur complement system the GPU level kernels + assembly produce equals the
    reference's own compute_schur + new_btd output (tests/golden: _factorize_level of the real
    reference), <= 1e-12 x the block scale."""
    i = 0
    while f"schur{i}_meta" in golden:
        N, n, seed, rho = (int(v) for v in golden[f"schur{i}_meta"])
        A, _ = pkg.generate_spd_btd(N, n, 1, seed)
        cfg = pkg.RecursionConfig(crossover=2, segment_length=rho)
        diag, sub = pkg.level_schur(A, 0, cfg)
        want_d, want_s = golden[f"schur{i}_diag"], golden[f"schur{i}_sub"]
        scale = np.abs(want_d).max()
        assert tuple(diag.shape) == want_d.shape and tuple(sub.shape) == want_s.shape
        assert np.abs(diag.cpu().numpy() - want_d).max() <= 1e-12 * scale, i
        assert np.abs(sub.cpu().numpy() - want_s).max() <= 1e-12 * scale, i
        i += 1
    assert i == 5


@pytest.mark.parametrize("case", [(30000, 64, 8, 1), (30000, 64, 8, 2), (200000, 8, 8, 0), (3000, 128, 8, 0),
                                  (5000, 32, 5, 1)], ids=str)
def test_level_schur_vs_oracle(case):
    """Every level's Schur system (levels 0..2) against the oracle's compute_schur at sizes beyond
    the golden fixtures (n = 8 / 32 / 64 / 128 kernel families)."""
    N, n, rho, level = case
    A, _ = pkg.generate_spd_btd(N, n, 1, seed=level + 5)
    cfg = pkg.RecursionConfig(crossover=64, segment_length=rho)
    diag, sub = pkg.level_schur(A, level, cfg)
    want_d, want_s = port.level_schur(A.diag, A.sub, level, 64, rho)
    scale = np.abs(want_d).max()
    assert np.abs(diag.cpu().numpy() - want_d).max() <= 1e-12 * scale
    assert np.abs(sub.cpu().numpy() - want_s).max() <= 1e-12 * scale


@pytest.mark.parametrize("case", [(20000, 16, 2, 2, 8, 3), (20000, 16, 2, 3, 8, 3), (30000, 64, 1, 4, 64, 8),
                                  (6000, 8, 3, 8, 64, 8), (2000, 128, 2, 2, 8, 3)],
                         ids=lambda c: f"N{c[0]}_n{c[1]}_G{c[3]}")
def test_sharded_gpu_matches_unsharded(case):
    """Multi-GPU path on one device: every rank's partial factor/solve kernels run in sequence,
    the reduced system is assembled exactly as the NCCL all-gather would, and the result equals the
    unsharded solve."""
    from paper_2509_03015_b200.sharded import CudaEngine, run_sharded_local, shard_plan
    N, n, d, G, cross, rho = case
    A, B = pkg.generate_spd_btd(N, n, d, seed=G)
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
    dB = pkg.BlockRhs(torch.from_numpy(B.blocks).cuda())
    cfg = pkg.RecursionConfig(crossover=cross, segment_length=rho)
    plan = shard_plan(N, G, cross, rho)
    X = run_sharded_local(plan, CudaEngine(), dA.diag, dA.sub, dB.blocks, cfg)
    ref = pkg.recursive_solve(pkg.recursive_factorize(dA, cfg), dB).blocks
    rel = float((X - ref).abs().max() / ref.abs().max())
    assert rel <= 1e-12, rel
    _, rres = pkg.residual_report(dA, pkg.BlockRhs(X), dB)
    assert rres <= REL_RES


@pytest.mark.parametrize("N,n,d", [(4096, 64, 1), (20000, 8, 2), (3000, 33, 1), (600, 128, 2), (2800, 128, 1)])
def test_host_input_overlapped_copy_is_bitwise_device_path(N, n, d):
    """btd_factorize_from_host (chunked H2D overlapping the level-0 kernels) == device-input path."""
    A, B = pkg.generate_spd_btd(N, n, d, seed=11)
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
    dB = pkg.BlockRhs(torch.from_numpy(B.blocks).cuda())
    x_dev = pkg.recursive_solve(pkg.recursive_factorize(dA), dB).blocks.cpu().numpy()
    x_np = pkg.recursive_solve(pkg.recursive_factorize(A), B).blocks
    pA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).pin_memory(), torch.from_numpy(A.sub).pin_memory())
    x_pin = pkg.recursive_solve(pkg.recursive_factorize(pA), dB).blocks.cpu().numpy()
    assert np.array_equal(x_dev, x_np) and np.array_equal(x_dev, x_pin)


def test_host_input_npd_coordinates_match_device_path():
    A, _ = pkg.generate_spd_btd(5000, 16, 1, seed=2)
    diag = A.diag.copy()
    diag[2345, 3, 3] = -50.0
    bad = pkg.BlockTridiagonalMatrix(diag, A.sub)
    with pytest.raises(pkg.NotPositiveDefinite) as e_host:
        pkg.recursive_factorize(bad)
    with pytest.raises(pkg.NotPositiveDefinite) as e_dev:
        pkg.recursive_factorize(pkg.BlockTridiagonalMatrix(torch.from_numpy(diag).cuda(), torch.from_numpy(A.sub).cuda()))
    a, b = e_host.value, e_dev.value
    assert (a.pivot, a.level, a.member, a.block) == (b.pivot, b.level, b.member, b.block)


@pytest.mark.parametrize("N,n,rho,cross,bad", [
    (3000, 64, 8, 64, [(1234, 5), (1500, 40)]),   # wide level: factor_level_kernel<64>
    (600, 64, 8, 64, [(301, 63)]),                 # single-wave levels: factor_stream_kernel
    (70, 64, 8, 64, [(20, 0), (61, 7)]),           # deep level + base
    (5000, 6, 8, 64, [(777, 2), (778, 0)]),        # n <= 8: factor_small_kernel
    (2000, 40, 3, 16, [(999, 17)]),                # n = 40 padded to 64
    (6000, 64, 8, 64, [(9 * 20, 3)]),              # a level-0 separator: fails at level 1
    # n > 64 tiled path (two half-level streams at K = 333): two members failing in the same step
    # at different 64-column tiles -> the lower member (tile 1) wins over the higher one (tile 0)
    (3000, 128, 8, 64, [(9 * 3 + 1 + 2, 100), (9 * 5 + 1 + 2, 5)]),
    # ... and an earlier step in the second half-level stream beats a later step in the first
    (3000, 128, 8, 64, [(9 * 3 + 1 + 4, 5), (9 * 200 + 1 + 1, 70)]),
    # a level-0 separator that fails in the serial base (cluster-resident base kernel, n = 128, 256)
    (70, 128, 8, 64, [(9 * 3, 5)]),
    (70, 256, 8, 64, [(9 * 4, 200), (9 * 6, 3)]),
])
def test_npd_coordinates_every_kernel_vs_oracle(N, n, rho, cross, bad):
    """A non-positive pivot reports the oracle's (pivot, level, member, block) -- the reference's
    earliest-step, lowest-member rule -- whichever factor kernel the level runs on."""
    A, _ = pkg.generate_spd_btd(N, n, 1, seed=9)
    diag = A.diag.copy()
    for blk, i in bad:
        diag[blk, i, i] = -1.0e3
    with pytest.raises(port.OracleNPD) as eo:
        port.factorize(diag, A.sub, cross, rho)
    with pytest.raises(pkg.NotPositiveDefinite) as eg:
        pkg.recursive_factorize(pkg.BlockTridiagonalMatrix(torch.from_numpy(diag).cuda(), torch.from_numpy(A.sub).cuda()),
                                pkg.RecursionConfig(crossover=cross, segment_length=rho))
    o, g = eo.value, eg.value
    assert (g.pivot, g.level, g.member, g.block) == (o.pivot, o.level, o.member, o.block)


def test_padded_block_size_npd_coordinates_and_introspection():
    """n = 100 runs padded to 128: a non-positive pivot reports the n x n system's coordinates, and
    level_factor returns n x n blocks (the embedded factor)."""
    N, n = 300, 100
    A, B = pkg.generate_spd_btd(N, n, 1, seed=4)
    diag = A.diag.copy()
    diag[123, 37, 37] = -80.0
    with pytest.raises(pkg.NotPositiveDefinite) as e:
        pkg.recursive_factorize(pkg.BlockTridiagonalMatrix(diag, A.sub))
    with pytest.raises(port.OracleNPD) as eo:
        port.factorize(diag, A.sub)
    want = (eo.value.pivot, eo.value.level, eo.value.member, eo.value.block)
    assert (e.value.pivot, e.value.level, e.value.member, e.value.block) == want
    h = pkg.recursive_factorize(A)
    linv, lsub = pkg.level_factor(h, 0)
    assert tuple(linv.shape) == (N, n, n) and tuple(lsub.shape) == (N - 1, n, n)
    X = pkg.recursive_solve(h, B)
    assert X.blocks.shape == (N, n, 1)
    assert pkg.residual_report(A, X, B)[1] <= REL_RES
