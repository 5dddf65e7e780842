"""Pin the CPU oracle (oracle/blocktri_port.py) against outputs of the real reference
(tests/golden/reference_golden.npz, produced by tests/golden/make_golden.py) and against the
reference test-suite's known-answer tests."""

import numpy as np
import pytest

from oracle import blocktri_port as port
from paper_2509_03015_b200.synthgen import generate_spd_btd


def _cases(golden, prefix):
    i = 0
    while f"{prefix}{i}_meta" in golden:
        yield i
        i += 1


def test_solutions_match_reference(golden):
    for i in _cases(golden, "solve"):
        N, n, d, seed, cross, rho, auto = golden[f"solve{i}_meta"]
        A, B = generate_spd_btd(int(N), int(n), int(d), int(seed))
        h = port.factorize(A.diag, A.sub, int(cross), int(rho), 32, bool(auto))
        X = port.solve(h, B.blocks)
        ref = golden[f"solve{i}_x"]
        rel = np.abs(X - ref).max() / max(np.abs(ref).max(), 1e-300)
        assert rel <= 1e-12, (i, rel)
        levels = [r["seps"][-1] + 1 for r in h["levels"]] + [h["base"][0].shape[1]]
        assert levels == list(golden[f"solve{i}_levels"]), i
        for li, r in enumerate(h["levels"]):
            assert r["seps"] == list(golden[f"solve{i}_seps{li}"])


def test_schur_matches_reference(golden):
    for i in _cases(golden, "schur"):
        N, n, seed, rho = (int(v) for v in golden[f"schur{i}_meta"])
        A, _ = generate_spd_btd(N, n, 1, seed)
        sd, ss = port.schur_level0(A.diag, A.sub, rho)
        rd, rs = golden[f"schur{i}_diag"], golden[f"schur{i}_sub"]
        scale = np.abs(rd).max()
        assert np.abs(sd - rd).max() <= 1e-13 * scale
        assert np.abs(ss - rs).max() <= 1e-13 * scale


def test_npd_coordinates_match_reference(golden):
    for i in _cases(golden, "npd"):
        N, n, seed, rho, cross = (int(v) for v in golden[f"npd{i}_meta"])
        A, _ = generate_spd_btd(N, n, 1, seed)
        for b in golden[f"npd{i}_bad"]:
            A.diag[b] = -A.diag[b]
        want = list(golden[f"npd{i}_coords"])
        with pytest.raises(port.OracleNPD) as e:
            port.factorize(A.diag, A.sub, cross, rho)
        got = [e.value.pivot, e.value.level, e.value.member, e.value.block]
        assert got == want, (i, got, want)


def test_plans_match_reference(golden):
    seps, offs = golden["plans_seps"], golden["plans_offsets"]
    idx = 0
    for rho in range(1, 21):
        for N in range(3, 701):
            ref = list(seps[offs[idx]:offs[idx + 1]])
            assert port.plan_separators(N, rho) == ref
            idx += 1


# ---- known-answer tests of the reference suite (pkg/tests/...) ----
def test_kat_scalar_chain_schur():
    # tests/test_schur.py:152-156: tridiag(1,4,1), N=3 -> S = [[3.75,-0.25],[-0.25,3.75]]
    N = 3
    diag = np.full((N, 1, 1), 4.0)
    sub = np.full((N - 1, 1, 1), 1.0)
    sd, ss = port.schur_level0(diag, sub, rho=8)
    assert np.allclose(sd[:, 0, 0], [3.75, 3.75], atol=1e-15)
    assert np.allclose(ss[:, 0, 0], [-0.25], atol=1e-15)


def test_kat_2x2_solve():
    # tests/test_block_cholesky.py:76-85: [[4,2],[2,5]] x = [6,7] -> x = [1,1]
    diag = np.array([[[4.0]], [[5.0]]])
    sub = np.array([[[2.0]]])
    h = port.factorize(diag, sub)
    x = port.solve(h, np.array([[[6.0]], [[7.0]]]))
    assert np.allclose(x.ravel(), [1.0, 1.0], atol=1e-15)


def test_kat_potrf():
    # tests/test_kernels.py:20-49
    a = np.array([[[4.0, 2.0], [2.0, 5.0]]])
    port.potrf_batch(a)
    assert np.allclose(a[0], [[2.0, 0.0], [1.0, 2.0]])
    b = np.array([[[1.0, 2.0], [2.0, 1.0]]])
    with pytest.raises(port.OracleNPD) as e:
        port.potrf_batch(b)
    assert e.value.pivot == 2


def test_oracle_vs_dense(rng):
    for N, n, d in [(7, 3, 2), (30, 2, 1), (12, 5, 3)]:
        A, B = generate_spd_btd(N, n, d, seed=int(rng.integers(1000)))
        h = port.factorize(A.diag, A.sub, crossover=2, rho=2)
        X = port.solve(h, B.blocks)
        dense = port.assemble_dense(A.diag, A.sub)
        ref = np.linalg.solve(dense, B.blocks.reshape(N * n, d)).reshape(N, n, d)
        assert np.abs(X - ref).max() <= 1e-12 * np.abs(ref).max()
