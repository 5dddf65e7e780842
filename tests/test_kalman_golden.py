"""Kalman front-end: the rotation-model generator is bit-identical to the
reference's (hashes from tests/golden/make_kalman_golden.py, which ran the real reference), the
model container validates like the reference (kalman.py:45-96), and -- on the GPU -- the
normal-equation assembly kernel matches the reference's build_normal_equations outputs and failure
coordinates."""

import hashlib
import os

import numpy as np
import pytest

import paper_2509_03015_b200 as pkg

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "kalman_golden.npz"))
FIELDS = ("transition", "observation", "process_cov", "measurement_cov", "observations", "prior_offsets")


def _h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def _cases(prefix):
    i = 0
    while f"{prefix}{i}_diag" in GOLD:
        yield i
        i += 1


def _rot_model(i):
    n, m, N, seed = (int(v) for v in GOLD[f"rot{i}_meta"])
    return pkg.generate_rotation_model(n, m, N, dt=float(GOLD[f"rot{i}_dt"][0]), seed=seed)


def _stored_model(prefix):
    return pkg.StateSpaceModel(**{f: np.array(GOLD[f"{prefix}_{f}"]) for f in FIELDS})


def _close(a, b, tol=1e-12):
    a = np.asarray(a)
    if a.shape != b.shape:
        return False
    return a.size == 0 or np.abs(a - b).max() <= tol * max(np.abs(b).max(), 1.0)


def test_rotation_model_bit_identical_to_reference():
    for i in _cases("rot"):
        mdl = _rot_model(i)
        got = [_h(mdl.transition), _h(mdl.observation[0]), _h(mdl.process_cov[0]), _h(mdl.measurement_cov[0]),
               _h(mdl.observations)]
        assert got == list(GOLD[f"rot{i}_hash"]), i
        assert mdl.observation.strides[0] == 0 and mdl.process_cov.strides[0] == 0


def test_model_validation_like_reference():
    mdl = _rot_model(1)
    with pytest.raises(ValueError):
        pkg.StateSpaceModel(transition=mdl.transition * 0.5, observation=mdl.observation, process_cov=mdl.process_cov,
                            measurement_cov=mdl.measurement_cov, observations=mdl.observations,
                            prior_offsets=mdl.prior_offsets)
    with pytest.raises(pkg.DimensionMismatch):
        pkg.StateSpaceModel(transition=mdl.transition, observation=mdl.observation, process_cov=mdl.process_cov,
                            measurement_cov=mdl.measurement_cov, observations=mdl.observations[:, :-1],
                            prior_offsets=mdl.prior_offsets)
    for bad in ((3, 4, 5), (4, 3, 5), (4, 4, 0)):
        with pytest.raises(pkg.InvalidDimensions):
            pkg.generate_rotation_model(*bad)


def test_cpu_port_pinned_to_reference_outputs():
    from oracle import kalman_port
    for prefix, make in [("rot", _rot_model), ("rnd", lambda i: _stored_model(f"rnd{i}"))]:
        for i in _cases(prefix):
            d, s, r = kalman_port.build_normal_equations(make(i))
            assert _close(d, GOLD[f"{prefix}{i}_diag"], 1e-11) and _close(s, GOLD[f"{prefix}{i}_sub"], 1e-11)
            assert _close(r, GOLD[f"{prefix}{i}_rhs"], 1e-11)


torch = pytest.importorskip("torch")


@pytest.mark.gpu
def test_gpu_assembly_matches_reference_outputs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    for prefix, make in [("rot", _rot_model), ("rnd", lambda i: _stored_model(f"rnd{i}"))]:
        for i in _cases(prefix):
            A, B = pkg.build_normal_equations(make(i))
            assert _close(A.diag, GOLD[f"{prefix}{i}_diag"]), (prefix, i)
            assert _close(A.sub, GOLD[f"{prefix}{i}_sub"]), (prefix, i)
            assert _close(B.blocks, GOLD[f"{prefix}{i}_rhs"]), (prefix, i)
            assert np.array_equal(A.diag, A.diag.transpose(0, 2, 1))  # new_btd symmetrisation


@pytest.mark.gpu
def test_gpu_assembly_failure_coordinates():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    for i, (pivot, block, kind) in enumerate(GOLD["err_coords"]):
        with pytest.raises(pkg.NotPositiveDefinite) as e:
            pkg.build_normal_equations(_stored_model(f"err{i}"))
        assert (e.value.pivot, e.value.block) == (pivot, block), i
        assert ("process" if kind == 0 else "measurement") in e.value.context


@pytest.mark.gpu
def test_gpu_kalman_pipeline_device_resident():
    """Assembly -> recursive factor/solve without leaving the device (the paper's application)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mdl = pkg.generate_rotation_model(8, 12, 5000, seed=7)
    A, B = pkg.build_normal_equations(mdl, device_out=True)
    X = pkg.recursive_solve(pkg.recursive_factorize(A), B)
    assert X.blocks.is_cuda
    assert pkg.residual_report(A, X, B)[1] <= 1e-12


@pytest.mark.gpu
def test_gpu_batched_assembly_matches_reference_outputs_and_coordinates():
    """The large-shape path (batched factorizations, n or dense m > 64) on the golden cases."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    for prefix, make in [("rot", _rot_model), ("rnd", lambda i: _stored_model(f"rnd{i}"))]:
        for i in _cases(prefix):
            A, B = pkg.build_normal_equations(make(i), _path="batched")
            assert _close(A.diag, GOLD[f"{prefix}{i}_diag"]), (prefix, i)
            assert _close(A.sub, GOLD[f"{prefix}{i}_sub"]), (prefix, i)
            assert _close(B.blocks, GOLD[f"{prefix}{i}_rhs"]), (prefix, i)
            assert np.array_equal(A.diag, A.diag.transpose(0, 2, 1))
    for i, (pivot, block, kind) in enumerate(GOLD["err_coords"]):
        with pytest.raises(pkg.NotPositiveDefinite) as e:
            pkg.build_normal_equations(_stored_model(f"err{i}"), _path="batched")
        assert (e.value.pivot, e.value.block) == (pivot, block), i
        assert ("process" if kind == 0 else "measurement") in e.value.context


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,diag_r", [(96, 128, True), (80, 160, False)])
def test_gpu_large_shape_assembly_vs_cpu_port(n, m, diag_r):
    """Shapes beyond the assembly kernel go through the batched path and match the CPU port of
    the reference loop (oracle/kalman_port.py); the smoothing pipeline then solves to 1e-12."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import kalman_port
    mdl = pkg.generate_rotation_model(n, m, 40, seed=3)
    if not diag_r:  # dense, time-varying R built from the diagonal one
        rng = np.random.default_rng(5)
        mix = rng.standard_normal((40, m, m)) * 0.05
        dense = np.einsum("kij,kjl->kil", mix, mix.transpose(0, 2, 1)) + np.eye(m) * mdl.measurement_cov[0]
        mdl = pkg.StateSpaceModel(mdl.transition, mdl.observation, mdl.process_cov, dense, mdl.observations,
                                  mdl.prior_offsets)
    A, B = pkg.build_normal_equations(mdl)
    ref = kalman_port.build_normal_equations(mdl)
    assert _close(A.diag, ref[0], 1e-11) and _close(A.sub, ref[1], 1e-11) and _close(B.blocks, ref[2], 1e-11)
    Ad, Bd = pkg.build_normal_equations(mdl, device_out=True)
    X = pkg.recursive_solve(pkg.recursive_factorize(Ad), Bd)
    assert pkg.residual_report(Ad, X, Bd)[1] <= 1e-12
