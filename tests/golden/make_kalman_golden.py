"""Golden fixtures for the Kalman normal-equation assembly, made by running the REAL reference.

    python tests/golden/make_kalman_golden.py     # needs /root/reference; writes kalman_golden.npz

Rotation models are regenerated from (state_dim, obs_dim, horizon, dt, seed) by the package's
bit-identical port of generate_rotation_model (checked against the stored hashes); the random
per-step models of the reference's test suite (tests/test_kalman.py:36-54) are stored verbatim.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import blocktri as bt  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

ROTATION = [(2, 2, 1, 0.1, 0), (4, 6, 50, 0.1, 1), (8, 12, 300, 0.05, 2), (16, 20, 64, 0.2, 3),
            (8, 8, 1000, 0.1, 4)]
RANDOM = [(6, 3, 4, 2, True), (6, 3, 4, 2, False), (8, 2, 3, 5, True), (32, 8, 10, 11, True),
          (20, 5, 7, 3, False), (17, 12, 16, 9, False)]


def random_model(horizon, n, m, seed, diag_r=True):  # tests/test_kalman.py:36-54
    rng = np.random.default_rng(seed)
    transition = rng.standard_normal((horizon, n, n)) * 0.3
    transition[0] = np.eye(n)
    q = rng.standard_normal((horizon, n, n))
    process = q @ q.transpose(0, 2, 1) + 2 * n * np.eye(n)
    if diag_r:
        meas = rng.uniform(0.5, 2.0, (horizon, m))
    else:
        r = rng.standard_normal((horizon, m, m))
        meas = r @ r.transpose(0, 2, 1) + 2 * m * np.eye(m)
    return bt.StateSpaceModel(transition=transition, observation=rng.standard_normal((horizon, m, n)),
                              process_cov=process, measurement_cov=meas,
                              observations=rng.standard_normal((horizon, m)), prior_offsets=np.zeros((horizon, n)))


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main():
    out = {}
    for i, (n, m, N, dt, seed) in enumerate(ROTATION):
        model = bt.generate_rotation_model(n, m, N, dt=dt, seed=seed)
        A, B = bt.build_normal_equations(model)
        out[f"rot{i}_meta"] = np.array([n, m, N, seed], dtype=np.int64)
        out[f"rot{i}_dt"] = np.array([dt])
        out[f"rot{i}_hash"] = np.array([h(model.transition), h(model.observation[0]), h(model.process_cov[0]),
                                        h(model.measurement_cov[0]), h(model.observations)])
        out[f"rot{i}_diag"], out[f"rot{i}_sub"], out[f"rot{i}_rhs"] = A.diag, A.sub, B.blocks
    for i, (N, n, m, seed, diag_r) in enumerate(RANDOM):
        model = random_model(N, n, m, seed, diag_r)
        A, B = bt.build_normal_equations(model)
        for f in ("transition", "observation", "process_cov", "measurement_cov", "observations", "prior_offsets"):
            out[f"rnd{i}_{f}"] = getattr(model, f)
        out[f"rnd{i}_diag"], out[f"rnd{i}_sub"], out[f"rnd{i}_rhs"] = A.diag, A.sub, B.blocks
    # failures: (case, what) -> (pivot, block, context)
    errs = []
    m1 = random_model(5, 2, 3, 1)
    m1.process_cov[3] = -np.eye(2)
    m2 = random_model(4, 2, 3, 1, diag_r=False)
    m2.measurement_cov[2] = np.array([[1.0, 2.0, 0.0], [2.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    m3 = random_model(4, 2, 3, 1, diag_r=True)
    m3.measurement_cov[1, 0] = -0.5
    m4 = random_model(9, 3, 4, 7, diag_r=False)
    m4.process_cov[6] = -np.eye(3)
    m4.measurement_cov[6] = -np.eye(4)
    m4.measurement_cov[2, 1, 1] = -10.0
    for i, mdl in enumerate((m1, m2, m3, m4)):
        try:
            bt.build_normal_equations(mdl)
            raise SystemExit("expected a failure")
        except bt.NotPositiveDefinite as e:
            errs.append((e.pivot, e.block, 0 if "process" in e.context else 1))
        for f in ("transition", "observation", "process_cov", "measurement_cov", "observations", "prior_offsets"):
            out[f"err{i}_{f}"] = getattr(mdl, f)
    out["err_coords"] = np.array(errs, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "kalman_golden.npz"), **out)
    print("wrote", len(out), "arrays; errors:", errs)


if __name__ == "__main__":
    main()
