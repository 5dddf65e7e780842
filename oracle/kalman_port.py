"""CPU restatement of the reference's Kalman normal-equation assembly -- TEST / BASELINE
INFRASTRUCTURE ONLY (tests/, bench CPU legs); the product path is the GPU kernel
(paper_2509_03015_b200/csrc/btd_kalman.cuh).

Follows build_normal_equations (/root/reference/pkg/src/blocktri/kalman.py:130-162) and
_observation_terms (kalman.py:105-127): per step k a Cholesky of Q_k (and of a dense R_k), every
inverse applied through two triangular solves.  Pinned against the reference's outputs in
tests/test_kalman_golden.py.
"""

from __future__ import annotations

import numpy as np


def _chol_solve(lower: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    y = np.linalg.solve(lower, rhs)          # L y = rhs
    return np.linalg.solve(lower.T, y)       # L^T x = y


def build_normal_equations(model):
    N, n = model.horizon, model.state_dim
    diag = np.empty((N, n, n))
    sub = np.empty((max(N - 1, 0), n, n))
    rhs = np.empty((N, n, 1))
    eye = np.eye(n)
    for k in range(N):
        lq = np.linalg.cholesky(model.process_cov[k])
        qi = _chol_solve(lq, eye)
        qig = _chol_solve(lq, model.transition[k])
        qiz = _chol_solve(lq, model.prior_offsets[k][:, None])
        h, z = model.observation[k], model.observations[k]
        if model.diagonal_measurement_cov:
            r = model.measurement_cov[k]
            hrh, hrz = h.T @ (h / r[:, None]), h.T @ (z / r)
        else:
            lr = np.linalg.cholesky(model.measurement_cov[k])
            wh, wz = np.linalg.solve(lr, h), np.linalg.solve(lr, z)
            hrh, hrz = wh.T @ wh, wh.T @ wz
        diag[k] = qi + hrh
        rhs[k] = hrz[:, None] + model.transition[k].T @ qiz
        if k > 0:
            diag[k - 1] += model.transition[k].T @ qig
            sub[k - 1] = -qig
    diag = (diag + diag.transpose(0, 2, 1)) / 2.0
    return diag, sub, rhs
