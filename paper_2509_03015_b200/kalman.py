"""Kalman MAP-smoothing front-end (drop-in for `blocktri.kalman`, /root/reference/pkg/src/blocktri/kalman.py).

`build_normal_equations` assembles the SPD block-tridiagonal normal equations of linear-Gaussian
trajectory smoothing on the GPU (C ABI `btd_kalman_normal_equations`, btd_kalman.cuh; the
reference's per-step Python loop, kalman.py:130-162).  `StateSpaceModel` and
`generate_rotation_model` keep the reference's container, validation and seeded generator
(bit-identical draw sequence, kalman.py:45-96, 165-228); the generator is host code like the
reference's.  Arrays that are constant over the horizon (stride-0 broadcast views) are passed to
the device once.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .core import BlockRhs, BlockTridiagonalMatrix
from .errors import DimensionMismatch, InvalidDimensions, NotPositiveDefinite

ROTATION_DAMPING = 0.98
PROCESS_COV_SCALE = 0.01
REFERENCE_DT = 0.1


@dataclass
class StateSpaceModel:
    """Linear-Gaussian state-space model over a fixed horizon (kalman.py:45-96)."""

    transition: np.ndarray       # (N, n, n)
    observation: np.ndarray      # (N, m, n)
    process_cov: np.ndarray      # (N, n, n) SPD
    measurement_cov: np.ndarray  # (N, m, m) SPD, or (N, m) diagonals
    observations: np.ndarray     # (N, m)
    prior_offsets: np.ndarray    # (N, n)
    dt: float = REFERENCE_DT
    seed: int | None = None

    def __post_init__(self):
        horizon, n = self.transition.shape[0], self.transition.shape[-1]
        m = self.observation.shape[1]
        if self.transition.shape != (horizon, n, n):
            raise DimensionMismatch("transition must be (N, n, n)")
        if self.observation.shape != (horizon, m, n):
            raise DimensionMismatch("observation must be (N, m, n)")
        if self.process_cov.shape != (horizon, n, n):
            raise DimensionMismatch("process_cov must be (N, n, n)")
        if self.measurement_cov.shape not in ((horizon, m, m), (horizon, m)):
            raise DimensionMismatch("measurement_cov must be (N, m, m) or (N, m)")
        if self.observations.shape != (horizon, m):
            raise DimensionMismatch("observations must be (N, m)")
        if self.prior_offsets.shape != (horizon, n):
            raise DimensionMismatch("prior_offsets must be (N, n)")
        if not np.array_equal(self.transition[0], np.eye(n)):
            raise ValueError("the first transition must be the identity")

    @property
    def horizon(self) -> int:
        return self.transition.shape[0]

    @property
    def state_dim(self) -> int:
        return self.transition.shape[1]

    @property
    def obs_dim(self) -> int:
        return self.observation.shape[1]

    @property
    def diagonal_measurement_cov(self) -> bool:
        return self.measurement_cov.ndim == 2


def _device_array(a: np.ndarray, dev):
    """(torch tensor on dev, shared?) -- a stride-0 leading axis goes up as a single block."""
    import torch
    shared = a.ndim >= 1 and a.shape[0] > 1 and a.strides[0] == 0
    src = np.ascontiguousarray(a[:1] if shared else a, dtype=np.float64)
    if not src.flags.writeable:  # broadcast views are read-only; torch wants writable memory
        src = src.copy()
    return torch.from_numpy(src).to(dev), shared


#: largest state / dense-measurement dimension of the hand-written assembly kernel (btd_kalman.cuh)
KERNEL_MAX_DIM = 64


def _raise_first_failure(info_q, info_r):
    """NotPositiveDefinite for the first failing time step in the reference's loop order (process
    covariance before measurement covariance at the same step, kalman.py:143-153); info_* are
    1-based first failing pivots per step (0: fine)."""
    import torch
    bad = (info_q > 0) | (info_r > 0)
    if not bool(bad.any()):
        return
    k = int(torch.nonzero(bad).flatten()[0])
    if int(info_q[k]) > 0:
        raise NotPositiveDefinite(int(info_q[k]), block=k, context="process covariance")
    raise NotPositiveDefinite(int(info_r[k]), block=k, context="measurement covariance")


def _build_batched(model: StateSpaceModel, dev):
    """Large shapes (n or dense m > KERNEL_MAX_DIM, e.g. the paper's n = 256, m = 1024 case,
    PAPER.md:632-641): the same algebra as the reference's per-step loop (kalman.py:99-162) as
    batched GPU factorizations and products over the horizon (torch.linalg: cuSOLVER / cuBLAS --
    harness code in front of the factor/solve path, not part of it).  Time-invariant H / Q / R
    (stride-0 broadcasts) are factored once.  Returns (diag, sub, rhs) on the device."""
    import torch
    N, n, m = model.horizon, model.state_dim, model.obs_dim
    G, _ = _device_array(model.transition, dev)
    H, _ = _device_array(model.observation, dev)
    Q, _ = _device_array(model.process_cov, dev)
    R, _ = _device_array(model.measurement_cov, dev)
    Z, _ = _device_array(model.observations, dev)
    P, _ = _device_array(model.prior_offsets, dev)
    # process covariance: Q^{-1}, Q^{-1} G_k, Q^{-1} zeta_k through its Cholesky factor
    Lq, info_q = torch.linalg.cholesky_ex(Q)
    if model.diagonal_measurement_cov:
        bad = R <= 0.0
        info_r = torch.where(bad.any(dim=1), bad.to(torch.int64).argmax(dim=1) + 1, 0)
    else:
        Lr, info_r = torch.linalg.cholesky_ex(R)
    info_q = info_q.expand(N) if info_q.shape[0] == 1 else info_q
    info_r = info_r.expand(N) if info_r.shape[0] == 1 else info_r
    _raise_first_failure(info_q.cpu(), info_r.cpu())
    eye = torch.eye(n, dtype=torch.float64, device=dev).expand(Lq.shape[0], n, n).contiguous()
    q_inv = torch.cholesky_solve(eye, Lq)
    q_inv_g = torch.cholesky_solve(G, Lq.expand(N, n, n) if Lq.shape[0] == 1 else Lq)
    q_inv_zeta = torch.cholesky_solve(P.unsqueeze(-1), Lq.expand(N, n, n) if Lq.shape[0] == 1 else Lq)
    # observation terms H^T R^{-1} H and H^T R^{-1} z (kalman.py:107-127)
    if model.diagonal_measurement_cov:
        weighted = H / R.unsqueeze(-1)
        ht_ri_h = H.transpose(1, 2) @ weighted
        ht_ri_z = H.transpose(1, 2) @ (Z / R).unsqueeze(-1)
    else:
        white_h = torch.linalg.solve_triangular(Lr, H, upper=False)
        Lr_n = Lr.expand(N, m, m) if Lr.shape[0] == 1 else Lr
        white_z = torch.linalg.solve_triangular(Lr_n, Z.unsqueeze(-1), upper=False)
        ht_ri_h = white_h.transpose(1, 2) @ white_h
        wh_n = white_h.expand(N, m, n) if white_h.shape[0] == 1 else white_h
        ht_ri_z = wh_n.transpose(1, 2) @ white_z
    diag = (q_inv + ht_ri_h).expand(N, n, n).clone()
    rhs = ht_ri_z.expand(N, n, 1) + G.transpose(1, 2) @ q_inv_zeta
    if N > 1:
        diag[:-1] += G[1:].transpose(1, 2) @ q_inv_g[1:]
    sub = -q_inv_g[1:].contiguous()
    return diag.contiguous(), sub, rhs.contiguous()


def build_normal_equations(model: StateSpaceModel, *, device_out: bool = False, _path: str = "auto"):
    """Smoothing normal equations (kalman.py:130-162), assembled on the GPU.

    Returns (BlockTridiagonalMatrix, BlockRhs) with numpy arenas (the reference's types), or torch
    CUDA tensors with ``device_out=True`` (ready for ``recursive_factorize`` without a round trip).
    Raises NotPositiveDefinite(pivot, block=k, context="process covariance" / "measurement
    covariance") for the first failing time step, like the reference.  Shapes up to
    KERNEL_MAX_DIM run in the hand-written assembly kernel; larger ones in batched library
    factorizations (``_path`` = "kernel" / "batched" forces one, for tests).
    """
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    N, n, m = model.horizon, model.state_dim, model.obs_dim
    batched = _path == "batched" or (_path == "auto" and (
        n > KERNEL_MAX_DIM or (m > KERNEL_MAX_DIM and not model.diagonal_measurement_cov)))
    if batched:
        from .core import new_btd
        diag, sub, rhs = _build_batched(model, dev)
        A = new_btd(N, n, diag, sub)  # the reference's symmetry check + (D + D^T)/2
        if device_out:
            return A, BlockRhs(rhs)
        return BlockTridiagonalMatrix(A.diag.cpu().numpy(), A.sub.cpu().numpy()), BlockRhs(rhs.cpu().numpy())
    G, _ = _device_array(model.transition, dev)
    H, sh = _device_array(model.observation, dev)
    Q, sq = _device_array(model.process_cov, dev)
    R, sr = _device_array(model.measurement_cov, dev)
    Z, _ = _device_array(model.observations, dev)
    P, _ = _device_array(model.prior_offsets, dev)
    flags = ((1 if model.diagonal_measurement_cov else 0) | (2 if sh else 0) | (4 if sq else 0) |
             (8 if sr else 0))
    diag = torch.empty((N, n, n), dtype=torch.float64, device=dev)
    sub = torch.empty((max(N - 1, 0), n, n), dtype=torch.float64, device=dev)
    rhs = torch.empty((N, n, 1), dtype=torch.float64, device=dev)
    L = _native.lib()
    ws = ctypes.c_size_t()
    L.btd_kalman_workspace(N, n, ctypes.byref(ws))
    work = torch.empty(ws.value, dtype=torch.uint8, device=dev)
    st = _native.BtdStatus()
    s = torch.cuda.current_stream(dev)
    rc = L.btd_kalman_normal_equations(N, n, m, G.data_ptr(), H.data_ptr(), Q.data_ptr(), R.data_ptr(),
                                       Z.data_ptr(), P.data_ptr(), flags, diag.data_ptr(),
                                       sub.data_ptr() if N > 1 else None, rhs.data_ptr(), work.data_ptr(),
                                       ctypes.c_void_p(s.cuda_stream), ctypes.byref(st))
    if rc == _native.BTD_ERR_NOT_POSITIVE_DEFINITE:
        ctx = "process covariance" if st.member == 0 else "measurement covariance"
        raise NotPositiveDefinite(int(st.pivot), block=int(st.block), context=ctx)
    if rc == _native.BTD_ERR_UNSUPPORTED:
        raise NotImplementedError(st.message.decode())
    if rc != _native.BTD_OK:
        raise RuntimeError(st.message.decode())
    if device_out:
        return BlockTridiagonalMatrix(diag, sub), BlockRhs(rhs)
    return BlockTridiagonalMatrix(diag.cpu().numpy(), sub.cpu().numpy()), BlockRhs(rhs.cpu().numpy())


def generate_rotation_model(state_dim: int, obs_dim: int, horizon: int, dt: float = REFERENCE_DT,
                            seed: int = 0) -> StateSpaceModel:
    """Damped-rotation dynamics with tall observations (kalman.py:165-228).

    Same random stream (one default_rng(seed): plane angles, mixing matrix, raw observation
    matrix, measurement variances, initial state, then per step process and measurement noise)
    and the same floating-point expressions, so the model is bitwise identical to the reference's
    for the same arguments (tests/test_kalman_golden.py checks the hashes)."""
    if state_dim < 2 or state_dim % 2:
        raise InvalidDimensions(f"state_dim must be even and >= 2, got {state_dim}")
    if obs_dim < state_dim:
        raise InvalidDimensions(f"obs_dim must be >= state_dim, got {obs_dim} < {state_dim}")
    if horizon < 1:
        raise InvalidDimensions(f"horizon must be >= 1, got {horizon}")
    n, m = state_dim, obs_dim
    draw = np.random.default_rng(seed)
    theta = draw.uniform(0.0, np.pi / 4.0, n // 2) * (dt / REFERENCE_DT)
    dyn = np.zeros((n, n))
    for p, t in enumerate(theta):  # one damped 2x2 rotation per plane
        cs, sn = np.cos(t), np.sin(t)
        dyn[2 * p:2 * p + 2, 2 * p:2 * p + 2] = ROTATION_DAMPING * np.array([[cs, -sn], [sn, cs]])
    G = np.empty((horizon, n, n))
    G[0] = np.eye(n)
    G[1:] = dyn
    mix = draw.standard_normal((n, n))
    Qc = PROCESS_COV_SCALE * (mix @ mix.T + n * np.eye(n)) / n
    u, sv, vt = np.linalg.svd(draw.standard_normal((m, n)), full_matrices=False)
    Hc = (u * np.clip(sv, 0.5, 2.0)) @ vt
    rvar = draw.uniform(0.1, 1.0, m)
    x = draw.standard_normal(n)
    lq, rstd = np.linalg.cholesky(Qc), np.sqrt(rvar)
    z = np.empty((horizon, m))
    for k in range(horizon):  # simulate the trajectory and its noisy observations
        x = G[k] @ x + lq @ draw.standard_normal(n)
        z[k] = Hc @ x + rstd * draw.standard_normal(m)
    return StateSpaceModel(transition=G, observation=np.broadcast_to(Hc, (horizon, m, n)),
                           process_cov=np.broadcast_to(Qc, (horizon, n, n)),
                           measurement_cov=np.broadcast_to(rvar, (horizon, m)), observations=z,
                           prior_offsets=np.zeros((horizon, n)), dt=dt, seed=seed)
