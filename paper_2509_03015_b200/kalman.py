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
#: diagonal-block size of the blocked triangular solves of the large-shape path (the seam kernel's
#: shared-memory limit, btd_seam.cuh kSeamSmemMaxN)
_TRSM_BLOCK = 128


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
    PAPER.md:632-641): the reference's per-step loop (kalman.py:99-162) batched over the horizon
    on this package's own seam kernels (btd_seam.cuh, the GPU kernels behind `kernels.py`): the
    reference calls exactly these primitives -- chol_factor, trsm_lower (twice for an SPD solve)
    and matrix products -- step by step.  Time-invariant H / Q / R (stride-0 broadcasts) are
    factored and multiplied once; only elementwise scaling / negation / broadcasting copies run
    as torch tensor ops.  Returns (diag, sub, rhs) on the device."""
    import torch
    from . import kernels as kn
    N, n, m = model.horizon, model.state_dim, model.obs_dim
    G, _ = _device_array(model.transition, dev)
    H, _ = _device_array(model.observation, dev)
    Q, _ = _device_array(model.process_cov, dev)
    R, _ = _device_array(model.measurement_cov, dev)
    Z, _ = _device_array(model.observations, dev)
    P, _ = _device_array(model.prior_offsets, dev)

    def over(x, count):  # a (1, ...) broadcast as `count` members (stride-0 view, no copy)
        return x.expand(count, *x.shape[1:]) if x.shape[0] != count else x

    def chol(x):  # (factor, (first failing member, pivot) or None)
        f = x.clone()
        if f.shape[1] > _TRSM_BLOCK and chol_blocked(f):
            return f, None
        f = x.clone()  # unblocked (or after a failure: the exact first failing member and pivot)
        err = kn._ErrWord()
        kn._chol_dev(kn._Dev(f, True), f.shape[0], f.shape[1], err)
        rc, st = err.read()
        if rc == _native.BTD_OK:
            return f, None
        if rc != _native.BTD_ERR_NOT_POSITIVE_DEFINITE:
            kn._check(rc, st)
        return f, (int(st.member), int(st.pivot))

    def gemm(out, a, b, ta=False, alpha=1.0, beta=0.0):  # out <- alpha op(a) @ b + beta out
        c = out.shape[0]
        am = a.shape[2] if ta else a.shape[1]
        kn._gemm_dev(kn._Dev(out, True), kn._Dev(over(a, c), False), kn._Dev(over(b, c), False), c, am, b.shape[1],
                     b.shape[2], ta, False, alpha, beta)
        return out

    def trsm1(f, panel, trans):  # one seam launch: panel <- L^{-1} panel / L^{-T} panel, in place
        err = kn._ErrWord()
        kn._trsm_dev(kn._Dev(over(f, panel.shape[0]), False), kn._Dev(panel, True), panel.shape[0], f.shape[1],
                     panel.shape[2], trans, err)
        kn._raise_err(err)

    def trsm(f, panel, trans):
        # blocked substitution over diagonal blocks of <= _TRSM_BLOCK rows (the seam kernel keeps
        # those in shared memory; larger factors would be read from global memory per FMA), the
        # off-diagonal coupling as seam GEMM updates (views: no copies)
        nn = f.shape[1]
        if nn <= _TRSM_BLOCK:
            trsm1(f, panel, trans)
            return panel
        starts = list(range(0, nn, _TRSM_BLOCK))
        for i0 in (reversed(starts) if trans else starts):
            i1 = min(nn, i0 + _TRSM_BLOCK)
            if not trans and i0 > 0:  # b_i -= L[i, :i] x_{:i}
                gemm(panel[:, i0:i1], f[:, i0:i1, :i0], panel[:, :i0], alpha=-1.0, beta=1.0)
            if trans and i1 < nn:  # b_i -= L[i1:, i]^T x_{i1:}
                gemm(panel[:, i0:i1], f[:, i1:, i0:i1], panel[:, i1:], ta=True, alpha=-1.0, beta=1.0)
            trsm1(f[:, i0:i1, i0:i1], panel[:, i0:i1], trans)
        return panel

    def chol_blocked(f):
        # right-looking blocked Cholesky over diagonal blocks of <= _TRSM_BLOCK (factored in shared
        # memory by the seam kernel), L21 = A21 L11^{-T} as a seam trsm on the transposed view, the
        # trailing update as a seam GEMM; True when every member is SPD (else the caller reruns the
        # unblocked kernel for the reference's first failing member and pivot)
        cnt, nn = f.shape[0], f.shape[1]
        err = kn._ErrWord()
        for i0 in range(0, nn, _TRSM_BLOCK):
            i1 = min(nn, i0 + _TRSM_BLOCK)
            d = f[:, i0:i1, i0:i1]
            kn._chol_dev(kn._Dev(d, True), cnt, i1 - i0, err)
            if i1 < nn:
                pan = f[:, i1:, i0:i1]
                kn._trsm_dev(kn._Dev(d, False), kn._Dev(pan.transpose(1, 2), True), cnt, i1 - i0, nn - i1, False, err)
                gemm(f[:, i1:, i1:], pan, pan.transpose(1, 2), alpha=-1.0, beta=1.0)
        if err.read()[0] != _native.BTD_OK:
            return False
        f.tril_()  # the original A12 and the square trailing updates above the diagonal
        return True

    def spd_solve(f, panel):  # _chol_solve_spd (kalman.py:99-104)
        trsm(f, panel, False)
        trsm(f, panel, True)
        return panel


    # failures in the reference's loop order: process covariance before measurement covariance at
    # the same step (kalman.py:143-153); a broadcast covariance fails at step 0
    Lq, fq = chol(Q)
    if model.diagonal_measurement_cov:
        bad = R <= 0.0
        rows = torch.nonzero(bad.any(dim=1)).flatten()
        fr = None
        if rows.numel():
            k = int(rows[0])
            fr = (k, int(bad[k].to(torch.int64).argmax()) + 1)
    else:
        Lr, fr = chol(R)
    if fq is not None and (fr is None or fq[0] <= fr[0]):
        raise NotPositiveDefinite(fq[1], block=fq[0], context="process covariance")
    if fr is not None:
        raise NotPositiveDefinite(fr[1], block=fr[0], context="measurement covariance")

    nq = Q.shape[0]
    q_inv = spd_solve(Lq, torch.eye(n, dtype=torch.float64, device=dev).expand(nq, n, n).contiguous())
    q_inv_g = spd_solve(Lq, G.expand(N, n, n).clone())
    q_inv_zeta = spd_solve(Lq, over(P, N).reshape(N, n, 1).clone())
    # observation terms H^T R^{-1} H and H^T R^{-1} z (kalman.py:107-127)
    if model.diagonal_measurement_cov:
        nb = max(H.shape[0], R.shape[0])
        white_h = over(H, nb) / over(R, nb).unsqueeze(-1)  # R^{-1} H (elementwise)
        lhs_h, rhs_h = H, white_h
        white_z = (over(Z, N) / over(R, N)).unsqueeze(-1)
        lhs_z = H
    else:
        nb = max(H.shape[0], R.shape[0])
        white_h = _white(Lr, H, nb, trsm)
        lhs_h = rhs_h = white_h
        white_z = over(Z, N).reshape(N, m, 1).clone()
        trsm(Lr, white_z, False)
        lhs_z = white_h
    # diag_k = Q_k^{-1} + H^T R^{-1} H, computed once over the distinct members
    nd = max(nq, nb)
    dsum = over(q_inv, nd).clone()
    gemm(dsum, over(lhs_h, nd), over(rhs_h, nd), ta=True, beta=1.0)
    diag = over(dsum, N).clone()
    rhs = gemm(torch.empty((N, n, 1), dtype=torch.float64, device=dev), over(lhs_z, N), white_z, ta=True)
    gemm(rhs, G.expand(N, n, n), q_inv_zeta, ta=True, beta=1.0)  # + G_k^T Q_k^{-1} zeta_k
    if N > 1:
        gemm(diag[:-1], G[1:], q_inv_g[1:], ta=True, beta=1.0)  # + G_{k+1}^T Q^{-1} G_{k+1}
    sub = torch.neg(q_inv_g[1:])
    return diag, sub, rhs


def _white(Lr, H, nb, trsm):
    """R^{-1/2} H = L_R^{-1} H over nb members (a fresh copy; H untouched)."""
    out = (H.expand(nb, *H.shape[1:]) if H.shape[0] != nb else H).clone()
    trsm(Lr, out, False)
    return out


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
