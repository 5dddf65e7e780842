"""CPU ORACLE -- test infrastructure only.

A numpy restatement of the reference hot path (arXiv 2509.03015 reference package `blocktri`,
/root/reference/pkg/src/blocktri, "bt/" below): the F-form recursive Schur-complement factor and
solve, with the reference's dense kernels (LAPACK potrf through numpy, row-sweep trsm, BLAS gemm)
and its thread-pool member chunking.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module, and only as the checker or the
timed CPU baseline -- never as the product path.

Pinned against the reference itself: tests/golden/make_golden.py runs the real reference in the
build container and stores its outputs (solutions, level-0 Schur complements, plans, error
coordinates) in tests/golden/*.npz; tests/test_oracle_golden.py checks this port against them.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np


class OracleNPD(Exception):
    """Mirror of NotPositiveDefinite (bt/errors.py:31-68): 1-based pivot + level-local coords."""

    def __init__(self, pivot, level=None, member=None, block=None):
        super().__init__(f"pivot {pivot} block {block} member {member} level {level}")
        self.pivot, self.level, self.member, self.block = pivot, level, member, block


class OracleLevelOverflow(Exception):
    """Mirror of LevelOverflow (bt/errors.py:89-90)."""


# ------------------------------------------------------------------------------------------
# partition plan: bt/schur.py:75-95 ; recursion test: bt/schur.py:321-326
# ------------------------------------------------------------------------------------------
def plan_separators(num_blocks: int, rho: int) -> list[int]:
    if num_blocks < 3:
        raise ValueError(f"cannot partition fewer than 3 block rows, got {num_blocks}")
    seps = list(range(0, num_blocks, rho + 1))
    if seps[-1] != num_blocks - 1:
        if seps[-1] == num_blocks - 2:
            seps.pop()
        seps.append(num_blocks - 1)
    return seps


def should_recurse(num_blocks: int, crossover: int, rho: int, auto: bool) -> bool:
    if num_blocks < 3:
        return False
    if auto:
        return len(plan_separators(num_blocks, rho)) - 1 >= 2
    return num_blocks > crossover


# ------------------------------------------------------------------------------------------
# dense kernels: bt/kernels.py
# ------------------------------------------------------------------------------------------
def _threads() -> int:
    env = os.environ.get("BLOCKTRI_THREADS", "").strip()
    if env:
        try:
            return max(1, int(env))
        except ValueError:
            pass
    return min(8, os.cpu_count() or 1)


_POOL: ThreadPoolExecutor | None = None


def _chunked(fn, count: int, elems: int, threads: int | None = None) -> None:
    """Member chunking over a thread pool (bt/kernels.py:72-101); failures remapped, lowest wins."""
    global _POOL
    cap = _threads() if threads is None else threads
    if cap <= 1 or count < 2 * cap or count * elems < (1 << 15):
        fn(0, count)
        return
    if _POOL is None or _POOL._max_workers < cap:
        _POOL = ThreadPoolExecutor(max_workers=cap)
    edges = np.linspace(0, count, cap + 1).astype(int)
    futs = [(lo, _POOL.submit(fn, lo, hi)) for lo, hi in zip(edges[:-1], edges[1:]) if hi > lo]
    errs = []
    for lo, f in futs:
        e = f.exception()
        if e is not None:
            if isinstance(e, OracleNPD) and e.member is not None:
                e = OracleNPD(e.pivot, e.level, e.member + lo, e.block)
            errs.append(((e.member if isinstance(e, OracleNPD) and e.member is not None else lo), e))
    if errs:
        errs.sort(key=lambda t: t[0])
        raise errs[0][1]


def first_bad_pivot(block: np.ndarray) -> int:
    """Naive elimination locating the first non-positive pivot (bt/kernels.py:136-152)."""
    a = np.array(block, dtype=np.float64)
    for j in range(a.shape[0]):
        d = a[j, j]
        if not (d > 0.0) or not np.isfinite(d):
            return j + 1
        col = a[j + 1:, j] / np.sqrt(d)
        a[j + 1:, j + 1:] -= np.outer(col, col)
    return 0


def potrf_batch(blocks: np.ndarray) -> None:
    """In-place lower Cholesky of each member, strict upper zeroed (bt/kernels.py:164-181)."""
    def body(lo, hi):
        v = blocks[lo:hi]
        try:
            v[:] = np.linalg.cholesky(v)
        except np.linalg.LinAlgError:
            for m in range(v.shape[0]):
                p = first_bad_pivot(v[m])
                if p:
                    raise OracleNPD(p, member=m) from None
            raise OracleNPD(v.shape[1], member=v.shape[0] - 1) from None
    _chunked(body, blocks.shape[0], blocks.shape[1] * blocks.shape[2])


def _fwd_rows(f, p, lo, hi):
    for i in range(lo, hi):
        if i > lo:
            p[:, i, :] -= np.matmul(f[:, i:i + 1, lo:i], p[:, lo:i, :])[:, 0, :]
        p[:, i, :] /= f[:, i, i, None]


def _bwd_rows(f, p, lo, hi):
    for i in range(hi - 1, lo - 1, -1):
        if i < hi - 1:
            p[:, i, :] -= np.matmul(f[:, i + 1:hi, i][:, None, :], p[:, i + 1:hi, :])[:, 0, :]
        p[:, i, :] /= f[:, i, i, None]


def trsm_batch(factors: np.ndarray, panels: np.ndarray, trans: bool = False) -> None:
    """panels <- L^{-1} panels (or L^{-T}); unblocked row sweeps for n <= 64, 32-wide tiles above
    (bt/kernels.py:199-259)."""
    n = factors.shape[1]

    def body(lo_k, hi_k):
        f, p = factors[lo_k:hi_k], panels[lo_k:hi_k]
        if not trans:
            if n <= 64:
                _fwd_rows(f, p, 0, n)
            else:
                for lo in range(0, n, 32):
                    hi = min(lo + 32, n)
                    if lo:
                        p[:, lo:hi, :] -= np.matmul(f[:, lo:hi, :lo], p[:, :lo, :])
                    _fwd_rows(f, p, lo, hi)
        else:
            if n <= 64:
                _bwd_rows(f, p, 0, n)
            else:
                for hi in range(n, 0, -32):
                    lo = max(hi - 32, 0)
                    if hi < n:
                        p[:, lo:hi, :] -= np.matmul(f[:, hi:, lo:hi].transpose(0, 2, 1), p[:, hi:, :])
                    _bwd_rows(f, p, lo, hi)
    _chunked(body, factors.shape[0], n * panels.shape[2])


def gemm_batch(out, a, b, ta=False, tb=False, alpha=1.0, beta=0.0) -> None:
    """out <- alpha op(a) op(b) + beta out (bt/kernels.py:270-310)."""
    oa = a.transpose(0, 2, 1) if ta else a
    ob = b.transpose(0, 2, 1) if tb else b

    def body(lo, hi):
        c = out[lo:hi]
        if alpha == 0.0:
            if beta == 0.0:
                c[:] = 0.0
            elif beta != 1.0:
                c *= beta
            return
        prod = np.matmul(oa[lo:hi], ob[lo:hi])
        if alpha != 1.0:
            prod *= alpha
        if beta == 0.0:
            c[:] = prod
        else:
            if beta != 1.0:
                c *= beta
            c += prod
    _chunked(body, out.shape[0], oa.shape[1] * oa.shape[2] + ob.shape[1] * ob.shape[2])


# ------------------------------------------------------------------------------------------
# block sweeps: bt/block_cholesky.py:24-57
# ------------------------------------------------------------------------------------------
def block_factor(diag: np.ndarray, sub: np.ndarray) -> None:
    """Alg. 1 over (K, J, n, n) / (K, J-1, n, n) arenas, in place (bt/block_cholesky.py:24-42)."""
    J = diag.shape[1]
    for j in range(J):
        if j > 0:
            c = sub[:, j - 1]
            trsm_batch(diag[:, j - 1], c.transpose(0, 2, 1))  # L_{j,j-1} = A_{j,j-1} L^{-T}
            gemm_batch(diag[:, j], c, c, tb=True, alpha=-1.0, beta=1.0)
        try:
            potrf_batch(diag[:, j])
        except OracleNPD as e:
            raise OracleNPD(e.pivot, member=e.member, block=j) from None


def block_solve(diag: np.ndarray, sub: np.ndarray, rhs: np.ndarray) -> None:
    """Alg. 2 forward/backward block substitution, in place (bt/block_cholesky.py:45-57)."""
    J = diag.shape[1]
    trsm_batch(diag[:, 0], rhs[:, 0])
    for j in range(1, J):
        gemm_batch(rhs[:, j], sub[:, j - 1], rhs[:, j - 1], alpha=-1.0, beta=1.0)
        trsm_batch(diag[:, j], rhs[:, j])
    trsm_batch(diag[:, J - 1], rhs[:, J - 1], trans=True)
    for j in range(J - 2, -1, -1):
        gemm_batch(rhs[:, j], sub[:, j], rhs[:, j + 1], ta=True, alpha=-1.0, beta=1.0)
        trsm_batch(diag[:, j], rhs[:, j], trans=True)


# ------------------------------------------------------------------------------------------
# one recursion level: permute_split (bt/schur.py:98-138), _coupling_panels (:141-153),
# factor + F panels (:329-343), compute_schur (:156-193)
# ------------------------------------------------------------------------------------------
def factor_level(diag: np.ndarray, sub: np.ndarray, rho: int, level: int):
    N, n = diag.shape[0], diag.shape[1]
    seps = plan_separators(N, rho)
    seg = [(a + 1, b) for a, b in zip(seps, seps[1:])]
    K = len(seg)
    lengths = np.array([b - a for a, b in seg], dtype=np.int64)
    J = int(lengths.max())
    D = np.broadcast_to(np.eye(n), (K, J, n, n)).copy()
    S = np.zeros((K, max(J - 1, 0), n, n))
    CL = np.empty((K, n, n))
    CR = np.empty((K, n, n))
    for k, (a, b) in enumerate(seg):
        D[k, :b - a] = diag[a:b]
        if b - a > 1:
            S[k, :b - a - 1] = sub[a:b - 1]
        CL[k] = sub[a - 1]
        CR[k] = sub[b - 1]
    try:
        block_factor(D, S)
    except OracleNPD as e:
        raise OracleNPD(e.pivot, level=level, member=e.member, block=e.block) from None
    F = np.zeros((K, J, n, 2 * n))
    F[:, 0, :, :n] = CL
    F[np.arange(K), lengths - 1, :, n:] = CR.transpose(0, 2, 1)
    block_solve(D, S, F)
    top = np.empty((K, n, 2 * n))
    gemm_batch(top, CL, F[:, 0], ta=True)
    bottom = np.empty((K, n, 2 * n))
    gemm_batch(bottom, CR, F[np.arange(K), lengths - 1])
    sdiag = diag[seps].copy()
    sdiag[:-1] -= top[:, :, :n]
    sdiag[1:] -= bottom[:, :, n:]
    ssub = -bottom[:, :, :n]
    sdiag = (sdiag + sdiag.transpose(0, 2, 1)) / 2.0  # new_btd symmetrisation (bt/core.py:211)
    rec = dict(seps=seps, seg=seg, lengths=lengths, D=D, S=S, CL=CL, CR=CR, F=F)
    return rec, sdiag, ssub


def factorize(diag, sub, crossover=64, rho=8, max_levels=32, auto=False):
    """recursive_factorize (bt/schur.py:289-318).  Returns a dict hierarchy."""
    levels = []
    cd, cs = diag, sub
    while True:
        lvl = len(levels)
        if not should_recurse(cd.shape[0], crossover, rho, auto):
            bd = cd.copy()[None]
            bs = cs.copy()[None]
            try:
                block_factor(bd, bs)
            except OracleNPD as e:
                raise OracleNPD(e.pivot, level=lvl, member=0, block=e.block) from None
            return dict(levels=levels, base=(bd, bs), N=diag.shape[0], n=diag.shape[1])
        if lvl >= max_levels:
            raise OracleLevelOverflow(f"recursion needs more than max_levels={max_levels} levels")
        rec, cd, cs = factor_level(cd, cs, rho, lvl)
        levels.append(rec)


def solve(h, rhs: np.ndarray) -> np.ndarray:
    """recursive_solve (bt/schur.py:346-374): split, fold (Alg. 5), recurse, boundary (Alg. 6),
    interior sweep, assemble."""
    return _solve_level(h, 0, rhs.copy())


def _solve_level(h, level, b):
    if level == len(h["levels"]):
        bd, bs = h["base"]
        x = b.copy()[None]
        block_solve(bd, bs, x)
        return x[0]
    r = h["levels"][level]
    seps, seg, lengths, F = r["seps"], r["seg"], r["lengths"], r["F"]
    K, J, n = F.shape[0], F.shape[1], F.shape[2]
    d = b.shape[2]
    interior = np.zeros((K, J, n, d))
    for k, (a, c) in enumerate(seg):
        interior[k, :c - a] = b[a:c]
    bsep = b[seps].copy()
    contrib = np.empty((K, 2 * n, d))
    gemm_batch(contrib, F.reshape(K, J * n, 2 * n), interior.reshape(K, J * n, d), ta=True, alpha=-1.0)
    bsep[:-1] += contrib[:, :n]
    bsep[1:] += contrib[:, n:]
    xsep = _solve_level(h, level + 1, bsep)
    gemm_batch(interior[:, 0], r["CL"], xsep[:-1], alpha=-1.0, beta=1.0)
    idx = np.arange(K)
    last = interior[idx, lengths - 1]
    gemm_batch(last, r["CR"], xsep[1:], ta=True, alpha=-1.0, beta=1.0)
    interior[idx, lengths - 1] = last
    block_solve(r["D"], r["S"], interior)
    out = np.empty_like(b)
    out[seps] = xsep
    for k, (a, c) in enumerate(seg):
        out[a:c] = interior[k, :c - a]
    return out


def schur_level0(diag, sub, rho=8):
    """Level-0 Schur complement (diag, sub) as the reference compute_schur builds it."""
    _, sd, ss = factor_level(diag, sub, rho, 0)
    return sd, ss


def level_schur(diag, sub, level, crossover=64, rho=8):
    """The Schur system level `level` hands to level + 1 (bt/schur.py:329-343 iterated)."""
    cd, cs = diag, sub
    for lvl in range(level + 1):
        if not should_recurse(cd.shape[0], crossover, rho, False):
            raise ValueError(f"level {lvl} does not recurse")
        _, cd, cs = factor_level(cd, cs, rho, lvl)
    return cd, cs


# ------------------------------------------------------------------------------------------
# dense checks: bt/oracle.py:26-74, bt/core.py:262-288, bt/report.py:20-38
# ------------------------------------------------------------------------------------------
def assemble_dense(diag, sub) -> np.ndarray:
    N, n = diag.shape[0], diag.shape[1]
    A = np.zeros((N * n, N * n))
    for i in range(N):
        A[i * n:(i + 1) * n, i * n:(i + 1) * n] = diag[i]
    for i in range(N - 1):
        A[(i + 1) * n:(i + 2) * n, i * n:(i + 1) * n] = sub[i]
        A[i * n:(i + 1) * n, (i + 1) * n:(i + 2) * n] = sub[i].T
    return A


def btd_matmul(diag, sub, x) -> np.ndarray:
    y = np.matmul(diag, x)
    if diag.shape[0] > 1:
        y[1:] += np.matmul(sub, x[:-1])
        y[:-1] += np.matmul(sub.transpose(0, 2, 1), x[1:])
    return y


def residual(diag, sub, x, b) -> tuple[float, float]:
    d = b.shape[2]
    r = (b - btd_matmul(diag, sub, x)).reshape(-1, d)
    rn = np.linalg.norm(r, axis=0)
    bn = np.linalg.norm(b.reshape(-1, d), axis=0)
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(bn > 0, rn / bn, np.where(rn > 0, np.inf, 0.0))
    return float(rn.max()), float(ratio.max())
