"""Recursive Schur-complement factor/solve on B200 (drop-in for `blocktri.schur`,
/root/reference/pkg/src/blocktri/schur.py).

``recursive_factorize`` / ``recursive_solve`` keep the reference signatures, argument meaning,
ownership rules (input matrix and rhs never mutated; the hierarchy is immutable after the factor
and safe for concurrent solves) and error behaviour (NotPositiveDefinite with level-local
coordinates, LevelOverflow, DimensionMismatch).  All arithmetic runs in the sm_100a kernels of
``libblocktri_b200.so`` behind the C ABI in include/blocktri_b200.h; this module only plans,
allocates device memory through torch's caching allocator and maps status codes to exceptions.
"""

from __future__ import annotations

import contextlib
import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .core import BlockRhs, BlockTridiagonalMatrix, FactorHierarchy, PartitionPlan, _is_torch
from .errors import DeviceError, DimensionMismatch, LevelOverflow, NotPositiveDefinite


@dataclass(frozen=True)
class RecursionConfig:
    """Tuning knobs of the recursive reduction (schur.py:43-64)."""

    crossover: int = 64
    segment_length: int = 8
    max_levels: int = 32
    auto_crossover: bool = False

    def __post_init__(self):
        if self.crossover < 1 or self.segment_length < 1 or self.max_levels < 1:
            raise ValueError("crossover, segment_length and max_levels must be >= 1")

    def _c(self) -> _native.BtdConfig:
        return _native.BtdConfig(int(self.crossover), int(self.segment_length), int(self.max_levels),
                                 1 if self.auto_crossover else 0, 0)


class FactorLevel:
    """One recursion level: its partition (schur.py:67-72). The factor blocks stay on the device.

    ``plan`` is materialised lazily (a 2^20-block level has ~10^5 separators; building the
    Python tuples eagerly would dominate the host time of a factorization)."""

    def __init__(self, num_blocks: int, num_separators: int, level: int, native):
        self.num_blocks = num_blocks
        self.num_separators = num_separators
        self.level = level
        self._native = native  # keeps the C handle alive for the lazy separator fetch
        self._seps = None
        self._plan = None

    @property
    def separators(self) -> np.ndarray:
        """Separator block indices of this level (fetched from the C plan on first use)."""
        if self._seps is None:
            seps = np.empty(self.num_separators, dtype=np.int64)
            _native.lib().btd_level_info(self._native.handle, self.level, None, None,
                                         seps.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
            self._seps = seps
        return self._seps

    @property
    def plan(self) -> PartitionPlan:
        if self._plan is None:
            self._plan = _plan_from_separators(self.num_blocks, self.separators.tolist())
        return self._plan

    def __repr__(self):
        return f"FactorLevel(level={self.level}, num_blocks={self.num_blocks}, separators={self.num_separators})"


@dataclass
class BaseFactor:
    """The serially factored base system (reference: FactorHierarchy.base, core.py:172)."""

    num_blocks: int
    block_size: int


def _plan_from_separators(num_blocks: int, seps) -> PartitionPlan:
    seps = tuple(int(s) for s in seps)
    segments = tuple((a + 1, b) for a, b in zip(seps, seps[1:]))
    return PartitionPlan(num_blocks, seps, segments)


def plan_partition(num_blocks: int, config: RecursionConfig) -> PartitionPlan:
    """Separators for one level (schur.py:75-95), computed by the native planner (bit-exact)."""
    L = _native.lib()
    st = _native.BtdStatus()
    cnt = ctypes.c_int64()
    cfg = config._c()
    rc = L.btd_plan_separators(int(num_blocks), ctypes.byref(cfg), None, ctypes.byref(cnt), ctypes.byref(st))
    if rc != _native.BTD_OK:
        raise ValueError(st.message.decode())
    out = (ctypes.c_int64 * cnt.value)()
    L.btd_plan_separators(int(num_blocks), ctypes.byref(cfg), out, ctypes.byref(cnt), ctypes.byref(st))
    plan = _plan_from_separators(num_blocks, out)
    plan.validate()
    return plan


def _raise_status(st: _native.BtdStatus, rc: int):
    msg = st.message.decode(errors="replace")
    if rc == _native.BTD_ERR_NOT_POSITIVE_DEFINITE:
        raise NotPositiveDefinite(int(st.pivot), level=int(st.level), member=int(st.member), block=int(st.block))
    if rc == _native.BTD_ERR_LEVEL_OVERFLOW:
        raise LevelOverflow(msg)
    if rc == _native.BTD_ERR_DIMENSION_MISMATCH:
        raise DimensionMismatch(msg)
    if rc in (_native.BTD_ERR_INVALID_ARGUMENT, _native.BTD_ERR_NOT_FACTORED):
        raise ValueError(msg)
    if rc == _native.BTD_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise DeviceError(msg)


class NativeFactor:
    """Owns the C handle and the device memory of one factorization."""

    def __init__(self, handle, persistent, device):
        self.handle = handle
        self.persistent = persistent
        self.device = device

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _native.lib().btd_destroy(h)
            except Exception:
                pass
            self.handle = None


def _device_matrix(matrix: BlockTridiagonalMatrix):
    import torch
    N, n = matrix.num_blocks, matrix.block_size
    if _is_torch(matrix.diag):
        dev = matrix.diag.device
        if dev.type != "cuda":
            diag = matrix.diag.to("cuda", non_blocking=True)
            sub = matrix.sub.to("cuda", non_blocking=True)
        else:
            diag, sub = matrix.diag, matrix.sub
        diag = diag.to(torch.float64).contiguous()
        sub = sub.to(torch.float64).contiguous()
    else:
        diag = torch.from_numpy(np.ascontiguousarray(matrix.diag, dtype=np.float64)).to("cuda")
        sub = torch.from_numpy(np.ascontiguousarray(matrix.sub, dtype=np.float64)).to("cuda")
    if tuple(diag.shape) != (N, n, n) or tuple(sub.shape) != (max(N - 1, 0), n, n):
        raise DimensionMismatch(f"matrix arenas {tuple(diag.shape)}, {tuple(sub.shape)} do not match (N={N}, n={n})")
    return diag, sub


def _host_matrix(matrix: BlockTridiagonalMatrix):
    """(diag ptr, sub ptr, keep-alive) for host-resident float64 contiguous arenas, else None."""
    N, n = matrix.num_blocks, matrix.block_size
    if _is_torch(matrix.diag):
        if matrix.diag.device.type != "cpu":
            return None
        import torch
        d = matrix.diag.to(torch.float64).contiguous()
        s = matrix.sub.to(torch.float64).contiguous()
        if tuple(d.shape) != (N, n, n) or tuple(s.shape) != (max(N - 1, 0), n, n):
            raise DimensionMismatch(f"matrix arenas {tuple(d.shape)}, {tuple(s.shape)} do not match (N={N}, n={n})")
        return d.data_ptr(), s.data_ptr(), (d, s)
    d = np.ascontiguousarray(matrix.diag, dtype=np.float64)
    s = np.ascontiguousarray(matrix.sub, dtype=np.float64)
    if d.shape != (N, n, n) or s.shape != (max(N - 1, 0), n, n):
        raise DimensionMismatch(f"matrix arenas {d.shape}, {s.shape} do not match (N={N}, n={n})")
    return d.ctypes.data, s.ctypes.data, (d, s)


def _padded_size(n: int) -> int:
    """Block size the kernels run at: n itself for n <= 64 (the level kernels pad in shared memory)
    and for multiples of 64 (tiled path); otherwise the next multiple of 64.  A block padded with
    an identity diagonal and zero couplings factors into the embedded original factor exactly (the
    extra terms are exact zeros), so results and NPD coordinates are those of the n x n system."""
    return n if n <= 64 or n % 64 == 0 else (n + 63) // 64 * 64


def _pad_matrix(diag, sub, n: int, npad: int):
    """Device arenas of size npad: identity on the padded diagonal, zero padded couplings."""
    import torch
    N = diag.shape[0]
    dp = torch.zeros((N, npad, npad), dtype=torch.float64, device=diag.device)
    dp[:, :n, :n] = diag
    idx = torch.arange(n, npad, device=diag.device)
    dp[:, idx, idx] = 1.0
    sp = torch.zeros((sub.shape[0], npad, npad), dtype=torch.float64, device=diag.device)
    sp[:, :n, :n] = sub
    return dp, sp


@contextlib.contextmanager
def _on_stream(device, stream):
    """Run the body with ``device`` current and every torch op / native launch on ``stream``.

    The stream waits for the caller's current stream on entry (inputs it produced) and the caller's
    current stream waits for ``stream`` on exit (outputs and the freed scratch), so passing a
    non-current stream is safe in both directions; the caching allocator attributes every
    temporary to ``stream``."""
    import torch
    if stream is None and device.index == torch.cuda.current_device():
        # the common call: nothing to switch (entering torch's stream context costs ~10 us of host
        # time, on the critical path between a factorization's error check and the solve launch)
        yield torch.cuda.current_stream(device)
        return
    with torch.cuda.device(device):
        cur = torch.cuda.current_stream(device)
        s = stream if stream is not None else cur
        if s != cur:
            s.wait_stream(cur)
        with torch.cuda.stream(s):
            yield s
        if s != cur:
            cur.wait_stream(s)


def _matrix_device(matrix: BlockTridiagonalMatrix):
    import torch
    if _is_torch(matrix.diag) and matrix.diag.device.type == "cuda":
        return matrix.diag.device
    return torch.device("cuda", torch.cuda.current_device())


def recursive_factorize(matrix: BlockTridiagonalMatrix, config: RecursionConfig | None = None,
                        *, stream=None, profile: bool = False) -> FactorHierarchy:
    """Factor an SPD block-tridiagonal system for repeated solves (schur.py:289-318).

    Never mutates ``matrix``. Raises NotPositiveDefinite(pivot, level, member, block) with the
    reference's level-local coordinates, LevelOverflow past ``max_levels``.  ``stream`` (optional)
    is the CUDA stream the work is ordered on (default: the current stream of the matrix's device).
    """
    with _on_stream(_matrix_device(matrix), stream) as s:
        return _factorize_on(matrix, config, s, profile)


def _factorize_on(matrix, config, s, profile, keep_scratch=False):
    import torch
    cfg = config or RecursionConfig()
    L = _native.lib()
    N, n_user = matrix.num_blocks, matrix.block_size
    n = _padded_size(n_user)
    st = _native.BtdStatus()
    handle = ctypes.c_void_p()
    c = cfg._c()
    rc = L.btd_create(N, n, ctypes.byref(c), ctypes.byref(handle), ctypes.byref(st))
    if rc != _native.BTD_OK:
        _raise_status(st, rc)
    host = _host_matrix(matrix) if n == n_user else None
    if host is None:
        diag, sub = _device_matrix(matrix)
        if n != n_user:
            diag, sub = _pad_matrix(diag, sub, n_user, n)
    else:  # host-resident input: the C ABI overlaps the H2D copy with the level-0 elimination
        diag = torch.empty((N, n, n), dtype=torch.float64, device=s.device)
        sub = torch.empty((max(N - 1, 0), n, n), dtype=torch.float64, device=s.device)
    pers_b, scr_b = ctypes.c_size_t(), ctypes.c_size_t()
    L.btd_factor_workspace(handle, ctypes.byref(pers_b), ctypes.byref(scr_b))
    dev = diag.device
    persistent = torch.empty(pers_b.value, dtype=torch.uint8, device=dev)
    scratch = torch.empty(scr_b.value, dtype=torch.uint8, device=dev)
    native = NativeFactor(handle, persistent, dev)
    native.padded = n  # kernel block size (> n_user when padded)
    if profile:
        L.btd_profile_kernels(handle, 1)
    if host is None:
        rc = L.btd_factorize(handle, diag.data_ptr(), sub.data_ptr() if N > 1 else None, persistent.data_ptr(),
                             scratch.data_ptr(), ctypes.c_void_p(s.cuda_stream), 1, ctypes.byref(st))
    else:
        hd, hs, _keep = host
        rc = L.btd_factorize_from_host(handle, hd, hs if N > 1 else None, diag.data_ptr(),
                                       sub.data_ptr() if N > 1 else None, persistent.data_ptr(),
                                       scratch.data_ptr(), ctypes.c_void_p(s.cuda_stream), 1, ctypes.byref(st))
    if keep_scratch:
        native.scratch = scratch
    del scratch
    if rc != _native.BTD_OK:
        _raise_status(st, rc)
    nl, nb, ov = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
    L.btd_num_levels(handle, ctypes.byref(nl), ctypes.byref(nb), ctypes.byref(ov))
    levels = []
    for lvl in range(nl.value):
        lnb, lp = ctypes.c_int64(), ctypes.c_int64()
        L.btd_level_info(handle, lvl, ctypes.byref(lnb), ctypes.byref(lp), None)
        levels.append(FactorLevel(lnb.value, lp.value, lvl, native))
    return FactorHierarchy(N, n_user, levels, BaseFactor(nb.value, n_user), native)


def recursive_solve(hierarchy: FactorHierarchy, rhs: BlockRhs, *, stream=None) -> BlockRhs:
    """Solve against a stored factorization (schur.py:346-359).

    Neither the hierarchy nor ``rhs`` is mutated.  numpy rhs -> numpy solution (host round
    trip); torch CUDA rhs -> torch CUDA solution (device resident).  ``stream`` as in
    recursive_factorize.
    """
    native = hierarchy._native
    if native is None or not native.handle:
        raise ValueError("hierarchy must be factorized before solving")
    with _on_stream(native.device, stream) as s:
        return _solve_on(hierarchy, rhs, s)


def _solve_on(hierarchy, rhs, s):
    import torch
    if rhs.num_blocks != hierarchy.num_blocks or rhs.block_size != hierarchy.block_size:
        raise DimensionMismatch(
            f"rhs ({rhs.num_blocks}, {rhs.block_size}) not conformal with "
            f"hierarchy ({hierarchy.num_blocks}, {hierarchy.block_size})")
    native = hierarchy._native
    if native is None or not native.handle:
        raise ValueError("hierarchy must be factorized before solving")
    L = _native.lib()
    host = not _is_torch(rhs.blocks)
    host_tensor = (not host) and rhs.blocks.device.type == "cpu"
    if host:
        b = torch.from_numpy(np.ascontiguousarray(rhs.blocks, dtype=np.float64)).to(native.device, non_blocking=True)
    else:
        b = rhs.blocks
        if b.device != native.device:
            b = b.to(native.device, non_blocking=True)
        if b.dtype != torch.float64 or not b.is_contiguous():
            b = b.to(torch.float64).contiguous()
    d = int(b.shape[2])
    npad = getattr(native, "padded", hierarchy.block_size)
    nu = hierarchy.block_size
    if npad != nu:  # zero rows for the padded unknowns; the solution is the leading n rows
        bp = torch.zeros((b.shape[0], npad, d), dtype=torch.float64, device=b.device)
        bp[:, :nu] = b
        b = bp
    x = torch.empty_like(b)
    scr_b = ctypes.c_size_t()
    L.btd_solve_workspace(native.handle, d, ctypes.byref(scr_b))
    scratch = torch.empty(scr_b.value, dtype=torch.uint8, device=native.device)
    st = _native.BtdStatus()
    rc = L.btd_solve(native.handle, b.data_ptr(), x.data_ptr(), d, scratch.data_ptr(),
                     ctypes.c_void_p(s.cuda_stream), ctypes.byref(st))
    if rc != _native.BTD_OK:
        _raise_status(st, rc)
    if npad != nu:
        x = x[:, :nu].contiguous()
    if host or host_tensor:
        # D2H into pinned memory (torch's caching host allocator): a pageable destination runs at a
        # fraction of the link bandwidth
        out = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        out.copy_(x, non_blocking=True)
        s.synchronize()
        return BlockRhs(out.numpy() if host else out)
    return BlockRhs(x)


def factor_kernel_times(matrix: BlockTridiagonalMatrix, config: RecursionConfig | None = None,
                        repeats: int = 3, rhs_cols: int = 1) -> dict:
    """Bench helper: median (over ``repeats``) device times of factor, solve (``rhs_cols``
    right-hand sides) and the level-0 factor kernel (CUDA events on the launching stream, C-ABI
    timing hook)."""
    import statistics

    import torch
    f_ms, s_ms, l0 = [], [], []
    rhs = BlockRhs(torch.ones((matrix.num_blocks, matrix.block_size, rhs_cols), dtype=torch.float64,
                              device=matrix.diag.device))
    h = None
    for _ in range(repeats):
        h = None  # release the previous factor before the next one is allocated
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        h = recursive_factorize(matrix, config, profile=True)
        e[1].record()
        recursive_solve(h, rhs)
        e[2].record()
        torch.cuda.synchronize()
        f_ms.append(e[0].elapsed_time(e[1]))
        s_ms.append(e[1].elapsed_time(e[2]))
        L = _native.lib()
        cnt = ctypes.c_int64()
        out = (ctypes.c_float * 64)()
        L.btd_kernel_times(h._native.handle, out, 64, ctypes.byref(cnt))
        l0.append(out[0])
    return {"factor_ms": statistics.median(f_ms), "solve_ms": statistics.median(s_ms),
            "level0_factor_ms": statistics.median(l0)}


def level_schur(matrix: BlockTridiagonalMatrix, level: int, config: RecursionConfig | None = None):
    """Debug view: the next-level Schur complement system (diag, sub) that level ``level`` of the
    recursion hands to level ``level + 1`` -- what the reference's ``compute_schur`` + ``new_btd``
    return (schur.py:156-193) -- as device tensors of the user's block size."""
    import torch
    with _on_stream(_matrix_device(matrix), None) as s:
        h = _factorize_on(matrix, config, s, False, keep_scratch=True)
        native = h._native
        if not 0 <= level < len(h.levels):
            raise ValueError(f"level {level} outside [0, {len(h.levels)})")
        P = h.levels[level].num_separators
        n = getattr(native, "padded", h.block_size)
        diag = torch.empty((P, n, n), dtype=torch.float64, device=native.device)
        sub = torch.empty((max(P - 1, 1), n, n), dtype=torch.float64, device=native.device)
        st = _native.BtdStatus()
        rc = _native.lib().btd_level_schur(native.handle, level, native.scratch.data_ptr(), diag.data_ptr(),
                                           sub.data_ptr(), ctypes.c_void_p(s.cuda_stream), ctypes.byref(st))
        if rc != _native.BTD_OK:
            _raise_status(st, rc)
        nu = h.block_size
        return diag[:, :nu, :nu], sub[:max(P - 1, 0), :nu, :nu]


def level_factor(hierarchy: FactorHierarchy, level: int):
    """Debug view: (Linv, Lsub) device tensors of one level (level == len(levels) is the base)."""
    import torch
    native = hierarchy._native
    L = _native.lib()
    nu = hierarchy.block_size
    n = getattr(native, "padded", nu)
    N = hierarchy.base.num_blocks if level == len(hierarchy.levels) else hierarchy.levels[level].num_blocks
    linv = torch.empty((N, n, n), dtype=torch.float64, device=native.device)
    lsub = torch.empty((max(N - 1, 0), n, n), dtype=torch.float64, device=native.device)
    st = _native.BtdStatus()
    rc = L.btd_level_factor(native.handle, level, linv.data_ptr(), lsub.data_ptr() if N > 1 else None,
                            ctypes.c_void_p(torch.cuda.current_stream(native.device).cuda_stream), ctypes.byref(st))
    if rc != _native.BTD_OK:
        _raise_status(st, rc)
    return linv[:, :nu, :nu], lsub[:, :nu, :nu]
