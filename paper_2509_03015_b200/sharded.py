"""Multi-GPU sharded factor/solve of one N-block chain.

The chain is cut into G contiguous chunks at level-L separators (global indices that are
multiples of (rho+1)^L), so every chunk's own plan for its first L levels is exactly the global
plan restricted to the chunk -- separator indexing stays bit-exact (checked by `shard_plan`).
Chunk g eliminates its interiors through L levels with no communication; the reduced system over
all level-L separators (P_L blocks, ~N/(rho+1)^L) is all-gathered -- the two partial Schur
diagonals of each shared boundary separator are summed in rank order -- and factored
redundantly on every rank with the ordinary recursion (whose plan is the global plan from level
L on).  The solve folds locally, all-gathers the reduced rhs partials, solves the reduced system
redundantly and back-substitutes locally: one all-gather per phase, no scatter.

A shared boundary block (diagonal block / rhs panel of separator b_g = a_{g+1}) is owned by the
left chunk; the right chunk passes zeros for it.

`engine` performs the per-rank linear algebra: `CudaEngine` (the sm_100a kernels through the C
ABI) is the product engine; tests inject a CPU restatement to check the host logic with gloo.
`comm` is `torch.distributed` (NCCL on B200, gloo in the CPU tests) or `LocalComm`, which plays all
ranks in one process.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native


def _seps(N: int, rho: int) -> list[int]:
    """plan_partition separators (bt/schur.py:75-95)."""
    s = list(range(0, N, rho + 1))
    if s[-1] != N - 1:
        if s[-1] == N - 2:
            s.pop()
        s.append(N - 1)
    return s


def global_level_sizes(N: int, crossover: int = 64, rho: int = 8) -> list[int]:
    sizes, cur = [], N
    while cur >= 3 and cur > crossover:
        sizes.append(cur)
        cur = len(_seps(cur, rho))
    return sizes + [cur]


def _local_plans(a: int, b: int, L: int, rho: int) -> list[list[int]]:
    """Global-index separators of chunk [a, b] after each of its L local levels."""
    idx = list(range(a, b + 1))
    out = []
    for _ in range(L):
        loc = _seps(len(idx), rho)
        idx = [idx[i] for i in loc]
        out.append(idx)
    return out


def _global_plans(N: int, L: int, rho: int) -> list[list[int]]:
    idx = list(range(N))
    out = []
    for _ in range(L):
        loc = _seps(len(idx), rho)
        idx = [idx[i] for i in loc]
        out.append(idx)
    return out


@dataclass
class ShardPlan:
    N: int
    G: int
    L: int                      # local levels per chunk
    cuts: list                  # c_0 = 0 < c_1 < ... < c_G = N - 1 ; chunk g = [c_g, c_{g+1}]
    reduced_sizes: list = field(default_factory=list)   # P_g (separators of chunk g after L levels)
    offsets: list = field(default_factory=list)         # first reduced index of chunk g
    reduced_N: int = 0
    crossover: int = 64         # RecursionConfig the cuts were planned for (the reduced sizes
    rho: int = 8                # depend on segment_length; the solver config must match)

    def config(self, config=None):
        """The RecursionConfig of this plan; a given ``config`` must agree with it."""
        from .schur import RecursionConfig
        if config is None:
            return RecursionConfig(crossover=self.crossover, segment_length=self.rho)
        if config.segment_length != self.rho or config.crossover != self.crossover or config.auto_crossover:
            raise ValueError(f"config (crossover={config.crossover}, segment_length={config.segment_length}, "
                             f"auto={config.auto_crossover}) differs from the shard plan's "
                             f"(crossover={self.crossover}, segment_length={self.rho})")
        return config

    def chunk(self, g: int) -> tuple[int, int]:
        return self.cuts[g], self.cuts[g + 1]


def shard_plan(N: int, G: int, crossover: int = 64, rho: int = 8, L: int | None = None) -> ShardPlan:
    """Cut points on the level-L separator grid, with a bit-exactness check of every chunk plan."""
    sizes = global_level_sizes(N, crossover, rho)
    levels = len(sizes) - 1
    if levels < 1 or G < 1:
        raise ValueError("the chain does not recurse; nothing to shard")
    if L is None:
        L = 1
        while L + 1 < levels and (rho + 1) ** (L + 1) * G * 2 <= N:
            L += 1
    if not 1 <= L < levels + 1:
        raise ValueError(f"local levels {L} outside [1, {levels}]")
    U = (rho + 1) ** L
    cuts = [0]
    for g in range(1, G):
        c = int(round(g * N / G / U)) * U
        c = min(max(c, cuts[-1] + U), N - 1 - U)
        if c <= cuts[-1]:
            raise ValueError(f"N={N} too small for {G} shards at L={L}")
        cuts.append(c)
    cuts.append(N - 1)
    glob = _global_plans(N, L, rho)
    plan = ShardPlan(N, G, L, cuts, crossover=crossover, rho=rho)
    off = 0
    for g in range(G):
        a, b = cuts[g], cuts[g + 1]
        loc = _local_plans(a, b, L, rho)
        for lvl in range(L):
            want = [s for s in glob[lvl] if a <= s <= b]
            if loc[lvl] != want:
                raise AssertionError(f"chunk {g} level {lvl}: local plan differs from the global plan")
        plan.reduced_sizes.append(len(loc[-1]))
        plan.offsets.append(off)
        off += len(loc[-1]) - 1
    plan.reduced_N = off + 1
    assert plan.reduced_N == len(glob[-1])
    return plan


def assemble_reduced(plan: ShardPlan, diags: list, subs: list):
    """Global reduced matrix from per-chunk partial reduced systems (boundary partials summed in
    rank order).  Works on numpy arrays or torch tensors."""
    like = diags[0]
    n = like.shape[1]
    if type(like).__module__.startswith("torch"):
        import torch
        D = torch.zeros((plan.reduced_N, n, n), dtype=like.dtype, device=like.device)
        S = torch.zeros((plan.reduced_N - 1, n, n), dtype=like.dtype, device=like.device)
    else:
        D = np.zeros((plan.reduced_N, n, n))
        S = np.zeros((plan.reduced_N - 1, n, n))
    for g in range(plan.G):
        o, P = plan.offsets[g], plan.reduced_sizes[g]
        D[o:o + P] += diags[g][:P]
        S[o:o + P - 1] = subs[g][:P - 1]
    return D, S


def assemble_reduced_rhs(plan: ShardPlan, parts: list):
    like = parts[0]
    if type(like).__module__.startswith("torch"):
        import torch
        R = torch.zeros((plan.reduced_N,) + tuple(like.shape[1:]), dtype=like.dtype, device=like.device)
    else:
        R = np.zeros((plan.reduced_N,) + like.shape[1:])
    for g in range(plan.G):
        o, P = plan.offsets[g], plan.reduced_sizes[g]
        R[o:o + P] += parts[g][:P]
    return R


def chunk_inputs(plan: ShardPlan, g: int, diag, sub, rhs=None):
    """Rank g's slice of the global arrays with the shared-boundary ownership rule applied."""
    a, b = plan.chunk(g)
    d = diag[a:b + 1].clone() if hasattr(diag, "clone") else diag[a:b + 1].copy()
    s = sub[a:b]
    if g > 0:
        d[0] = 0.0
    r = None
    if rhs is not None:
        r = rhs[a:b + 1].clone() if hasattr(rhs, "clone") else rhs[a:b + 1].copy()
        if g > 0:
            r[0] = 0.0
    return d, s, r


# ------------------------------------------------------------------------------------------
# engines
# ------------------------------------------------------------------------------------------
def _on_device(fn):
    """Run an engine method with the engine's device current (the C ABI launches on the current
    device; the tensors live on ``self.device``)."""
    def wrapped(self, *a, **k):
        with self.torch.cuda.device(self.device):
            return fn(self, *a, **k)
    wrapped.__name__, wrapped.__doc__ = fn.__name__, fn.__doc__
    return wrapped


class CudaEngine:
    """Per-rank linear algebra on the sm_100a kernels (C ABI partial entry points)."""

    def __init__(self, device=None):
        import torch
        self.torch = torch
        self.device = device or torch.device("cuda", torch.cuda.current_device())

    def _cfg(self, cfg):
        return cfg._c()

    @_on_device
    def factor_partial(self, diag, sub, L, cfg):
        torch = self.torch
        lib = _native.lib()
        N, n = diag.shape[0], diag.shape[1]
        h = ctypes.c_void_p()
        st = _native.BtdStatus()
        c = self._cfg(cfg)
        rc = lib.btd_create_partial(N, n, ctypes.byref(c), L, ctypes.byref(h), ctypes.byref(st))
        if rc:
            from .schur import _raise_status
            _raise_status(st, rc)
        P = ctypes.c_int64()
        lib.btd_reduced_size(h, ctypes.byref(P))
        pb, sb = ctypes.c_size_t(), ctypes.c_size_t()
        lib.btd_factor_workspace(h, ctypes.byref(pb), ctypes.byref(sb))
        pers = torch.empty(pb.value, dtype=torch.uint8, device=self.device)
        scr = torch.empty(sb.value, dtype=torch.uint8, device=self.device)
        rd = torch.empty((P.value, n, n), dtype=torch.float64, device=self.device)
        rs = torch.empty((max(P.value - 1, 1), n, n), dtype=torch.float64, device=self.device)
        s = torch.cuda.current_stream(self.device)
        rc = lib.btd_factorize_partial(h, diag.data_ptr(), sub.data_ptr(), pers.data_ptr(), scr.data_ptr(),
                                       rd.data_ptr(), rs.data_ptr(), ctypes.c_void_p(s.cuda_stream), 1,
                                       ctypes.byref(st))
        if rc:
            lib.btd_destroy(h)
            from .schur import _raise_status
            _raise_status(st, rc)
        state = {"h": h, "pers": pers, "N": N, "n": n, "P": P.value}
        return state, rd, rs[:max(P.value - 1, 0)]

    @_on_device
    def solve_down(self, state, rhs):
        torch = self.torch
        lib = _native.lib()
        d = rhs.shape[2]
        sb = ctypes.c_size_t()
        lib.btd_solve_workspace(state["h"], d, ctypes.byref(sb))
        state["scr"] = torch.empty(sb.value, dtype=torch.uint8, device=self.device)
        state["x"] = torch.empty_like(rhs)
        red = torch.empty((state["P"], state["n"], d), dtype=torch.float64, device=self.device)
        st = _native.BtdStatus()
        s = torch.cuda.current_stream(self.device)
        rc = lib.btd_solve_down(state["h"], rhs.data_ptr(), state["x"].data_ptr(), d, state["scr"].data_ptr(),
                                red.data_ptr(), ctypes.c_void_p(s.cuda_stream), ctypes.byref(st))
        if rc:
            from .schur import _raise_status
            _raise_status(st, rc)
        return red

    @_on_device
    def solve_up(self, state, rhs, red_x):
        torch = self.torch
        lib = _native.lib()
        d = rhs.shape[2]
        st = _native.BtdStatus()
        s = torch.cuda.current_stream(self.device)
        red_x = red_x.contiguous()
        rc = lib.btd_solve_up(state["h"], rhs.data_ptr(), red_x.data_ptr(), state["x"].data_ptr(), d,
                              state["scr"].data_ptr(), ctypes.c_void_p(s.cuda_stream), ctypes.byref(st))
        if rc:
            from .schur import _raise_status
            _raise_status(st, rc)
        return state["x"]

    def factor_full(self, diag, sub, cfg):
        from .core import BlockTridiagonalMatrix
        from .schur import recursive_factorize
        return recursive_factorize(BlockTridiagonalMatrix(diag.contiguous(), sub.contiguous()), cfg)

    def solve_full(self, h, rhs):
        from .core import BlockRhs
        from .schur import recursive_solve
        return recursive_solve(h, BlockRhs(rhs.contiguous())).blocks

    def release(self, state):
        """Drop this rank's partial factor (C handle and device buffers); the solution returned by
        solve_up stays valid."""
        if state.get("h"):
            _native.lib().btd_destroy(state["h"])
            state["h"] = None
        for key in ("pers", "scr", "x"):
            state.pop(key, None)


# ------------------------------------------------------------------------------------------
# communication
# ------------------------------------------------------------------------------------------
class TorchComm:
    """All-gather of variable-length block stacks over torch.distributed (padded to the max)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def all_gather_blocks(self, x, counts):
        import torch
        if isinstance(x, np.ndarray):  # CPU engines (gloo tests)
            return [o.numpy() for o in self.all_gather_blocks(torch.from_numpy(np.ascontiguousarray(x)), counts)]
        if x.is_cuda and self.dist.get_backend(self.group) == "gloo":  # gloo: stage through the host
            return [o.to(x.device) for o in self.all_gather_blocks(x.cpu(), counts)]
        m = max(counts)
        pad = torch.zeros((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        pad[:x.shape[0]] = x
        out = [torch.empty_like(pad) for _ in range(self.size)]
        self.dist.all_gather(out, pad, group=self.group)
        return [o[:c] for o, c in zip(out, counts)]


class ShardedSolver:
    """One rank's view of the sharded factorization (all ranks call the same methods)."""

    def __init__(self, plan: ShardPlan, rank: int, comm, engine, config=None):
        from .schur import RecursionConfig
        self.plan, self.rank, self.comm, self.engine = plan, rank, comm, engine
        self.cfg = plan.config(config)

    def factorize(self, diag_chunk, sub_chunk):
        """diag/sub of this rank's chunk, ownership rule applied (see chunk_inputs)."""
        self.state, rd, rs = self.engine.factor_partial(diag_chunk, sub_chunk, self.plan.L, self.cfg)
        counts = self.plan.reduced_sizes
        if rd.shape[0] != counts[self.rank]:
            raise AssertionError(f"rank {self.rank}: reduced size {rd.shape[0]} != planned {counts[self.rank]}")
        diags = self.comm.all_gather_blocks(rd, counts)
        subs = self.comm.all_gather_blocks(rs, [max(c - 1, 0) for c in counts])
        D, S = assemble_reduced(self.plan, diags, subs)
        self.reduced = self.engine.factor_full(D, S, self.cfg)
        return self

    def solve(self, rhs_chunk):
        red = self.engine.solve_down(self.state, rhs_chunk)
        parts = self.comm.all_gather_blocks(red, self.plan.reduced_sizes)
        R = assemble_reduced_rhs(self.plan, parts)
        X = self.engine.solve_full(self.reduced, R)
        o, P = self.plan.offsets[self.rank], self.plan.reduced_sizes[self.rank]
        return self.engine.solve_up(self.state, rhs_chunk, X[o:o + P])


def run_sharded_local(plan: ShardPlan, engine, diag, sub, rhs, config=None):
    """All G ranks of the sharded algorithm played sequentially in one process (single-GPU check
    of the per-rank kernels and the assembly; the collective is the identity).

    Torch inputs are not copied chunk by chunk (a config-5 matrix is 64 GiB): chunk g > 0 sees its
    shared boundary block zeroed only while its factor is enqueued, and the block is restored
    right after on the same stream (stream order keeps both neighbours' reads correct)."""
    cfg = plan.config(config)
    states, rds, rss, rhs_c = [], [], [], []
    is_torch = type(diag).__module__.startswith("torch")
    for g in range(plan.G):
        if is_torch:
            a, b = plan.chunk(g)
            d, s = diag[a:b + 1], sub[a:b]
            r = rhs[a:b + 1].clone()
            saved = None
            if g > 0:
                saved = d[0].clone()
                d[0].zero_()
                r[0] = 0.0
            st, rd, rs = engine.factor_partial(d, s, plan.L, cfg)
            if saved is not None:
                d[0].copy_(saved)
        else:
            d, s, r = chunk_inputs(plan, g, diag, sub, rhs)
            st, rd, rs = engine.factor_partial(d, s, plan.L, cfg)
        if rd.shape[0] != plan.reduced_sizes[g]:
            raise AssertionError(f"chunk {g}: reduced size {rd.shape[0]} != planned {plan.reduced_sizes[g]}")
        states.append(st)
        rds.append(rd)
        rss.append(rs)
        rhs_c.append(r)
    D, S = assemble_reduced(plan, rds, rss)
    red = engine.factor_full(D, S, cfg)
    parts = [engine.solve_down(states[g], rhs_c[g]) for g in range(plan.G)]
    X = engine.solve_full(red, assemble_reduced_rhs(plan, parts))
    xs = []
    for g in range(plan.G):
        o, P = plan.offsets[g], plan.reduced_sizes[g]
        xs.append(engine.solve_up(states[g], rhs_c[g], X[o:o + P]).clone()
                  if hasattr(X, "clone") else engine.solve_up(states[g], rhs_c[g], X[o:o + P]))
    return gather_solution(plan, xs)


def gather_solution(plan: ShardPlan, chunks: list):
    """Global solution from per-rank chunk solutions (shared boundaries taken from the left)."""
    parts = []
    for g, x in enumerate(chunks):
        parts.append(x if g == 0 else x[1:])
    if type(chunks[0]).__module__.startswith("torch"):
        import torch
        return torch.cat(parts)
    return np.concatenate(parts)
