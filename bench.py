"""Benchmark: fp64 block-tridiagonal SPD factor+solve (recursive Schur complement) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

One "step" = recursive_factorize + recursive_solve of one synthetic SPD system (the reference
generator's seeded instance, bit-identical).  Workload (N=1): BASELINE.json configs[1],
N=65536 blocks, n=64, d=1, default RecursionConfig.  Inputs are 4.3 GB (> 126 MB L2), so no
L2 flush is needed between steps.

value      = W_sub / t  (GFLOP/s, whole job over all ranks; W_sub = structure-exploiting
             substructuring flops, SURVEY.md §8(d) / BASELINE.md §3), inputs resident in HBM.
e2e        = same metric through the public API with pinned HOST buffers (H2D of A and B and
             D2H of X inside the timed region; the diagonal blocks' H2D sends the row bands that
             cover their lower triangle, the only part any kernel reads).
roofline   = the dominant kernel (level-0 factor_level_kernel<64>), fp64 DMMA-bound, timed
             with CUDA events on the launching stream (C-ABI timing hook).
Multi-GPU (N > 1; `--gpus N` self-launches N ranks through torch.distributed.run when WORLD_SIZE
is unset): strong scaling of BASELINE config 5 (N = 2^20, n = 64, d = 4) -- the ONE seed-0
instance is cut into G contiguous chunks at level-L separators, every rank
generates exactly its slice of that instance (bit-identical, synthgen.generate_spd_btd_slice),
eliminates its interiors locally, the reduced separator system is all-gathered over NCCL and
solved redundantly; value = W_sub of the global chain / max-over-ranks time.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {  # BASELINE.json configs
    "cfg1": (1024, 32, 1),
    "cfg2": (65536, 64, 1),
    "cfg3": (1048576, 8, 1),
    "cfg4": (4096, 256, 64),
    "cfg5": (1048576, 64, 4),
}
DEFAULT_SINGLE, DEFAULT_MULTI = "cfg2", "cfg5"
# CPU (reference-port) sample per config: the full instance where one factor+solve takes <~30 s on
# the GPU hosts' cores (cfg1, cfg2: same config as the GPU arm), else a bounded prefix-sized sample
CPU_SAMPLE = {"cfg1": (1024, 32, 1), "cfg2": (65536, 64, 1), "cfg3": (131072, 8, 1), "cfg4": (512, 256, 64),
              "cfg5": (32768, 64, 4)}


# ------------------------------------------------------------------------------------------
# algorithmic counts
# ------------------------------------------------------------------------------------------
def plan_levels(N, crossover=64, rho=8):
    """[(N_l, segment lengths)], base blocks -- same integer rules as plan_partition."""
    levels, cur = [], N
    while cur >= 3 and cur > crossover:
        seps = list(range(0, cur, rho + 1))
        if seps[-1] != cur - 1:
            if seps[-1] == cur - 2:
                seps.pop()
            seps.append(cur - 1)
        lens = np.diff(np.array(seps)) - 1
        levels.append((cur, lens))
        cur = len(seps)
    return levels, cur


def w_sub(N, n, d):
    """(factor flops, solve flops, level-0 factor flops) of the Y-form substructuring."""
    levels, nb = plan_levels(N)
    f = s = 0.0
    f0 = 0.0
    for i, (_, lens) in enumerate(levels):
        J = float(lens.sum())
        f += 19.0 / 3.0 * J * n ** 3
        s += 10.0 * J * n * n * d
        if i == 0:
            f0 = 19.0 / 3.0 * J * n ** 3
    f += nb * n ** 3 / 3.0 + 2.0 * max(nb - 1, 0) * n ** 3
    s += (6.0 * nb - 4.0) * n * n * d
    return f, s, f0


def diag_h2d_bytes(N, n):
    """Bytes the host-input path sends for the diagonal blocks (copy_diag_h2d, btd_capi.cu): G row
    bands, band g only its first (g+1) n/G columns (every kernel reads just the lower triangle)."""
    G = 4 if n >= 64 else 2 if n >= 32 else 1
    while G > 1 and n % G:
        G -= 1
    band = n // G
    return N * 8 * band * band * G * (G + 1) // 2


def q_min(N, n, d):
    return 8.0 * (3.0 * (2 * N - 1) * n * n + 2.0 * N * n * d)


def packed_stride(n):
    k = n >> 1
    return 2 * (k + 1) * (k + 1) if n & 1 else 2 * k * (k + 1)


def level0_bytes(N, n, rho=8):
    """Algorithmic HBM bytes of one level-0 factor launch: read the interior diagonal blocks and
    every sub block, write Linv (packed) of the interior rows, L_sub / the coupling copies, and
    S_L, S_R, S_sub per segment (btd_factor.cuh / btd_small.cuh)."""
    levels, _ = plan_levels(N, rho=rho)
    N0, lens = levels[0]
    K = len(lens)
    interior = int(lens.sum())
    nn = n * n
    return 8.0 * (interior * nn + (N0 - 1) * nn + interior * packed_stride(n) + (N0 - 1) * nn + 3 * K * nn)


def bound_of(N, n, d, peak_tflops, hbm_gbs):
    """'tensor' (fp64 pipe) or 'hbm': whichever roofline term is larger."""
    f, s_, _ = w_sub(N, n, d)
    return "tensor" if (f + s_) / (peak_tflops * 1e12) >= q_min(N, n, d) / (hbm_gbs * 1e9) else "hbm"


def measured_peaks():
    """(fp64 DMMA TFLOP/s, HBM GB/s, source note)."""
    fp = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak_r01.json")))["dmma_m8n8k4_tflops"]
    hbm, src = 6556.2, "fallback 6556.2 GB/s"
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        hbm, src = float(json.load(open(mp))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    return fp, hbm, src


# ------------------------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md clocks line)
# ------------------------------------------------------------------------------------------
class ClockSampler:
    def __init__(self):
        self.rows, self.proc = [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self, gpu_index=0):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 9 and r[0] == str(gpu_index)]
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [v for v in sm if mx and v > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------------------------------
# CPU baseline (oracle port of the reference algorithm, timed on the host cores)
# ------------------------------------------------------------------------------------------
def _cpu_instance(cfg_name):
    from paper_2509_03015_b200.synthgen import generate_spd_btd
    N, n, d = CPU_SAMPLE[cfg_name]
    A, B = generate_spd_btd(N, n, d, seed=0)
    return (N, n, d), A, B


def _cpu_step(A, B):
    from oracle import blocktri_port as port
    t0 = time.perf_counter()
    h = port.factorize(A.diag, A.sub)
    port.solve(h, B.blocks)
    return time.perf_counter() - t0


def _cpu_sample_note(cfg_name, runs, sec):
    from oracle import blocktri_port as port
    N, n, d = CPU_SAMPLE[cfg_name]
    same = CPU_SAMPLE[cfg_name] == CONFIGS[cfg_name]
    what = "the full instance (same config as the GPU arm)" if same else f"a bounded sample N={N}"
    return (f"{what}: N={N} n={n} d={d}, reference generator seed 0, {runs} run(s), median {sec * 1e3:.0f} ms "
            f"factor+solve; oracle/blocktri_port.py F-form restatement of the reference, pool={port._threads()} "
            f"threads, BLAS threads default, host cpus={os.cpu_count()}")


def cpu_baseline(cfg_name, runs=1):
    from oracle import blocktri_port as port
    (N, n, d), A, B = _cpu_instance(cfg_name)
    sec = statistics.median([_cpu_step(A, B) for _ in range(runs)])
    f, s, _ = w_sub(N, n, d)
    return {"value": (f + s) / sec / 1e9, "unit": "GFLOP/s", "cores": port._threads(), "kind": "port",
            "same_config": CPU_SAMPLE[cfg_name] == CONFIGS[cfg_name], "sample": _cpu_sample_note(cfg_name, runs, sec)}


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm (oracle port, pinned to the real reference's
    outputs) on the host cores, rank 0 only; each step is one factor+solve of the CPU sample."""
    if rank != 0:
        return
    from oracle import blocktri_port as port
    cfg = args.config
    N, n, d = CONFIGS[cfg]
    (Ns, ns, ds), A, B = _cpu_instance(cfg)
    for _ in range(min(args.warmup, 1)):  # a CPU step needs no graph/allocator warm-up beyond one
        _cpu_step(A, B)
    budget, times = 300.0, []  # bound the arm to ~5 minutes of timed steps
    t_start = time.perf_counter()
    while len(times) < args.steps:
        times.append(_cpu_step(A, B))
        if time.perf_counter() - t_start + times[-1] > budget:
            break
    sec = statistics.median(times)
    fs, ss, _ = w_sub(Ns, ns, ds)
    v = (fs + ss) / sec / 1e9
    same = (Ns, ns, ds) == (N, n, d)
    line = {
        "impl": "reference", "metric": "fp64 factor+solve GFLOP/s (W_sub), block-tridiagonal SPD N x n",
        "value": round(v, 4), "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": len(times),
        "steps_requested": args.steps, "warmup": min(args.warmup, 1),
        "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True, "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generate_spd_btd, seed 0)",
        "config": {"workload": f"{cfg}: N={N} n={n} d={d}" + ("" if same else f" (CPU step = bounded sample N={Ns})"),
                   "crossover": 64, "segment_length": 8},
        "same_config": same,
        "cpu_baseline": {"value": round(v, 4), "unit": "GFLOP/s", "cores": port._threads(), "kind": "port",
                         "sample": _cpu_sample_note(cfg, len(times), sec)},
        "e2e": {"value": round(v, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------
def kernel_name(n):
    if n <= 8:
        return "factor_small_kernel level 0 (8-lane group per segment, btd_small.cuh)"
    if n > 64:
        return "level-0 tiled factor (big_potrf_kernel + bt_gemm_kernel sequence, btd_big.cuh)"
    nt = 8 if n <= 8 else 16 if n <= 16 else 32 if n <= 32 else 64
    return f"factor_level_kernel<{nt}> level 0"


def run_ours(args, rank, world):
    import torch
    import paper_2509_03015_b200 as pkg
    from paper_2509_03015_b200 import _native

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    cfg = args.config
    N, n, d = CONFIGS[cfg]
    # pinned host inputs (bit-identical reference generator), then a resident device copy
    hd = torch.empty((N, n, n), dtype=torch.float64).pin_memory()
    hs = torch.empty((N - 1, n, n), dtype=torch.float64).pin_memory()
    hb = torch.empty((N, n, d), dtype=torch.float64).pin_memory()
    pkg.generate_spd_btd(N, n, d, seed=0, out=(hd.numpy(), hs.numpy(), hb.numpy()))
    dA = pkg.BlockTridiagonalMatrix(hd.to(dev), hs.to(dev))
    dB = pkg.BlockRhs(hb.to(dev))
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)

    def step():
        h = pkg.recursive_factorize(dA)
        return h, pkg.recursive_solve(h, dB)

    h = X = None
    for _ in range(max(args.warmup, 3)):
        h = X = None  # release the previous factor first (cfg5's hierarchy is ~55 GB)
        h, X = step()
    torch.cuda.synchronize()
    _, rres = pkg.residual_report(dA, X, dB)

    dist = None
    if world > 1:
        import torch.distributed as dist
    sampler = ClockSampler() if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    launches0 = _native.lib().btd_launch_count()
    ev[0].record(stream)
    for _ in range(args.steps):
        h = X = None
        h, X = step()
    ev[1].record(stream)
    torch.cuda.synchronize()
    launches = _native.lib().btd_launch_count() - launches0
    ms = ev[0].elapsed_time(ev[1]) / args.steps
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t)
        dist.barrier()

    # per-launch timing of the dominant kernel (level-0 factor) through the C-ABI timing hook
    h = X = None
    kt = pkg.schur.factor_kernel_times(dA, repeats=3, rhs_cols=d)
    clocks = sampler.stop(dev.index) if sampler else None
    del dA, dB
    torch.cuda.empty_cache()  # the host-input path below allocates its own device arenas

    # end to end: pinned host buffers -> public API -> host solution
    hA = pkg.BlockTridiagonalMatrix(hd, hs)
    hB = pkg.BlockRhs(hb)
    for _ in range(2):  # untimed warm-up of the host-buffer path (workspaces, pinned staging, graphs)
        Xh = None
        Xh = pkg.recursive_solve(pkg.recursive_factorize(hA), hB)
    torch.cuda.synchronize()
    hh = Xh = None
    # every step ends with the solution on the host (a host sync), so each step is timed on its own;
    # the median over the K steps is reported (PCIe throughput of a fresh box fluctuates step to step)
    e2e_each = []
    for _ in range(args.steps):
        hh = Xh = None
        t0 = time.perf_counter()
        hh = pkg.recursive_factorize(hA)
        Xh = pkg.recursive_solve(hh, hB)
        assert Xh.blocks.device.type == "cpu"
        torch.cuda.synchronize()
        e2e_each.append((time.perf_counter() - t0) * 1e3)
    e2e_ms = statistics.median(e2e_each)
    e2e_mean = statistics.fmean(e2e_each)
    if dist:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t)

    f, s, f0 = w_sub(N, n, d)
    gflops = (f + s) / (ms * 1e-3) / 1e9 * world
    e2e = (f + s) / (e2e_ms * 1e-3) / 1e9 * world
    if rank != 0:
        return
    peak_fp, hbm, hbm_src = measured_peaks()
    bound = bound_of(N, n, d, peak_fp, hbm)
    l0_ms = kt["level0_factor_ms"]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"ncu_{cfg}_factor_l0.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
    if bound == "tensor":
        achieved, peak, unit = f0 / (l0_ms * 1e-3) / 1e12, peak_fp, "TFLOP/s"
        peak_source = "profiles/fp64_peak_r01.json (measured fp64 DMMA; MEASURED_PEAKS.json has no fp64)"
        whole = (f + s) / (ms * 1e-3) / 1e12 / peak_fp
        algo = {"algorithmic_flops": f0}
    else:
        b0 = level0_bytes(N, n)
        achieved, peak, unit = b0 / (l0_ms * 1e-3) / 1e9, hbm, "GB/s"
        peak_source = hbm_src
        whole = q_min(N, n, d) / (ms * 1e-3) / 1e9 / hbm
        algo = {"algorithmic_bytes": b0}
    cpu = cpu_baseline(cfg) if world == 1 and not args.no_cpu else None
    line = {
        "metric": "fp64 factor+solve GFLOP/s (W_sub), block-tridiagonal SPD N x n",
        "value": round(gflops, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generate_spd_btd stream, seed 0; inputs > L2, no flush)",
        "config": {"workload": f"{cfg}: N={N} n={n} d={d}", "crossover": 64, "segment_length": 8,
                   "parallelism": "single GPU", "l2": "inputs larger than L2"},
        "factor_ms": round(kt["factor_ms"], 4), "solve_ms": round(kt["solve_ms"], 4),
        "rel_residual": rres, "w_sub_gflop": round((f + s) / 1e9, 3), "q_min_gb": round(q_min(N, n, d) / 1e9, 3),
        "roofline": {"bound": bound, "kernel": kernel_name(n),
                     "achieved": round(achieved, 3), "peak": peak, "unit": unit,
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "peak_source": peak_source, "launch_ms": round(l0_ms, 4), **algo,
                     "whole_step_frac": round(whole, 4),
                     **({"note": "n > 64: the level-0 sequence is host-issued in the timing-hook mode (no "
                                 "graph), so launch_ms includes host launch gaps and varies with the box's "
                                 "CPU; whole_step_frac (graph-replayed step) is the stable figure"}
                        if n > 64 else {})},
        "e2e": {"value": round(e2e, 3), "unit": "GFLOP/s", "ms_per_step": round(e2e_ms, 3),
                "ms_per_step_mean": round(e2e_mean, 3), "timing": f"median of {args.steps} host-timed steps",
                "h2d_bytes_per_step": int(diag_h2d_bytes(N, n) + hs.numel() * 8 + hb.numel() * 8),
                "d2h_bytes_per_step": int(hb.numel() * 8)},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# N > 1: strong scaling of config 5 over the sharded chain -- every rank slices
# its chunk of the ONE global seed-0 instance; the reduced separator system is all-gathered
# ------------------------------------------------------------------------------------------
def sharded_residual(plan, rank, dd, ds, db, x, dist):
    """Global max-column ||b - A x|| / ||b|| of the distributed solution.  Each rank owns the rows
    (a_g, b_g] of its chunk (rank 0 also row 0); the coupling term A_{b+1,b}^T x_{b+1} of a chunk's
    last row lives on the right neighbour and is all-gathered (one n x d panel per rank)."""
    import torch
    from paper_2509_03015_b200 import report
    y = report.btd_matmul(sh_matrix(dd, ds), sh_rhs(x)).blocks
    G = plan.G
    part = (ds[0].transpose(0, 1) @ x[1]) if rank > 0 else torch.zeros_like(x[0])
    parts = [torch.empty_like(part) for _ in range(G)]
    dist.all_gather(parts, part.contiguous())
    lo = 0 if rank == 0 else 1
    r = db[lo:] - y[lo:]
    if rank < G - 1:
        r[-1] -= parts[rank + 1]
    d = x.shape[2]
    sums = torch.stack([(r.reshape(-1, d) ** 2).sum(0), (db[lo:].reshape(-1, d) ** 2).sum(0)])
    dist.all_reduce(sums)
    return float((sums[0] / sums[1]).sqrt().max())


def run_sharded(args, rank, world):
    import torch
    import torch.distributed as dist
    from paper_2509_03015_b200 import _native
    from paper_2509_03015_b200 import sharded as sh
    from paper_2509_03015_b200.synthgen import generate_spd_btd_slice

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    cfg = args.config
    N, n, d = CONFIGS[cfg]
    plan = sh.shard_plan(N, world)
    a, b = plan.chunk(rank)
    Nc = b - a + 1
    # this rank's slice of the global instance (bit-identical to the unsharded generator); the
    # shared boundary block / rhs panel is owned by the left rank (sharded.chunk_inputs rule)
    hd = torch.empty((Nc, n, n), dtype=torch.float64).pin_memory()
    hs = torch.empty((Nc - 1, n, n), dtype=torch.float64).pin_memory()
    hb = torch.empty((Nc, n, d), dtype=torch.float64).pin_memory()
    generate_spd_btd_slice(N, n, d, 0, a, b, out=(hd.numpy(), hs.numpy(), hb.numpy()))
    if rank > 0:
        hd[0] = 0.0
        hb[0] = 0.0
    dd, ds, db = hd.to(dev), hs.to(dev), hb.to(dev)
    comm = sh.TorchComm()
    solver = sh.ShardedSolver(plan, rank, comm, sh.CudaEngine(dev))

    def step(d_, s_, b_):
        solver.factorize(d_, s_)
        x = solver.solve(b_)
        solver.engine.release(solver.state)  # one partial factor alive at a time (config 5 is large)
        solver.reduced = None
        return x

    x = None
    for _ in range(max(args.warmup, 3)):
        x = None
        x = step(dd, ds, db)
    torch.cuda.synchronize()
    rres = sharded_residual(plan, rank, dd, ds, db, x, dist)

    sampler = ClockSampler() if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    stream = torch.cuda.current_stream(dev)
    launches0 = _native.lib().btd_launch_count()
    dist.barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(stream)
    for _ in range(args.steps):
        x = None
        x = step(dd, ds, db)
    ev[1].record(stream)
    torch.cuda.synchronize()
    launches = _native.lib().btd_launch_count() - launches0
    ms = ev[0].elapsed_time(ev[1]) / args.steps
    t = torch.tensor([ms], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t)
    dist.barrier()
    clocks = sampler.stop(dev.index) if sampler else None

    # end to end: pinned host chunk -> device -> sharded factor + solve -> host solution chunk
    x = None
    del dd, ds, db
    torch.cuda.empty_cache()  # the e2e leg copies its own device chunk (config 5: 34 GB per rank at N=2)
    hx = torch.empty_like(hb)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_steps = max(1, args.steps // 2)
    for _ in range(e2e_steps):
        xx = None
        xx = step(hd.to(dev, non_blocking=True), hs.to(dev, non_blocking=True), hb.to(dev, non_blocking=True))
        hx.copy_(xx)
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    t = torch.tensor([e2e_ms], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t)
    h2d = torch.tensor([(hd.numel() + hs.numel() + hb.numel()) * 8, hb.numel() * 8], device=dev, dtype=torch.float64)
    dist.all_reduce(h2d)
    f, s_, _ = w_sub(N, n, d)
    if rank != 0:
        return
    line = {
        "metric": "fp64 factor+solve GFLOP/s (W_sub), block-tridiagonal SPD N x n",
        "value": round((f + s_) / (ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (the reference generator's seed-0 instance, each rank its own slice; inputs > L2, no flush)",
        "config": {"workload": f"{cfg}: N={N} n={n} d={d}, one chain sharded over {world} GPUs",
                   "crossover": 64, "segment_length": 8, "parallelism": f"chain sharded x{world}",
                   "local_levels": plan.L, "reduced_blocks": plan.reduced_N, "cuts": plan.cuts,
                   "l2": "inputs larger than L2"},
        "rel_residual": rres, "w_sub_gflop": round((f + s_) / 1e9, 3),
        "e2e": {"value": round((f + s_) / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s", "ms_per_step": round(e2e_ms, 3),
                "h2d_bytes_per_step": int(h2d[0]), "d2h_bytes_per_step": int(h2d[1])},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "collective": f"torch.distributed ({dist.get_backend()}) all_gather of the reduced separator system "
                      "(factor) and of the reduced rhs (solve)",
    }
    print(json.dumps(line), flush=True)


def sh_matrix(d, s):
    from paper_2509_03015_b200.core import BlockTridiagonalMatrix
    return BlockTridiagonalMatrix(d, s)


def sh_rhs(x):
    from paper_2509_03015_b200.core import BlockRhs
    return BlockRhs(x)


def self_launch(args):
    """`--gpus N` with N > 1 and no torchrun environment: re-run this script as N ranks."""
    import socket
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help=f"default: {DEFAULT_SINGLE} on one GPU, {DEFAULT_MULTI} (strong scaling) on N > 1")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.config is None:
        args.config = DEFAULT_SINGLE if world == 1 else DEFAULT_MULTI
    dist_on = world > 1 and args.impl == "ours"
    if dist_on:
        import torch
        import torch.distributed as dist
        ndev = torch.cuda.device_count()
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % ndev)
        # more ranks than GPUs (a dry run of N ranks on one device): NCCL refuses duplicate GPUs, so
        # the collectives are host-staged over gloo; BTD_BENCH_GLOO=1 forces that
        gloo = os.environ.get("BTD_BENCH_GLOO") == "1" or world > ndev
        dist.init_process_group("gloo" if gloo else "nccl")
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif world > 1:
        run_sharded(args, rank, world)
    else:
        run_ours(args, rank, world)
    if dist_on:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
