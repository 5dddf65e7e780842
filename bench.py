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
Multi-GPU (torchrun, N > 1): the chain is sharded -- every rank owns a chunk of the
configuration's size (weak scaling: N_global = N x chunk), eliminates its interiors locally and the
reduced separator system is all-gathered over NCCL and solved redundantly; value = W_sub of the
global chain / max-over-ranks time.
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
}
CPU_SAMPLE = {"cfg1": (1024, 32, 1), "cfg2": (8192, 64, 1), "cfg3": (131072, 8, 1), "cfg4": (512, 256, 64)}


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
def cpu_baseline(cfg_name, runs=1):
    from oracle import blocktri_port as port
    from paper_2509_03015_b200.synthgen import generate_spd_btd
    N, n, d = CPU_SAMPLE[cfg_name]
    A, B = generate_spd_btd(N, n, d, seed=0)
    t = []
    for _ in range(runs):
        t0 = time.perf_counter()
        h = port.factorize(A.diag, A.sub)
        port.solve(h, B.blocks)
        t.append(time.perf_counter() - t0)
    f, s, _ = w_sub(N, n, d)
    sec = statistics.median(t)
    return {"value": (f + s) / sec / 1e9, "unit": "GFLOP/s", "cores": port._threads(), "kind": "port",
            "sample": f"N={N} n={n} d={d} (same generator/seed, {runs} run(s), median {sec * 1e3:.0f} ms "
                      f"factor+solve; oracle/blocktri_port.py F-form restatement, pool={port._threads()} threads, "
                      f"BLAS threads default, host cpus={os.cpu_count()})"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = args.config
    N, n, d = CONFIGS[cfg]
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(cfg, runs=1)
        if i >= args.warmup:
            vals.append(r["value"])
    v = statistics.median(vals)
    Ns, ns, ds = CPU_SAMPLE[cfg]
    fs, ss, _ = w_sub(Ns, ns, ds)
    line = {
        "impl": "reference", "metric": "fp64 factor+solve GFLOP/s (W_sub), block-tridiagonal SPD N x n",
        "value": round(v, 4), "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round((fs + ss) / (v * 1e9) * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generate_spd_btd, seed 0)",
        "config": {"workload": f"{cfg}: N={N} n={n} d={d} (CPU step = bounded sample N={Ns})",
                   "crossover": 64, "segment_length": 8},
        "cpu_baseline": {"value": round(v, 4), "unit": "GFLOP/s", "cores": r["cores"], "kind": "port",
                         "sample": r["sample"]},
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
    pkg.generate_spd_btd(N, n, d, seed=rank, out=(hd.numpy(), hs.numpy(), hb.numpy()))
    dA = pkg.BlockTridiagonalMatrix(hd.to(dev), hs.to(dev))
    dB = pkg.BlockRhs(hb.to(dev))
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)

    def step():
        h = pkg.recursive_factorize(dA)
        return h, pkg.recursive_solve(h, dB)

    for _ in range(max(args.warmup, 3)):
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
    L = _native.lib()
    kt = pkg.schur.factor_kernel_times(dA, repeats=3)
    clocks = sampler.stop(dev.index) if sampler else None

    # end to end: pinned host buffers -> public API -> host solution
    hA = pkg.BlockTridiagonalMatrix(hd, hs)
    hB = pkg.BlockRhs(hb)
    for _ in range(2):  # untimed warm-up of the host-buffer path (workspaces, pinned staging, graphs)
        pkg.recursive_solve(pkg.recursive_factorize(hA), hB)
    torch.cuda.synchronize()
    # every step ends with the solution on the host (a host sync), so each step is timed on its own;
    # the median over the K steps is reported (PCIe throughput of a fresh box fluctuates step to step)
    e2e_each = []
    for _ in range(args.steps):
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
    peaks = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak_r01.json")))
    peak = peaks["dmma_m8n8k4_tflops"]
    l0_ms = kt["level0_factor_ms"]
    achieved = f0 / (l0_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"ncu_{cfg}_factor_l0.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
    cpu = cpu_baseline(cfg) if world == 1 and not args.no_cpu else None
    line = {
        "metric": "fp64 factor+solve GFLOP/s (W_sub), block-tridiagonal SPD N x n",
        "value": round(gflops, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generate_spd_btd stream, seed=rank; inputs 4.3 GB > L2, no flush)",
        "config": {"workload": f"{cfg}: N={N} n={n} d={d}", "crossover": 64, "segment_length": 8,
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": "inputs larger than L2"},
        "factor_ms": round(kt["factor_ms"], 4), "solve_ms": round(kt["solve_ms"], 4),
        "rel_residual": rres, "w_sub_gflop": round((f + s) / 1e9, 3), "q_min_gb": round(q_min(N, n, d) / 1e9, 3),
        "roofline": {"bound": "tensor", "kernel": kernel_name(n),
                     "achieved": round(achieved, 3), "peak": peak, "unit": "TFLOP/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "peak_source": "profiles/fp64_peak_r01.json (measured fp64 DMMA; MEASURED_PEAKS.json has no fp64)",
                     "launch_ms": round(l0_ms, 4), "algorithmic_flops": f0,
                     "whole_step_frac": round((f + s) / (ms * 1e-3) / 1e12 / peak, 4)},
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
# N > 1: the sharded chain, weak scaling -- every rank owns a chunk of the
# configuration's size, the reduced separator system is all-gathered over NCCL
# ------------------------------------------------------------------------------------------
def run_sharded(args, rank, world):
    import torch
    import torch.distributed as dist
    from paper_2509_03015_b200 import sharded as sh
    from paper_2509_03015_b200.synthgen import generate_spd_btd

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    cfg = args.config
    N1, n, d = CONFIGS[cfg]
    plan = sh.shard_plan(N1 * world, world)
    a, b = plan.chunk(rank)
    Nc = b - a + 1
    # synthetic chunk: the reference generator's stream with seed = rank; the shared boundary
    # block is owned by the left rank (diagonal shifted by n so it also dominates the right
    # neighbour's coupling, |A_{b+1,b}| row sums <= n), the right rank passes zeros for it
    hd = torch.empty((Nc, n, n), dtype=torch.float64).pin_memory()
    hs = torch.empty((Nc - 1, n, n), dtype=torch.float64).pin_memory()
    hb = torch.empty((Nc, n, d), dtype=torch.float64).pin_memory()
    generate_spd_btd(Nc, n, d, seed=rank, out=(hd.numpy(), hs.numpy(), hb.numpy()))
    if rank < world - 1:
        hd[-1] += n * torch.eye(n, dtype=torch.float64)
    if rank > 0:
        hd[0] = 0.0
        hb[0] = 0.0
    dd, ds, db = hd.to(dev), hs.to(dev), hb.to(dev)
    comm = sh.TorchComm()
    solver = sh.ShardedSolver(plan, rank, comm, sh.CudaEngine(dev))

    def step(d_, s_, b_):
        solver.factorize(d_, s_)
        x = solver.solve(b_)
        solver.engine.release(solver.state)
        return x

    for _ in range(max(args.warmup, 3)):
        x = step(dd, ds, db)
    torch.cuda.synchronize()
    # residual of this rank's interior rows (rows 1..Nc-2 only involve the chunk's own blocks)
    from paper_2509_03015_b200 import report
    y = report.btd_matmul(sh_matrix(dd, ds), sh_rhs(x)).blocks
    r = (db[1:-1] - y[1:-1]).reshape(-1, d)
    rres = float((torch.linalg.vector_norm(r, dim=0) / torch.linalg.vector_norm(db[1:-1].reshape(-1, d), dim=0)).max())
    t = torch.tensor([rres], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    rres = float(t)

    sampler = ClockSampler() if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    stream = torch.cuda.current_stream(dev)
    from paper_2509_03015_b200 import _native
    launches0 = _native.lib().btd_launch_count()
    dist.barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(stream)
    for _ in range(args.steps):
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
    hx = torch.empty_like(hb)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_steps = max(1, args.steps // 2)
    for _ in range(e2e_steps):
        xx = step(hd.to(dev, non_blocking=True), hs.to(dev, non_blocking=True), hb.to(dev, non_blocking=True))
        hx.copy_(xx)
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    t = torch.tensor([e2e_ms], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t)
    f, s_, _ = w_sub(plan.N, n, d)
    if rank != 0:
        return
    line = {
        "metric": "fp64 factor+solve GFLOP/s (W_sub), block-tridiagonal SPD N x n",
        "value": round((f + s_) / (ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generate_spd_btd stream per chunk, seed=rank; inputs > L2, no flush)",
        "config": {"workload": f"{cfg} chunk per GPU, sharded chain: N={plan.N} (={world} x ~{N1}) n={n} d={d}",
                   "crossover": 64, "segment_length": 8, "parallelism": f"chain sharded x{world}",
                   "local_levels": plan.L, "reduced_blocks": plan.reduced_N, "l2": "inputs larger than L2"},
        "rel_residual_interior": rres, "w_sub_gflop": round((f + s_) / 1e9, 3),
        "e2e": {"value": round((f + s_) / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s", "ms_per_step": round(e2e_ms, 3),
                "h2d_bytes_per_step": int((hd.numel() + hs.numel() + hb.numel()) * 8) * world,
                "d2h_bytes_per_step": int(hb.numel() * 8) * world},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "collective": "torch.distributed all_gather of the reduced separator system (factor) and rhs (solve)",
    }
    print(json.dumps(line), flush=True)


def sh_matrix(d, s):
    from paper_2509_03015_b200.core import BlockTridiagonalMatrix
    return BlockTridiagonalMatrix(d, s)


def sh_rhs(x):
    from paper_2509_03015_b200.core import BlockRhs
    return BlockRhs(x)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and args.impl == "ours":
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
        # BTD_BENCH_GLOO=1: host-staged gloo collectives (lets N ranks share one GPU for a dry run)
        dist.init_process_group("gloo" if os.environ.get("BTD_BENCH_GLOO") == "1" else "nccl")
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif world > 1:
        run_sharded(args, rank, world)
    else:
        run_ours(args, rank, world)
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
