"""Measurement of the Kalman front-end: GPU normal-equation assembly
(btd_kalman_normal_equations, model resident on the device) and the full smoothing pipeline
(assembly -> recursive factor -> solve, all on the device) against the CPU port of the reference
assembly (oracle/kalman_port.py) on a bounded sample of the same model.  One JSON line.

    python tools/bench_kalman.py [--horizon 1048576] [--state 8] [--obs 12]
"""
import argparse, json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_03015_b200 as pkg
from paper_2509_03015_b200 import kalman

ap = argparse.ArgumentParser()
ap.add_argument("--horizon", type=int, default=1 << 20)
ap.add_argument("--state", type=int, default=8)
ap.add_argument("--obs", type=int, default=12)
ap.add_argument("--cpu-sample", type=int, default=20000)
args = ap.parse_args()
mdl = pkg.generate_rotation_model(args.state, args.obs, args.horizon, seed=0)
N, n, m = mdl.horizon, mdl.state_dim, mdl.obs_dim
for _ in range(2):
    A, B = kalman.build_normal_equations(mdl, device_out=True)
for _ in range(2):
    X = pkg.recursive_solve(pkg.recursive_factorize(A), B)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
reps = 5
e[0].record()
for _ in range(reps):
    A, B = kalman.build_normal_equations(mdl, device_out=True)
e[1].record()
for _ in range(reps):
    X = pkg.recursive_solve(pkg.recursive_factorize(A), B)
e[2].record()
torch.cuda.synchronize()
asm_ms = e[0].elapsed_time(e[1]) / reps
solve_ms = e[1].elapsed_time(e[2]) / reps
rres = pkg.residual_report(A, X, B)[1]
from oracle import kalman_port
small = pkg.generate_rotation_model(args.state, args.obs, args.cpu_sample, seed=0)
t0 = time.perf_counter()
kalman_port.build_normal_equations(small)
cpu_s = time.perf_counter() - t0
print(json.dumps({
    "what": "Kalman normal equations (build_normal_equations) on B200 vs CPU port of the reference",
    "model": f"generate_rotation_model(state_dim={n}, obs_dim={m}, horizon={N}, seed=0)",
    "gpu_assembly_ms": round(asm_ms, 4), "gpu_steps_per_s": round(N / (asm_ms * 1e-3)),
    "gpu_factor_solve_ms": round(solve_ms, 4), "rel_residual": rres,
    "note": "assembly timed with the model resident on the device except for the per-call H2D of the"
            " per-step arrays (transition, observations, prior offsets); shared H/Q/R go up once",
    "cpu_baseline": {"steps_per_s": round(args.cpu_sample / cpu_s), "cores": 1, "kind": "port",
                     "sample": f"horizon {args.cpu_sample} of the same model, oracle/kalman_port.py"}}), flush=True)
