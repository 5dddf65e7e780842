"""BASELINE config 5 (N = 2^20, n = 64, d = 4) on ONE GPU: the unsharded factor+solve (GPU residual)
and the sharded algorithm played with G = 2 / 4 / 8 ranks on the same device (run_sharded_local:
the per-rank partial kernels + the reduced-system assembly an all-gather would produce), whose
solution must equal the unsharded one to <= 1e-12.  Writes gpurun_out/cfg5_check.json.

    python tools/cfg5_check.py [N n d]
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_03015_b200 as pkg  # noqa: E402
from paper_2509_03015_b200.sharded import CudaEngine, run_sharded_local, shard_plan  # noqa: E402
from paper_2509_03015_b200.synthgen import generate_spd_btd_slice  # noqa: E402

N, n, d = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (1048576, 64, 4)
dev = torch.device("cuda", 0)
out = {"N": N, "n": n, "d": d}
t0 = time.time()
diag = torch.empty((N, n, n), dtype=torch.float64, device=dev)
sub = torch.empty((N - 1, n, n), dtype=torch.float64, device=dev)
rhs = torch.empty((N, n, d), dtype=torch.float64, device=dev)
step = 65536
f = 0
while f < N - 1:  # slices [f, l] overlapping by one row, so every sub block is covered
    l = min(f + step, N - 1)
    dg, sb, rh = generate_spd_btd_slice(N, n, d, 0, f, l)
    diag[f:l + 1].copy_(torch.from_numpy(dg))
    sub[f:l].copy_(torch.from_numpy(sb))
    rhs[f:l + 1].copy_(torch.from_numpy(rh))
    f = l
torch.cuda.synchronize()
out["generate_s"] = round(time.time() - t0, 1)
A, B = pkg.BlockTridiagonalMatrix(diag, sub), pkg.BlockRhs(rhs)
h = pkg.recursive_factorize(A)
X = pkg.recursive_solve(h, B).blocks
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
h = None
ev[0].record()
h = pkg.recursive_factorize(A)
ev[1].record()
X = pkg.recursive_solve(h, B).blocks
ev[2].record()
torch.cuda.synchronize()
out["unsharded"] = {"factor_ms": ev[0].elapsed_time(ev[1]), "solve_ms": ev[1].elapsed_time(ev[2]),
                    "levels": [lv.num_blocks for lv in h.levels] + [h.base.num_blocks],
                    "rel_residual": pkg.residual_report(A, pkg.BlockRhs(X), B)[1]}
h = None
torch.cuda.empty_cache()
out["sharded_local"] = {}
for G in (2, 4, 8):
    plan = shard_plan(N, G)
    Xs = run_sharded_local(plan, CudaEngine(dev), diag, sub, rhs)
    rel = float((Xs - X).abs().max() / X.abs().max())
    out["sharded_local"][G] = {"L": plan.L, "reduced_N": plan.reduced_N, "cuts": plan.cuts,
                               "rel_vs_unsharded": rel,
                               "rel_residual": pkg.residual_report(A, pkg.BlockRhs(Xs), B)[1]}
    Xs = None
    torch.cuda.empty_cache()
    print(G, out["sharded_local"][G], flush=True)
out["peak_mem_gb"] = torch.cuda.max_memory_allocated() / 1e9
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "cfg5_check.json"), "w"), indent=1)
print(json.dumps(out))
