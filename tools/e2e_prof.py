"""Where the end-to-end (pinned host in -> host solution out) step of a config spends its time:
host wall time of factorize / solve and the CUDA activity (copies, kernels) under torch.profiler.
    python tools/e2e_prof.py N,n,d"""
import sys, time
from collections import defaultdict
sys.path.insert(0, '.')
import torch
import paper_2509_03015_b200 as pkg
N, n, d = (int(v) for v in sys.argv[1].split(','))
hd = torch.empty((N, n, n), dtype=torch.float64).pin_memory()
hs = torch.empty((N - 1, n, n), dtype=torch.float64).pin_memory()
hb = torch.empty((N, n, d), dtype=torch.float64).pin_memory()
pkg.generate_spd_btd(N, n, d, seed=0, out=(hd.numpy(), hs.numpy(), hb.numpy()))
A, B = pkg.BlockTridiagonalMatrix(hd, hs), pkg.BlockRhs(hb)
for _ in range(3):
    X = pkg.recursive_solve(pkg.recursive_factorize(A), B)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    h = pkg.recursive_factorize(A)
    t1 = time.perf_counter()
    X = pkg.recursive_solve(h, B)
    t2 = time.perf_counter()
    print(f"host wall: factorize {1e3*(t1-t0):.2f} ms  solve {1e3*(t2-t1):.2f} ms  total {1e3*(t2-t0):.2f} ms", flush=True)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    h = pkg.recursive_factorize(A)
    X = pkg.recursive_solve(h, B)
    torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
span = [1e30, 0]
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        agg[ev.name[:60]][0] += 1
        agg[ev.name[:60]][1] += ev.device_time_total
        span[0] = min(span[0], ev.time_range.start); span[1] = max(span[1], ev.time_range.end)
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"{t/1e3:9.3f} ms  x{c:4d}  {k}")
print(f"device activity span {1e-3*(span[1]-span[0]):.2f} ms")
