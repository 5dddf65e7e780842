"""Device timeline of a few public-API factor+solve steps (torch.profiler / CUPTI): per-kernel start
and end, idle gaps between kernels, step span.  python tools/trace_steps.py N,n,d [steps]"""
import json, os, sys, tempfile
sys.path.insert(0, '.')
import torch
import paper_2509_03015_b200 as pkg
N, n, d = (int(v) for v in sys.argv[1].split(','))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
A, B = pkg.generate_spd_btd(N, n, d, seed=0)
dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
dB = pkg.BlockRhs(torch.from_numpy(B.blocks).cuda())
for _ in range(3):
    h = pkg.recursive_factorize(dA); X = pkg.recursive_solve(h, dB)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as p:
    for _ in range(steps):
        h = pkg.recursive_factorize(dA); X = pkg.recursive_solve(h, dB)
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "t.json")
p.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
k = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
t0 = k[0]["ts"]
prev_end = None
busy = 0.0
for e in k:
    gap = 0.0 if prev_end is None else e["ts"] - prev_end
    busy += e["dur"]
    print(f"{e['ts'] - t0:9.1f} us  dur {e['dur']:7.1f}  gap {gap:6.1f}  {e['name'][:60]}")
    prev_end = e["ts"] + e["dur"]
span = prev_end - t0
print(f"span {span:.1f} us for {steps} steps ({span / steps:.1f} us/step), device busy {busy:.1f} us "
      f"({busy / span:.0%})")
