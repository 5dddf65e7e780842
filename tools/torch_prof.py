"""Kernel-time breakdown of one factor or solve call via torch.profiler (CUPTI), grouped by kernel
name and grid size.   python tools/torch_prof.py N,n,d [factor|solve]"""
import sys
from collections import defaultdict
sys.path.insert(0, '.')
import torch
import paper_2509_03015_b200 as pkg
N, n, d = (int(v) for v in sys.argv[1].split(','))
what = sys.argv[2] if len(sys.argv) > 2 else 'solve'
A, B = pkg.generate_spd_btd(N, n, d, seed=0)
dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
dB = pkg.BlockRhs(torch.from_numpy(B.blocks).cuda())
for _ in range(2):
    h = pkg.recursive_factorize(dA)
    X = pkg.recursive_solve(h, dB)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    if what == 'factor':
        h = pkg.recursive_factorize(dA)
    else:
        X = pkg.recursive_solve(h, dB)
    torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        key = ev.name[:70]
        agg[key][0] += 1
        agg[key][1] += ev.device_time_total if hasattr(ev, 'device_time_total') else ev.cuda_time_total
tot = sum(v[1] for v in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:15]:
    print(f"{t/1e3:9.3f} ms  x{c:5d}  {k}")
print(f"{tot/1e3:9.3f} ms total")
