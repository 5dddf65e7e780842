"""Per-kernel device times of the large-shape Kalman assembly (kalman._build_batched) on the
paper's case (n = 256, m = 1024, N = 100) via torch.profiler.  Diagnostic only."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_03015_b200 as pkg
from paper_2509_03015_b200 import kalman
n, m, N = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (256, 1024, 100)))
mdl = pkg.generate_rotation_model(n, m, N, seed=0)
for _ in range(2):
    kalman.build_normal_equations(mdl, device_out=True)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as p:
    kalman.build_normal_equations(mdl, device_out=True)
    torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=25))
