"""Break down the end-to-end (host buffers) step: pure pinned H2D bandwidth vs the e2e call."""
import sys, time
import torch
sys.path.insert(0, '.')
import paper_2509_03015_b200 as pkg
N, n, d = 65536, 64, 1
hd = torch.empty((N, n, n), dtype=torch.float64).pin_memory()
hs = torch.empty((N - 1, n, n), dtype=torch.float64).pin_memory()
hb = torch.empty((N, n, d), dtype=torch.float64).pin_memory()
pkg.generate_spd_btd(N, n, d, seed=0, out=(hd.numpy(), hs.numpy(), hb.numpy()))
dd = torch.empty_like(hd, device='cuda'); ds = torch.empty_like(hs, device='cuda')
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dd.copy_(hd, non_blocking=True); ds.copy_(hs, non_blocking=True); torch.cuda.synchronize()
    t = time.perf_counter() - t0
print(f"pinned H2D {hd.numel()*8/1e9 + hs.numel()*8/1e9:.2f} GB in {t*1e3:.1f} ms = {(hd.numel()+hs.numel())*8/t/1e9:.1f} GB/s", flush=True)
A = pkg.BlockTridiagonalMatrix(hd, hs); B = pkg.BlockRhs(hb)
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = pkg.recursive_factorize(A); t1 = time.perf_counter()
    X = pkg.recursive_solve(h, B); t2 = time.perf_counter()
print(f"e2e factor {1e3*(t1-t0):.1f} ms, solve {1e3*(t2-t1):.1f} ms", flush=True)
