"""Pinned host -> device copy bandwidth on this box: one stream vs two / four concurrent streams,
contiguous and 2D-pitched (the banded diagonal copies).  python tools/h2d_bw.py"""
import torch, time
n = 2 * 1024**3 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
def run(ns, chunks=16):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    torch.cuda.synchronize()
    t = time.perf_counter()
    step = n // chunks
    for i in range(chunks):
        with torch.cuda.stream(ss[i % ns]):
            d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
    torch.cuda.synchronize()
    return n * 8 / (time.perf_counter() - t) / 1e9
for ns in (1, 2, 4):
    run(ns)
    print(f"streams={ns}: {max(run(ns) for _ in range(3)):.1f} GB/s", flush=True)
# pitched (cudaMemcpy2DAsync, like the banded diagonal copies): 64 x 64 blocks, the first w columns
from cuda.bindings import runtime as cudart
N = 65536
for w in (32, 48, 64):
    for ns in (1, 2):
        ss = [torch.cuda.Stream() for _ in range(ns)]
        for rep in range(2):
            torch.cuda.synchronize(); t = time.perf_counter()
            rows = N * 64 // 16
            for i in range(16):
                off = i * rows * 64 * 8
                cudart.cudaMemcpy2DAsync(d.data_ptr() + off, 512, h.data_ptr() + off, 512, w * 8, rows,
                                         cudart.cudaMemcpyKind.cudaMemcpyHostToDevice, ss[i % ns].cuda_stream)
            torch.cuda.synchronize()
            bw = N * 64 * w * 8 / (time.perf_counter() - t) / 1e9
        print(f"2D copy, {w * 8} B rows of 512 B, streams={ns}: {bw:.1f} GB/s", flush=True)
