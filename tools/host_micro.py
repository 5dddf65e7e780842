"""Host-side cost of the public-API pieces around the launches (per call, perf_counter, no profiler):
recursive_factorize / recursive_solve wall at a small config, and the torch / ctypes primitives
they use.   python tools/host_micro.py [N,n,d]"""
import ctypes, sys, time
sys.path.insert(0, '.')
import torch
import paper_2509_03015_b200 as pkg
from paper_2509_03015_b200 import _native, schur
N, n, d = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1024,32,1").split(','))
A, B = pkg.generate_spd_btd(N, n, d, seed=0)
dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
dB = pkg.BlockRhs(torch.from_numpy(B.blocks).cuda())
dev = dA.diag.device
for _ in range(5):
    h = pkg.recursive_factorize(dA); X = pkg.recursive_solve(h, dB)
torch.cuda.synchronize()


def per_call(fn, reps=2000):
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e6


def ctx_dev():
    with torch.cuda.device(dev):
        pass


def ctx_stream():
    with torch.cuda.stream(torch.cuda.current_stream(dev)):
        pass


def ctx_on():
    with schur._on_stream(dev, None):
        pass


L = _native.lib()
print(f"torch.cuda.device ctx   {per_call(ctx_dev):7.2f} us")
print(f"torch.cuda.stream ctx   {per_call(ctx_stream):7.2f} us")
print(f"_on_stream ctx          {per_call(ctx_on):7.2f} us")
print(f"current_stream          {per_call(lambda: torch.cuda.current_stream(dev)):7.2f} us")
print(f"torch.empty (cuda)      {per_call(lambda: torch.empty(4096, dtype=torch.uint8, device=dev)):7.2f} us")
print(f"ctypes call             {per_call(lambda: L.btd_launch_count()):7.2f} us")
# wall of the API calls, device work included (factor syncs on its error word; solve is async)
tf, ts, tt = [], [], []
for _ in range(200):
    h = X = None
    t0 = time.perf_counter()
    h = pkg.recursive_factorize(dA)
    t1 = time.perf_counter()
    X = pkg.recursive_solve(h, dB)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    tf.append(t1 - t0); ts.append(t2 - t1); tt.append(t3 - t0)
med = lambda v: sorted(v)[len(v) // 2] * 1e6
print(f"factorize wall {med(tf):.1f} us, solve call {med(ts):.1f} us, step incl. sync {med(tt):.1f} us")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
torch.cuda.synchronize()
ev[0].record()
for _ in range(200):
    h = X = None
    h = pkg.recursive_factorize(dA); X = pkg.recursive_solve(h, dB)
ev[1].record(); torch.cuda.synchronize()
print(f"back-to-back step {ev[0].elapsed_time(ev[1]) / 200 * 1e3:.1f} us")
