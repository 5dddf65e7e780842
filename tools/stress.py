"""Randomised parity stress run (GPU engine vs the CPU oracle) over shapes, configs and input kinds
(numpy host, pinned torch, device torch), repeated calls (graph replays).  python tools/stress.py [cases] [seed]"""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2509_03015_b200 as pkg
from oracle import blocktri_port as port

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
ns = [1, 2, 3, 5, 8, 12, 16, 31, 32, 33, 48, 63, 64, 65, 80, 100, 128, 150, 192, 256]
worst = 0.0
t0 = time.time()
for i in range(cases):
    n = int(rng.choice(ns))
    nmax = max(3, int(float(sys.argv[3]) if len(sys.argv) > 3 else 4e6) // (n * n * 8 * 3))  # keep the oracle quick
    N = int(rng.integers(1, min(3000, nmax) + 1))
    d = int(rng.integers(1, 6))
    cross = int(rng.choice([1, 2, 4, 8, 16, 64]))
    rho = int(rng.choice([1, 2, 3, 5, 8, 12]))
    A, B = pkg.generate_spd_btd(N, n, d, seed=i)
    cfg = pkg.RecursionConfig(crossover=cross, segment_length=rho, max_levels=64)
    kind = i % 3
    if kind == 0:
        AA, BB = A, B
    elif kind == 1:
        AA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).pin_memory(), torch.from_numpy(A.sub).pin_memory())
        BB = pkg.BlockRhs(torch.from_numpy(B.blocks).pin_memory())
    else:
        AA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
        BB = pkg.BlockRhs(torch.from_numpy(B.blocks).cuda())
    for rep in range(3):
        X = pkg.recursive_solve(pkg.recursive_factorize(AA, cfg), BB).blocks
    X = X.cpu().numpy() if hasattr(X, 'cpu') else X
    ref = port.solve(port.factorize(A.diag, A.sub, cross, rho, 64), B.blocks)
    rel = float(np.abs(X - ref).max() / max(np.abs(ref).max(), 1e-300))
    _, rres = pkg.residual_report(A, pkg.BlockRhs(X), B)
    worst = max(worst, rel)
    ok = rel <= 1e-10 and rres <= 1e-12
    print(f"{i:3d} N={N:5d} n={n:3d} d={d} cross={cross:2d} rho={rho:2d} kind={kind} rel={rel:.2e} res={rres:.2e} {'ok' if ok else 'FAIL'}", flush=True)
    assert ok
print(f"all {cases} ok, worst rel {worst:.2e}, {time.time() - t0:.0f} s")
