"""d > 1 solve paths at n <= 64 (two-CTA wide levels, narrow levels, base, column slices): a
residual workload meant for compute-sanitizer (closed on this pool in the last session of round 2,
so it ran only as a plain residual check inside tests/test_gpu_parity.py's sweep cases)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2509_03015_b200 as pkg

cases = [(1500, 64, 4, 64, 8), (1500, 64, 3, 64, 8), (1500, 64, 7, 64, 8), (200, 64, 4, 8, 4),
         (1600, 50, 4, 64, 8), (1400, 64, 2, 64, 8)]
for N, n, d, cross, rho in cases:
    A, B = pkg.generate_spd_btd(N, n, d, seed=1)
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
    dB = pkg.BlockRhs(torch.from_numpy(B.blocks).cuda())
    cfg = pkg.RecursionConfig(crossover=cross, segment_length=rho)
    X = pkg.recursive_solve(pkg.recursive_factorize(dA, cfg), dB)
    rr = pkg.residual_report(dA, X, dB)[1]
    print(N, n, d, f"{rr:.2e}", flush=True)
    assert rr <= 1e-12
