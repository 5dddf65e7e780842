"""Small factor + solve runs covering every kernel family, for compute-sanitizer (memcheck / racecheck)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2509_03015_b200 as pkg
from paper_2509_03015_b200 import _native

cases = [(40, 8, 2, 8, 4), (200, 8, 1, 8, 8), (150, 5, 4, 8, 8), (90, 6, 2, 8, 3),  # n <= 8: small kernels (DC 1/2/4, odd n)
          (60, 32, 1, 8, 4), (300, 64, 1, 64, 8), (600, 64, 1, 8, 8),  # small / level / stream / 2-CTA solve
         (80, 128, 2, 8, 4), (700, 128, 1, 64, 8), (30, 100, 1, 8, 4), (20, 256, 3, 4, 3)]  # tiled, wide solve, padded
for N, n, d, cross, rho in cases:
    A, B = pkg.generate_spd_btd(N, n, d, seed=1)
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
    dB = pkg.BlockRhs(torch.from_numpy(B.blocks).cuda())
    cfg = pkg.RecursionConfig(crossover=cross, segment_length=rho)
    for _ in range(2):
        X = pkg.recursive_solve(pkg.recursive_factorize(dA, cfg), dB)
    rr = pkg.residual_report(dA, X, dB)[1]
    print(N, n, d, f"{rr:.2e}", flush=True)
    assert rr <= 1e-12
# host-input path with the chunked / banded H2D
A, B = pkg.generate_spd_btd(2000, 64, 1, seed=2)
X = pkg.recursive_solve(pkg.recursive_factorize(A), B)
print("host", f"{pkg.residual_report(A, X, B)[1]:.2e}")
