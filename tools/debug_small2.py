import sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2509_03015_b200 as pkg
N, n, d, seed, cross, rho = 10, 3, 2, 3, 2, 3
A, B = pkg.generate_spd_btd(N, n, d, seed)
cfg = pkg.RecursionConfig(crossover=cross, segment_length=rho)
h = pkg.recursive_factorize(A, cfg)
print("factor ok", flush=True)
X = pkg.recursive_solve(h, B).blocks
print("solve ok", flush=True)
