import sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2509_03015_b200 as pkg
g = np.load('tests/golden/reference_golden.npz')
i = 0
while f'solve{i}_meta' in g:
    N, n, d, seed, cross, rho, auto = (int(v) for v in g[f'solve{i}_meta'])
    if n <= 8:
        A, B = pkg.generate_spd_btd(N, n, d, seed)
        cfg = pkg.RecursionConfig(crossover=cross, segment_length=rho, auto_crossover=bool(auto))
        try:
            h = pkg.recursive_factorize(A, cfg)
            X = pkg.recursive_solve(h, B).blocks
            ref = g[f'solve{i}_x']
            print(i, (N, n, d, cross, rho), 'rel', np.abs(X - ref).max() / np.abs(ref).max(), flush=True)
        except Exception as e:
            print(i, (N, n, d, cross, rho), 'ERR', repr(e), flush=True)
    i += 1
