import sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2509_03015_b200 as pkg
g = np.load('tests/golden/reference_golden.npz')
i = 0
while f'solve{i}_meta' in g:
    N, n, d, seed, cross, rho, auto = (int(v) for v in g[f'solve{i}_meta'])
    A, B = pkg.generate_spd_btd(N, n, d, seed)
    cfg = pkg.RecursionConfig(crossover=cross, segment_length=rho, auto_crossover=bool(auto))
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
    try:
        xd = pkg.recursive_solve(pkg.recursive_factorize(dA, cfg), B).blocks
        ed = None
    except Exception as e:
        ed = repr(e)
    try:
        xh = pkg.recursive_solve(pkg.recursive_factorize(A, cfg), B).blocks
        eh = None
    except Exception as e:
        eh = repr(e)
    print(i, (N, n, d, cross, rho), 'dev err', ed, 'host err', eh, 'equal', (ed is None and eh is None and np.array_equal(xd, xh)), flush=True)
    i += 1
