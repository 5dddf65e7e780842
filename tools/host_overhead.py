"""Host-side cost of recursive_factorize / recursive_solve (device inputs) vs device time."""
import cProfile, pstats, sys, time
import torch
sys.path.insert(0, '.')
import paper_2509_03015_b200 as pkg
for cfg in sys.argv[1:]:
    N, n, d = (int(v) for v in cfg.split(','))
    A, B = pkg.generate_spd_btd(N, n, d, seed=0)
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
    dB = pkg.BlockRhs(torch.from_numpy(B.blocks).cuda())
    for _ in range(3):
        h = pkg.recursive_factorize(dA); X = pkg.recursive_solve(h, dB)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    for _ in range(5):
        h = pkg.recursive_factorize(dA); X = pkg.recursive_solve(h, dB)
    torch.cuda.synchronize()
    pr.disable()
    print(cfg, f"wall per step {(time.perf_counter()-t0)/5*1e3:.3f} ms", flush=True)
    pstats.Stats(pr).sort_stats('tottime').print_stats(8)
