"""Quick device-resident timing of recursive_factorize + recursive_solve (dev tool)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2509_03015_b200 as pkg

def run(N, n, d, reps=5):
    A, B = pkg.generate_spd_btd(N, n, d, seed=0)
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
    dB = pkg.BlockRhs(torch.from_numpy(B.blocks).cuda())
    for _ in range(2):
        h = pkg.recursive_factorize(dA); X = pkg.recursive_solve(h, dB)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf, ts = [], []
    for _ in range(reps):
        e[0].record(); h = pkg.recursive_factorize(dA); e[1].record(); X = pkg.recursive_solve(h, dB); e[2].record()
        torch.cuda.synchronize(); tf.append(e[0].elapsed_time(e[1])); ts.append(e[1].elapsed_time(e[2]))
    _, rres = pkg.residual_report(dA, X, dB)
    print(f"N={N} n={n} d={d}: factor {np.median(tf):.3f} ms  solve {np.median(ts):.3f} ms  rel_res {rres:.2e}", flush=True)

for cfg in sys.argv[1:]:
    N, n, d = (int(v) for v in cfg.split(','))
    run(N, n, d)
