import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2509_03015_b200 as pkg
from paper_2509_03015_b200 import kalman
mdl = pkg.generate_rotation_model(8, 12, 1 << 20, seed=0)
A, B = kalman.build_normal_equations(mdl, device_out=True)
A2, B2 = pkg.generate_spd_btd(1 << 20, 8, 1, seed=0)
dA2 = pkg.BlockTridiagonalMatrix(torch.from_numpy(A2.diag).cuda(), torch.from_numpy(A2.sub).cuda())
dB2 = pkg.BlockRhs(torch.from_numpy(B2.blocks).cuda())
for name, a, b in (("kalman", A, B), ("synthetic", dA2, dB2)):
    for _ in range(2):
        h = pkg.recursive_factorize(a); X = pkg.recursive_solve(h, b)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(); h = pkg.recursive_factorize(a); e[1].record(); X = pkg.recursive_solve(h, b); e[2].record()
    torch.cuda.synchronize()
    print(name, a.diag.shape, a.diag.dtype, a.diag.is_contiguous(), b.blocks.shape, b.blocks.stride(), "factor", e[0].elapsed_time(e[1]), "solve", e[1].elapsed_time(e[2]), flush=True)
