"""One factor+solve at a given config (for ncu)."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2509_03015_b200 as pkg
N, n, d = (int(v) for v in sys.argv[1].split(','))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
A, B = pkg.generate_spd_btd(N, n, d, seed=0)
dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
dB = pkg.BlockRhs(torch.from_numpy(B.blocks).cuda())
for _ in range(reps):
    h = pkg.recursive_factorize(dA)
    X = pkg.recursive_solve(h, dB)
torch.cuda.synchronize()
