"""Probe: NotPositiveDefinite on the n > 64 tiled path (two half-level streams), each case in its
own process under a timeout (gpu_r02_pair.sh).  python tools/npd_probe.py CASE"""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2509_03015_b200 as pkg

CASES = {
    "one_tile1": [(9 * 3 + 1 + 2, 100)],
    "one_tile0": [(9 * 5 + 1 + 2, 5)],
    "two": [(9 * 3 + 1 + 2, 100), (9 * 5 + 1 + 2, 5)],
    "halfB": [(9 * 200 + 1 + 1, 70)],
}
name = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
A, _ = pkg.generate_spd_btd(N, 128, 1, seed=9)
diag = A.diag.copy()
for blk, i in CASES[name]:
    diag[blk, i, i] = -1.0e3
t = time.time()
try:
    pkg.recursive_factorize(pkg.BlockTridiagonalMatrix(torch.from_numpy(diag).cuda(), torch.from_numpy(A.sub).cuda()))
    print(name, "no error", flush=True)
except pkg.NotPositiveDefinite as e:
    print(name, "npd", e.pivot, e.level, e.member, e.block, f"{time.time() - t:.2f}s", flush=True)
