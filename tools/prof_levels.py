"""Per-level factor kernel times (C-ABI timing hook, CUDA events on the launching stream)."""
import ctypes, sys
sys.path.insert(0, '.')
import torch
import paper_2509_03015_b200 as pkg
from paper_2509_03015_b200 import _native
for cfg in sys.argv[1:]:
    N, n, d = (int(v) for v in cfg.split(','))
    A, B = pkg.generate_spd_btd(N, n, d, seed=0)
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
    for rep in range(3):
        h = pkg.recursive_factorize(dA, profile=True)
        torch.cuda.synchronize()
    L = _native.lib()
    cnt = ctypes.c_int64()
    out = (ctypes.c_float * 64)()
    L.btd_kernel_times(h._native.handle, out, 64, ctypes.byref(cnt))
    print(cfg, "factor kernel ms per level:", [round(out[i], 4) for i in range(cnt.value)], flush=True)
