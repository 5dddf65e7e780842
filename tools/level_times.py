"""Per-level factor times (C-ABI timing hook, CUDA events on the launching stream).
    python tools/level_times.py N,n,d ..."""
import ctypes, sys
sys.path.insert(0, '.')
import torch
import paper_2509_03015_b200 as pkg
from paper_2509_03015_b200 import _native
for cfg in sys.argv[1:]:
    N, n, d = (int(v) for v in cfg.split(','))
    A, B = pkg.generate_spd_btd(N, n, d, seed=0)
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
    for _ in range(2):
        h = pkg.recursive_factorize(dA, profile=True)
    torch.cuda.synchronize()
    out = (ctypes.c_float * 64)(); cnt = ctypes.c_int64()
    _native.lib().btd_kernel_times(h._native.handle, out, 64, ctypes.byref(cnt))
    print(cfg, 'levels', [lv.num_blocks for lv in h.levels], 'base', h.base.num_blocks,
          'ms per level (last = base):', [round(out[i], 3) for i in range(cnt.value)], flush=True)
