"""Per-phase cycle breakdown of factor_level_kernel CTA 0 (debug build with -DBTD_PHASE_PROF).

    python tools/phase_prof.py N,n,d[,crossover] ...
Phases (btd_factor.cuh BTD_PHASE ids) are summed over CTA 0 of every factor launch.
"""
import ctypes, os, sys
sys.path.insert(0, '.')
from paper_2509_03015_b200 import _native
_native.LIB_PATH = os.path.abspath(os.environ.get('BTD_PROF_LIB', os.path.join('tools', 'libblocktri_b200_prof.so')))
import torch
import paper_2509_03015_b200 as pkg
L = _native.lib()
L.btd_debug_phase_cycles.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
names = {1: 'phase1', 2: 'pt_gemm', 3: 'D tiles', 4: 'panel chains', 5: 'crit tile upd',
         9: 'leaves', 10: 'doubling', 11: 'S potrf', 12: 'S B-pre (fill+SL)', 13: 'S B-trsm done', 14: 'S step', 15: 'p15'}
for cfg in sys.argv[1:]:
    v = [int(x) for x in cfg.split(',')]
    N, n, d = v[:3]
    cross = v[3] if len(v) > 3 else 64
    A, B = pkg.generate_spd_btd(N, n, d, seed=0)
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
    c = pkg.RecursionConfig(crossover=cross)
    pkg.recursive_factorize(dA, c)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 16)()
    L.btd_debug_phase_cycles(buf, 1)
    pkg.recursive_factorize(dA, c)
    torch.cuda.synchronize()
    L.btd_debug_phase_cycles(buf, 1)
    print(cfg, {names.get(i, str(i)): int(buf[i]) for i in range(16) if buf[i]}, flush=True)
