"""Per-phase cycle breakdown of factor_level_kernel CTA 0 (debug build with -DBTD_PHASE_PROF)."""
import ctypes, os, subprocess, sys
sys.path.insert(0, '.')
from paper_2509_03015_b200 import _native
dbg = os.path.join('tools', 'libblocktri_b200_prof.so')
_native.LIB_PATH = os.path.abspath(dbg)
import torch
import paper_2509_03015_b200 as pkg
L = _native.lib()
L.btd_debug_phase_cycles.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
names = ['-', 'phase1 (A: potrf | B: SL+fill)', 'phase2 pt_gemm', 'phase2 D tiles', '4', '5', '6', '7', '8', '9']
for cfg in sys.argv[1:]:
    N, n, d = (int(v) for v in cfg.split(','))
    A, B = pkg.generate_spd_btd(N, n, d, seed=0)
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
    pkg.recursive_factorize(dA)
    buf = (ctypes.c_ulonglong * 16)()
    L.btd_debug_phase_cycles(buf, 1)
    pkg.recursive_factorize(dA)
    L.btd_debug_phase_cycles(buf, 1)
    print(cfg, {names[i]: int(buf[i]) for i in range(10)})
