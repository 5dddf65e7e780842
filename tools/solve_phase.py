"""Per-phase cycle breakdown of solve_tma_kernel CTA 0, consumer thread 0 (debug build -DBTD_PHASE_PROF).
    python tools/solve_phase.py N,n,d
0: step bookkeeping, 1: wait for the slot, 2: F first mat-vec, 3: F barrier 1, 4: F second mat-vec,
5: F barrier 2, 6: B first mat-vec, 7: B barrier 1, 8: B second mat-vec, 9: B barrier 2,
10: fold/up steps, 11: slot release."""
import ctypes, os, sys
sys.path.insert(0, '.')
from paper_2509_03015_b200 import _native
_native.LIB_PATH = os.path.abspath(os.path.join('tools', 'libblocktri_b200_prof.so'))
import torch
import paper_2509_03015_b200 as pkg
L = _native.lib()
L.btd_debug_phase_cycles.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
for cfg in sys.argv[1:]:
    N, n, d = (int(x) for x in cfg.split(','))
    A, B = pkg.generate_spd_btd(N, n, d, seed=0)
    dA = pkg.BlockTridiagonalMatrix(torch.from_numpy(A.diag).cuda(), torch.from_numpy(A.sub).cuda())
    dB = pkg.BlockRhs(torch.from_numpy(B.blocks).cuda())
    h = pkg.recursive_factorize(dA)
    pkg.recursive_solve(h, dB)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 16)()
    L.btd_debug_phase_cycles(buf, 1)
    pkg.recursive_solve(h, dB)
    torch.cuda.synchronize()
    L.btd_debug_phase_cycles(buf, 1)
    tot = sum(buf[i] for i in range(12))
    print(cfg, 'total', tot, {i: f"{100*buf[i]/tot:.1f}%" for i in range(12)}, flush=True)
