import ctypes, sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2509_03015_b200 as pkg
from paper_2509_03015_b200 import _native
L = _native.lib()
for (N, n, cross, rho) in [(40, 4, 4, 2), (300, 64, 64, 8), (1024, 32, 64, 8)]:
    A, B = pkg.generate_spd_btd(N, n, 1, 3)
    cfg = pkg.RecursionConfig(crossover=cross, segment_length=rho)
    st = _native.BtdStatus(); h = ctypes.c_void_p(); c = cfg._c()
    L.btd_create(N, n, ctypes.byref(c), ctypes.byref(h), ctypes.byref(st))
    pb, sb = ctypes.c_size_t(), ctypes.c_size_t()
    L.btd_factor_workspace(h, ctypes.byref(pb), ctypes.byref(sb))
    pers = torch.empty(pb.value, dtype=torch.uint8, device='cuda'); scr = torch.empty(sb.value, dtype=torch.uint8, device='cuda')
    dd = torch.full((N, n, n), -7.0, dtype=torch.float64, device='cuda'); ds = torch.full((N - 1, n, n), -7.0, dtype=torch.float64, device='cuda')
    s = torch.cuda.current_stream()
    rc = L.btd_factorize_from_host(h, A.diag.ctypes.data, A.sub.ctypes.data, dd.data_ptr(), ds.data_ptr(), pers.data_ptr(), scr.data_ptr(), ctypes.c_void_p(s.cuda_stream), 1, ctypes.byref(st))
    torch.cuda.synchronize()
    bd = np.where(np.abs(dd.cpu().numpy() - A.diag).reshape(N, -1).max(1) > 0)[0]
    bs = np.where(np.abs(ds.cpu().numpy() - A.sub).reshape(N - 1, -1).max(1) > 0)[0]
    print((N, n), 'rc', rc, st.message.decode(), 'bad diag rows', bd[:20], len(bd), 'bad sub rows', bs[:20], len(bs), flush=True)
