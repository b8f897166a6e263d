import os, sys, threading, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2005_05436_b200 as P
from paper_2005_05436_b200.configs import CONFIGS, make_inputs
from paper_2005_05436_b200.dist import ThreadHostComm, make_rank_context, slab_views
cfg = CONFIGS[2].scaled(150, 50)
x, u, st = make_inputs(cfg)
def dev_copy(ptr, n):
    t = torch.empty(n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    cudart = ctypes.CDLL("libcudart.so.12")
    cudart.cudaMemcpy(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(ptr), ctypes.c_size_t(8 * n), 3)
    return t.cpu().numpy()
with P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu, state=st) as ctx:
    p, n = ctx.device_buffer(100); cw_full = dev_copy(p, n)
comm = ThreadHostComm(2); res = {}
def work(r):
    j0, j1, xs, us, s_ = slab_views(cfg, x, u, st, r, 2)
    ctx = make_rank_context(cfg, s_, r, 2, comm=comm.for_rank(r))
    p, n = ctx.device_buffer(100); res[(r,'cw')] = dev_copy(p, n)
    p, n = ctx.device_buffer(101); res[(r,'hs_st')] = dev_copy(p, n)
    res[(r,'j')] = (j0, j1)
ts = [threading.Thread(target=work, args=(r,)) for r in range(2)]
[t.start() for t in ts]; [t.join() for t in ts]
S = cfg.nely
for r in range(2):
    j0, j1 = res[(r,'j')]; cw = res[(r,'cw')]
    print(r, "cw nan", np.isnan(cw).sum(), "maxdiff", np.nanmax(np.abs(cw - cw_full[j0*S:j1*S])), "hs_st range", res[(r,'hs_st')].min(), res[(r,'hs_st')].max())
