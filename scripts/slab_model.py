"""Compute-side model of strong scaling on one GPU: the C5 grid cut into N
x-slabs, ONE slab timed as a single-rank pass (mirror faces instead of halos:
the same kernels and traffic per rank, no communication). Prints the slab pass
time and the efficiency bound t1 / (N tN) that the compute side alone allows;
NCCL halos (2 x 0.9 MB + 2 x 1.8 MB per pass at N = 8) and 5 small allreduces
come on top. Development aid for DESIGN.md §6 (the pool leases one GPU)."""
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2005_05436_b200 as P
from paper_2005_05436_b200 import _lib as L
from paper_2005_05436_b200.configs import CONFIGS

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
base = CONFIGS[cid]
t1 = None
for n in (1, 2, 4, 8):
    cfg = base.scaled(base.nelx // n, base.nely, base.nelz)
    rng = np.random.default_rng(1)
    xd = torch.from_numpy(rng.uniform(0.01, 1.0, cfg.m)).cuda()
    ud = torch.from_numpy(rng.normal(size=cfg.n)).cuda()
    with P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu) as ctx:
        stream = torch.cuda.Stream()
        ctx.set_stream(stream.cuda_stream)
        pp = L.PassParams(P.SimpParams().c(), cfg.beta, cfg.eta0, cfg.move, cfg.volfrac, math.nan,
                          L.VOL_FILTERED, 1)
        xnew = torch.empty(cfg.m, dtype=torch.float64, device="cuda")
        po = L.PassOut(None, None, None, None, None, xnew.data_ptr(), None)
        ts = []
        for it in range(12):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            assert ctx.lib.topo_design_pass_begin(ctx.h, xd.data_ptr(), ud.data_ptr(), C.byref(pp),
                                                  C.byref(po)) == 0
            e1.record(stream)
            assert ctx.lib.topo_design_pass_end(ctx.h, C.byref(po)) == 0
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = float(np.median(ts[4:]))
    t1 = t1 or t
    print(f"N {n}: slab {cfg.nelx}x{cfg.nely}x{cfg.nelz}  {t:.4f} ms per pass  "
          f"compute-side efficiency bound {t1 / (n * t):.3f}", flush=True)
    del xd, ud, xnew
    torch.cuda.empty_cache()
