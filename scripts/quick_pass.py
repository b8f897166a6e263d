"""Rough per-config pass timing (device-resident inputs, wall clock around the
synchronous C-ABI call). Development aid; bench.py is the measurement."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2005_05436_b200 as P
from paper_2005_05436_b200.configs import CONFIGS, make_inputs

args = [a for a in sys.argv[1:] if not a.startswith('--')]
npass = int(next((a.split('=')[1] for a in sys.argv[1:] if a.startswith('--passes=')), 6))
cids = [int(c) for c in args] or [1, 2, 3, 4, 5]
for cid in cids:
    cfg = CONFIGS[cid]
    t0 = time.time()
    x, u, st = make_inputs(cfg)
    xd, ud = torch.from_numpy(x).cuda(), torch.from_numpy(u).cuda()
    with P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu, state=st) as ctx:
        t1 = time.time()
        r = None
        ts = []
        for it in range(npass):
            torch.cuda.synchronize()
            a = time.perf_counter()
            r = ctx.design_pass(xd, ud, beta=cfg.beta, move=cfg.move, volfrac=cfg.volfrac, outputs=False)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - a)
        t = float(np.median(ts[2:] if len(ts) > 2 else ts))
        print(f"{cfg.name}: setup {t1-t0:.2f}s pass {t*1e3:.3f} ms  {cfg.m/t/1e6:.1f} Melem/s "
              f"eta {r.eta:.10f} it {r.eta_iters} lam {r.lam:.6e} bis {r.bisections} ev {r.evaluations} "
              f"c {r.c:.6e} launches {r.launches}", flush=True)
