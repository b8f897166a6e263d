"""Workloads for compute-sanitizer (scripts/sanitize.sh): one fused design pass
on C1 and on C4 (device inputs, default schedule incl. the CUDA graph on the
second call), one multigrid state solve, one Anderson step and the loop
records. Exits non-zero on any library error."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2005_05436_b200 as P
from paper_2005_05436_b200.configs import CONFIGS, fixed_dofs, load_vector, make_inputs

what = sys.argv[1] if len(sys.argv) > 1 else "all"
if what in ("all", "pass"):
    for cid in (1, 4):
        cfg = CONFIGS[cid]
        x, u, st = make_inputs(cfg)
        with P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu, state=st) as ctx:
            xd, ud = torch.from_numpy(x).cuda(), torch.from_numpy(u).cuda()
            for _ in range(2):  # eager, then captured into the pass graph
                r = ctx.design_pass(xd, ud, beta=cfg.beta, move=cfg.move, volfrac=cfg.volfrac,
                                    return_sk=True)
            print(cfg.name, "eta", r.eta, "lambda", r.lam, flush=True)
if what in ("all", "solve"):
    cfg = CONFIGS[5].scaled(32, 16, 16)
    sK = 1e-9 + np.random.default_rng(7).uniform(0.05, 1.0, cfg.m) ** 3
    with P.Context(*cfg.grid, rmin=1.0, nu=cfg.nu) as ctx:
        uu, it, rr = ctx.solve_state(sK, load_vector(cfg), fixed_dofs(cfg), rtol=1e-8,
                                     multigrid=True)
        print("MG solve", it, rr, flush=True)
torch.cuda.synchronize()
print("ok")
