"""Stage times (CUDA events) of one config's pass, for overlap experiments."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2005_05436_b200 as P
from paper_2005_05436_b200.configs import CONFIGS, make_inputs
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = CONFIGS[cid]
x, u, st = make_inputs(cfg)
xd, ud = torch.from_numpy(x).cuda(), torch.from_numpy(u).cuda()
with P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu, state=st) as ctx:
    kw = dict(beta=cfg.beta, move=cfg.move, volfrac=cfg.volfrac, outputs=False)
    for _ in range(3):
        ctx.design_pass(xd, ud, **kw)
    ctx.set_timing(True)
    acc = {}
    for _ in range(5):
        ctx.design_pass(xd, ud, **kw)
        for k, v in ctx.stage_times().items():
            acc[k] = acc.get(k, 0.0) + v / 5
    print(os.environ.get("TAG", ""), " ".join(f"{k} {v:.3f}" for k, v in acc.items()), flush=True)
