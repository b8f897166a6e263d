import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["TOPO_DEBUG"] = "1"
import numpy as np
import paper_2005_05436_b200 as P
from paper_2005_05436_b200.configs import CONFIGS, make_inputs
from tests.test_gpu_multirank import run_ranks
cfg = CONFIGS[2].scaled(150, 50)
x, u, st = make_inputs(cfg)
os.environ["TOPO_OC_HOST"] = "1"
with P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu, state=st) as ctx:
    r = ctx.design_pass(x, u, beta=cfg.beta, move=cfg.move, volfrac=cfg.volfrac)
    print("single", r.lam, r.bisections, flush=True)
rs = run_ranks(P, cfg, x, u, st, 2)
print("ranks", rs[0].lam, rs[0].bisections)
