import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2005_05436_b200 as P
from paper_2005_05436_b200.configs import CONFIGS, make_inputs
for cfg in (CONFIGS[2].scaled(150, 50), CONFIGS[1]):
    x, u, st = make_inputs(cfg)
    with P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu, state=st) as ctx:
        r = ctx.design_pass(x, u, beta=cfg.beta, move=cfg.move, volfrac=cfg.volfrac)
        ro = ctx.bisect_update(x, r.dc, r.dV, P.OcParams(move=cfg.move, volfrac=cfg.volfrac), volume_mode=3)
        print(cfg.name, os.environ.get("TOPO_OC_HOST"), r.lam, r.bisections, r.evaluations, "| standalone", ro.lam, ro.bisections)
