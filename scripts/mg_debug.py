import os, sys
sys.path.insert(0, os.getcwd())
os.environ["TOPO_MG_MIN_DOFS"] = "50"
import numpy as np
import paper_2005_05436_b200 as P
from paper_2005_05436_b200.configs import CONFIGS, fixed_dofs, load_vector
cfg = CONFIGS[1].scaled(16, 8, 0)
sK = 1e-9 + np.random.default_rng(3).uniform(0.3, 1.0, cfg.m) ** 3
with P.Context(*cfg.grid, rmin=1.0, nu=cfg.nu) as ctx:
    u, it, rr = ctx.solve_state(sK, load_vector(cfg), fixed_dofs(cfg), rtol=1e-13, multigrid=True)
    print(it, rr)
