"""A few multigrid-PCG iterations on C4 (for a kernel launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2005_05436_b200 as P
from paper_2005_05436_b200.configs import CONFIGS, fixed_dofs, load_vector
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
x = np.random.default_rng(1).uniform(0.01, 1.0, cfg.m)
sK = torch.from_numpy(1e-9 + x ** 3).cuda()
f = torch.from_numpy(load_vector(cfg)).cuda()
with P.Context(*cfg.grid, rmin=1.0, nu=cfg.nu) as ctx:
    u, it, rr = ctx.solve_state(sK, f, fixed_dofs(cfg), rtol=1e-30, maxit=2, multigrid=True)
    print(it, rr)
