"""Device state solve timing on a config grid (sK = SIMP moduli of x ~ U(0.01, 1)):
Jacobi-PCG and multigrid-PCG to relres 1e-6 (plus a fixed-iteration cost probe)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2005_05436_b200 as P
from paper_2005_05436_b200.configs import CONFIGS, fixed_dofs, load_vector
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["jacobi", "mg"]
cfg = CONFIGS[cid]
x = np.random.default_rng(1).uniform(0.01, 1.0, cfg.m)
sK = torch.from_numpy(1e-9 + x ** 3 * (1 - 1e-9)).cuda()
f = torch.from_numpy(load_vector(cfg)).cuda()
fixed = fixed_dofs(cfg)
with P.Context(*cfg.grid, rmin=1.0, nu=cfg.nu) as ctx:
    for mode in modes:
        mg = mode == "mg"
        ctx.solve_state(sK, f, fixed, rtol=1e-30, maxit=2, multigrid=mg)
        torch.cuda.synchronize()
        t = time.perf_counter()
        u, it, rr = ctx.solve_state(sK, f, fixed, rtol=1e-6, maxit=20000, multigrid=mg)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(f"{cfg.name} n {cfg.n} [{mode}] to relres 1e-6: {it} iterations, {dt:.3f} s "
              f"({dt/it*1e3:.2f} ms/iter incl. setup), relres {rr:.2e}", flush=True)
