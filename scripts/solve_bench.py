"""Device state solve timing: per-iteration cost of the matrix-free PCG on a
config grid (sK = SIMP moduli of x ~ U(0.01, 1)), fixed iteration budget."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2005_05436_b200 as P
from paper_2005_05436_b200.configs import CONFIGS, fixed_dofs, load_vector
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = CONFIGS[cid]
x = np.random.default_rng(1).uniform(0.01, 1.0, cfg.m)
sK = torch.from_numpy(1e-9 + x ** 3 * (1 - 1e-9)).cuda()
f = torch.from_numpy(load_vector(cfg)).cuda()
fixed = fixed_dofs(cfg)
with P.Context(*cfg.grid, rmin=1.0, nu=cfg.nu) as ctx:
    ctx.solve_state(sK, f, fixed, rtol=1e-30, maxit=5)
    torch.cuda.synchronize()
    t = time.perf_counter()
    u, it, rr = ctx.solve_state(sK, f, fixed, rtol=1e-30, maxit=iters)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{cfg.name}: n {cfg.n} {it} PCG iterations {dt*1e3:.1f} ms  {dt/it*1e3:.3f} ms/iter "
          f"relres {rr:.3e}  ({cfg.n/(dt/it)/1e9:.2f} G DOF/s per iteration)")
    t = time.perf_counter()
    u, it, rr = ctx.solve_state(sK, f, fixed, rtol=1e-6, maxit=20000)
    torch.cuda.synchronize()
    print(f"  to relres 1e-6: {it} iterations, {time.perf_counter()-t:.2f} s, relres {rr:.2e}")
