"""Lower-triangle CSC on C5 (or another config): pattern setup time, value
kernel time (CUDA events) and its HBM rate; the pass with Kval instead of sK."""
import os, sys, time
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
    t0 = time.time()
    cp, ri = ctx.csc_pattern(device=True)
    torch.cuda.synchronize()
    nnz = ri.numel()
    print(f"{cfg.name}: n {ctx.n} nnz {nnz} pattern setup {time.time()-t0:.2f} s", flush=True)
    del cp, ri
    E = torch.rand(cfg.m, dtype=torch.float64, device="cuda")
    vals = ctx.csc_values(E)
    for _ in range(2):
        ctx.csc_values(E)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a = time.perf_counter()
        ctx.csc_values(E)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - a)
    t = min(ts)
    print(f"csc values: {t*1e3:.3f} ms  {nnz*8/t/1e9:.0f} GB/s written  ({nnz/t/1e9:.2f} G slots/s)")
    del vals
    kw = dict(beta=cfg.beta, move=cfg.move, volfrac=cfg.volfrac, outputs=False)
    for mode in ("sK", "Kval", "both"):
        ts = []
        for it in range(4):
            torch.cuda.synchronize()
            a = time.perf_counter()
            ctx.design_pass(xd, ud, write_sk=mode != "Kval", return_K=mode != "sK", out_device=True, **kw)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - a)
        print(f"pass with {mode}: {min(ts[1:])*1e3:.3f} ms", flush=True)
