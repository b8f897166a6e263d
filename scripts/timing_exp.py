import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2005_05436_b200 as P
from paper_2005_05436_b200.configs import CONFIGS, make_inputs
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 5]
x, u, st = make_inputs(cfg)
xd, ud = torch.from_numpy(x).cuda(), torch.from_numpy(u).cuda()
kw = dict(beta=cfg.beta, move=cfg.move, volfrac=cfg.volfrac, outputs=False)
for use_stream in (False, True):
    for timing in (False, True):
        with P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu, state=st) as ctx:
            s = torch.cuda.Stream()
            if use_stream: ctx.set_stream(s.cuda_stream)
            ctx.set_timing(timing)
            for _ in range(3): ctx.design_pass(xd, ud, **kw)
            torch.cuda.synchronize()
            ev = []; wall = []
            for _ in range(8):
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                t0 = time.perf_counter(); e0.record(s); r = ctx.design_pass(xd, ud, **kw); e1.record(s); e1.synchronize()
                wall.append((time.perf_counter() - t0) * 1e3); ev.append(e0.elapsed_time(e1))
            print(f"stream={use_stream} timing={timing}: events {np.median(ev):.3f} ms wall {np.median(wall):.3f} ms internal {ctx.stage_times()['pass'] if timing else 0:.3f}", flush=True)
