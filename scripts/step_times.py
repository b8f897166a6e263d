"""Per-step pass times with the bench's L2 flush (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2005_05436_b200 as P
from paper_2005_05436_b200.configs import CONFIGS, make_inputs

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
flush_on = "--noflush" not in sys.argv
if "--nogc" in sys.argv:
    import gc
    gc.disable()
cfg = CONFIGS[cid]
x, u, state = make_inputs(cfg)
ctx = P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu, device=0, state=state)
xd, ud = torch.from_numpy(x).cuda(), torch.from_numpy(u).cuda()
st = torch.cuda.Stream()
ctx.set_stream(st.cuda_stream)
kw = dict(beta=cfg.beta, eta0=cfg.eta0, move=cfg.move, volfrac=cfg.volfrac, outputs=False)
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for _ in range(3):
    ctx.design_pass(xd, ud, **kw)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    if flush_on:
        with torch.cuda.stream(st):
            flush.fill_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    r = ctx.design_pass(xd, ud, **kw)
    e1.record(st)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print(cfg.name, "flush" if flush_on else "noflush", " ".join(f"{t:.3f}" for t in ts))

if "--variants" in sys.argv:
    import gc
    import ctypes as C
    from paper_2005_05436_b200 import _lib as L
    # (a) gc disabled
    gc.disable()
    ts = []
    for _ in range(20):
        with torch.cuda.stream(st):
            flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ctx.design_pass(xd, ud, **kw)
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    gc.enable()
    print("gc off ", " ".join(f"{t:.3f}" for t in ts))
    # (b) direct C-ABI call, preallocated outputs
    xn = torch.empty(cfg.m, dtype=torch.float64, device="cuda")
    pp = L.PassParams(L.Simp(cfg.e0, cfg.emin, cfg.penal), cfg.beta, cfg.eta0, cfg.move,
                      cfg.volfrac, float("nan"), L.VOL_FILTERED, 1)
    po = L.PassOut(None, None, None, None, None, xn.data_ptr(), None)
    ts = []
    for _ in range(20):
        with torch.cuda.stream(st):
            flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ctx.lib.topo_design_pass(ctx.h, xd.data_ptr(), ud.data_ptr(), C.byref(pp), C.byref(po))
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print("c-abi  ", " ".join(f"{t:.3f}" for t in ts))
