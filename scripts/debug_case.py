import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2005_05436_b200 as P
from oracle.oracle import Oracle
from tests.common import rand_case, rel
O = Oracle("port")
for grid, rmin, beta, seed in [((6, 5, 4), 4.0, 4.0, 9), ((30, 10, 0), 2.4, 2.0, 1)]:
    x, u, st = rand_case(grid, seed, False)
    f = O.filter(grid, rmin)
    with P.Context(*grid, rmin=rmin) as ctx:
        g = ctx.design_pass(x, u, beta=beta, move=0.2, volfrac=0.5)
        r = O.design_pass(grid, rmin, x, u, None, beta=beta, move=0.2, volfrac=0.5, filt=f, eta_override=g.eta)
        print(grid, "gpu", g.lam, g.bisections, g.evaluations, "orc", r.lam, r.bisections, r.evaluations)
        print("  hs", rel(ctx.hs(), f.hs()), "xNew", rel(g.xNew, r.xNew))
        xo, lo, bo, eo = O.bisect_update(x, g.dc, g.dV, None, move=0.2, volfrac=0.5, mode=3, filt=f)
        print("  oracle OC on gpu dc/dV:", lo, bo, eo, rel(g.xNew, xo))
        ro = ctx.bisect_update(x, g.dc, g.dV, P.OcParams(), volume_mode=3)
        print("  gpu standalone OC:", ro.lam, ro.bisections, ro.evaluations, rel(ro.xNew, xo))
        ro = ctx.bisect_update(x, g.dc, g.dV, P.OcParams(), volume_mode=1)
        xo, lo, bo, eo = O.bisect_update(x, g.dc, g.dV, None, move=0.2, volfrac=0.5, mode=1)
        print("  mean mode gpu/orc:", ro.lam, ro.bisections, lo, bo, rel(ro.xNew, xo))
