"""Device state solve: K(sK) u = f on the free DOFs,
matrix-free Jacobi-PCG, against the reference's solve_equilibrium
(fea.hpp:205-239, a Cholesky factorisation) on small grids. The solutions
agree to the solver tolerance, not bitwise (direct vs iterative)."""
import numpy as np
import pytest

from tests.common import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2005_05436_b200 as P
    return P


@pytest.mark.parametrize("cid,grid,lo", [(1, (12, 6, 0), 0.3), (1, (20, 9, 0), 0.05),
                                         (4, (6, 4, 4), 0.3), (5, (8, 5, 4), 0.1)])
def test_solve_matches_reference(P, oracle_ref, cid, grid, lo):
    from paper_2005_05436_b200.configs import CONFIGS, fixed_dofs, load_vector
    cfg = CONFIGS[cid].scaled(*grid)
    sK = 1e-9 + np.random.default_rng(2).uniform(lo, 1.0, cfg.m) ** 3  # SIMP moduli
    f, fixed = load_vector(cfg), fixed_dofs(cfg)
    ur = oracle_ref.solve_state(cfg.grid, cfg.nu, sK, f, fixed)
    with P.Context(*cfg.grid, rmin=1.0, nu=cfg.nu) as ctx:
        u, it, rr = ctx.solve_state(sK, f, fixed, rtol=1e-13)
    assert rr <= 1e-13 and it > 0
    assert np.all(u[fixed] == 0.0)
    assert rel(u, ur) <= 1e-8, rel(u, ur)


def test_solve_edge_cases(P):
    from paper_2005_05436_b200.configs import CONFIGS, fixed_dofs
    cfg = CONFIGS[4].scaled(4, 3, 3)
    sK = np.ones(cfg.m)
    with P.Context(*cfg.grid, rmin=1.0) as ctx:
        u, it, rr = ctx.solve_state(sK, np.zeros(cfg.n), fixed_dofs(cfg))
        assert it == 0 and np.all(u == 0)
        with pytest.raises(P.InvalidArgument):
            ctx.solve_state(sK, np.ones(cfg.n), [cfg.n])


@pytest.mark.parametrize("cid,grid,lo", [(1, (16, 8, 0), 0.3), (1, (32, 16, 0), 0.05),
                                         (4, (8, 4, 4), 0.3), (5, (16, 8, 8), 0.1)])
def test_multigrid_solve_matches_reference(P, oracle_ref, cid, grid, lo, monkeypatch):
    from paper_2005_05436_b200.configs import CONFIGS, fixed_dofs, load_vector
    monkeypatch.setenv("TOPO_MG_MIN_DOFS", "50")  # coarsen these small grids
    cfg = CONFIGS[cid].scaled(*grid)
    sK = 1e-9 + np.random.default_rng(3).uniform(lo, 1.0, cfg.m) ** 3
    f, fixed = load_vector(cfg), fixed_dofs(cfg)
    ur = oracle_ref.solve_state(cfg.grid, cfg.nu, sK, f, fixed)
    with P.Context(*cfg.grid, rmin=1.0, nu=cfg.nu) as ctx:
        u, it, rr = ctx.solve_state(sK, f, fixed, rtol=1e-13, multigrid=True)
        uj, itj, _ = ctx.solve_state(sK, f, fixed, rtol=1e-13)
    assert rr <= 1e-13 and 0 < it < itj  # the V-cycle cuts the iteration count
    assert np.all(u[fixed] == 0.0)
    assert rel(u, ur) <= 1e-8, rel(u, ur)


def _numpy_apply(P, cfg, sK, x):
    """y = sum_e sK_e Ke x_e over the element DOF table (fea.hpp:162-174)."""
    Ke, _ = P.element_stiffness(3, cfg.nu)
    with P.Context(*cfg.grid, rmin=1.0, nu=cfg.nu) as ctx:
        dofs = np.asarray(ctx.build_connectivity()).reshape(cfg.m, -1).astype(np.int64)
    y = np.zeros(cfg.n)
    np.add.at(y, dofs.ravel(), (sK[:, None] * (x[dofs] @ Ke.T)).ravel())
    return y


# grids around the tile shape (31 x 7 nodes in y, z; x split in chunks)
@pytest.mark.parametrize("grid", [(3, 2, 2), (7, 5, 9), (12, 30, 6), (17, 31, 7), (40, 33, 17),
                                  (96, 48, 48)])
def test_stiffness_operator_variants(P, grid):
    from paper_2005_05436_b200.configs import CONFIGS
    cfg = CONFIGS[4].scaled(*grid)
    rng = np.random.default_rng(11)
    sK = 1e-9 + rng.uniform(0.01, 1.0, cfg.m) ** 3
    x = rng.standard_normal(cfg.n)
    with P.Context(*cfg.grid, rmin=1.0, nu=cfg.nu) as ctx:
        y0 = ctx.apply_stiffness(sK, x, 0)
        y1 = ctx.apply_stiffness(sK, x, 1)
        y2 = ctx.apply_stiffness(sK, x, 2)
    assert np.array_equal(y0, y1)  # one-launch tiles == colour launches, bit for bit
    assert rel(y0, y2) <= 1e-13, rel(y0, y2)
    if cfg.m <= 20000:
        yr = _numpy_apply(P, cfg, sK, x)
        assert rel(y0, yr) <= 1e-13, rel(y0, yr)


_VARIANT_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2005_05436_b200 as P
from paper_2005_05436_b200.configs import CONFIGS, fixed_dofs, load_vector
cfg = CONFIGS[5].scaled(32, 16, 16)
sK = 1e-9 + np.random.default_rng(7).uniform(0.05, 1.0, cfg.m) ** 3
with P.Context(*cfg.grid, rmin=1.0, nu=cfg.nu) as ctx:
    u, it, rr = ctx.solve_state(sK, load_vector(cfg), fixed_dofs(cfg), rtol=1e-12, multigrid=True)
np.save(sys.argv[2], u)
print(it, rr)
"""


# the multigrid's alternative code paths (env switches, read once per process):
# each must solve to the same answer
@pytest.mark.parametrize("env", [{}, {"TOPO_MG_MF1": "0"},
                                 {"TOPO_MG_NODE": "0"}, {"TOPO_MG_TILE": "0"},
                                 {"TOPO_MG_DENSE_COARSE": "0"}, {"TOPO_MG_LANES_MAX": "0"},
                                 {"TOPO_MG_DENSE_MAX": "100"}, {"TOPO_MG_BLOCK": "0"},
                                 {"TOPO_MG_GRAPH": "0"}])
def test_multigrid_variants_agree(P, tmp_path, env):
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "u.npy"
    e = dict(os.environ, TOPO_MG_MIN_DOFS="500", **env)
    r = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT, root, str(out)], env=e,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    it, rr = r.stdout.split()
    assert float(rr) <= 1e-12 and 0 < int(it) < 200
    u = np.load(out)
    from paper_2005_05436_b200.configs import CONFIGS, fixed_dofs, load_vector
    cfg = CONFIGS[5].scaled(32, 16, 16)
    sK = 1e-9 + np.random.default_rng(7).uniform(0.05, 1.0, cfg.m) ** 3
    with P.Context(*cfg.grid, rmin=1.0, nu=cfg.nu) as ctx:
        uj, _, _ = ctx.solve_state(sK, load_vector(cfg), fixed_dofs(cfg), rtol=1e-12)
    assert rel(u, uj) <= 1e-9, rel(u, uj)


def test_multigrid_state_reused_across_solves(P):
    # the context keeps its multigrid level storage between solves (the coarse
    # inverse and the captured PCG-iteration graph are rebuilt per solve, they
    # depend on the moduli): solving A, B, A on one context equals fresh
    # contexts bit for bit
    from paper_2005_05436_b200.configs import CONFIGS, fixed_dofs, load_vector
    cfg = CONFIGS[5].scaled(32, 16, 16)
    f, fixed = load_vector(cfg), fixed_dofs(cfg)
    rng = np.random.default_rng(21)
    sA = 1e-9 + rng.uniform(0.05, 1.0, cfg.m) ** 3
    sB = 1e-9 + rng.uniform(0.01, 1.0, cfg.m) ** 3

    def fresh(sK):
        with P.Context(*cfg.grid, rmin=1.0, nu=cfg.nu) as c:
            return c.solve_state(sK, f, fixed, rtol=1e-10, multigrid=True)

    ra, rb = fresh(sA), fresh(sB)
    with P.Context(*cfg.grid, rmin=1.0, nu=cfg.nu) as ctx:
        seq = [ctx.solve_state(s, f, fixed, rtol=1e-10, multigrid=True) for s in (sA, sB, sA)]
    for (u, it, rr), (u0, it0, rr0) in zip(seq, (ra, rb, ra)):
        assert it == it0 and rr == rr0
        assert np.array_equal(u, u0)


def test_pass_c_abi_matches_python_api(P):
    # bench.py times topo_design_pass through ctypes with prebuilt arguments:
    # the same call as Context.design_pass, bit for bit
    import ctypes as C
    import math
    import torch
    from paper_2005_05436_b200 import _lib as L
    from paper_2005_05436_b200.configs import CONFIGS, make_inputs
    cfg = CONFIGS[4].scaled(24, 12, 12)
    x, u, state = make_inputs(cfg)
    with P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu, state=state) as ctx:
        xd, ud = torch.from_numpy(x).cuda(), torch.from_numpy(u).cuda()
        r = ctx.design_pass(xd, ud, beta=cfg.beta, eta0=cfg.eta0, move=cfg.move,
                            volfrac=cfg.volfrac, outputs=False)
        pp = L.PassParams(P.SimpParams().c(), cfg.beta, cfg.eta0, cfg.move, cfg.volfrac,
                          math.nan, L.VOL_FILTERED, 1)
        xn = torch.empty(cfg.m, dtype=torch.float64, device="cuda")
        po = L.PassOut(None, None, None, None, None, xn.data_ptr(), None)
        assert ctx.lib.topo_design_pass(ctx.h, xd.data_ptr(), ud.data_ptr(), C.byref(pp),
                                        C.byref(po)) == 0
        assert torch.equal(xn, r.xNew) and po.eta == r.eta and po.c == r.c
