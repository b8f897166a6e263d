"""Lower-triangle CSC of K on the device: the matrix
assemble_lower builds with setFromTriplets (fea.hpp:154-176). Pattern and
values are compared bit for bit with reference-generated fixtures
(tests/golden/csc.npz, golden_meta.json) and with the oracle."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

from tests.common import rel

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def P():
    import paper_2005_05436_b200 as P
    return P


@pytest.fixture(scope="module")
def meta():
    with open(os.path.join(GOLD, "golden_meta.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", ["5x4", "4x3x2", "3x1x2", "C1", "C4"])
def test_csc_matches_reference_fixture(P, meta, name):
    g = meta["csc"][name]
    grid = tuple(g["grid"])
    m = grid[0] * grid[1] * (grid[2] or 1)
    sK = np.random.default_rng(2005).uniform(0.01, 1.0, m)
    with P.Context(*grid, rmin=1.0) as ctx:
        cp, ri = ctx.csc_pattern()
        va = ctx.csc_values(sK)
        vd = ctx.csc_values(torch.from_numpy(sK).cuda()).cpu().numpy()  # device in / out
    assert ri.size == g["nnz"] and cp[-1] == g["nnz"]
    assert sha(cp.astype(np.int64)) == g["sha_col_ptr"]
    assert sha(ri) == g["sha_row_idx"]
    assert sha(va) == g["sha_values"]
    np.testing.assert_array_equal(va, vd)


@pytest.mark.parametrize("grid", [(7, 5, 0), (1, 1, 0), (5, 3, 4), (1, 1, 1), (2, 9, 1)])
def test_csc_matches_oracle(P, oracle_port, grid):
    m = grid[0] * grid[1] * (grid[2] or 1)
    sK = np.random.default_rng(7).uniform(0.01, 1.0, m)
    with P.Context(*grid, rmin=1.0) as ctx:
        cp, ri = ctx.csc_pattern()
        va = ctx.csc_values(sK)
    rc, rr, rv = oracle_port.assemble_lower_csc(grid, 0.3, sK)
    np.testing.assert_array_equal(cp, rc.astype(np.int64))
    np.testing.assert_array_equal(ri, rr)
    np.testing.assert_array_equal(va.view(np.int64), rv.view(np.int64))


@pytest.mark.parametrize("cid,grid", [(1, (40, 20, 0)), (4, (16, 10, 8))])
def test_pass_returns_csc_values(P, oracle_port, cid, grid):
    from paper_2005_05436_b200.configs import CONFIGS
    cfg = CONFIGS[cid].scaled(*grid)
    rng = np.random.default_rng(3)
    x, u = rng.uniform(0.01, 1.0, cfg.m), rng.normal(size=cfg.n)
    with P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu) as ctx:
        g = ctx.design_pass(x, u, beta=cfg.beta, move=cfg.move, volfrac=cfg.volfrac,
                            return_K=True)
        cp, ri = ctx.csc_pattern()
    ro = oracle_port.design_pass(cfg.grid, cfg.rmin, x, u, None, beta=cfg.beta, move=cfg.move,
                                 volfrac=cfg.volfrac, eta_override=g.eta)
    rc, rr, rv = oracle_port.assemble_lower_csc(cfg.grid, cfg.nu, ro.sKe)
    np.testing.assert_array_equal(ri, rr)
    assert rel(g.Kval, rv) <= 1e-12


def test_csc_rejects_multi_rank(P):
    from paper_2005_05436_b200.dist import ThreadHostComm  # noqa: F401
    with P.Context(8, 4, 0, rmin=1.5, rank=0, nranks=2) as ctx:
        with pytest.raises(P.InvalidArgument):
            ctx.csc_pattern()


def _restrict(cp, ri, va, fixed, n):
    """the reduced matrix of solve_equilibrium / EquilibriumSolver (fea.hpp:206-239,
    :316-361): entries with a fixed row or column dropped, free DOFs renumbered."""
    free = np.ones(n, bool)
    free[fixed] = False
    mp = np.cumsum(free) - 1
    cols = np.repeat(np.arange(n), np.diff(cp))
    keep = free[ri] & free[cols]
    rc = mp[cols[keep]]
    ncols = int(free.sum())
    cpr = np.zeros(ncols + 1, np.int64)
    np.add.at(cpr, rc + 1, 1)
    return np.cumsum(cpr), mp[ri[keep]].astype(np.int32), va[keep]


@pytest.mark.parametrize("cid,grid", [(1, (12, 6, 0)), (4, (7, 5, 4)), (5, (9, 6, 5))])
def test_reduced_csc_matches_reference(P, oracle_ref, cid, grid):
    from paper_2005_05436_b200.configs import CONFIGS, fixed_dofs
    cfg = CONFIGS[cid].scaled(*grid)
    fixed = fixed_dofs(cfg)
    sK = np.random.default_rng(9).uniform(0.01, 1.0, cfg.m)
    cp, ri, va = oracle_ref.assemble_lower_csc(cfg.grid, cfg.nu, sK)
    rcp, rri, rva = _restrict(cp.astype(np.int64), ri, va, fixed, cfg.n)
    with P.Context(*cfg.grid, rmin=1.0, nu=cfg.nu) as ctx:
        nf = ctx.csc_set_fixed(fixed)
        gcp, gri = ctx.csc_pattern()
        gva = ctx.csc_values(sK)
        assert nf == rcp.size - 1
        ctx.csc_set_fixed(None)  # back to the full matrix
        fcp, _ = ctx.csc_pattern()
        assert fcp.size == cfg.n + 1
        with pytest.raises(P.InvalidArgument):
            ctx.csc_set_fixed([cfg.n])
    np.testing.assert_array_equal(gcp, rcp)
    np.testing.assert_array_equal(gri, rri)
    np.testing.assert_array_equal(gva.view(np.int64), rva.view(np.int64))
