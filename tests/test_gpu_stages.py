"""GPU parity of every stage entry point against the CPU oracle (C restatement
of the reference), on seeded inputs at sizes the oracle finishes in seconds.
Integer work bit-exact; floating point <= 1e-12 relative (max|a-b|/max|b|)
unless a test states otherwise."""
import math

import numpy as np
import pytest

from tests.common import rand_case, rel

pytestmark = pytest.mark.gpu

GRIDS_2D = [(3, 2, 0), (7, 5, 0), (30, 10, 0), (41, 17, 0)]
GRIDS_3D = [(1, 1, 1), (4, 3, 2), (6, 5, 7), (12, 7, 6)]


@pytest.fixture(scope="module")
def P():
    import paper_2005_05436_b200 as P
    return P


# ------------------------------------------------------------------ K0
@pytest.mark.parametrize("grid", GRIDS_2D + GRIDS_3D + [(300, 100, 0), (96, 48, 48)])
def test_index_pairs_bit_exact(P, oracle_port, grid):
    with P.Context(*grid, rmin=1.5) as ctx:
        iK, jK = ctx.build_symmetric_index_pairs()
        conn = ctx.build_connectivity()
    riK, rjK = oracle_port.index_pairs(grid)
    assert np.array_equal(iK, riK) and np.array_equal(jK, rjK)
    assert np.array_equal(conn, oracle_port.connectivity(grid))
    assert np.all(iK >= jK)


def test_connectivity_golden_3x2(P):
    # test_grid.cpp:35-46 hand enumeration
    expected = [[2, 3, 8, 9, 6, 7, 0, 1], [4, 5, 10, 11, 8, 9, 2, 3],
                [8, 9, 14, 15, 12, 13, 6, 7], [10, 11, 16, 17, 14, 15, 8, 9],
                [14, 15, 20, 21, 18, 19, 12, 13], [16, 17, 22, 23, 20, 21, 14, 15]]
    with P.Context(3, 2, 0, rmin=1.0) as ctx:
        assert ctx.build_connectivity().tolist() == expected


def test_pair_counts(P):
    # test_grid.cpp:54-73
    for grid, total in [((1, 1, 0), 72), ((1, 1, 1), 600), ((120, 120, 0), 1036800),
                        ((8, 8, 8), 307200)]:
        with P.Context(*grid, rmin=1.0) as ctx:
            iK, jK = ctx.build_symmetric_index_pairs()
            assert iK.size + jK.size == total


def test_index_pairs_on_device(P, oracle_port):
    import torch
    with P.Context(5, 4, 3, rmin=1.0) as ctx:
        iK, jK = ctx.build_symmetric_index_pairs(device=True)
        assert iK.is_cuda
        riK, rjK = oracle_port.index_pairs((5, 4, 3))
        assert np.array_equal(iK.cpu().numpy(), riK) and np.array_equal(jK.cpu().numpy(), rjK)
        ctx.build_symmetric_index_pairs(keep=True)
        p, cnt = ctx.device_buffer(P._lib.BUF_IK)
        assert p and cnt == riK.size


def test_overflow_rejected(P):
    # test_grid.cpp:48-52
    with pytest.raises(OverflowError):
        P.Context(40000, 40000, 0, rmin=1.0)


# ----------------------------------------------------------- filter.hpp
@pytest.mark.parametrize("bc", [0, 1])
@pytest.mark.parametrize("grid,rmin", [((6, 4, 0), 2.2), ((7, 5, 0), 3.0), ((30, 10, 0), 8.75),
                                       ((41, 17, 0), 4.6), ((3, 2, 0), 4.5), ((4, 3, 2), 1.5),
                                       ((6, 5, 7), 2.3), ((12, 7, 6), math.sqrt(3.0)),
                                       ((9, 8, 8), 4.0), ((2, 2, 2), 3.5)])
def test_filter_forward_adjoint(P, oracle_port, grid, rmin, bc):
    x, _, state = rand_case(grid, 11, passives=True)
    g = np.random.default_rng(5).uniform(-1, 1, x.size)
    f = oracle_port.filter(grid, rmin, bc)
    with P.Context(*grid, rmin=rmin, bc=bc, state=state) as ctx:
        assert ctx.ntaps == f.ntaps
        di, dj, dk, w = ctx.taps()
        odi, odj, odk, ow = f.taps()
        assert np.array_equal(di, odi) and np.array_equal(dj, odj) and np.array_equal(dk, odk)
        assert np.array_equal(w, ow)
        assert rel(ctx.hs(), f.hs()) <= 1e-13
        assert rel(ctx.apply_filter(x), oracle_port.apply_filter(f, x)) <= 1e-12
        xt = oracle_port.apply_filter(f, x)
        xt[state == 1] = 1.0
        xt[state == 2] = 0.0
        assert rel(ctx.apply_filter(x, pin=True), xt) <= 1e-12
        assert rel(ctx.apply_filter_adjoint(g), oracle_port.apply_filter_adjoint(f, g)) <= 1e-12
        for on in (False, True):
            got = ctx.backfilter(g, x, 0.45, 3.0, on)
            assert rel(got, oracle_port.backfilter(f, g, x, 0.45, 3.0, on)) <= 1e-12


def test_filter_tap_counts(P):
    # C1 241, C2 973, C3 3841, C4 19, C5 251
    for grid, rmin, T in [((300, 100, 0), 8.75, 241), ((600, 200, 0), 17.5, 973),
                          ((1200, 400, 0), 35.0, 3841), ((96, 48, 48), math.sqrt(3.0), 19),
                          ((24, 24, 24), 4.0, 251), ((8, 8, 8), 1.73205081, 27)]:
        with P.Context(*grid, rmin=rmin) as ctx:
            assert ctx.ntaps == T


def test_filter_rejects_small_radius(P):
    with pytest.raises(ValueError):  # test_filter.cpp:14-16
        P.Context(4, 4, 0, rmin=0.5)


def test_filter_length_mismatch(P):
    with P.Context(4, 4, 0, rmin=1.5) as ctx:
        with pytest.raises(ValueError):
            ctx.apply_filter(np.zeros(15))


def test_filter_device_arrays(P, oracle_port):
    import torch
    grid, rmin = (30, 10, 0), 2.4
    x, _, _ = rand_case(grid, 3)
    f = oracle_port.filter(grid, rmin)
    with P.Context(*grid, rmin=rmin) as ctx:
        xd = torch.from_numpy(x).cuda()
        out = ctx.apply_filter(xd)
        assert out.is_cuda
        assert rel(out.cpu().numpy(), oracle_port.apply_filter(f, x)) <= 1e-12


# ----------------------------------------------------------- projection
def test_project_and_derivatives(P, oracle_port):
    x = np.random.default_rng(29).uniform(0, 1, 1000)
    with P.Context(1000, 1, 0, rmin=1.0) as ctx:
        for eta, beta in [(0.5, 2.0), (0.45, 6.0), (0.3, 3.0), (0.55, 32.0), (0.4, 1e-6)]:
            assert rel(ctx.project(x, eta, beta), oracle_port.project(x, eta, beta)) <= 1e-14
            assert rel(ctx.project_derivative(x, eta, beta),
                       oracle_port.project_derivative(x, eta, beta)) <= 1e-13


def test_project_endpoints_bitwise(P):
    # SURVEY.md §7 hard part 6: pinned 0 / 1 land exactly on 0 / 1
    rng = np.random.default_rng(1)
    with P.Context(2, 1, 0, rmin=1.0) as ctx:
        for _ in range(200):
            eta, beta = rng.uniform(0.3, 0.7), rng.uniform(0.5, 32)
            p = ctx.project(np.array([0.0, 1.0]), eta, beta)
            assert p[0] == 0.0 and p[1] == 1.0


# -------------------------------------------------------------------- eta
@pytest.mark.parametrize("grid,beta,seed,passives", [((10, 10, 0), 2.0, 41, False),
                                                     ((10, 10, 0), 2.5, 42, True),
                                                     ((30, 10, 0), 4.0, 1, False),
                                                     ((120, 40, 0), 4.0, 7, False),
                                                     ((6, 5, 7), 8.0, 3, True)])
def test_eta_solve(P, oracle_port, grid, beta, seed, passives):
    x, _, state = rand_case(grid, seed, passives)
    with P.Context(*grid, rmin=1.0, state=state) as ctx:
        eta, it = ctx.solve_volume_preserving_eta(x, beta, 0.5)
    reta, rit = oracle_port.solve_eta(x, beta, 0.5, state)
    assert abs(eta - reta) <= 5e-8
    assert abs(oracle_port.eta_mismatch(x, beta, eta, state)) <= 1e-6


def test_eta_uniform_half(P):
    # test_filter.cpp:226-232
    with P.Context(10, 10, 0, rmin=1.0) as ctx:
        for beta in (0.7, 2.0, 9.0):
            eta, _ = ctx.solve_volume_preserving_eta(np.full(100, 0.5), beta, 0.3)
            assert abs(eta - 0.5) <= 1e-5


def test_eta_bad_beta(P):
    with P.Context(4, 4, 0, rmin=1.0) as ctx:
        with pytest.raises(ValueError):
            ctx.solve_volume_preserving_eta(np.full(16, 0.5), 0.0, 0.5)


# -------------------------------------------------------------------- fea
def test_simp_known_answers(P):
    # test_fea.cpp:81-90
    with P.Context(3, 1, 0, rmin=1.0) as ctx:
        sK, dsK = ctx.simp_interpolate(np.array([1.0, 0.0, 0.5]))
    assert sK[0] == pytest.approx(1.0) and sK[1] == pytest.approx(1e-9)
    assert sK[2] == pytest.approx(1e-9 + 0.125 * (1 - 1e-9))
    assert dsK[2] == pytest.approx(3.0 * 0.25 * (1 - 1e-9))


@pytest.mark.parametrize("grid", [(7, 5, 0), (30, 10, 0), (4, 3, 2), (12, 7, 6)])
def test_simp_assembly_sensitivity(P, oracle_port, grid):
    x, u, state = rand_case(grid, 23, passives=True)
    dim = 3 if grid[2] else 2
    kf, kl = oracle_port.element_stiffness(dim, 0.3)
    with P.Context(*grid, rmin=1.0, state=state) as ctx:
        sK, dsK = ctx.simp_interpolate(x)
        rsK, rdsK = oracle_port.simp(x)
        assert rel(sK, rsK) <= 1e-12 and rel(dsK, rdsK) <= 1e-12
        vals = ctx.assemble_values(rsK)
        assert rel(vals, oracle_port.assemble_values(rsK, kl)) <= 1e-15
        c, dc = ctx.compliance_and_sensitivity(u, x)
        rc, rdc = oracle_port.compliance_sensitivity(grid, kf, u, x, state)
        assert abs(c - rc) <= 1e-12 * abs(rc)
        assert rel(dc, rdc) <= 1e-12
        assert np.all(dc[state != 0] == 0.0)


def test_assembly_pattern_matches_reference_csc(P, oracle_ref):
    # lower-triangle values + index pairs, duplicate-summed, equal the
    # reference's assemble_lower CSC (fea.hpp:154-176)
    import scipy.sparse as sp
    for grid in [(3, 2, 0), (2, 2, 2)]:
        rng = np.random.default_rng(3)
        m = grid[0] * grid[1] * (grid[2] or 1)
        sKe = rng.uniform(0.1, 2.0, m)
        with P.Context(*grid, rmin=1.0) as ctx:
            iK, jK = ctx.build_symmetric_index_pairs()
            vals = ctx.assemble_values(sKe)
            n = ctx.n
        K = sp.coo_matrix((vals, (iK, jK)), shape=(n, n)).tocsc()
        cp, ri, va = oracle_ref.assemble_lower_csc(grid, 0.3, sKe)
        R = sp.csc_matrix((va, ri, cp), shape=(n, n))
        assert abs(K - R).max() <= 1e-14 * abs(R).max()


# --------------------------------------------------------------------- oc
def _oc_instance(m, seed, passives=False):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.1, 0.9, m)
    dc = -rng.uniform(0.05, 2.0, m)
    dV = np.full(m, 1.0 / m)
    state = None
    if passives:
        state = np.zeros(m, np.uint8)
        state[:2] = 1
        state[-2:] = 2
        x[:2] = 1.0
        x[-2:] = 0.0
        dc[:2] = dc[-2:] = 0.0
    return x, dc, dV, state


def test_lambda_and_candidate(P, oracle_port):
    x, dc, dV, _ = _oc_instance(1000, 3)
    with P.Context(1000, 1, 0, rmin=1.0) as ctx:
        assert ctx.lambda_upper_estimate(x, dc, dV, 0.5, 1000) == pytest.approx(
            oracle_port.lambda_upper(x, dc, dV, 0.5, 1000), rel=1e-13)
        for lam in (1e-3, 0.7, 5.0, 1e4):
            assert rel(ctx.oc_candidate(x, dc, dV, lam, 0.2),
                       oracle_port.oc_candidate(x, dc, dV, lam, 0.2)) == 0.0
        with pytest.raises(ValueError):
            ctx.oc_candidate(x, dc, dV, 0.0, 0.2)
        # test_oc.cpp:94-105 golden values
        c = ctx.oc_candidate(np.full(3, 0.5), np.array([-100.0, -1e-8, -0.3025]),
                             np.full(3, 0.25), 1.0, 0.2)
        assert c[0] == pytest.approx(0.7) and c[1] == pytest.approx(0.3)
        assert c[2] == pytest.approx(0.55)
        # test_oc.cpp:44-51 collapse to s, and zero
        s = 3.7
        assert ctx.lambda_upper_estimate(np.full(12, 0.4), np.full(12, -s / 12),
                                         np.full(12, 1 / 12), 0.4, 12) == pytest.approx(s, rel=1e-14)
        assert ctx.lambda_upper_estimate(np.full(5, 0.5), np.zeros(5), np.full(5, 0.2), 0.5,
                                         5) == 0.0


@pytest.mark.parametrize("m,seed,passives,move,volfrac", [(10, 17, False, 0.2, 0.5),
                                                          (20, 18, False, 0.2, 0.5),
                                                          (12, 19, True, 0.2, 0.5),
                                                          (5000, 20, False, 0.2, 0.5),
                                                          (5000, 21, True, 0.1, 0.12),
                                                          (3000, 22, False, 0.05, 0.9)])
def test_bisect_mean_mode(P, oracle_port, m, seed, passives, move, volfrac):
    x, dc, dV, state = _oc_instance(m, seed, passives)
    with P.Context(m, 1, 0, rmin=1.0, state=state) as ctx:
        r = ctx.bisect_update(x, dc, dV, P.OcParams(move=move, volfrac=volfrac),
                              volume_mode=P.VOL_MEAN)
    xo, lo, bo, eo = oracle_port.bisect_update(x, dc, dV, state, move=move, volfrac=volfrac)
    assert r.bisections == bo and r.evaluations == eo
    assert abs(r.lam - lo) <= 1e-10 * abs(lo)
    assert rel(r.xNew, xo) <= 1e-12
    if state is not None:
        assert np.array_equal(r.xNew[state != 0], x[state != 0])


def test_bisect_lambda_space_and_max(P, oracle_port):
    x, dc, dV, _ = _oc_instance(10, 3)
    with P.Context(10, 1, 0, rmin=1.0) as ctx:
        for kw in [dict(lambdaSpace=True, absTol=1e-10, lambdaMax=1e9),
                   dict(lambdaSpace=True, absTol=1e-8), dict(lambdaMax=50.0)]:
            prm = P.OcParams(move=0.95 if kw.get("lambdaMax") == 1e9 else 0.2, **kw)
            r = ctx.bisect_update(x, dc, dV, prm, volume_mode=P.VOL_MEAN)
            xo, lo, bo, eo = oracle_port.bisect_update(
                x, dc, dV, None, move=prm.move, lambda_space=prm.lambdaSpace,
                abs_tol=prm.absTol, lambda_max=prm.lambdaMax)
            assert r.bisections == bo
            assert abs(r.lam - lo) <= 1e-10 * abs(lo)
            assert rel(r.xNew, xo) <= 1e-12


def test_bisect_nonmonotone_callback_throws(P):
    # test_oc.cpp:179-188
    x, dc, dV, _ = _oc_instance(10, 5)
    seq = [0.2, 0.6, 0.9, 0.1, 0.8]
    calls = {"n": 0}

    def fake(_x):
        v = seq[min(calls["n"], 4)]
        calls["n"] += 1
        return v

    with P.Context(10, 1, 0, rmin=1.0) as ctx:
        with pytest.raises(RuntimeError):
            ctx.bisect_update(x, dc, dV, P.OcParams(volfrac=0.5), physical_volume=fake)


def test_bisect_callback_matches_mean(P, oracle_port):
    x, dc, dV, _ = _oc_instance(50, 9)
    with P.Context(50, 1, 0, rmin=1.0) as ctx:
        r = ctx.bisect_update(x, dc, dV, P.OcParams(), physical_volume=lambda v: v.mean())
    xo, lo, bo, _ = oracle_port.bisect_update(x, dc, dV)
    assert r.bisections == bo and abs(r.lam - lo) <= 1e-10 * lo and rel(r.xNew, xo) <= 1e-12


@pytest.mark.parametrize("mode", [2, 3])
@pytest.mark.parametrize("grid,rmin,passives", [((30, 10, 0), 2.4, False),
                                                ((40, 17, 0), 4.6, True),
                                                ((12, 7, 6), 2.3, True)])
def test_bisect_filtered_modes(P, oracle_port, grid, rmin, passives, mode):
    x, _, state = rand_case(grid, 31, passives)
    m = x.size
    rng = np.random.default_rng(4)
    dc = -rng.uniform(0.05, 2.0, m)
    dV = rng.uniform(0.5, 1.5, m) / m
    if state is not None:
        dc[state != 0] = 0.0
    f = oracle_port.filter(grid, rmin)
    with P.Context(*grid, rmin=rmin, state=state) as ctx:
        r = ctx.bisect_update(x, dc, dV, P.OcParams(), volume_mode=mode, eta=0.45, beta=2.0)
    xo, lo, bo, eo = oracle_port.bisect_update(x, dc, dV, state, mode=mode, filt=f, eta=0.45,
                                               beta=2.0)
    assert r.bisections == bo and r.evaluations == eo
    assert abs(r.lam - lo) <= 1e-10 * abs(lo)
    assert rel(r.xNew, xo) <= 1e-12


# ------------------------------------------------------------ primal-dual
@pytest.mark.parametrize("m,seed,move,volfrac,passives", [(400, 1, 0.2, 0.5, False),
                                                          (1000, 2, 0.05, 0.3, True),
                                                          (5000, 3, 0.1, 0.12, False),
                                                          (257, 4, 0.45, 0.5, True)])
def test_primal_dual_matches_oracle(P, oracle_port, m, seed, move, volfrac, passives):
    x, dc, dV, state = _oc_instance(m, seed, passives)
    ro = oracle_port.primal_dual_update(x, dc, dV, state, move=move, volfrac=volfrac)
    with P.Context(m, 1, 0, rmin=1.0, state=state) as ctx:
        r = ctx.primal_dual_update(x, dc, dV, P.OcParams(move=move, volfrac=volfrac))
    assert r.fell_back == bool(ro[3])
    assert r.bisections == ro[2]
    assert abs(r.lam - ro[1]) <= 1e-10 * abs(ro[1])
    assert rel(r.xNew, ro[0]) <= 1e-12


def test_primal_dual_reference_known_answers(P):  # test_oc.cpp:195-240
    rng = np.random.default_rng(5)
    m = 200
    x = np.full(m, 0.5)
    dV = np.full(m, 1.0 / m)
    dc = -rng.uniform(0.9, 1.1, m) / m
    with P.Context(m, 1, 0, rmin=1.0) as ctx:
        # wide box, nothing clamps: <= 3 iterations, lambda = lambda#
        r = ctx.primal_dual_update(x, dc, dV, P.OcParams(move=0.45, volfrac=0.5))
        lam_hash = ctx.lambda_upper_estimate(x, dc, dV, 0.5, m)
        assert r.bisections <= 3 and not r.fell_back
        assert abs(r.lam - lam_hash) <= 1e-6 * lam_hash
        # agrees with a tight bisection
        t = ctx.bisect_update(x, dc, dV, P.OcParams(move=0.2, volfrac=0.5, bisectRelTol=1e-12,
                                                    volumeTol=1e-9))
        p2 = ctx.primal_dual_update(x, dc, dV, P.OcParams(move=0.2, volfrac=0.5))
        assert np.max(np.abs(p2.xNew - t.xNew)) <= 1e-6
        assert abs(p2.xNew.mean() - 0.5) <= 1e-9
    # every element clamps: falls back to bisection
    m = 10
    x = np.full(m, 0.5)
    dV = np.full(m, 1.0 / m)
    dc = np.where(np.arange(m) % 2 == 0, -1e8, -1e-8)
    with P.Context(m, 1, 0, rmin=1.0) as ctx:
        r = ctx.primal_dual_update(x, dc, dV, P.OcParams(move=0.01, volfrac=0.5))
    assert abs(r.xNew.mean() - 0.5) <= 1e-3
    assert np.all(np.abs(r.xNew - x) <= 0.01 + 1e-14)


def test_primal_dual_device_loop_is_bitwise_host_loop(P, monkeypatch):
    """k_oc_pd (the dual fixed-point iteration in one cooperative launch) takes
    the reductions and decisions of the host-driven loop (TOPO_OC_PD_DEVICE=0,
    the multi-rank path) in the same order: same multiplier bits, iteration
    count and update, with and without the bisection fallback."""
    rng = np.random.default_rng(5)
    m = 48 * 24
    for move, volfrac in ((0.2, 0.5), (0.45, 0.3), (0.01, 0.5)):
        x = rng.uniform(0.05, 1.0, m)
        dc = -rng.uniform(0.1, 2.0, m)
        dV = np.full(m, 1.0 / m)
        res = []
        for dev in ("1", "0"):
            monkeypatch.setenv("TOPO_OC_PD_DEVICE", dev)
            with P.Context(48, 24, 0, rmin=1.5) as ctx:
                res.append(ctx.primal_dual_update(x, dc, dV, P.OcParams(move=move, volfrac=volfrac)))
        a, b = res
        assert (a.lam, a.bisections, a.fell_back) == (b.lam, b.bisections, b.fell_back)
        assert np.array_equal(a.xNew, b.xNew)
