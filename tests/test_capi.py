"""CPU-only checks of the product boundary: the C-ABI library loads and exports
every symbol include/*.h declares; host setup helpers (element matrices,
Appendix-B generator, partition, configs) and the host replays of the scalar
control flow (the code the multi-GPU path runs on the host, and the device
kernels run per block) agree with the oracle. No compute call needs a GPU."""
import ctypes as C
import glob
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def P():
    import paper_2005_05436_b200 as P
    return P


@pytest.fixture(scope="module")
def lib(P):
    return P._lib.load()


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(topo_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


def test_library_exports_every_declared_symbol(P):
    lib = C.CDLL(P._lib.LIB_PATH)
    decl = declared_functions()
    assert len(decl) >= 30
    missing = [n for n in decl if not hasattr(lib, n)]
    assert not missing, missing
    assert set(P._lib.EXPORTS) <= set(decl)


def test_library_is_sm100a(P):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", P._lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_element_stiffness_bits_equal_reference_fixture(P):
    d = np.load(os.path.join(ROOT, "tests", "golden", "ke.npz"))
    for dim, f, l in ((2, "q4_full", "q4_lower"), (3, "h8_full", "h8_lower")):
        full, lower = P.element_stiffness(dim, 0.3)
        np.testing.assert_array_equal(full, d[f])
        np.testing.assert_array_equal(lower, d[l])
    with pytest.raises(ValueError):
        P.element_stiffness(2, 0.5)


def test_generator_is_counter_based(P):
    a = P.generate(7, 1, "uniform", 0.01, 1.0, 1000)
    b = P.generate(7, 1, "uniform", 0.01, 1.0, 300, offset=700)
    np.testing.assert_array_equal(a[700:], b)
    assert a.min() >= 0.01 and a.max() < 1.0
    z = P.generate(7, 2, "normal", 0.0, 1.0, 200000)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01
    z2 = P.generate(7, 2, "normal", 0.0, 1.0, 1001, offset=99)
    np.testing.assert_array_equal(z[99:1100], z2)


def test_configs_and_inputs(P):
    from paper_2005_05436_b200.configs import CONFIGS, fixed_dofs, make_inputs, passive_state
    st = passive_state(CONFIGS[2])
    assert np.bincount(st).tolist() == [82290, 24000, 13710]
    x, u, s = make_inputs(CONFIGS[2])
    assert np.all(x[s == 1] == 1.0) and np.all(x[s == 2] == 0.0)
    x1, u1, _ = make_inputs(CONFIGS[1])
    x1b, _, _ = make_inputs(CONFIGS[1])
    np.testing.assert_array_equal(x1, x1b)
    assert np.all(u1[fixed_dofs(CONFIGS[1])] == 0)
    assert fixed_dofs(CONFIGS[4]).size == 3 * 49 * 49
    assert [CONFIGS[c].m for c in range(1, 6)] == [30000, 120000, 480000, 221184, 14155776]
    assert CONFIGS[5].n == 43022595 and CONFIGS[5].m * 300 > 2 ** 31  # int64 offsets needed


def test_partition_domain_errors(P):
    with pytest.raises(ValueError):
        P.partition_domain((4, 3, 0), [0], [0])
    with pytest.raises(ValueError):
        P.partition_domain((4, 3, 0), [12], [])
    st = P.partition_domain((4, 3, 0), [3, 1], [5])
    assert (st == 1).sum() == 2 and (st == 2).sum() == 1


def test_context_without_gpu_fails_loudly(P):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.TopoError):
        P.Context(4, 4, 0, rmin=1.5)


# ------------------------------------------------ host control replays
def _oc_setup(m, seed, move, volfrac, passives=False):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.1, 0.9, m)
    dc = -rng.uniform(0.05, 2.0, m)
    dV = np.full(m, 1.0 / m)
    state = None
    if passives:
        state = np.zeros(m, np.uint8)
        state[:2] = 1
        state[-2:] = 2
        x[:2], x[-2:] = 1.0, 0.0
        dc[:2] = dc[-2:] = 0.0
    act = np.ones(m, bool) if state is None else state == 0
    ocP = x[act] * np.sqrt(np.maximum(0.0, -dc[act] / dV[act]))
    lo = np.maximum(0.0, x[act] - move)
    hi = np.minimum(1.0, x[act] + move)

    def volume(s):  # mean(xc) with the reference's sequential sum (cumsum is sequential)
        f = ocP / s if s > 0 else np.where(ocP > 0, np.inf, 0.0)
        full = x.copy()
        full[act] = np.minimum(np.maximum(f, lo), hi)
        return float(np.cumsum(full)[-1] / m)

    s = 0.0
    for v in ocP:  # lambda# with the reference's sequential sum (oc.hpp:34-36)
        s += v
    root = s / (m * volfrac)
    return x, dc, dV, state, volume, root * root


@pytest.mark.parametrize("m,seed,move,volfrac,pas", [(10, 1, 0.2, 0.5, False),
                                                      (50, 2, 0.2, 0.5, True),
                                                      (400, 3, 0.1, 0.12, False),
                                                      (400, 4, 0.05, 0.9, False),
                                                      (1000, 5, 0.2, 0.3, True)])
@pytest.mark.parametrize("speculative", [0, 1, 2])
def test_host_oc_replay_matches_oracle(P, lib, oracle_port, m, seed, move, volfrac, pas,
                                       speculative):
    x, dc, dV, state, volume, lam0 = _oc_setup(m, seed, move, volfrac, pas)
    xo, lo, bo, eo = oracle_port.bisect_update(x, dc, dV, state, move=move, volfrac=volfrac)
    prm = P._lib.OcParams(move, volfrac, 1e-4, 1e-3, 0, 1e-8, 0.0)
    cb = P._lib.SFUN(lambda _u, s: volume(s))
    lam, bis, ev, sf, nb = C.c_double(), C.c_int32(), C.c_int32(), C.c_double(), C.c_int32()
    st = lib.topo_host_oc_replay(C.byref(prm), lam0, cb, None, speculative, C.byref(lam),
                                 C.byref(bis), C.byref(ev), C.byref(sf), C.byref(nb))
    assert st == 0
    assert (lam.value, bis.value, ev.value) == (lo, bo, eo)
    if speculative:
        per = 4 if speculative == 1 else 5  # bisection levels per batch
        assert nb.value <= max(2, (bo + per - 2) // (per - 1) + 2)


def test_host_oc_replay_nonmonotone(P, lib):
    seq = iter([0.2, 0.6, 0.9, 0.1, 0.8] + [0.8] * 1000)
    prm = P._lib.OcParams(0.2, 0.5, 1e-4, 1e-3, 0, 1e-8, 0.0)
    cb = P._lib.SFUN(lambda _u, s: next(seq))
    st = lib.topo_host_oc_replay(C.byref(prm), 2.0, cb, None, 0, None, None, None, None, None)
    assert st == 3  # TOPO_ENONMONO, oc.hpp:160-161


@pytest.mark.parametrize("beta,seed", [(2.0, 1), (4.0, 2), (8.0, 3), (1.0, 4)])
def test_host_eta_replay_matches_oracle(P, lib, oracle_port, beta, seed):
    x = np.random.default_rng(seed).uniform(0.05, 0.95, 500)
    eta_o, it_o = oracle_port.solve_eta(x, beta, 0.5)
    m = x.size

    def g_gp(_u, eta, g, gp):  # filter.hpp:187-201 with sequential sums
        a = math.tanh(beta * eta)
        den = a + math.tanh(beta * (1.0 - eta))
        gs = 0.0
        ps = 0.0
        for t in x:
            gs += (a + math.tanh(beta * (t - eta))) / den - t
            sech = 1.0 / math.cosh(beta * (t - eta))
            ps += -beta / math.sinh(beta) * sech * sech * math.sinh(beta * t) * math.sinh(beta * (1 - t))
        g[0] = gs / m
        gp[0] = ps / m

    cb = P._lib.GFUN(g_gp)
    eta, it = C.c_double(), C.c_int32()
    lib.topo_host_eta_replay(0.5, cb, None, C.byref(eta), C.byref(it))
    assert abs(eta.value - eta_o) <= 1e-15 and it.value == it_o


@pytest.mark.parametrize("sign", [1.0, -1.0])
@pytest.mark.parametrize("lam0,move,volfrac,ls", [(9.3e4, 0.2, 0.5, 0), (2.2e31, 0.1, 0.12, 0),
                                                  (1.0, 0.05, 0.3, 1), (5e-3, 0.2, 0.9, 0),
                                                  (1e300, 0.2, 0.5, 0)])
def test_host_oc_known_outcome_replay(P, lib, sign, lam0, move, volfrac, ls):
    # the bound-shortcut replay (OcCtl::replay_known, used by the device OC
    # kernel) ends in the state of feeding +-inf to every evaluation
    prm = P._lib.OcParams(move, volfrac, 1e-4, 1e-3, ls, 1e-8, 0.0)
    cb = P._lib.SFUN(lambda _u, s: sign * math.inf)
    outs = []
    for spec in (0, -1):
        lam, bis, ev, sf = C.c_double(), C.c_int32(), C.c_int32(), C.c_double()
        st = lib.topo_host_oc_replay(C.byref(prm), lam0, cb, None, spec, C.byref(lam),
                                     C.byref(bis), C.byref(ev), C.byref(sf), None)
        assert st == 0
        outs.append((lam.value, bis.value, ev.value, sf.value))
    assert outs[0] == outs[1]
