"""x-slab decomposition on the GPU: N rank contexts (threads, one GPU, host
exchange through ThreadHostComm) reproduce the single-context pass. The
kernels of different ranks never wait on one another; every exchange and
allreduce happens on the host between launches. With >= 2 GPUs the same
ranks also run over NCCL."""
import threading

import numpy as np
import pytest

from tests.common import rand_case, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2005_05436_b200 as P
    return P


def run_ranks(P, cfg, x, u, state, nranks, nccl=False):
    from paper_2005_05436_b200.dist import ThreadHostComm, make_rank_context, slab_views
    comm = ThreadHostComm(nranks)
    out = [None] * nranks
    err = [None] * nranks

    def work(r):
        try:
            j0, j1, xs, us, st = slab_views(cfg, x, u, state, r, nranks)
            ctx = make_rank_context(cfg, st, r, nranks, comm=comm.for_rank(r))
            try:
                out[r] = ctx.design_pass(xs, us, beta=cfg.beta, move=cfg.move, volfrac=cfg.volfrac,
                                         return_sk=True)
            finally:
                ctx.close()
        except Exception as e:  # noqa: BLE001
            import traceback
            err[r] = traceback.format_exc()
            comm.barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in err:
        assert e is None, e
    return out


def cat(rs, k):
    return np.concatenate([getattr(r, k) for r in rs])


@pytest.mark.parametrize("case,nranks", [("c4", 2), ("c4", 4), ("c2s", 2), ("c2s", 3),
                                         ("c5s", 2), ("c3s", 2), ("c1", 4)])
def test_slab_ranks_match_single_context(P, oracle_port, case, nranks):
    from paper_2005_05436_b200.configs import CONFIGS, make_inputs
    if case == "c4":
        cfg = CONFIGS[4]
    elif case == "c2s":
        cfg = CONFIGS[2].scaled(150, 50)
    elif case == "c5s":
        cfg = CONFIGS[5].scaled(24, 24, 24)
    elif case == "c3s":
        cfg = CONFIGS[3].scaled(160, 80)
    else:
        cfg = CONFIGS[1]
    x, u, state = make_inputs(cfg)
    with P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu, state=state) as ctx:
        ref = ctx.design_pass(x, u, beta=cfg.beta, move=cfg.move, volfrac=cfg.volfrac,
                              return_sk=True)
    rs = run_ranks(P, cfg, x, u, state, nranks)
    eta = rs[0].eta
    assert all(r.eta == eta for r in rs)  # every rank takes the same decisions
    assert abs(eta - ref.eta) <= 5e-8
    assert rel(cat(rs, "xTilde"), ref.xTilde) <= 1e-12
    assert all(r.c == rs[0].c for r in rs)  # c is allreduced
    if eta == ref.eta:  # (else: a rounding-ill-conditioned Newton exit)
        assert abs(rs[0].c - ref.c) <= 1e-12 * abs(ref.c)
        for k in ("xPhys", "dcPhys", "dc", "dV", "sK"):
            assert rel(cat(rs, k), getattr(ref, k)) <= 1e-12, k
    # conditioned on the ranks' eta: the oracle of the whole domain
    rc = oracle_port.design_pass(cfg.grid, cfg.rmin, x, u, state, beta=cfg.beta, move=cfg.move,
                                 volfrac=cfg.volfrac, eta_override=eta, volume_mode=4)
    for k in ("xPhys", "dc", "dV", "xNew"):
        assert rel(cat(rs, k), getattr(rc, k)) <= 1e-12, k
    assert abs(rs[0].c - rc.c) <= 1e-12 * abs(rc.c)
    assert all(r.bisections == rc.bisections and r.lam == rs[0].lam for r in rs)
    assert abs(rs[0].lam - rc.lam) <= 1e-10 * abs(rc.lam)


def test_slab_narrower_than_reach_rejected(P):
    with pytest.raises(ValueError):
        P.Context(64, 10, 0, rmin=35.0, rank=1, nranks=4)


@pytest.mark.parametrize("cid,scale", [(4, None), (5, (48, 48, 48)), (2, (150, 50))])
def test_nccl_two_gpus(P, oracle_port, tmp_path, cid, scale):
    """Two processes, one GPU each, over a real NCCL clique (halo send/recv,
    on-stream allreduces, device-resident eta and OC replays): the slabs
    together equal the single-context pass and the oracle."""
    import os
    import subprocess
    import sys
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (NCCL ranks cannot share a GPU)")
    from paper_2005_05436_b200.configs import CONFIGS, make_inputs
    cfg = CONFIGS[cid] if scale is None else CONFIGS[cid].scaled(*scale)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + cid),
           os.path.join(root, "tests", "helpers", "nccl_rank.py"), str(cid), str(tmp_path)]
    if scale is not None:
        cmd.append(",".join(str(v) for v in scale))
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    rs = [np.load(tmp_path / f"rank{q}.npz") for q in range(2)]
    x, u, state = make_inputs(cfg)
    with P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu, state=state) as ctx:
        ref = ctx.design_pass(x, u, beta=cfg.beta, move=cfg.move, volfrac=cfg.volfrac,
                              return_sk=True)
    eta = float(rs[0]["eta"])
    assert float(rs[1]["eta"]) == eta and abs(eta - ref.eta) <= 5e-8
    cat2 = lambda k: np.concatenate([q[k] for q in rs])  # noqa: E731
    assert rel(cat2("xTilde"), ref.xTilde) <= 1e-12
    rc = oracle_port.design_pass(cfg.grid, cfg.rmin, x, u, state, beta=cfg.beta, move=cfg.move,
                                 volfrac=cfg.volfrac, eta_override=eta, volume_mode=4)
    for k in ("xPhys", "dc", "dV", "xNew"):
        assert rel(cat2(k), getattr(rc, k)) <= 1e-12, k
    assert all(int(q["bisections"]) == rc.bisections for q in rs)
    assert abs(float(rs[0]["lam"]) - rc.lam) <= 1e-10 * abs(rc.lam)


def test_nccl_single_rank_clique_matches_plain_pass():
    """The NCCL communicator path (dlopen'ed libnccl, unique id, halo send/recv
    groups, allreduces, host-driven eta / OC replays) on a one-rank clique:
    nothing waits on another GPU, and the pass must equal the plain one."""
    import numpy as np
    import paper_2005_05436_b200 as P
    from paper_2005_05436_b200.configs import CONFIGS
    from tests.common import rel
    for cid, grid in ((4, (16, 10, 8)), (2, (60, 20, 0))):
        cfg = CONFIGS[cid].scaled(*grid)
        rng = np.random.default_rng(4)
        x, u = rng.uniform(0.01, 1.0, cfg.m), rng.normal(size=cfg.n)
        kw = dict(beta=cfg.beta, move=cfg.move, volfrac=cfg.volfrac, return_sk=True)
        with P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu) as ctx:
            a = ctx.design_pass(x, u, **kw)
        with P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu, rank=0, nranks=1) as ctx:
            ctx.comm_init(P.nccl_unique_id())
            b0 = ctx.design_pass(x, u, **kw)  # eta over NCCL allreduces
            b = ctx.design_pass(x, u, eta_override=a.eta, **kw)
        assert abs(a.eta - b0.eta) <= 5e-8
        assert a.bisections == b.bisections and abs(a.lam - b.lam) <= 1e-10 * abs(a.lam)
        for k in ("xTilde", "xPhys", "dc", "dV", "xNew", "sK"):
            assert rel(getattr(b, k), getattr(a, k)) <= 1e-12, k


@pytest.mark.parametrize("nranks", [2, 3])
def test_slab_ranks_with_overlapped_sk_stream(P, nranks, monkeypatch):
    """Per-slab sK stream on the aux stream beside K3a/K4 and the host-driven
    OC (the default on large slabs): bitwise equal to the serial schedule."""
    from paper_2005_05436_b200.configs import CONFIGS, make_inputs
    cfg = CONFIGS[5].scaled(30, 16, 12)
    x, u, state = make_inputs(cfg)
    monkeypatch.setenv("TOPO_SK_OVERLAP", "0")
    a = run_ranks(P, cfg, x, u, state, nranks)
    monkeypatch.setenv("TOPO_SK_OVERLAP", "1")
    b = run_ranks(P, cfg, x, u, state, nranks)
    for k in ("xTilde", "xPhys", "dc", "dV", "xNew", "sK"):
        np.testing.assert_array_equal(cat(a, k), cat(b, k), err_msg=k)
    assert [r.lam for r in a] == [r.lam for r in b]


@pytest.mark.parametrize("spec_rounds", ["1", "2"])
def test_slab_ranks_recentred_eta(P, monkeypatch, spec_rounds):
    """A design whose eta lies far from eta0 (x ~ U^3: the moment series must
    re-centre): with one speculative eta round the pass detects the unfinished
    solve after its final synchronisation and re-runs with a host check per
    round; either way the ranks match the single context."""
    from paper_2005_05436_b200.configs import CONFIGS
    cfg = CONFIGS[4].scaled(24, 12, 12)
    rng = np.random.default_rng(8)
    x = 0.01 + 0.99 * rng.uniform(0, 1, cfg.m) ** 3
    u = rng.normal(size=cfg.n)
    with P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu) as ctx:
        ref = ctx.design_pass(x, u, beta=8.0, move=cfg.move, volfrac=cfg.volfrac, return_sk=True)
    assert abs(ref.eta - 0.5) > 0.03  # far enough to need a re-centred pass
    monkeypatch.setenv("TOPO_ETA_SPEC_ROUNDS", spec_rounds)
    from paper_2005_05436_b200.dist import ThreadHostComm, make_rank_context, slab_views
    comm = ThreadHostComm(2)
    out, err = [None, None], [None, None]

    def work(r):
        try:
            _, _, xs, us, st = slab_views(cfg, x, u, None, r, 2)
            with make_rank_context(cfg, st, r, 2, comm=comm.for_rank(r)) as c:
                out[r] = c.design_pass(xs, us, beta=8.0, move=cfg.move, volfrac=cfg.volfrac)
        except Exception:  # noqa: BLE001
            import traceback
            err[r] = traceback.format_exc()
            comm.barrier.abort()

    import threading
    ts = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert err == [None, None], err
    assert out[0].eta == out[1].eta and abs(out[0].eta - ref.eta) <= 5e-8
    assert out[0].eta_iters == ref.eta_iters
    assert rel(np.concatenate([o.xNew for o in out]), ref.xNew) <= 1e-10


def test_slab_ranks_adaptive_eta_speculation(P):
    """The number of eta rounds a multi-rank pass enqueues without a host check
    adapts: two at first, one after four passes in a row that converged in
    their first round (fewer launches), two again after a design that needs a
    re-centred round (detected after the pass, which is re-run). Every pass
    matches the single context."""
    import threading
    from paper_2005_05436_b200.configs import CONFIGS
    from paper_2005_05436_b200.dist import ThreadHostComm, make_rank_context, slab_views
    cfg = CONFIGS[4].scaled(24, 12, 12)
    rng = np.random.default_rng(8)
    calm = rng.uniform(0.01, 1.0, cfg.m)
    far = 0.01 + 0.99 * rng.uniform(0, 1, cfg.m) ** 3
    u = rng.normal(size=cfg.n)
    seq = [calm] * 6 + [far, calm]
    kw = dict(beta=4.0, move=cfg.move, volfrac=cfg.volfrac)  # calm: d = 0.017, far: d = -0.44
    with P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu) as ctx:
        ref = [ctx.design_pass(x, u, outputs=False, **kw) for x in (calm, far)]
    assert abs(ref[1].eta - 0.5) > 0.03  # `far` needs a re-centred round
    comm = ThreadHostComm(2)
    out, err = [[], []], [None, None]

    def work(r):
        try:
            views = {id(x): slab_views(cfg, x, u, None, r, 2) for x in (calm, far)}
            st = views[id(calm)][4]
            with make_rank_context(cfg, st, r, 2, comm=comm.for_rank(r)) as c:
                for x in seq:
                    _, _, xs, us, _ = views[id(x)]
                    out[r].append(c.design_pass(xs, us, outputs=False, **kw))
        except Exception:  # noqa: BLE001
            import traceback
            err[r] = traceback.format_exc()
            comm.barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert err == [None, None], err
    for k, x in enumerate(seq):
        want = ref[0] if x is calm else ref[1]
        a, b = out[0][k], out[1][k]
        assert a.eta == b.eta and abs(a.eta - want.eta) <= 5e-8 and a.eta_iters == want.eta_iters, k
        assert rel(np.concatenate([a.xNew, b.xNew]), want.xNew) <= 1e-10, k
    launches = [o.launches for o in out[0]]
    assert launches[5] < launches[0]   # the second speculative round was dropped
    assert launches[7] == launches[0]  # and came back after the re-centred pass
