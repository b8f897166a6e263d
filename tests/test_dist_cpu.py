"""Multi-rank x-slab protocol on CPU (gloo, world size 2 and 4): the slab plan
of the library (topo_slab_plan), halo exchange and allreduce through
torch.distributed, and the distributed filter / OC bisection rebuilt from
per-rank pieces — equal to the single-domain oracle. The same plan and the
same host replays (topo_host_oc_replay) drive the library's NCCL path."""
import ctypes as C
import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_slab_plans_tile_the_domain():
    import paper_2005_05436_b200 as P
    for grid, rmin, n in [((384, 192, 192), 4.0, 8), ((1200, 400, 0), 35.0, 8),
                          ((96, 48, 48), math.sqrt(3.0), 4), ((600, 200, 0), 17.5, 2),
                          ((300, 100, 0), 8.75, 4)]:
        plans = [P.slab_plan(*grid, rmin, r, n) for r in range(n)]
        assert plans[0]["j0"] == 0 and plans[-1]["j1"] == grid[0]
        for a, b in zip(plans, plans[1:]):
            assert a["j1"] == b["j0"]
            assert a["send_right"] == b["recv_left"] and b["send_left"] == a["recv_right"]
        reach = math.ceil(rmin) - 1
        for p in plans:
            assert p["sj0"] == max(0, p["j0"] - reach) and p["sj1"] == min(grid[0], p["j1"] + reach)
    with pytest.raises(ValueError):
        P.slab_plan(64, 10, 0, 35.0, 1, 4)  # slabs narrower than the reach


def _filter_slab(x_st, sj0, j0, j1, grid, taps):
    """Direct cone stencil of the owned columns from a halo-extended slab
    (half-sample mirror at the global x ends, full extent in y/z)."""
    nelx, nely, nelz = grid
    nz = max(nelz, 1)
    X = x_st.reshape(-1, nz, nely)
    out = np.zeros((j1 - j0, nz, nely))
    fold = lambda t, n: (t % (2 * n)) if (t % (2 * n)) < n else 2 * n - 1 - (t % (2 * n))
    for j in range(j0, j1):
        for k in range(nz):
            for i in range(nely):
                acc = 0.0
                for di, dj, dk, w in taps:
                    jj, kk, ii = fold(j + dj, nelx), fold(k + dk, nz), fold(i + di, nely)
                    acc += w * X[jj - sj0, kk, ii]
                out[j - j0, k, i] = acc
    return out.reshape(-1)


def _worker(rank, world, port, grid, rmin, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, ROOT)
        import paper_2005_05436_b200 as P
        from oracle.oracle import Oracle
        from paper_2005_05436_b200.dist import TorchHostComm
        orc = Oracle("port")
        nelx, nely, nelz = grid
        S = nely * max(nelz, 1)
        m = nelx * S
        rng = np.random.default_rng(5)
        x = rng.uniform(0.01, 1.0, m)
        dc = -rng.uniform(0.05, 2.0, m)
        dV = np.full(m, 1.0 / m)
        plan = P.slab_plan(*grid, rmin, rank, world)
        j0, j1, sj0, sj1 = plan["j0"], plan["j1"], plan["sj0"], plan["sj1"]
        comm = TorchHostComm(rank, world)
        # 1. halo exchange exactly as the library plans it
        x_st = np.zeros((sj1 - sj0) * S)
        own = x[j0 * S:j1 * S]
        x_st[(j0 - sj0) * S:(j1 - sj0) * S] = own
        sl = own[:plan["send_left"] * S]
        sr = own[len(own) - plan["send_right"] * S:] if plan["send_right"] else own[:0]
        rl = np.zeros(plan["recv_left"] * S)
        rr = np.zeros(plan["recv_right"] * S)
        comm.exchange(sl, sr, rl, rr)
        x_st[:rl.size] = rl
        if rr.size:
            x_st[(j1 - sj0) * S:] = rr
        np.testing.assert_array_equal(x_st, x[sj0 * S:sj1 * S])
        # 2. distributed filter of the owned columns == full-domain oracle filter
        f = orc.filter(grid, rmin)
        di, dj, dk, w = f.taps()
        taps = list(zip(di.tolist(), dj.tolist(), dk.tolist(), w.tolist()))
        mine = _filter_slab(x_st, sj0, j0, j1, grid, taps)
        full = orc.apply_filter(f, x) * f.hs()
        assert np.abs(mine - full[j0 * S:j1 * S]).max() <= 1e-12 * np.abs(full).max()
        # 3. distributed OC: per-rank partial volumes, allreduced, replayed on
        #    the host with the library's controller == single-domain bisection
        sl_ = slice(j0 * S, j1 * S)
        ocP = x[sl_] * np.sqrt(np.maximum(0.0, -dc[sl_] / dV[sl_]))
        lo, hi = np.maximum(0, x[sl_] - 0.2), np.minimum(1, x[sl_] + 0.2)
        part = np.array([ocP.sum()])
        comm.allreduce_sum(part)
        root = part[0] / (m * 0.5)

        def vol(_u, s):
            f_ = ocP / s if s > 0 else np.where(ocP > 0, np.inf, 0.0)
            v = np.array([np.minimum(np.maximum(f_, lo), hi).sum()])
            comm.allreduce_sum(v)
            return float(v[0] / m)

        lib = P._lib.load()
        prm = P._lib.OcParams(0.2, 0.5, 1e-4, 1e-3, 0, 1e-8, 0.0)
        cb = P._lib.SFUN(vol)
        lam, bis, ev = C.c_double(), C.c_int32(), C.c_int32()
        lib.topo_host_oc_replay(C.byref(prm), root * root, cb, None, 1, C.byref(lam), C.byref(bis),
                                C.byref(ev), None, None)
        xo, lo_, bo, eo = orc.bisect_update(x, dc, dV)
        assert bis.value == bo and ev.value == eo
        assert abs(lam.value - lo_) <= 1e-10 * lo_
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,grid,rmin", [(2, (12, 6, 0), 3.5), (4, (16, 5, 4), 2.3),
                                             (2, (9, 4, 3), 4.0)])
def test_distributed_protocol_gloo(world, grid, rmin):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, grid, rmin, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}:\n{msg}"
