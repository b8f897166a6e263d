"""Redesign-loop helpers on the device: the record
reductions (driver.hpp:189, :249-251) and the Anderson extrapolation
(accel.hpp:21-95 as driver.hpp:235-244 applies it) against numpy
restatements on the same inputs, through the C-ABI on device arrays."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


class AndersonRef:
    """accel.hpp:21-95, restated in numpy (test infrastructure)."""

    def __init__(self, depth, period, mix_plain, mix_accel):
        self.depth, self.period, self.mp, self.ma = depth, period, mix_plain, mix_accel
        self.dx = self.dr = None
        self.cols = self.next = self.counter = 0
        self.has_prev = False

    def step(self, x, r):
        if self.dx is None or self.dx.shape[0] != x.size:
            self.dx = np.zeros((x.size, self.depth))
            self.dr = np.zeros((x.size, self.depth))
        t = self.counter
        self.counter += 1
        if self.has_prev:
            self.dx[:, self.next] = x - self.px
            self.dr[:, self.next] = r - self.pr
            self.next = (self.next + 1) % self.depth
            self.cols = min(self.cols + 1, self.depth)
        self.px, self.pr, self.has_prev = x.copy(), r.copy(), True
        extra = t % self.period == 0 and self.cols >= 2
        mix = self.ma if extra else self.mp
        out = x + mix * r
        if extra:
            X, R = self.dx[:, :self.cols], self.dr[:, :self.cols]
            G, rhs = R.T @ R, R.T @ r
            ev, V = np.linalg.eigh(G)
            cut = np.abs(ev).max() * 1e-13
            g = np.zeros(self.cols)
            if cut > 0:
                for i in range(ev.size):
                    if ev[i] > cut:
                        g += V[:, i] * (V[:, i] @ rhs / ev[i])
            out = out - (X + mix * R) @ g
        return out


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def test_loop_records_match_numpy():
    import paper_2005_05436_b200 as P
    rng = np.random.default_rng(3)
    with P.Context(40, 20, 10, rmin=1.5) as ctx:
        m = ctx.m
        xp, xprev, x = rng.uniform(0, 1, m), rng.uniform(0, 1, m), rng.uniform(0, 1, m)
        d = [torch.from_numpy(a.copy()).cuda() for a in (xp, xprev, x)]
        out = (C.c_double * 3)()
        assert ctx.lib.topo_loop_records(ctx.h, _ptr(d[0]), _ptr(d[1]), _ptr(d[2]),
                                         C.addressof(out)) == 0
        ch = np.linalg.norm(xp - xprev) / np.sqrt(m)
        assert abs(out[0] - ch) <= 1e-14 * ch
        assert abs(out[1] - xp.mean()) <= 1e-14
        assert abs(out[2] - 400.0 * np.sum(x * (1 - x)) / m) <= 1e-12
        np.testing.assert_array_equal(d[1].cpu().numpy(), xp)  # xPrev <- xPhys


@pytest.mark.parametrize("depth,period", [(4, 4), (3, 2), (5, 1)])
def test_anderson_steps_match_accel_hpp(depth, period):
    import paper_2005_05436_b200 as P
    from paper_2005_05436_b200 import _lib as L
    rng = np.random.default_rng(depth * 10 + period)
    nelx, nely = 30, 12
    state = np.zeros(nelx * nely, np.uint8)
    state[rng.choice(state.size, 40, replace=False)] = L.PASSIVE_SOLID  # passives untouched
    with P.Context(nelx, nely, 0, rmin=2.0, state=state) as ctx:
        m = ctx.m
        act = state == 0
        ref = AndersonRef(depth, period, 0.9, 1.0)

        class Opt(C.Structure):
            _fields_ = [("depth", C.c_int32), ("period", C.c_int32), ("mix_plain", C.c_double),
                        ("mix_accel", C.c_double)]
        o = Opt(depth, period, 0.9, 1.0)
        assert ctx.lib.topo_anderson_reset(ctx.h) == 0
        x = rng.uniform(0.2, 0.8, m)
        for it in range(12):  # a contracting fixed-point map with noise
            xnew = np.clip(0.5 + 0.6 * (x - 0.5) + 0.05 * rng.normal(size=m), 0, 1)
            xnew[~act] = x[~act]
            xb_d = torch.from_numpy(x.copy()).cuda()
            xn_d = torch.from_numpy(xnew.copy()).cuda()
            assert ctx.lib.topo_anderson_step(ctx.h, C.addressof(o), _ptr(xb_d), _ptr(xn_d)) == 0
            got = xn_d.cpu().numpy()
            want = xnew.copy()
            want[act] = np.clip(ref.step(x[act], xnew[act] - x[act]), 0, 1)
            err = np.max(np.abs(got - want))
            assert err <= 1e-12, (it, err)
            np.testing.assert_array_equal(got[~act], x[~act])
            x = got
