"""Stream ordering at the Python boundary: device inputs produced by async torch
kernels on torch's current stream (default or a side stream) must be complete
before the library's own stream reads them (api._FencedLib ->
topo_wait_stream), and a second context on the same process keeps its device."""
import numpy as np
import pytest

from tests.common import rand_case, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2005_05436_b200 as P
    return P


def _delay(torch, n=24):
    # ~ms of queued work on the current stream before the input is written
    a = torch.randn(4096, 4096, device="cuda")
    for _ in range(n):
        a = a @ a
        a = a / a.abs().max()
    return a


@pytest.mark.parametrize("side_stream", [False, True])
def test_input_from_async_torch_kernel(P, oracle_port, side_stream):
    import torch
    grid = (40, 30, 20)
    x, u, _ = rand_case(grid, 31)
    f = oracle_port.filter(grid, 2.5)
    ref = oracle_port.apply_filter(f, x)
    src = torch.from_numpy(x).cuda()
    torch.cuda.synchronize()
    s = torch.cuda.Stream() if side_stream else torch.cuda.current_stream()
    with P.Context(*grid, rmin=2.5) as ctx, torch.cuda.stream(s):
        xd = torch.zeros_like(src)
        _delay(torch)
        xd.copy_(src)          # queued behind the delay on the current stream
        y = ctx.apply_filter(xd)
        assert rel(y.cpu().numpy(), ref) <= 1e-12
        # a pass whose inputs come from torch kernels on the same stream
        xd2 = torch.zeros_like(src)
        ud = torch.zeros(u.size, dtype=torch.float64, device="cuda")
        _delay(torch)
        xd2.copy_(src)
        ud.copy_(torch.from_numpy(u).cuda(non_blocking=True))
        g = ctx.design_pass(xd2, ud, beta=2.0, move=0.2, volfrac=0.5)
    gh = P.Context(*grid, rmin=2.5).design_pass(x, u, beta=2.0, move=0.2, volfrac=0.5)
    assert g.eta == gh.eta and g.lam == gh.lam
    assert np.array_equal(g.xNew.cpu().numpy(), gh.xNew)


def test_rand_on_device_input(P, oracle_port):
    import torch
    grid = (64, 32, 0)
    with P.Context(*grid, rmin=3.0) as ctx:
        _delay(torch, 8)
        xd = torch.rand(grid[0] * grid[1], dtype=torch.float64, device="cuda")
        y = ctx.apply_filter(xd)
        x = xd.cpu().numpy()
    f = oracle_port.filter(grid, 3.0)
    assert rel(y.cpu().numpy(), oracle_port.apply_filter(f, x)) <= 1e-12
