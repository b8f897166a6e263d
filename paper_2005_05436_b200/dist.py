"""Multi-rank plumbing of the x-slab decomposition.

One process (or thread) per GPU owns element columns [j0, j1) of the global
grid. Between kernels the ranks exchange `reach` filter-halo columns with
their neighbours and allreduce scalar sums (eta Newton terms, lambda#, batched
OC volumes, compliance). The library does this itself over NCCL
(Context.comm_init with a unique id broadcast here), or through host
callbacks (Context.comm_init_host), implemented below over torch.distributed
(gloo on CPU tensors) and over threads sharing one process (tests).
"""
from __future__ import annotations

import threading
from typing import Optional

import numpy as np

from .api import Context, nccl_unique_id, slab_plan


def slab_bounds(nelx: int, rank: int, nranks: int):
    """Even split of the nelx element columns (remainder to the first ranks)."""
    base, rem = divmod(nelx, nranks)
    j0 = rank * base + min(rank, rem)
    return j0, j0 + base + (1 if rank < rem else 0)


def slab_views(cfg, x, u, state, rank: int, nranks: int):
    """Rank-local inputs: elements of columns [j0, j1), U on node planes [j0, j1]."""
    j0, j1 = slab_bounds(cfg.nelx, rank, nranks)
    S = cfg.nely * (cfg.nelz or 1)
    plane = (cfg.nely + 1) * ((cfg.nelz + 1) if cfg.nelz else 1) * (3 if cfg.nelz else 2)
    xs = x[j0 * S:j1 * S]
    us = u[j0 * plane:(j1 + 1) * plane]
    st = None if state is None else state[j0 * S:j1 * S]
    return j0, j1, xs, us, st


class TorchHostComm:
    """Host-callback communicator over torch.distributed (CPU tensors, gloo)."""

    def __init__(self, rank: int, nranks: int, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.rank = rank
        self.nranks = nranks
        self.group = group

    def exchange(self, send_left, send_right, recv_left, recv_right):
        import torch
        d = self.dist
        ops = []
        if send_left.size:
            ops.append(d.P2POp(d.isend, torch.from_numpy(np.ascontiguousarray(send_left)),
                               self.rank - 1, self.group))
        if send_right.size:
            ops.append(d.P2POp(d.isend, torch.from_numpy(np.ascontiguousarray(send_right)),
                               self.rank + 1, self.group))
        rl = torch.from_numpy(recv_left) if recv_left.size else None
        rr = torch.from_numpy(recv_right) if recv_right.size else None
        if rl is not None:
            ops.append(d.P2POp(d.irecv, rl, self.rank - 1, self.group))
        if rr is not None:
            ops.append(d.P2POp(d.irecv, rr, self.rank + 1, self.group))
        if ops:
            for r in d.batch_isend_irecv(ops):
                r.wait()

    def allreduce_sum(self, values):
        import torch
        t = torch.from_numpy(values)
        self.dist.all_reduce(t, group=self.group)


class ThreadHostComm:
    """Ranks as threads of one process (tests: several contexts on one GPU,
    exchanges through host memory; kernels never wait on one another)."""

    def __init__(self, nranks: int):
        self.nranks = nranks
        self.barrier = threading.Barrier(nranks)
        self.box = {}

    def for_rank(self, rank: int):
        outer = self

        class _R:
            def exchange(self, sl, sr, rl, rr):
                outer.box[(rank, "L")] = sl.copy()
                outer.box[(rank, "R")] = sr.copy()
                outer.barrier.wait()
                if rl.size:
                    rl[:] = outer.box[(rank - 1, "R")]
                if rr.size:
                    rr[:] = outer.box[(rank + 1, "L")]
                outer.barrier.wait()

            def allreduce_sum(self, v):
                outer.box[(rank, "A")] = v.copy()
                outer.barrier.wait()
                tot = outer.box[(0, "A")].copy()
                for r in range(1, outer.nranks):  # fixed rank order
                    tot = tot + outer.box[(r, "A")]
                outer.barrier.wait()
                v[:] = tot

        return _R()


def init_nccl(ctx: Context, rank: int, group=None) -> None:
    """Create the NCCL clique: rank 0's unique id is broadcast with
    torch.distributed (any backend), then every rank joins."""
    import torch
    import torch.distributed as dist
    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        uid = torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8).clone()
    dist.broadcast(uid, 0, group=group)
    ctx.comm_init(bytes(uid.numpy()))


def make_rank_context(cfg, state_slab, rank: int, nranks: int, device: int = -1,
                      comm: Optional[object] = None, nccl_group=None) -> Context:
    """Context for one x-slab of cfg's grid, with its communicator attached."""
    j0, j1 = slab_bounds(cfg.nelx, rank, nranks)
    ctx = Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu, state=state_slab, device=device,
                  rank=rank, nranks=nranks, j0=j0, j1=j1)
    if nranks > 1:
        if comm is not None:
            ctx.comm_init_host(comm.exchange, comm.allreduce_sum)
        else:
            init_nccl(ctx, rank, nccl_group)
    return ctx


__all__ = ["slab_bounds", "slab_views", "slab_plan", "TorchHostComm", "ThreadHostComm",
           "init_nccl", "make_rank_context"]
