"""One rank of the 2-GPU NCCL parity test (tests/test_gpu_multirank.py):
started by torch.distributed.run, rank r on cuda:r, gloo for the NCCL unique
id broadcast; writes its slab outputs to <out>/rank<r>.npz."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    from paper_2005_05436_b200.configs import CONFIGS, make_inputs
    from paper_2005_05436_b200.dist import make_rank_context, slab_views
    cid, out = int(sys.argv[1]), sys.argv[2]
    scale = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else None
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group(backend="gloo")
    cfg = CONFIGS[cid] if not scale else CONFIGS[cid].scaled(*scale)
    x, u, state = make_inputs(cfg)
    _, _, xs, us, st = slab_views(cfg, x, u, state, rank, world)
    ctx = make_rank_context(cfg, st, rank, world, device=rank)  # NCCL clique
    try:
        r = ctx.design_pass(torch.from_numpy(np.ascontiguousarray(xs)).cuda(),
                            torch.from_numpy(np.ascontiguousarray(us)).cuda(), beta=cfg.beta,
                            move=cfg.move, volfrac=cfg.volfrac, return_sk=True)
        res = {k: getattr(r, k).cpu().numpy() for k in ("xTilde", "xPhys", "dc", "dV", "xNew", "sK")}
        np.savez(os.path.join(out, f"rank{rank}.npz"), eta=r.eta, lam=r.lam, c=r.c,
                 bisections=r.bisections, **res)
    finally:
        ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
