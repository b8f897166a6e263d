"""Generate tests/golden/*.npz from the REFERENCE itself: the reference's own
headers (/root/reference/proj/include/topopt/{grid,fea,filter,oc}.hpp)
compiled verbatim against oracle/eigen_shim into oracle/_ref/libtopo_ref.so.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The fixtures travel with the repo; nothing on the GPU box reads the reference.
"""
import hashlib
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

# small pass cases: (name, grid, rmin, beta, move, volfrac, passives, seed)
PASS_CASES = [
    ("mbb_30x10_r2.4", (30, 10, 0), 2.4, 2.0, 0.2, 0.5, False, 1),
    ("mbb_40x17_r4.6_pas_b8", (40, 17, 0), 4.6, 8.0, 0.2, 0.5, True, 4),
    ("mbb_24x12_r8.75_b2", (24, 12, 0), 8.75, 2.0, 0.2, 0.5, False, 12),
    ("h8_12x7x6_r2.3_pas", (12, 7, 6), 2.3, 2.0, 0.2, 0.5, True, 7),
    ("h8_8x8x8_rsqrt3", (8, 8, 8), math.sqrt(3.0), 2.0, 0.1, 0.12, False, 8),
    ("h8_10x6x6_r4_b4", (10, 6, 6), 4.0, 4.0, 0.1, 0.12, False, 13),
]


def rand_case(grid, seed, passives):
    rng = np.random.default_rng(seed)
    nelx, nely, nelz = grid
    m = nelx * nely * (nelz if nelz else 1)
    n = (3 if nelz else 2) * (nelx + 1) * (nely + 1) * ((nelz + 1) if nelz else 1)
    x = rng.uniform(0.01, 1.0, m)
    u = rng.normal(size=n)
    state = None
    if passives:
        state = np.zeros(m, np.uint8)
        idx = rng.permutation(m)
        state[idx[: max(1, m // 10)]] = 1
        state[idx[max(1, m // 10): max(2, m // 10 + m // 12)]] = 2
        x[state == 1] = 1.0
        x[state == 2] = 0.0
    return x, u, state


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    O.build()
    ref = O.Oracle("reference")
    meta = {"generator": "tests/golden/make_golden.py",
            "source": "oracle/_ref (reference headers compiled against oracle/eigen_shim)"}
    # element matrices
    kq, lq = ref.element_stiffness(2, 0.3)
    kh, lh = ref.element_stiffness(3, 0.3)
    np.savez(os.path.join(HERE, "ke.npz"), q4_full=kq, q4_lower=lq, h8_full=kh, h8_lower=lh)
    # index pairs: checksums on the config grids (C5 as its first 8 x-layers)
    idx = {}
    for name, grid in [("C1", (300, 100, 0)), ("C2", (600, 200, 0)), ("C3", (1200, 400, 0)),
                       ("C4", (96, 48, 48)), ("C5_first8", (8, 192, 192)), ("3x2", (3, 2, 0)),
                       ("2x2x2", (2, 2, 2))]:
        iK, jK = ref.index_pairs(grid)
        idx[name] = {"grid": grid, "pairs": int(iK.size), "sha_iK": sha(iK), "sha_jK": sha(jK),
                     "iK_head": iK[:40].tolist(), "jK_head": jK[:40].tolist()}
    meta["index_pairs"] = idx
    # filter taps / hs on the config radii
    taps = {}
    for name, grid, rmin in [("C1", (300, 100, 0), 8.75), ("C2", (600, 200, 0), 17.5),
                             ("C3", (64, 40, 0), 35.0), ("C4", (12, 8, 8), math.sqrt(3.0)),
                             ("C5", (12, 10, 10), 4.0)]:
        f = ref.filter(grid, rmin)
        di, dj, dk, w = f.taps()
        taps[name] = {"ntaps": int(f.ntaps), "w_sum": float(w.sum()), "hs0": float(f.hs()[0]),
                      "sha_w": sha(w)}
    meta["taps"] = taps
    # lower-triangle CSC of assemble_lower (fea.hpp:154-176): small grids in
    # full, the C1 / C4 patterns and values as checksums
    csc = {}
    arrays = {}
    for name, grid in [("5x4", (5, 4, 0)), ("4x3x2", (4, 3, 2)), ("3x1x2", (3, 1, 2)),
                       ("C1", (300, 100, 0)), ("C4", (96, 48, 48))]:
        m = grid[0] * grid[1] * (grid[2] or 1)
        sK = np.random.default_rng(2005).uniform(0.01, 1.0, m)
        cp, ri, va = ref.assemble_lower_csc(grid, 0.3, sK)
        csc[name] = {"grid": grid, "nnz": int(ri.size), "sha_col_ptr": sha(cp.astype(np.int64)),
                     "sha_row_idx": sha(ri), "sha_values": sha(va),
                     "sK": "numpy default_rng(2005).uniform(0.01, 1.0, m)"}
        if m < 100:
            arrays.update({f"{name}_sK": sK, f"{name}_col_ptr": cp, f"{name}_row_idx": ri,
                           f"{name}_values": va})
    np.savez(os.path.join(HERE, "csc.npz"), **arrays)
    meta["csc"] = csc
    # pass cases
    for name, grid, rmin, beta, move, volfrac, pas, seed in PASS_CASES:
        x, u, state = rand_case(grid, seed, pas)
        r = ref.design_pass(grid, rmin, x, u, state, beta=beta, move=move, volfrac=volfrac)
        np.savez(os.path.join(HERE, f"pass_{name}.npz"), x=x, u=u,
                 state=state if state is not None else np.zeros(0, np.uint8),
                 grid=np.array(grid), params=np.array([rmin, beta, move, volfrac]),
                 xTilde=r.xTilde, xPhys=r.xPhys, sKe=r.sKe, dcPhys=r.dcPhys, dc=r.dc, dV=r.dV,
                 xNew=r.xNew,
                 scalars=np.array([r.eta, r.c, r.lam, r.eta_iters, r.bisections, r.evaluations]))
    with open(os.path.join(HERE, "golden_meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print("wrote fixtures to", HERE)


if __name__ == "__main__":
    main()
