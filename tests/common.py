"""Shared helpers for the parity tests (SURVEY.md §8(c) protocol)."""
from __future__ import annotations

import numpy as np


def rel(a, b) -> float:
    """max|a - b| / max|b| (the "<= 1e-12" metric of SURVEY.md §8(c))."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise AssertionError(f"shape {a.shape} != {b.shape}")
    den = np.max(np.abs(b)) if b.size else 0.0
    num = np.max(np.abs(a - b)) if b.size else 0.0
    return float(num / den) if den > 0 else float(num)


def elem_rel(a, b) -> float:
    """element-wise max relative error over |b| > 1e-300 (reported alongside)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    mask = np.abs(b) > 1e-300
    if not mask.any():
        return 0.0
    return float(np.max(np.abs(a[mask] - b[mask]) / np.abs(b[mask])))


def rand_case(grid, seed, passives=False):
    """Small random case: x ~ U(0.01, 1), U ~ N(0, 1), optional passive sets."""
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
