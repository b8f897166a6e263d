"""The five BASELINE.json configurations and their seeded synthetic inputs
(SURVEY.md §8(d) and Appendix B — frozen here; the GPU path, the CPU oracle
and the reference arm all consume the same arrays).

Inputs are synthetic stand-ins with the configs' shapes and distributions:
x ~ U(0.01, 1) (C3: smoothed by one 3x3 mirror-padded box pass), passive
elements pinned (C2), U ~ N(0, 1) with the MBB (driver.hpp:293-295) or
cantilever (driver.hpp:357-363) fixed DOFs set to 0.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Optional, Tuple

import numpy as np

SEED_BASE = 20050543
STREAM_X, STREAM_U = 0, 1


@dataclass(frozen=True)
class Config:
    cid: int
    name: str
    nelx: int
    nely: int
    nelz: int
    rmin: float
    beta: float
    move: float
    volfrac: float
    penal: float = 3.0
    eta0: float = 0.5
    e0: float = 1.0
    emin: float = 1e-9
    nu: float = 0.3
    passives: bool = False
    smooth: bool = False
    problem: str = "mbb"

    @property
    def grid(self) -> Tuple[int, int, int]:
        return (self.nelx, self.nely, self.nelz)

    @property
    def is3d(self) -> bool:
        return self.nelz > 0

    @property
    def m(self) -> int:
        return self.nelx * self.nely * (self.nelz if self.nelz else 1)

    @property
    def n(self) -> int:
        nn = (self.nelx + 1) * (self.nely + 1) * ((self.nelz + 1) if self.nelz else 1)
        return (3 if self.nelz else 2) * nn

    @property
    def P(self) -> int:
        return 300 if self.nelz else 36

    @property
    def seed(self) -> int:
        return SEED_BASE + self.cid

    def scaled(self, nelx: int, nely: Optional[int] = None, nelz: Optional[int] = None,
               name: Optional[str] = None) -> "Config":
        """Same physics / filter / OC parameters on a different grid (tests, samples)."""
        return replace(self, nelx=nelx, nely=self.nely if nely is None else nely,
                       nelz=self.nelz if nelz is None else nelz,
                       name=name or f"{self.name}@{nelx}x{nely or self.nely}x{nelz or self.nelz}")


CONFIGS = {
    1: Config(1, "C1 MBB 300x100", 300, 100, 0, 8.75, 2.0, 0.2, 0.5),
    2: Config(2, "C2 MBB 600x200 + passives", 600, 200, 0, 17.5, 2.0, 0.2, 0.5, passives=True),
    3: Config(3, "C3 MBB 1200x400 beta 8", 1200, 400, 0, 35.0, 8.0, 0.2, 0.5, smooth=True),
    4: Config(4, "C4 cantilever 96x48x48", 96, 48, 48, math.sqrt(3.0), 2.0, 0.1, 0.12,
              problem="cantilever"),
    5: Config(5, "C5 cantilever 384x192x192", 384, 192, 192, 4.0, 4.0, 0.1, 0.12,
              problem="cantilever"),
}


def passive_state(cfg: Config) -> Optional[np.ndarray]:
    """C2 passive sets: solid band i < 0.2 nely along the
    top edge; void disc of radius nely/3 at the domain centre; the band wins
    where they overlap (the natural reading overlaps, which grid.hpp:173-176
    rejects)."""
    if not cfg.passives:
        return None
    nelx, nely = cfg.nelx, cfg.nely
    j, i = np.meshgrid(np.arange(nelx), np.arange(nely), indexing="ij")  # e = j * nely + i
    band = i < 0.2 * nely
    r = nely / 3.0
    disc = (j + 0.5 - nelx / 2.0) ** 2 + (i + 0.5 - nely / 2.0) ** 2 <= r * r
    state = np.zeros((nelx, nely), np.uint8)
    state[band] = 1
    state[disc & ~band] = 2
    return state.reshape(-1)


_GENERATOR = None  # override of the library's topo_generate (same bits), see set_generator


def set_generator(fn) -> None:
    """Use fn(seed, stream, kind, a, b, count, offset) instead of the library's
    generator: lets a process that must not load the product library (bench.py's
    CPU reference arm, which loads this file standalone) build identical inputs."""
    global _GENERATOR
    _GENERATOR = fn


def _gen(kind, seed, stream, a, b, count, offset=0):
    if _GENERATOR is not None:
        return _GENERATOR(seed, stream, kind, a, b, count, offset)
    from .api import generate
    return generate(seed, stream, kind, a, b, count, offset)


def design_field(cfg: Config, state: Optional[np.ndarray] = None) -> np.ndarray:
    x = _gen("uniform", cfg.seed, STREAM_X, 0.01, 1.0, cfg.m)
    if cfg.smooth:  # one 3x3 box pass, half-sample mirror (filter.hpp:43-48), fixed order
        X = x.reshape(cfg.nelx, cfg.nely)
        jj = np.arange(cfg.nelx)
        ii = np.arange(cfg.nely)
        fold = lambda t, n: np.where(t < 0, -t - 1, np.where(t >= n, 2 * n - 1 - t, t))
        s = np.zeros_like(X)
        for dj in (-1, 0, 1):
            for di in (-1, 0, 1):
                s = s + X[fold(jj + dj, cfg.nelx)][:, fold(ii + di, cfg.nely)]
        x = (s / 9.0).reshape(-1)
    if state is not None:  # driver.hpp:165 pin
        x = x.copy()
        x[state == 1] = 1.0
        x[state == 2] = 0.0
    return x


def fixed_dofs(cfg: Config) -> np.ndarray:
    nelx, nely, nelz = cfg.grid
    if not cfg.is3d:  # driver.hpp:293-295 (MBB)
        node = lambda i, j: j * (nely + 1) + i
        f = [2 * node(i, 0) for i in range(nely + 1)] + [2 * node(nely, nelx) + 1]
        return np.array(sorted(f), dtype=np.int64)
    ii, kk = np.meshgrid(np.arange(nely + 1), np.arange(nelz + 1), indexing="ij")
    nodes = (kk * (nely + 1) + ii).reshape(-1)  # node(i, k, 0), driver.hpp:357-363
    return np.sort(np.concatenate([3 * nodes, 3 * nodes + 1, 3 * nodes + 2]))


def load_vector(cfg: Config) -> np.ndarray:
    """The presets' unit loads: MBB downward at the top-left node (driver.hpp:
    289-290); cantilever downward along the x = nelx, y = nely edge (:353-354)."""
    nelx, nely, nelz = cfg.grid
    f = np.zeros(cfg.n)
    if not cfg.is3d:
        f[2 * 0 + 1] = -1.0  # node(0, 0)
        return f
    for k in range(nelz + 1):
        node = (nelx * (nelz + 1) + k) * (nely + 1) + nely
        f[3 * node + 1] = -1.0
    return f


def displacement(cfg: Config) -> np.ndarray:
    u = _gen("normal", cfg.seed, STREAM_U, 0.0, 1.0, cfg.n)
    u[fixed_dofs(cfg)] = 0.0
    return u


def make_inputs(cfg: Config):
    """(x, U, state) for a configuration, reproducible bit-for-bit."""
    state = passive_state(cfg)
    return design_field(cfg, state), displacement(cfg), state


def slab_of(cfg: Config, arr_elem: np.ndarray, arr_dof: np.ndarray, j0: int, j1: int):
    """Per-rank views: elements of columns [j0, j1) and node planes [j0, j1]."""
    S = cfg.nely * (cfg.nelz if cfg.nelz else 1)
    plane = (cfg.nely + 1) * ((cfg.nelz + 1) if cfg.nelz else 1) * (3 if cfg.nelz else 2)
    return arr_elem[j0 * S:j1 * S], arr_dof[j0 * plane:(j1 + 1) * plane]
