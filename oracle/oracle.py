"""TEST INFRASTRUCTURE ONLY — ctypes front end of the CPU oracle.

Two interchangeable back ends with identical method names:

* ``Oracle("port")``      -> oracle/_build/libtopo_oracle.so, the C restatement
  (oracle/topo_oracle.c) of the reference hot path;
* ``Oracle("reference")`` -> oracle/_ref/libtopo_ref.so, the reference's own
  headers (/root/reference/proj/include/topopt/*.hpp) compiled verbatim
  against oracle/eigen_shim (oracle/ref_pass.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module, and only as the checker or the timed CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "_build", "libtopo_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libtopo_ref.so")

VOL_CALLBACK, VOL_MEAN, VOL_PROJECTED, VOL_FILTERED, VOL_IDENTITY = 0, 1, 2, 3, 4


def build(quiet: bool = True) -> None:
    """Run oracle/Makefile (port always; reference only if its headers exist)."""
    out = subprocess.run(["make", "-C", HERE, "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


class Grid(C.Structure):
    _fields_ = [("nelx", C.c_int32), ("nely", C.c_int32), ("nelz", C.c_int32)]


class OcParams(C.Structure):
    _fields_ = [("move", C.c_double), ("volfrac", C.c_double), ("bisect_rel_tol", C.c_double),
                ("volume_tol", C.c_double), ("lambda_space", C.c_int), ("abs_tol", C.c_double),
                ("lambda_max", C.c_double)]


class PassParams(C.Structure):
    _fields_ = [("e0", C.c_double), ("emin", C.c_double), ("penal", C.c_double),
                ("beta", C.c_double), ("eta0", C.c_double), ("move", C.c_double),
                ("volfrac", C.c_double), ("eta_override", C.c_double), ("volume_mode", C.c_int)]


class PassOut(C.Structure):
    _fields_ = [("xTilde", C.c_void_p), ("xPhys", C.c_void_p), ("sKe", C.c_void_p),
                ("dcPhys", C.c_void_p), ("dc", C.c_void_p), ("dV", C.c_void_p),
                ("xNew", C.c_void_p), ("eta", C.c_double), ("c", C.c_double),
                ("lambda_", C.c_double), ("eta_iters", C.c_int), ("bisections", C.c_int),
                ("evaluations", C.c_int)]


VOLUME_FN = C.CFUNCTYPE(C.c_double, C.c_void_p, C.POINTER(C.c_double), C.c_int64)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class PassResult:
    xTilde: np.ndarray
    xPhys: np.ndarray
    sKe: np.ndarray
    dcPhys: np.ndarray
    dc: np.ndarray
    dV: np.ndarray
    xNew: np.ndarray
    eta: float
    c: float
    lam: float
    eta_iters: int
    bisections: int
    evaluations: int


class Filter:
    def __init__(self, owner: "Oracle", grid, rmin: float, bc: int = 0):
        self.o = owner
        self.grid = tuple(grid)
        self.m = _num_elements(self.grid)
        self.h = owner._filter_create(Grid(*self.grid), rmin, bc)
        if not self.h:
            raise OracleError(1, owner._err())

    def __del__(self):
        if getattr(self, "h", None):
            self.o._filter_destroy(self.h)
            self.h = None

    @property
    def ntaps(self) -> int:
        return self.o._filter_ntaps(self.h)

    def taps(self):
        T = self.ntaps
        di = np.empty(T, np.int32)
        dj = np.empty(T, np.int32)
        dk = np.empty(T, np.int32)
        w = np.empty(T, np.float64)
        self.o._filter_taps(self.h, _p(di), _p(dj), _p(dk), _p(w))
        return di, dj, dk, w

    def hs(self) -> np.ndarray:
        out = np.empty(self.m)
        if self.o.kind == "port":
            src = self.o.lib.orc_filter_hs(self.h)
            C.memmove(out.ctypes.data, src, 8 * self.m)
        else:
            self.o.lib.ref_filter_hs(self.h, _p(out))
        return out


def _num_elements(grid) -> int:
    nelx, nely, nelz = grid
    return nelx * nely * (nelz if nelz > 0 else 1)


def _num_dofs(grid) -> int:
    nelx, nely, nelz = grid
    nn = (nelx + 1) * (nely + 1) * ((nelz + 1) if nelz > 0 else 1)
    return (3 if nelz > 0 else 2) * nn


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (run oracle.build())")
        self.lib = L = C.CDLL(path)
        pre = "orc_" if kind == "port" else "ref_"
        self.pre = pre
        vp, i32p, f64p, u8p = C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p

        def fn(name, res, *args):
            f = getattr(L, pre + name)
            f.restype = res
            f.argtypes = list(args)
            return f

        self._err_f = fn("last_error", C.c_char_p)
        fn("build_connectivity", C.c_int, Grid, i32p)
        fn("build_index_pairs", C.c_int, Grid, i32p, i32p)
        fn("partition", C.c_int, Grid, i32p, C.c_int64, i32p, C.c_int64, u8p)
        fn("simp", None, C.c_int64, f64p, C.c_double, C.c_double, C.c_double, f64p, f64p)
        self._filter_create = fn("filter_create", C.c_void_p, Grid, C.c_double, C.c_int)
        self._filter_destroy = fn("filter_destroy", None, C.c_void_p)
        self._filter_ntaps = fn("filter_ntaps", C.c_int, C.c_void_p)
        self._filter_taps = fn("filter_taps", None, C.c_void_p, i32p, i32p, i32p, f64p)
        fn("project", None, C.c_int64, f64p, C.c_double, C.c_double, f64p)
        fn("project_derivative", None, C.c_int64, f64p, C.c_double, C.c_double, f64p)
        fn("project_eta_derivative", C.c_double, C.c_double, C.c_double, C.c_double)
        fn("lambda_upper", C.c_double, C.c_int64, f64p, f64p, f64p, C.c_double, C.c_int64)
        fn("oc_candidate", C.c_int, C.c_int64, f64p, f64p, f64p, C.c_double, C.c_double, f64p)
        if kind == "port":
            L.orc_filter_hs.restype = C.c_void_p
            L.orc_filter_hs.argtypes = [C.c_void_p]
            L.orc_set_threads.restype = C.c_int
            L.orc_set_threads.argtypes = [C.c_int]
            L.orc_generate.restype = None
            L.orc_generate.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_double, C.c_double,
                                       C.c_int64, C.c_int64, C.c_void_p]
            fn("element_stiffness", C.c_int, C.c_int, C.c_double, f64p, f64p)
            fn("assemble_values", None, C.c_int64, C.c_int, f64p, f64p, f64p)
            fn("assemble_lower", C.c_int, Grid, C.c_double, f64p, i32p, i32p, f64p,
               C.POINTER(C.c_int64))
            fn("compliance_sensitivity", C.c_int, Grid, f64p, f64p, f64p, C.c_double,
               C.c_double, C.c_double, u8p, C.POINTER(C.c_double), f64p)
            fn("apply_filter", None, C.c_void_p, f64p, f64p)
            fn("apply_filter_adjoint", None, C.c_void_p, f64p, f64p)
            fn("backfilter", None, C.c_void_p, f64p, f64p, C.c_double, C.c_double, C.c_int, f64p)
            fn("solve_eta", C.c_int, C.c_int64, f64p, C.c_double, C.c_double, u8p,
               C.POINTER(C.c_double), C.POINTER(C.c_int))
            fn("eta_mismatch", C.c_double, C.c_int64, f64p, C.c_double, C.c_double, u8p)
            fn("bisect_update", C.c_int, C.c_int64, f64p, f64p, f64p, u8p, C.POINTER(OcParams),
               C.c_int, C.c_void_p, C.c_double, C.c_double, VOLUME_FN, C.c_void_p, f64p,
               C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int))
            fn("design_pass", C.c_int, Grid, C.c_void_p, f64p, u8p, f64p, f64p,
               C.POINTER(PassParams), C.POINTER(PassOut))
            fn("primal_dual_update", C.c_int, C.c_int64, f64p, f64p, f64p, u8p,
               C.POINTER(OcParams), C.c_double, f64p, C.POINTER(C.c_double),
               C.POINTER(C.c_int), C.POINTER(C.c_int))
        else:
            L.ref_filter_hs.restype = None
            L.ref_filter_hs.argtypes = [C.c_void_p, f64p]
            fn("element_stiffness", C.c_int, C.c_int, C.c_double, f64p, f64p)
            fn("assemble_lower", C.c_int, Grid, C.c_double, f64p, i32p, i32p, f64p,
               C.POINTER(C.c_int64))
            fn("compliance_sensitivity", C.c_int, Grid, C.c_double, f64p, f64p, C.c_double,
               C.c_double, C.c_double, u8p, C.POINTER(C.c_double), f64p)
            fn("apply_filter", C.c_int, C.c_void_p, f64p, f64p)
            fn("apply_filter_adjoint", C.c_int, C.c_void_p, f64p, f64p)
            fn("backfilter", C.c_int, C.c_void_p, f64p, f64p, C.c_double, C.c_double, C.c_int,
               f64p)
            fn("solve_eta", C.c_int, Grid, f64p, C.c_double, C.c_double, u8p,
               C.POINTER(C.c_double), C.POINTER(C.c_int))
            fn("bisect_update", C.c_int, Grid, f64p, f64p, f64p, u8p, C.POINTER(OcParams),
               C.c_int, C.c_void_p, C.c_double, C.c_double, VOLUME_FN, C.c_void_p, f64p,
               C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int))
            fn("primal_dual_update", C.c_int, Grid, f64p, f64p, f64p, u8p, C.POINTER(OcParams),
               C.c_double, f64p, C.POINTER(C.c_double), C.POINTER(C.c_int))
            fn("solve_state", C.c_int, Grid, C.c_double, f64p, f64p, i32p, C.c_int64, f64p)
            fn("problem_create", C.c_void_p, Grid, C.c_double, C.c_int, C.c_double, u8p)
            fn("problem_destroy", None, C.c_void_p)
            fn("design_pass", C.c_int, C.c_void_p, f64p, f64p, C.POINTER(PassParams),
               C.POINTER(PassOut))

    # ----------------------------------------------------------------- utils
    def _err(self) -> str:
        return (self._err_f() or b"").decode()

    def _check(self, st: int):
        if st:
            raise OracleError(st, self._err())

    def _call(self, name, *args):
        return getattr(self.lib, self.pre + name)(*args)

    def generate(self, seed: int, stream: int, kind: str, a: float, b: float, count: int,
                 offset: int = 0) -> np.ndarray:
        """port only: SURVEY.md Appendix B generator (same bits as topo_generate)."""
        out = np.empty(count)
        self.lib.orc_generate(seed, stream, 0 if kind == "uniform" else 1, a, b, offset, count,
                              out.ctypes.data)
        return out

    def set_threads(self, n: int) -> int:
        return self.lib.orc_set_threads(n) if self.kind == "port" else 1

    # ------------------------------------------------------------- grid.hpp
    def connectivity(self, grid) -> np.ndarray:
        d = 24 if grid[2] > 0 else 8
        out = np.empty(_num_elements(grid) * d, np.int32)
        self._check(self._call("build_connectivity", Grid(*grid), _p(out)))
        return out.reshape(-1, d)

    def index_pairs(self, grid):
        P = 300 if grid[2] > 0 else 36
        n = _num_elements(grid) * P
        iK = np.empty(n, np.int32)
        jK = np.empty(n, np.int32)
        self._check(self._call("build_index_pairs", Grid(*grid), _p(iK), _p(jK)))
        return iK, jK

    def partition(self, grid, pasS=(), pasV=()) -> np.ndarray:
        s = np.ascontiguousarray(pasS, np.int32)
        v = np.ascontiguousarray(pasV, np.int32)
        st = np.empty(_num_elements(grid), np.uint8)
        self._check(self._call("partition", Grid(*grid), _p(s), len(s), _p(v), len(v), _p(st)))
        return st

    # -------------------------------------------------------------- fea.hpp
    def element_stiffness(self, dim: int, nu: float):
        d = 24 if dim == 3 else 8
        full = np.empty(d * d)
        lower = np.empty(d * (d + 1) // 2)
        self._check(self._call("element_stiffness", dim, nu, _p(full), _p(lower)))
        return full.reshape(d, d, order="F"), lower

    def simp(self, xhat, e0=1.0, emin=1e-9, p=3.0):
        x = _f64(xhat)
        sK = np.empty_like(x)
        dsK = np.empty_like(x)
        self._call("simp", len(x), _p(x), e0, emin, p, _p(sK), _p(dsK))
        return sK, dsK

    def assemble_values(self, sK, ke_lower):
        sK = _f64(sK)
        kl = _f64(ke_lower)
        out = np.empty(len(sK) * len(kl))
        self.lib.orc_assemble_values(len(sK), len(kl), _p(sK), _p(kl), _p(out))
        return out

    def assemble_lower_csc(self, grid, nu, sK):
        """duplicate-summed lower CSC of assemble_lower (fea.hpp:154-176)."""
        sK = _f64(sK)
        nnz = C.c_int64()
        f = getattr(self.lib, self.pre + "assemble_lower")
        self._check(f(Grid(*grid), nu, _p(sK), None, None, None, C.byref(nnz)))
        n = _num_dofs(grid)
        cp = np.empty(n + 1, np.int32)
        ri = np.empty(nnz.value, np.int32)
        va = np.empty(nnz.value)
        self._check(f(Grid(*grid), nu, _p(sK), _p(cp), _p(ri), _p(va), C.byref(nnz)))
        return cp, ri, va

    def compliance_sensitivity(self, grid, ke_full_or_nu, u, xhat, state=None, e0=1.0,
                               emin=1e-9, p=3.0):
        u = _f64(u)
        x = _f64(xhat)
        dc = np.empty_like(x)
        c = C.c_double()
        st = None if state is None else np.ascontiguousarray(state, np.uint8)
        if self.kind == "port":
            kf = _f64(np.asarray(ke_full_or_nu).reshape(-1, order="F"))
            self._check(self.lib.orc_compliance_sensitivity(Grid(*grid), _p(kf), _p(u), _p(x),
                                                            e0, emin, p, _p(st), C.byref(c),
                                                            _p(dc)))
        else:
            self._check(self.lib.ref_compliance_sensitivity(Grid(*grid), float(ke_full_or_nu),
                                                            _p(u), _p(x), e0, emin, p, _p(st),
                                                            C.byref(c), _p(dc)))
        return c.value, dc

    # ----------------------------------------------------------- filter.hpp
    def filter(self, grid, rmin: float, bc: int = 0) -> Filter:
        return Filter(self, grid, rmin, bc)

    def apply_filter(self, f: Filter, x):
        x = _f64(x)
        out = np.empty_like(x)
        r = self._call("apply_filter", f.h, _p(x), _p(out))
        if self.kind != "port":
            self._check(r)
        return out

    def apply_filter_adjoint(self, f: Filter, g):
        g = _f64(g)
        out = np.empty_like(g)
        r = self._call("apply_filter_adjoint", f.h, _p(g), _p(out))
        if self.kind != "port":
            self._check(r)
        return out

    def project(self, xt, eta, beta):
        xt = _f64(xt)
        out = np.empty_like(xt)
        self._call("project", len(xt), _p(xt), eta, beta, _p(out))
        return out

    def project_derivative(self, xt, eta, beta):
        xt = _f64(xt)
        out = np.empty_like(xt)
        self._call("project_derivative", len(xt), _p(xt), eta, beta, _p(out))
        return out

    def project_eta_derivative(self, xt, eta, beta):
        return self._call("project_eta_derivative", xt, eta, beta)

    def backfilter(self, f: Filter, g, xt, eta, beta, on=True):
        g = _f64(g)
        xt = _f64(xt)
        out = np.empty_like(g)
        r = self._call("backfilter", f.h, _p(g), _p(xt), eta, beta, int(on), _p(out))
        if self.kind != "port":
            self._check(r)
        return out

    def solve_eta(self, xt, beta, eta0, state=None, grid=None):
        xt = _f64(xt)
        st = None if state is None else np.ascontiguousarray(state, np.uint8)
        eta = C.c_double()
        it = C.c_int()
        if self.kind == "port":
            self._check(self.lib.orc_solve_eta(len(xt), _p(xt), beta, eta0, _p(st), C.byref(eta),
                                               C.byref(it)))
        else:
            g = grid if grid is not None else (len(xt), 1, 0)
            self._check(self.lib.ref_solve_eta(Grid(*g), _p(xt), beta, eta0, _p(st),
                                               C.byref(eta), C.byref(it)))
        return eta.value, it.value

    def eta_mismatch(self, xt, beta, eta, state=None):
        """port only: g(eta) of filter.hpp:187-196 (already divided by m)."""
        xt = _f64(xt)
        st = None if state is None else np.ascontiguousarray(state, np.uint8)
        return self.lib.orc_eta_mismatch(len(xt), _p(xt), beta, eta, _p(st))

    # --------------------------------------------------------------- oc.hpp
    def lambda_upper(self, x, dc, dV, volfrac, mtotal):
        x, dc, dV = _f64(x), _f64(dc), _f64(dV)
        return self._call("lambda_upper", len(x), _p(x), _p(dc), _p(dV), volfrac, mtotal)

    def oc_candidate(self, x, dc, dV, lam, move):
        x, dc, dV = _f64(x), _f64(dc), _f64(dV)
        out = np.empty_like(x)
        self._check(self._call("oc_candidate", len(x), _p(x), _p(dc), _p(dV), lam, move, _p(out)))
        return out

    def bisect_update(self, x, dc, dV, state=None, move=0.2, volfrac=0.5, rel_tol=1e-4,
                      vol_tol=1e-3, lambda_space=False, abs_tol=1e-8, lambda_max=0.0,
                      mode=VOL_MEAN, filt: Filter | None = None, eta=0.5, beta=1.0,
                      callback=None, grid=None):
        x, dc, dV = _f64(x), _f64(dc), _f64(dV)
        m = len(x)
        st = None if state is None else np.ascontiguousarray(state, np.uint8)
        prm = OcParams(move, volfrac, rel_tol, vol_tol, int(lambda_space), abs_tol, lambda_max)
        xNew = np.empty_like(x)
        lam = C.c_double()
        bis = C.c_int()
        ev = C.c_int()
        if callback is not None:
            def _cb(_u, ptr, n):
                return float(callback(np.ctypeslib.as_array(ptr, shape=(n,)).copy()))
            cb = VOLUME_FN(_cb)
            mode = VOL_CALLBACK
        else:
            cb = VOLUME_FN(0)
        fh = filt.h if filt is not None else None
        if self.kind == "port":
            r = self.lib.orc_bisect_update(m, _p(x), _p(dc), _p(dV), _p(st), C.byref(prm), mode,
                                           fh, eta, beta, cb, None, _p(xNew), C.byref(lam),
                                           C.byref(bis), C.byref(ev))
        else:
            g = grid if grid is not None else (filt.grid if filt is not None else (m, 1, 0))
            r = self.lib.ref_bisect_update(Grid(*g), _p(x), _p(dc), _p(dV), _p(st), C.byref(prm),
                                           mode, fh, eta, beta, cb, None, _p(xNew), C.byref(lam),
                                           C.byref(bis), C.byref(ev))
        self._check(r)
        return xNew, lam.value, bis.value, ev.value

    def primal_dual_update(self, x, dc, dV, state=None, move=0.2, volfrac=0.5, rel_tol=1e-4,
                           vol_tol=1e-3, pd_tol=1e-10, grid=None):
        """oc.hpp:181-241. Returns (xNew, lambda, iterations, fell_back); the
        reference does not report a fallback (-1)."""
        x, dc, dV = _f64(x), _f64(dc), _f64(dV)
        m = len(x)
        st = None if state is None else np.ascontiguousarray(state, np.uint8)
        prm = OcParams(move, volfrac, rel_tol, vol_tol, 0, 1e-8, 0.0)
        xNew = np.empty_like(x)
        lam, it, fb = C.c_double(), C.c_int(), C.c_int(-1)
        if self.kind == "port":
            r = self.lib.orc_primal_dual_update(m, _p(x), _p(dc), _p(dV), _p(st), C.byref(prm),
                                                pd_tol, _p(xNew), C.byref(lam), C.byref(it),
                                                C.byref(fb))
        else:
            g = grid if grid is not None else (m, 1, 0)
            r = self.lib.ref_primal_dual_update(Grid(*g), _p(x), _p(dc), _p(dV), _p(st),
                                                C.byref(prm), pd_tol, _p(xNew), C.byref(lam),
                                                C.byref(it))
        self._check(r)
        return xNew, lam.value, it.value, fb.value

    def solve_state(self, grid, nu, sK, f, fixed):
        """reference only: fea.hpp:205-239 solve_equilibrium (dense Cholesky of
        the Eigen shim: small grids)."""
        sK, f = _f64(sK), _f64(f)
        fx = np.ascontiguousarray(fixed, np.int32)
        u = np.empty_like(f)
        self._check(self.lib.ref_solve_state(Grid(*grid), nu, _p(sK), _p(f), _p(fx), fx.size,
                                             _p(u)))
        return u

    # ----------------------------------------------------------- driver glue
    def design_pass(self, grid, rmin, x, u, state=None, *, nu=0.3, e0=1.0, emin=1e-9, penal=3.0,
                    beta=2.0, eta0=0.5, move=0.2, volfrac=0.5, eta_override=math.nan,
                    volume_mode=VOL_FILTERED, bc=0, filt: Filter | None = None,
                    problem=None) -> PassResult:
        m = _num_elements(grid)
        x, u = _f64(x), _f64(u)
        st = None if state is None else np.ascontiguousarray(state, np.uint8)
        arrs = {k: np.empty(m) for k in ("xTilde", "xPhys", "sKe", "dcPhys", "dc", "dV", "xNew")}
        out = PassOut(*[arrs[k].ctypes.data for k in
                        ("xTilde", "xPhys", "sKe", "dcPhys", "dc", "dV", "xNew")])
        prm = PassParams(e0, emin, penal, beta, eta0, move, volfrac, eta_override, volume_mode)
        if self.kind == "port":
            f = filt if filt is not None else self.filter(grid, rmin, bc)
            kf, _ = self.element_stiffness(3 if grid[2] > 0 else 2, nu)
            kf = _f64(kf.reshape(-1, order="F"))
            self._check(self.lib.orc_design_pass(Grid(*grid), f.h, _p(kf), _p(st), _p(x), _p(u),
                                                 C.byref(prm), C.byref(out)))
        else:
            h = problem if problem is not None else self.problem(grid, rmin, bc, nu, st)
            self._check(self.lib.ref_design_pass(h.h, _p(x), _p(u), C.byref(prm), C.byref(out)))
        return PassResult(eta=out.eta, c=out.c, lam=out.lambda_, eta_iters=out.eta_iters,
                          bisections=out.bisections, evaluations=out.evaluations, **arrs)

    def problem(self, grid, rmin, bc=0, nu=0.3, state=None):
        """reference only: cached grid / Ke / filter / partition handle."""
        owner = self

        class _H:
            def __init__(s):
                st = None if state is None else np.ascontiguousarray(state, np.uint8)
                s.h = owner.lib.ref_problem_create(Grid(*grid), rmin, bc, nu, _p(st))
                if not s.h:
                    raise OracleError(1, owner._err())

            def __del__(s):
                if getattr(s, "h", None):
                    owner.lib.ref_problem_destroy(s.h)

        return _H()
