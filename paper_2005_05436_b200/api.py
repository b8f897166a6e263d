"""Host-side mirror of the reference operator API for the design-update path.

Same names, argument meaning and error behaviour as the reference's free
functions in /root/reference/proj/include/topopt/{grid,fea,filter,oc}.hpp,
bound to a `Context` (one GPU / one x-slab rank) instead of Eigen objects:

    reference (C++ / Eigen)                          this module (Context method)
    build_connectivity            grid.hpp:89          build_connectivity()
    build_symmetric_index_pairs   grid.hpp:133         build_symmetric_index_pairs()
    partition_domain              grid.hpp:155         partition_domain()  (module level)
    element_stiffness_q4/h8       fea.hpp:51,73        element_stiffness() (module level)
    simp_interpolate              fea.hpp:135          simp_interpolate()
    assemble_lower (values)       fea.hpp:154-176      assemble_values()
    compliance_and_sensitivity    fea.hpp:248          compliance_and_sensitivity()
    build_filter / hs / taps      filter.hpp:95        taps(), hs()
    apply_filter                  filter.hpp:119       apply_filter()
    apply_filter_adjoint          filter.hpp:126       apply_filter_adjoint()
    project / project_derivative  filter.hpp:137,146   project(), project_derivative()
    backfilter                    filter.hpp:166       backfilter()
    solve_volume_preserving_eta   filter.hpp:182       solve_volume_preserving_eta()
    lambda_upper_estimate         oc.hpp:31            lambda_upper_estimate()
    oc_candidate                  oc.hpp:72            oc_candidate()
    bisect_update                 oc.hpp:93            bisect_update()
    run_optimization pass body    driver.hpp:183-231   design_pass()

Errors follow the reference's exception types: std::invalid_argument ->
ValueError, std::overflow_error -> OverflowError, std::runtime_error ->
RuntimeError (all subclasses of TopoError).

Arrays: numpy float64 (host; results come back as numpy) or torch float64
CUDA tensors (device; used in place, results come back as CUDA tensors).
"""
from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _lib as L


class TopoError(RuntimeError):
    code = -1


class InvalidArgument(TopoError, ValueError):
    code = L.TOPO_EINVAL


class IndexOverflow(TopoError, OverflowError):
    code = L.TOPO_EOVERFLOW


class NonMonotone(TopoError):
    code = L.TOPO_ENONMONO


class CudaError(TopoError):
    code = L.TOPO_ECUDA


_EXC = {L.TOPO_EINVAL: InvalidArgument, L.TOPO_EOVERFLOW: IndexOverflow,
        L.TOPO_ENONMONO: NonMonotone, L.TOPO_ECUDA: CudaError}


def _raise(code: int, msg: str):
    raise _EXC.get(code, TopoError)(f"[topo status {code}] {msg}")


# ------------------------------------------------------------------ arrays
def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


# Device arrays reach the library by raw pointer, but the library works on its
# own (non-blocking) stream. Every CUDA tensor an entry point is about to see
# (an input, or an output block torch.empty just handed out) marks the calling
# thread; the next library call first orders the context's stream after the
# tensor's current torch stream (topo_wait_stream). Entry points are
# synchronous at return, so results need no fence back.
_tls = threading.local()


def _note_cuda(t) -> None:
    _tls.pending = t.device


class _FencedLib:
    """The ctypes library of one Context: calls taking the context handle are
    preceded by the stream fence when CUDA tensors were staged for them."""

    def __init__(self, lib, owner: "Context"):
        self._lib = lib
        self._owner = owner

    def __getattr__(self, name):
        f = getattr(self._lib, name)
        if not name.startswith("topo_") or name in ("topo_last_error", "topo_wait_stream"):
            return f

        def call(*args):
            dev = getattr(_tls, "pending", None)
            h = getattr(self._owner, "h", None)
            if dev is not None and h:
                _tls.pending = None
                import torch
                s = torch.cuda.current_stream(dev).cuda_stream
                st = self._lib.topo_wait_stream(h, s)
                if st:
                    _raise(st, self._lib.topo_last_error(h).decode())
            return f(*args)

        return call


class _Arr:
    """Keeps a contiguous float64 / int32 / uint8 buffer alive and exposes its pointer."""

    def __init__(self, a, dtype=np.float64, n: Optional[int] = None, name: str = "array"):
        if _is_torch(a):
            import torch
            tdt = {np.float64: torch.float64, np.int32: torch.int32, np.uint8: torch.uint8}[dtype]
            if a.dtype != tdt:
                a = a.to(tdt)
            a = a.contiguous()
            if a.is_cuda:
                _note_cuda(a)
            self.obj = a
            self.ptr = a.data_ptr()
            self.size = a.numel()
            self.device = a.is_cuda
        else:
            a = np.ascontiguousarray(a, dtype=dtype)
            self.obj = a
            self.ptr = a.ctypes.data
            self.size = a.size
            self.device = False
        if n is not None and self.size != n:
            raise InvalidArgument(f"{name}: length {self.size} != expected {n}")


def _empty(n: int, like_device: bool, dtype=np.float64):
    if like_device:
        import torch
        tdt = {np.float64: torch.float64, np.int32: torch.int32, np.int64: torch.int64}[dtype]
        t = torch.empty(n, dtype=tdt, device="cuda")
        _note_cuda(t)
        return t, t.data_ptr()
    a = np.empty(n, dtype=dtype)
    return a, a.ctypes.data


# ---------------------------------------------------------------- structs
@dataclass
class SimpParams:  # fea.hpp:124-128
    e0: float = 1.0
    eMin: float = 1e-9
    p: float = 3.0

    def c(self):
        return L.Simp(self.e0, self.eMin, self.p)


@dataclass
class OcParams:  # oc.hpp:14-20 (+ BisectOptions oc.hpp:81-85)
    move: float = 0.2
    volfrac: float = 0.5
    bisectRelTol: float = 1e-4
    volumeTol: float = 1e-3
    lambdaSpace: bool = False
    absTol: float = 1e-8
    lambdaMax: float = 0.0
    pdTol: float = 1e-10  # primal-dual multiplier stagnation tolerance

    def c(self):
        return L.OcParams(self.move, self.volfrac, self.bisectRelTol, self.volumeTol,
                          int(self.lambdaSpace), self.absTol, self.lambdaMax)


@dataclass
class UpdateResult:  # oc.hpp:22-26
    xNew: object
    lam: float
    bisections: int
    evaluations: int = 0
    fell_back: bool = False  # primal_dual_update: the bisection fallback ran


@dataclass
class PassResult:
    xTilde: object
    xPhys: object
    dcPhys: object
    dc: object
    dV: object
    xNew: object
    sK: object
    eta: float
    c: float
    lam: float
    eta_iters: int
    bisections: int
    evaluations: int
    launches: int
    Kval: object = None  # lower-triangle CSC values of K (return_K=True)


# ---------------------------------------------------------- module helpers
def element_stiffness(dim: int, nu: float = 0.3):
    """fea.hpp:51-68 (dim 2, Q4) / fea.hpp:73-121 (dim 3, H8): (full d x d, lower)."""
    lib = L.load()
    d = 24 if dim == 3 else 8
    full = np.empty(d * d)
    lower = np.empty(d * (d + 1) // 2)
    st = lib.topo_element_stiffness(dim, nu, full.ctypes.data, lower.ctypes.data)
    if st:
        _raise(st, "element stiffness: Poisson ratio must lie in (-1, 0.5)")
    return full.reshape(d, d, order="F"), lower


def generate(seed: int, stream: int, kind: str, a: float, b: float, count: int,
             offset: int = 0) -> np.ndarray:
    """SURVEY.md Appendix B counter-based generator (uniform [a, b) or normal(a, b))."""
    lib = L.load()
    out = np.empty(count)
    lib.topo_generate(seed, stream, 0 if kind == "uniform" else 1, a, b, offset, count,
                      out.ctypes.data)
    return out


def nccl_unique_id() -> bytes:
    """128-byte NCCL clique id (rank 0 creates it, the caller broadcasts it)."""
    lib = L.load()
    buf = (C.c_char * 128)()
    st = lib.topo_nccl_unique_id(buf)
    if st:
        _raise(st, "ncclGetUniqueId failed (is libnccl.so.2 loadable?)")
    return bytes(buf)


def slab_plan(nelx: int, nely: int, nelz: int, rmin: float, rank: int, nranks: int,
              j0: int = 0, j1: int = 0) -> dict:
    """x-slab of a rank (host only): owned / stored columns and the halo columns
    exchanged with the neighbours (the plan the library's halo exchange uses)."""
    lib = L.load()
    desc = L.GridDesc(nelx, nely, nelz, rmin, 0, 0.3, -1, rank, nranks, j0, j1)
    out = np.zeros(8, np.int64)
    st = lib.topo_slab_plan(C.byref(desc), out.ctypes.data)
    keys = ["j0", "j1", "sj0", "sj1", "send_left", "send_right", "recv_left", "recv_right"]
    plan = dict(zip(keys, (int(v) for v in out)))
    if st:
        _raise(st, f"slab {plan['j0']}..{plan['j1']} narrower than the filter reach")
    return plan


def fp64_peak(device: int = 0) -> float:
    """Measured FP64 FMA throughput of `device` in TFLOP/s (DFMA loop)."""
    lib = L.load()
    t = C.c_double()
    st = lib.topo_fp64_peak(device, C.byref(t))
    if st:
        _raise(st, "fp64 peak probe failed")
    return t.value


def partition_domain(grid, pasS=(), pasV=()) -> np.ndarray:
    """grid.hpp:155-188 as a per-element state byte array (0 act / 1 solid / 2 void)."""
    nelx, nely, nelz = grid
    if nelx < 1 or nely < 1 or nelz < 0:
        raise InvalidArgument("grid: element counts must be >= 1 per active axis")
    m = nelx * nely * (nelz if nelz > 0 else 1)
    s = np.unique(np.asarray(pasS, dtype=np.int64))
    v = np.unique(np.asarray(pasV, dtype=np.int64))
    for name, ids in (("pasS", s), ("pasV", v)):
        if ids.size and (ids[0] < 0 or ids[-1] >= m):
            raise InvalidArgument(f"partition: {name} contains an element index outside [0, m)")
    state = np.zeros(m, np.uint8)
    state[s] = L.PASSIVE_SOLID
    clash = v[state[v] != 0] if v.size else v
    if clash.size:
        raise InvalidArgument(
            f"partition: passive solid and void sets overlap at element {int(clash[0])}")
    state[v] = L.PASSIVE_VOID
    return state


# ----------------------------------------------------------------- context
class Context:
    """One GPU (one x-slab rank) bound to a structured grid, a filter radius,
    an element stiffness and a domain partition (the reference's immutable
    setup objects StructuredGrid / FilterOperator / ElementStiffness /
    DomainPartition)."""

    def __init__(self, nelx: int, nely: int, nelz: int = 0, rmin: float = 2.0,
                 bc: int = L.BC_NEUMANN, nu: float = 0.3, state=None, device: int = -1,
                 rank: int = 0, nranks: int = 1, j0: int = 0, j1: int = 0,
                 ke_full=None, ke_lower=None):
        self.lib = _FencedLib(L.load(), self)
        self.grid = (nelx, nely, nelz)
        desc = L.GridDesc(nelx, nely, nelz, rmin, bc, nu, device, rank, nranks, j0, j1)
        h = C.c_void_p()
        self._keep = []
        st_ptr = None
        if state is not None:
            sa = _Arr(state, np.uint8, name="state")
            self._keep.append(sa)
            st_ptr = sa.ptr
        kf = kl = None
        if ke_full is not None:
            kfa = _Arr(np.asarray(ke_full).reshape(-1, order="F"))
            kla = _Arr(ke_lower)
            self._keep += [kfa, kla]
            kf, kl = kfa.ptr, kla.ptr
        status = self.lib.topo_ctx_create(C.byref(desc), kf, kl, st_ptr, C.byref(h))
        self.h = h.value
        if status:
            msg = self.lib.topo_last_error(self.h).decode() if self.h else "create failed"
            self.close()
            _raise(status, msg)
        m, n = C.c_int64(), C.c_int64()
        P, T, R, a, b = (C.c_int32() for _ in range(5))
        self.lib.topo_ctx_info(self.h, C.byref(m), C.byref(n), C.byref(P), C.byref(T),
                               C.byref(R), C.byref(a), C.byref(b))
        self.m, self.n, self.P = m.value, n.value, P.value
        self.ntaps, self.reach, self.j0, self.j1 = T.value, R.value, a.value, b.value
        self.m_total = nelx * nely * (nelz if nelz > 0 else 1)
        self.d = 24 if nelz > 0 else 8

    # lifecycle
    def close(self):
        if getattr(self, "h", None):
            self.lib.topo_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, st: int):
        if st:
            _raise(st, self.lib.topo_last_error(self.h).decode())

    @property
    def launches(self) -> int:
        return int(self.lib.topo_last_launch_count(self.h))

    def set_timing(self, on: bool = True):
        """Per-stage CUDA-event timing of design_pass (events on each kernel's stream)."""
        self._check(self.lib.topo_set_timing(self.h, int(on)))

    @property
    def graph_replays(self) -> int:
        """Design passes served by the captured CUDA graph so far."""
        n = C.c_int64()
        self._check(self.lib.topo_pass_graph_replays(self.h, C.byref(n)))
        return int(n.value)

    def stage_times(self) -> dict:
        t = np.zeros(len(L.STAGES))
        self._check(self.lib.topo_stage_times(self.h, t.ctypes.data))
        return dict(zip(L.STAGES, t.tolist()))

    def comm_init(self, unique_id: bytes):
        """Join the NCCL clique of this x-slab decomposition (all ranks call it)."""
        buf = (C.c_char * 128).from_buffer_copy(unique_id)
        self._check(self.lib.topo_comm_init_nccl(self.h, buf))

    def comm_init_host(self, exchange, allreduce_sum):
        """Host-callback communicator: exchange(send_left, send_right, recv_left,
        recv_right) with numpy views (recv_* to be filled in place) and
        allreduce_sum(values) in place."""

        def _ex(_u, sl, nsl, sr, nsr, rl, nrl, rr, nrr):
            try:
                view = lambda p, n: np.ctypeslib.as_array(p, shape=(n,)) if n else np.zeros(0)
                exchange(view(sl, nsl), view(sr, nsr), view(rl, nrl), view(rr, nrr))
                return 0
            except Exception:  # noqa: BLE001 - reported as a status code
                import traceback
                traceback.print_exc()
                return 1

        def _ar(_u, p, n):
            try:
                allreduce_sum(np.ctypeslib.as_array(p, shape=(n,)))
                return 0
            except Exception:  # noqa: BLE001
                import traceback
                traceback.print_exc()
                return 1

        self._host_comm_cbs = (L.EXCHANGE_FN(_ex), L.ALLREDUCE_FN(_ar))
        hc = L.HostComm(None, *self._host_comm_cbs)
        self._check(self.lib.topo_comm_init_host(self.h, C.byref(hc)))

    def set_stream(self, cuda_stream_handle: int):
        self._check(self.lib.topo_set_stream(self.h, cuda_stream_handle))

    def device_buffer(self, which: int):
        p, n = C.c_void_p(), C.c_int64()
        self._check(self.lib.topo_device_buffer(self.h, which, C.byref(p), C.byref(n)))
        return p.value, n.value

    # grid.hpp
    def build_connectivity(self, device: bool = False):
        out, ptr = _empty(self.m * self.d, device, np.int32)
        self._check(self.lib.topo_build_connectivity(self.h, ptr))
        return out.reshape(-1, self.d) if not device else out.view(-1, self.d)

    def build_symmetric_index_pairs(self, device: bool = False, keep: bool = False):
        """grid.hpp:133-153. keep=True leaves iK/jK in the context only."""
        if keep:
            self._check(self.lib.topo_build_index_pairs(self.h, None, None))
            return None
        iK, pi = _empty(self.m * self.P, device, np.int32)
        jK, pj = _empty(self.m * self.P, device, np.int32)
        self._check(self.lib.topo_build_index_pairs(self.h, pi, pj))
        return iK, jK

    # filter.hpp
    def taps(self):
        T = self.ntaps
        di, dj, dk = (np.empty(T, np.int32) for _ in range(3))
        w = np.empty(T)
        self._check(self.lib.topo_filter_taps(self.h, di.ctypes.data, dj.ctypes.data,
                                              dk.ctypes.data, w.ctypes.data))
        return di, dj, dk, w

    def hs(self):
        out = np.empty(self.m)
        self._check(self.lib.topo_filter_hs(self.h, out.ctypes.data))
        return out

    def apply_filter(self, x, pin: bool = False):
        a = _Arr(x, n=self.m, name="filter: field")
        out, ptr = _empty(self.m, a.device)
        self._check(self.lib.topo_filter(self.h, a.ptr, ptr, int(pin)))
        return out

    def apply_filter_adjoint(self, g):
        a = _Arr(g, n=self.m, name="filter: field")
        out, ptr = _empty(self.m, a.device)
        self._check(self.lib.topo_filter_adjoint(self.h, a.ptr, ptr))
        return out

    def project(self, xt, eta: float, beta: float):
        a = _Arr(xt)
        out, ptr = _empty(a.size, a.device)
        self._check(self._proj_len(a) or self.lib.topo_project(self.h, a.ptr, eta, beta, ptr))
        return out

    def project_derivative(self, xt, eta: float, beta: float):
        a = _Arr(xt)
        out, ptr = _empty(a.size, a.device)
        self._check(self._proj_len(a) or
                    self.lib.topo_project_derivative(self.h, a.ptr, eta, beta, ptr))
        return out

    def _proj_len(self, a):
        if a.size != self.m:
            raise InvalidArgument(f"project: length {a.size} != {self.m}")
        return 0

    def backfilter(self, g, xt, eta: float, beta: float, projection_on: bool = True):
        ga = _Arr(g, n=self.m, name="filter: field")
        xa = _Arr(xt, n=self.m, name="filter: field")
        out, ptr = _empty(self.m, ga.device)
        self._check(self.lib.topo_backfilter(self.h, ga.ptr, xa.ptr, eta, beta,
                                             int(projection_on), ptr))
        return out

    def solve_volume_preserving_eta(self, xTilde, beta: float, eta0: float):
        if not beta > 0:
            raise InvalidArgument("eta solve: beta must be positive")
        a = _Arr(xTilde, n=self.m, name="eta: field")
        eta, it = C.c_double(), C.c_int32()
        self._check(self.lib.topo_solve_eta(self.h, a.ptr, beta, eta0, C.byref(eta),
                                            C.byref(it)))
        return eta.value, it.value

    # fea.hpp
    def simp_interpolate(self, xhat, prm: SimpParams = SimpParams()):
        a = _Arr(xhat, n=self.m, name="simp: field")
        sK, p1 = _empty(self.m, a.device)
        dsK, p2 = _empty(self.m, a.device)
        sp = prm.c()
        self._check(self.lib.topo_simp_interpolate(self.h, a.ptr, C.byref(sp), p1, p2))
        return sK, dsK

    def assemble_values(self, sK, device: bool = False):
        """fea.hpp:162-169 triplet values, t = e * P + q (length m * P)."""
        a = _Arr(sK, n=self.m, name="assemble: index pairs do not match element count; sK")
        out, ptr = _empty(self.m * self.P, device or a.device)
        self._check(self.lib.topo_assemble_values(self.h, a.ptr, ptr))
        return out

    def csc_set_fixed(self, fixed=None) -> int:
        """Reduced (free-DOF) CSC mode of EquilibriumSolver (fea.hpp:316-361) for
        the load case's fixed DOFs; None / empty returns to the full matrix.
        Returns the number of free DOFs (columns)."""
        nf = C.c_int64()
        if fixed is None or len(fixed) == 0:
            self._check(self.lib.topo_csc_set_fixed(self.h, None, 0, C.byref(nf)))
        else:
            f = np.ascontiguousarray(fixed, dtype=np.int32)
            self._check(self.lib.topo_csc_set_fixed(self.h, f.ctypes.data, f.size, C.byref(nf)))
        self._csc_cols = nf.value
        return nf.value

    def csc_pattern(self, device: bool = False):
        """Lower-triangle CSC pattern of K (assemble_lower / setFromTriplets,
        fea.hpp:154-176): (col_ptr int64 ncols+1, row_idx int32 nnz); ncols = n,
        or the free-DOF count after csc_set_fixed."""
        nnz = C.c_int64()
        self._check(self.lib.topo_csc_pattern(self.h, None, None, C.byref(nnz)))
        cp, pc = _empty(getattr(self, "_csc_cols", self.n) + 1, device, np.int64)
        ri, pr = _empty(nnz.value, device, np.int32)
        self._check(self.lib.topo_csc_pattern(self.h, pc, pr, None))
        return cp, ri

    def csc_values(self, sK, device: bool = False):
        """Duplicate-summed CSC values from the per-element modulus sK (m)."""
        a = _Arr(sK, n=self.m, name="csc: sK")
        nnz = C.c_int64()
        self._check(self.lib.topo_csc_pattern(self.h, None, None, C.byref(nnz)))
        out, ptr = _empty(nnz.value, device or a.device)
        self._check(self.lib.topo_csc_values(self.h, a.ptr, ptr))
        return out

    def compliance_and_sensitivity(self, u, xhat, prm: SimpParams = SimpParams()):
        ua = _Arr(u, n=self.n, name="sensitivity: displacement")
        xa = _Arr(xhat, n=self.m, name="sensitivity: field")
        dc, ptr = _empty(self.m, xa.device)
        c = C.c_double()
        sp = prm.c()
        self._check(self.lib.topo_sensitivity(self.h, ua.ptr, xa.ptr, C.byref(sp), C.byref(c),
                                              ptr))
        return c.value, dc

    # oc.hpp
    def lambda_upper_estimate(self, xAct, dcAct, dVAct, volfrac: float, mTotal: int) -> float:
        x, dc, dV = _Arr(xAct), _Arr(dcAct), _Arr(dVAct)
        lam = C.c_double()
        self._check(self.lib.topo_lambda_upper(self.h, x.size, x.ptr, dc.ptr, dV.ptr, volfrac,
                                               mTotal, C.byref(lam)))
        return lam.value

    def oc_candidate(self, xAct, dcAct, dVAct, lam: float, move: float):
        x, dc, dV = _Arr(xAct), _Arr(dcAct), _Arr(dVAct)
        out, ptr = _empty(x.size, x.device)
        self._check(self.lib.topo_oc_candidate(self.h, x.size, x.ptr, dc.ptr, dV.ptr, lam, move,
                                               ptr))
        return out

    def bisect_update(self, x, dc, dV, prm: OcParams = OcParams(),
                      volume_mode: int = L.VOL_MEAN,
                      physical_volume: Optional[Callable[[np.ndarray], float]] = None,
                      eta: float = 0.5, beta: float = 1.0) -> UpdateResult:
        """oc.hpp:93-174. `physical_volume` (a Python callable on the full host
        candidate) stands in for the reference's std::function callback; the
        built-in modes are driver.hpp:214-229's ft = 1 / 2 / 3 volumes."""
        xa = _Arr(x, n=self.m, name="oc: x")
        ca = _Arr(dc, n=self.m, name="oc: dc")
        va = _Arr(dV, n=self.m, name="oc: dV")
        out, ptr = _empty(self.m, xa.device)
        lam, bis, ev = C.c_double(), C.c_int32(), C.c_int32()
        op = prm.c()
        if physical_volume is not None:
            volume_mode = L.VOL_CALLBACK

            def _cb(_user, p, n):
                return float(physical_volume(np.ctypeslib.as_array(p, shape=(n,)).copy()))
            cb = L.VOLUME_FN(_cb)
        else:
            cb = L.VOLUME_FN(0)
        self._check(self.lib.topo_oc_bisect(self.h, xa.ptr, ca.ptr, va.ptr, C.byref(op),
                                            volume_mode, eta, beta, cb, None, ptr, C.byref(lam),
                                            C.byref(bis), C.byref(ev)))
        return UpdateResult(out, lam.value, bis.value, ev.value)

    def primal_dual_update(self, x, dc, dV, prm: OcParams = OcParams()) -> UpdateResult:
        """oc.hpp:181-241 (ft = 1): dual-map iteration with the reference's
        fallback to the mean-volume bisection; bisections = iterations."""
        xa = _Arr(x, n=self.m, name="oc: x")
        ca = _Arr(dc, n=self.m, name="oc: dc")
        va = _Arr(dV, n=self.m, name="oc: dV")
        out, ptr = _empty(self.m, xa.device)
        lam, it, fb = C.c_double(), C.c_int32(), C.c_int32()
        op = prm.c()
        self._check(self.lib.topo_oc_primal_dual(self.h, xa.ptr, ca.ptr, va.ptr, C.byref(op),
                                                 prm.pdTol, ptr, C.byref(lam), C.byref(it),
                                                 C.byref(fb)))
        return UpdateResult(out, lam.value, it.value, 0, bool(fb.value))

    def solve_state(self, sK, f, fixed, rtol: float = 1e-10, maxit: int = 100000,
                    multigrid: bool = False):
        """fea.hpp:205-239 solve_equilibrium on the device: K(sK) u = f with u = 0
        on `fixed`; matrix-free PCG, Jacobi or geometric-multigrid (V-cycle)
        preconditioned. Returns (u, iterations, relres)."""
        sa = _Arr(sK, n=self.m, name="solve: sK")
        fa = _Arr(f, n=self.n, name="solve: load vector")
        fx = np.ascontiguousarray(fixed if fixed is not None else [], dtype=np.int32)
        out, ptr = _empty(self.n, fa.device)
        it, rr = C.c_int32(), C.c_double()
        fn = self.lib.topo_solve_state_mg if multigrid else self.lib.topo_solve_state
        self._check(fn(self.h, sa.ptr, fa.ptr, fx.ctypes.data, fx.size, rtol, maxit, ptr,
                       C.byref(it), C.byref(rr)))
        return out, it.value, rr.value

    def apply_stiffness(self, sK, x, variant: int = 0):
        """y = K(sK) x, the solves' matrix-free operator (no fixed DOFs)."""
        sa = _Arr(sK, n=self.m, name="apply: sK")
        xa = _Arr(x, n=self.n, name="apply: x")
        out, ptr = _empty(self.n, xa.device)
        self._check(self.lib.topo_apply_stiffness(self.h, sa.ptr, xa.ptr, ptr, variant))
        return out

    # driver.hpp:183-231
    def design_pass(self, x, U, *, beta: float = 2.0, eta0: float = 0.5, move: float = 0.2,
                    volfrac: float = 0.5, simp: SimpParams = SimpParams(),
                    eta_override: float = math.nan, volume_mode: int = L.VOL_FILTERED,
                    write_sk: bool = True, return_sk: bool = False, outputs: bool = True,
                    out_device: Optional[bool] = None, return_K: bool = False) -> PassResult:
        xa = _Arr(x, n=self.m, name="pass: x")
        ua = _Arr(U, n=self.n, name="pass: U")
        dev = xa.device if out_device is None else out_device
        res = {}
        ptrs = {}
        for k in ("xTilde", "xPhys", "dcPhys", "dc", "dV", "xNew"):
            if outputs or k == "xNew":
                res[k], ptrs[k] = _empty(self.m, dev)
            else:
                res[k], ptrs[k] = None, None
        if return_sk:
            res["sK"], ptrs["sK"] = _empty(self.m * self.P, dev)
        else:
            res["sK"], ptrs["sK"] = None, None
        kv, pk = None, None
        if return_K:
            nnz = C.c_int64()
            self._check(self.lib.topo_csc_pattern(self.h, None, None, C.byref(nnz)))
            kv, pk = _empty(nnz.value, dev)
        pp = L.PassParams(simp.c(), beta, eta0, move, volfrac, eta_override, volume_mode,
                          int(write_sk))
        po = L.PassOut(ptrs["xTilde"], ptrs["xPhys"], ptrs["dcPhys"], ptrs["dc"], ptrs["dV"],
                       ptrs["xNew"], ptrs["sK"])
        po.Kval = pk
        self._check(self.lib.topo_design_pass(self.h, xa.ptr, ua.ptr, C.byref(pp), C.byref(po)))
        return PassResult(eta=po.eta, c=po.c, lam=po.lambda_, eta_iters=po.eta_iters,
                          bisections=po.bisections, evaluations=po.evaluations,
                          launches=self.launches, Kval=kv, **res)
