"""ctypes binding of include/topo_capi.h (libtopo_b200.so, built in-tree).

Loading the library needs no GPU; every compute entry point does. There is no
CPU fallback: if the library is missing, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

# TOPO_LIB_PATH: load another build of the same library (A/B experiments)
LIB_PATH = os.environ.get("TOPO_LIB_PATH") or _build.LIB

TOPO_OK, TOPO_EINVAL, TOPO_EOVERFLOW, TOPO_ENONMONO, TOPO_ECUDA, TOPO_ENCCL, TOPO_ENOMEM = range(7)
BC_NEUMANN, BC_DIRICHLET = 0, 1
ACTIVE, PASSIVE_SOLID, PASSIVE_VOID = 0, 1, 2
VOL_CALLBACK, VOL_MEAN, VOL_PROJECTED, VOL_FILTERED = 0, 1, 2, 3
BUF_SK, BUF_IK, BUF_JK, BUF_XNEW, BUF_XPHYS = range(5)

# every symbol include/topo_capi.h declares
EXPORTS = [
    "topo_ctx_create", "topo_ctx_destroy", "topo_last_error", "topo_set_stream", "topo_sync",
    "topo_wait_stream",
    "topo_device_buffer", "topo_ctx_info", "topo_comm_init_nccl", "topo_element_stiffness",
    "topo_generate", "topo_build_connectivity", "topo_build_index_pairs",
    "topo_simp_interpolate", "topo_assemble_values", "topo_sensitivity", "topo_filter",
    "topo_filter_adjoint", "topo_project", "topo_project_derivative", "topo_backfilter",
    "topo_solve_eta", "topo_filter_taps", "topo_filter_hs", "topo_lambda_upper",
    "topo_oc_candidate", "topo_oc_bisect", "topo_design_pass", "topo_design_pass_begin",
    "topo_design_pass_end", "topo_last_launch_count",
    "topo_set_timing", "topo_stage_times", "topo_pass_graph_replays", "topo_loop_records",
    "topo_anderson_step", "topo_anderson_reset", "topo_host_oc_replay", "topo_host_eta_replay",
    "topo_nccl_unique_id", "topo_comm_init_host", "topo_slab_plan", "topo_fp64_peak",
    "topo_csc_pattern", "topo_csc_values", "topo_csc_set_fixed", "topo_oc_primal_dual",
    "topo_solve_state", "topo_solve_state_mg", "topo_apply_stiffness",
    "topo_device_alloc", "topo_device_free", "topo_copy",
]
STAGES = ["filter", "eta", "elem", "adjoint", "oc", "sk_store", "pass"]


class GridDesc(C.Structure):
    _fields_ = [("nelx", C.c_int32), ("nely", C.c_int32), ("nelz", C.c_int32),
                ("rmin", C.c_double), ("bc", C.c_int32), ("nu", C.c_double),
                ("device", C.c_int32), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("j0", C.c_int32), ("j1", C.c_int32)]


class Simp(C.Structure):
    _fields_ = [("e0", C.c_double), ("emin", C.c_double), ("penal", C.c_double)]


class OcParams(C.Structure):
    _fields_ = [("move", C.c_double), ("volfrac", C.c_double), ("bisect_rel_tol", C.c_double),
                ("volume_tol", C.c_double), ("lambda_space", C.c_int32), ("abs_tol", C.c_double),
                ("lambda_max", C.c_double)]


class PassParams(C.Structure):
    _fields_ = [("simp", Simp), ("beta", C.c_double), ("eta0", C.c_double),
                ("move", C.c_double), ("volfrac", C.c_double), ("eta_override", C.c_double),
                ("volume_mode", C.c_int32), ("write_sk", C.c_int32)]


class PassOut(C.Structure):
    _fields_ = [("xTilde", C.c_void_p), ("xPhys", C.c_void_p), ("dcPhys", C.c_void_p),
                ("dc", C.c_void_p), ("dV", C.c_void_p), ("xNew", C.c_void_p),
                ("sK", C.c_void_p), ("eta", C.c_double), ("c", C.c_double),
                ("lambda_", C.c_double), ("eta_iters", C.c_int32), ("bisections", C.c_int32),
                ("evaluations", C.c_int32), ("Kval", C.c_void_p)]


VOLUME_FN = C.CFUNCTYPE(C.c_double, C.c_void_p, C.POINTER(C.c_double), C.c_int64)
SFUN = C.CFUNCTYPE(C.c_double, C.c_void_p, C.c_double)
GFUN = C.CFUNCTYPE(None, C.c_void_p, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double))
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int64,
                          C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_double), C.c_int64,
                          C.POINTER(C.c_double), C.c_int64)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int)


class HostComm(C.Structure):
    _fields_ = [("user", C.c_void_p), ("exchange", EXCHANGE_FN), ("allreduce_sum", ALLREDUCE_FN)]

_lib = None


def load(build_if_missing: bool = True) -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if not build_if_missing:
            raise ImportError(f"{LIB_PATH} is missing; run `python -m paper_2005_05436_b200.build`")
        _build.build()
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    p = C.POINTER
    sig = {
        "topo_ctx_create": (C.c_int, [p(GridDesc), vp, vp, vp, p(vp)]),
        "topo_ctx_destroy": (None, [vp]),
        "topo_last_error": (C.c_char_p, [vp]),
        "topo_set_stream": (C.c_int, [vp, vp]),
        "topo_sync": (C.c_int, [vp]),
        "topo_wait_stream": (C.c_int, [vp, vp]),
        "topo_device_buffer": (C.c_int, [vp, C.c_int, p(vp), p(C.c_int64)]),
        "topo_ctx_info": (C.c_int, [vp, p(C.c_int64), p(C.c_int64), p(C.c_int32), p(C.c_int32),
                                    p(C.c_int32), p(C.c_int32), p(C.c_int32)]),
        "topo_comm_init_nccl": (C.c_int, [vp, vp]),
        "topo_element_stiffness": (C.c_int, [C.c_int, C.c_double, vp, vp]),
        "topo_generate": (None, [C.c_uint64, C.c_uint64, C.c_int, C.c_double, C.c_double,
                                 C.c_int64, C.c_int64, vp]),
        "topo_build_connectivity": (C.c_int, [vp, vp]),
        "topo_build_index_pairs": (C.c_int, [vp, vp, vp]),
        "topo_simp_interpolate": (C.c_int, [vp, vp, p(Simp), vp, vp]),
        "topo_assemble_values": (C.c_int, [vp, vp, vp]),
        "topo_sensitivity": (C.c_int, [vp, vp, vp, p(Simp), p(C.c_double), vp]),
        "topo_filter": (C.c_int, [vp, vp, vp, C.c_int]),
        "topo_filter_adjoint": (C.c_int, [vp, vp, vp]),
        "topo_project": (C.c_int, [vp, vp, C.c_double, C.c_double, vp]),
        "topo_project_derivative": (C.c_int, [vp, vp, C.c_double, C.c_double, vp]),
        "topo_backfilter": (C.c_int, [vp, vp, vp, C.c_double, C.c_double, C.c_int, vp]),
        "topo_solve_eta": (C.c_int, [vp, vp, C.c_double, C.c_double, p(C.c_double),
                                     p(C.c_int32)]),
        "topo_filter_taps": (C.c_int, [vp, vp, vp, vp, vp]),
        "topo_filter_hs": (C.c_int, [vp, vp]),
        "topo_lambda_upper": (C.c_int, [vp, C.c_int64, vp, vp, vp, C.c_double, C.c_int64,
                                        p(C.c_double)]),
        "topo_oc_candidate": (C.c_int, [vp, C.c_int64, vp, vp, vp, C.c_double, C.c_double, vp]),
        "topo_oc_bisect": (C.c_int, [vp, vp, vp, vp, p(OcParams), C.c_int, C.c_double,
                                     C.c_double, VOLUME_FN, vp, vp, p(C.c_double), p(C.c_int32),
                                     p(C.c_int32)]),
        "topo_design_pass": (C.c_int, [vp, vp, vp, p(PassParams), p(PassOut)]),
        "topo_design_pass_begin": (C.c_int, [vp, vp, vp, p(PassParams), p(PassOut)]),
        "topo_design_pass_end": (C.c_int, [vp, p(PassOut)]),
        "topo_last_launch_count": (C.c_int64, [vp]),
        "topo_set_timing": (C.c_int, [vp, C.c_int]),
        "topo_stage_times": (C.c_int, [vp, vp]),
        "topo_pass_graph_replays": (C.c_int, [vp, vp]),
        "topo_loop_records": (C.c_int, [vp, vp, vp, vp, vp]),
        "topo_anderson_step": (C.c_int, [vp, vp, vp, vp]),
        "topo_anderson_reset": (C.c_int, [vp]),
        "topo_fp64_peak": (C.c_int, [C.c_int, vp]),
        "topo_csc_pattern": (C.c_int, [vp, vp, vp, vp]),
        "topo_csc_values": (C.c_int, [vp, vp, vp]),
        "topo_csc_set_fixed": (C.c_int, [vp, vp, C.c_int64, vp]),
        "topo_oc_primal_dual": (C.c_int, [vp, vp, vp, vp, vp, C.c_double, vp, vp, vp, vp]),
        "topo_solve_state": (C.c_int, [vp, vp, vp, vp, C.c_int64, C.c_double, C.c_int32, vp, vp,
                                       vp]),
        "topo_solve_state_mg": (C.c_int, [vp, vp, vp, vp, C.c_int64, C.c_double, C.c_int32, vp,
                                          vp, vp]),
        "topo_apply_stiffness": (C.c_int, [vp, vp, vp, vp, C.c_int32]),
        "topo_device_alloc": (C.c_int, [vp, C.c_int64, vp]),
        "topo_device_free": (C.c_int, [vp, vp]),
        "topo_copy": (C.c_int, [vp, vp, vp, C.c_int64]),
        "topo_host_oc_replay": (C.c_int, [p(OcParams), C.c_double, SFUN, vp, C.c_int,
                                          p(C.c_double), p(C.c_int32), p(C.c_int32),
                                          p(C.c_double), p(C.c_int32)]),
        "topo_host_eta_replay": (C.c_int, [C.c_double, GFUN, vp, p(C.c_double), p(C.c_int32)]),
        "topo_nccl_unique_id": (C.c_int, [vp]),
        "topo_comm_init_host": (C.c_int, [vp, p(HostComm)]),
        "topo_slab_plan": (C.c_int, [p(GridDesc), vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L
