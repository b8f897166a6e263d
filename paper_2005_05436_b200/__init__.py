"""B200-native design-update hot path of top99neo / top3D125 (arXiv 2005.05436).

density filter -> volume-preserving Heaviside projection -> SIMP + lower-
triangle stiffness values -> compliance sensitivity from a supplied U ->
back-filter -> OC bisection update, as hand-written sm_100a CUDA behind the
C-ABI in include/topo_capi.h. See DESIGN.md.
"""
from . import _lib
from .api import (Context, CudaError, IndexOverflow, InvalidArgument, NonMonotone, OcParams,
                  PassResult, SimpParams, TopoError, UpdateResult, element_stiffness, fp64_peak,
                  generate, nccl_unique_id, partition_domain, slab_plan)
from .configs import CONFIGS, Config, make_inputs

BC_NEUMANN, BC_DIRICHLET = _lib.BC_NEUMANN, _lib.BC_DIRICHLET
VOL_CALLBACK, VOL_MEAN, VOL_PROJECTED, VOL_FILTERED = (_lib.VOL_CALLBACK, _lib.VOL_MEAN,
                                                      _lib.VOL_PROJECTED, _lib.VOL_FILTERED)

_lib.load()  # fail loudly at import if the native library is missing

__all__ = ["Context", "SimpParams", "OcParams", "PassResult", "UpdateResult", "TopoError",
           "InvalidArgument", "IndexOverflow", "NonMonotone", "CudaError", "element_stiffness",
           "generate", "partition_domain", "fp64_peak", "CONFIGS", "Config", "make_inputs", "BC_NEUMANN",
           "BC_DIRICHLET", "VOL_CALLBACK", "VOL_MEAN", "VOL_PROJECTED", "VOL_FILTERED"]
