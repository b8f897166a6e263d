// Multi-GPU plumbing of the x-slab decomposition: halo
// exchange of filter inputs and allreduce of the scalar sums inside the eta
// and OC bisections. Implemented in capi.cu over NCCL (loaded with dlopen, so
// single-GPU use has no NCCL dependency).
#pragma once

#include "../../include/topo_capi.h"

struct topo_ctx;
struct Comm;

topo_status comm_halo(Comm* c, topo_ctx* ctx, double* storage, double* storage2 = nullptr);
topo_status comm_allreduce(Comm* c, topo_ctx* ctx, double* dev, int n);
topo_status comm_allreduce_host(Comm* c, topo_ctx* ctx, double* host, int n);
void comm_destroy(Comm* c);
