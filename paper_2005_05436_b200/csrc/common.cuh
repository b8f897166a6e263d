// Shared device helpers for the sm_100a design-update kernels.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

namespace topo {

namespace cg = cooperative_groups;

// Bounds checks of the checked build (-DTOPO_CHECKED, libtopo_b200_checked.so,
// tests/test_gpu_checked.py): a computed index outside its array traps the
// kernel with a message. compute-sanitizer is unavailable on the GPU pool, so
// these asserts on the computed (gather / scatter / mirror-folded) indices
// stand in for memcheck. No code in the default build.
#ifdef TOPO_CHECKED
#define TOPO_CHECK(cond)                                                             \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      printf("TOPO_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, \
             __LINE__, int(blockIdx.x), int(threadIdx.x));                           \
      __trap();                                                                      \
    }                                                                                \
  } while (0)
#else
#define TOPO_CHECK(cond) \
  do {                   \
  } while (0)
#endif

// std::max / std::min argument semantics (oc.hpp:36,49-51,59): the first
// argument wins unless the second compares strictly greater / smaller. CUDA's
// fmax/fmin differ on NaN, so they are not used on the OC path.
__host__ __device__ __forceinline__ double std_max(double a, double b) { return (a < b) ? b : a; }
__host__ __device__ __forceinline__ double std_min(double a, double b) { return (b < a) ? b : a; }

// half-sample mirror fold onto [0, n) (filter.hpp:43-48)
__host__ __device__ __forceinline__ int reflect_index(int t, int n) {
  const int period = 2 * n;
  t %= period;
  if (t < 0) t += period;
  return t < n ? t : period - 1 - t;
}

/// Geometry of one rank's x-slab. 2D grids run as 3D with nz = 1 and no z
/// taps, so element (i, k, j) has index (j * nz + k) * nely + i for both
/// (grid.hpp:42-45). "Owned" columns are [j0, j0 + jn); per-element arrays are
/// indexed from j0. Halo-extended arrays ("storage") cover global columns
/// [sj0, sj0 + sjn) and are indexed from sj0.
struct Geo {
  int nelx, nely, nelz;  // global; nelz == 0 for 2D
  int nz;                // max(nelz, 1)
  int is3d, dim, d, P;   // dim 2/3, DOFs per element, lower pairs per element
  int j0, jn;            // owned columns
  int sj0, sjn;          // stored columns of halo-extended arrays
  long long S;           // elements per x column = nely * nz
  long long m;           // owned elements = jn * S
  int bc;                // 0 Neumann (mirror), 1 Dirichlet (zero)
};

// Per-element state byte: 0 active, 1 passive solid, 2 passive void.
__device__ __forceinline__ int elem_state(const uint8_t* st, long long e) {
  return st ? int(st[e]) : 0;
}

// ---------------------------------------------------------------- reductions
// Deterministic: fixed shuffle tree inside a warp, fixed warp order in a block.
template <int N>
__device__ __forceinline__ void warp_sum(double (&v)[N]) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], off);
}

// Sums v over the block; the result is valid in thread 0 (and returned to
// every thread of warp 0). `scratch` needs N * 32 doubles.
template <int N>
__device__ __forceinline__ void block_sum(double (&v)[N], double* scratch) {
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int nthr = blockDim.x * blockDim.y * blockDim.z;
  const int lane = tid & 31, warp = tid >> 5, nw = (nthr + 31) >> 5;
  warp_sum<N>(v);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < N; ++q) scratch[q * 32 + warp] = v[q];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = lane < nw ? scratch[q * 32 + lane] : 0.0;
    warp_sum<N>(v);
  }
  __syncthreads();
}

// Fixed-order sum of p[start], p[start + step], ... (< n), read through L2
// (__ldcg: written by other blocks) with 8 loads in flight.
__device__ __forceinline__ double strided_sum_l2(const double* p, int n, int start, int step,
                                                 int elem_stride = 1, int comp = 0) {
  double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int i = start;
  for (; i + 7 * step < n; i += 8 * step)
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] += __ldcg(p + (long long)(i + u * step) * elem_stride + comp);
  for (int u = 0; i < n; i += step, ++u) a[u] += __ldcg(p + (long long)i * elem_stride + comp);
  return ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
}

// Sum `count` partial records of stride `stride` (component q at p[i*stride+q])
// with one warp, in a fixed order; every lane of the calling warp gets the
// totals. Used identically by every block of a cooperative kernel so that all
// blocks take the same control decisions.
template <int N>
__device__ __forceinline__ void warp_sum_partials(const double* p, int count, int stride,
                                                  double (&out)[N]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < N; ++q) out[q] = strided_sum_l2(p, count, lane, 32, stride, q);
  warp_sum<N>(out);
}

}  // namespace topo
