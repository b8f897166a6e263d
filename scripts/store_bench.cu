// Store-stream microbenchmark behind K3b's design: how fast can
// an SM with a SMALL footprint (few warps, few registers, some shared memory)
// stream a contiguous FP64 array to HBM?
//   A: per-warp 1 KB `st.global.cs.v4.f64` stores (STG.256), W warps per SM
//   B: bulk (TMA engine) shared -> global copies of C-byte chunks, D in flight
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/_build/store_bench scripts/store_bench.cu
// Run:   scripts/_build/store_bench [GB]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      printf("%s: %s\n", #x, cudaGetErrorString(e_));                             \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

__device__ __forceinline__ void st256_cs(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}

// A: warp w writes 1 KB rows w, w + W, ... (U stores issued back to back)
template <int U>
__global__ void k_stg(double* out, long long rows, double s) {
  const int lane = threadIdx.x & 31;
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long W = ((long long)gridDim.x * blockDim.x) >> 5;
  const double a = s * lane, b = a + 1, c = a + 2, d = a + 3;
  for (long long r = w * U; r < rows; r += W * U) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r + u < rows) st256_cs(out + (r + u) * 128 + 4 * lane, a, b, c, d);
  }
}


// A2: warp w writes whole 76.8 KB groups (75 x 1 KB rows) w, w + W, ... like K3b
__global__ void k_stg_groups(double* out, long long groups, double s) {
  const int lane = threadIdx.x & 31;
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long W = ((long long)gridDim.x * blockDim.x) >> 5;
  const double a = s * lane, b = a + 1, c = a + 2, d = a + 3;
  for (long long g = w; g < groups; g += W) {
    double* o = out + g * 9600 + 4 * lane;
#pragma unroll 5
    for (int r = 0; r < 75; ++r) st256_cs(o + r * 128, a, b, c, d);
  }
}

// A3: cache-operator / eviction-policy variants of the per-warp contiguous stream
template <int V>
__device__ __forceinline__ void st256_v(double* p, double a, double b, double c, double d,
                                        unsigned long long pol) {
  if (V == 0)
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
  else if (V == 1)
    asm volatile("st.global.cg.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
  else if (V == 2)
    asm volatile("st.global.wt.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
  else if (V == 3)
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
  else if (V == 4)
    asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d), "l"(pol) : "memory");
  else {
    asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b) : "memory");
    asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p + 2), "d"(c), "d"(d) : "memory");
  }
}
template <int V, int POL>
__global__ void k_stg_policy(double* out, long long groups, double s) {
  const int lane = threadIdx.x & 31;
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long W = ((long long)gridDim.x * blockDim.x) >> 5;
  const double a = s * lane, b = a + 1, c = a + 2, d = a + 3;
  unsigned long long pol = 0;
  if (POL == 0) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (POL == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  if (POL == 2) asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol));
  if (POL == 3) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  for (long long g = w; g < groups; g += W) {
    double* o = out + g * 9600 + 4 * lane;
#pragma unroll 5
    for (int r = 0; r < 75; ++r) st256_v<V>(o + r * 128, a, b, c, d, pol);
  }
}
// A4: every SM writes one contiguous region of the buffer (its warps interleave 1 KB rows in it)
__global__ void k_stg_sm_region(double* out, long long rows_per_block, double s) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const double a = s * lane, b = a + 1, c = a + 2, d = a + 3;
  double* base = out + (long long)blockIdx.x * rows_per_block * 128 + 4 * lane;
  for (long long r = wib; r < rows_per_block; r += wpb) st256_cs(base + r * 128, a, b, c, d);
}

// A5: does the write rate depend on the data? (linear grid-stride sweep, 16 B per lane like a memset kernel)
__global__ void k_fill128(double2* out, long long n, double2 v, int vary) {
  const long long S = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += S) {
    double2 w = v;
    if (vary) { w.x = __longlong_as_double(i * 0x9E3779B97F4A7C15ull); w.y = __longlong_as_double(~i * 0xD1B54A32D192ED03ull); }
    out[i] = w;
  }
}

// A6: per-warp contiguous 76.8 KB groups with 128-bit stores (512 B per warp instruction)
__global__ void k_stg_groups128(double* out, long long groups, double s) {
  const int lane = threadIdx.x & 31;
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long W = ((long long)gridDim.x * blockDim.x) >> 5;
  const double a = s * lane, b = a + 1;
  for (long long g = w; g < groups; g += W) {
    double2* o = reinterpret_cast<double2*>(out + g * 9600) + lane;
#pragma unroll 10
    for (int r = 0; r < 150; ++r) o[r * 32] = make_double2(a, b);
  }
}
// A7: linear grid-stride sweep with 256-bit stores
__global__ void k_fill256(double* out, long long n4, double s) {
  const long long S = (long long)gridDim.x * blockDim.x;
  const double a = s * threadIdx.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += S)
    st256_cs(out + 4 * i, a, a + 1, a + 2, a + 3);
}

// A8: persistent grid, 76.8 KB groups claimed from a counter (dynamic balance)
__global__ void k_stg_groups_dyn(double* out, long long groups, double s, unsigned long long* ctr) {
  const int lane = threadIdx.x & 31;
  const double a = s * lane, b = a + 1, c = a + 2, d = a + 3;
  for (;;) {
    unsigned long long g = 0;
    if (lane == 0) g = atomicAdd(ctr, 1ull);
    g = __shfl_sync(0xffffffffu, g, 0);
    if ((long long)g >= groups) break;
    double* o = out + g * 9600 + 4 * lane;
#pragma unroll 5
    for (int r = 0; r < 75; ++r) st256_cs(o + r * 128, a, b, c, d);
  }
}
// A9: non-persistent: one group per warp, groups / 8 blocks (the block scheduler balances)
__global__ void k_stg_groups_np(double* out, long long groups, double s) {
  const int lane = threadIdx.x & 31;
  const long long g = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (g >= groups) return;
  const double a = s * lane, b = a + 1, c = a + 2, d = a + 3;
  double* o = out + g * 9600 + 4 * lane;
#pragma unroll 5
  for (int r = 0; r < 75; ++r) st256_cs(o + r * 128, a, b, c, d);
}
// B4: warp-private rings with 4800 B chunks, 76.8 KB groups claimed from a counter
template <int D>
__global__ void k_bulk_warp_dyn(double* out, long long groups, double s, unsigned long long* ctr) {
  extern __shared__ __align__(128) unsigned char ring[];
  constexpr int C = 4800;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* mine = ring + (size_t)wib * D * C;
  int stage = 0;
  for (;;) {
    unsigned long long g = 0;
    if (lane == 0) g = atomicAdd(ctr, 1ull);
    g = __shfl_sync(0xffffffffu, g, 0);
    if ((long long)g >= groups) break;
    for (int k = 0; k < 16; ++k) {
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(D - 1) : "memory");
      __syncwarp();
      double2* st = reinterpret_cast<double2*>(mine + (size_t)stage * C);
      const double v = s * double(g + k);
      for (int q = lane; q < C / 16; q += 32) st[q] = make_double2(v, v + 1.0);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(st);
        double* gp = out + g * 9600 + k * 600;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gp), "r"(sa), "n"(C) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      stage = stage + 1 == D ? 0 : stage + 1;
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// B: block fills a ring of D = DW + 1 stages of C bytes in shared memory; one
// thread issues cp.async.bulk shared -> global per stage and lets DW groups
// stay in flight. Chunks are assigned round-robin over blocks.
template <int DW>
__global__ void k_bulk2(double* out, long long chunks, int C, int D, double s) {
  extern __shared__ __align__(128) unsigned char ring[];
  const int T = blockDim.x;
  int it = 0;
  for (long long c = blockIdx.x; c < chunks; c += gridDim.x, ++it) {
    const int stage = it % D;
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(DW) : "memory");
    __syncthreads();
    double2* st = reinterpret_cast<double2*>(ring + (size_t)stage * C);
    const double v = s * double(c);
    for (int q = threadIdx.x; q < C / 16; q += T) st[q] = make_double2(v, v + 1.0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(st);
      double* g = out + c * (long long)(C / 8);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(sa),
                   "r"(C)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// B3: warp-private rings (no block barriers): each warp fills its own C-byte
// stage and lane 0 issues the copy; D stages per warp, D - 1 in flight.
template <int DW>
__global__ void k_bulk_warp(double* out, long long chunks, int C, double s) {
  extern __shared__ __align__(128) unsigned char ring[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const long long w = (long long)blockIdx.x * wpb + wib, W = (long long)gridDim.x * wpb;
  unsigned char* mine = ring + (size_t)wib * (DW + 1) * C;
  int it = 0;
  for (long long c = w; c < chunks; c += W, ++it) {
    const int stage = it % (DW + 1);
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(DW) : "memory");
    __syncwarp();
    double2* st = reinterpret_cast<double2*>(mine + (size_t)stage * C);
    const double v = s * double(c);
    for (int q = lane; q < C / 16; q += 32) st[q] = make_double2(v, v + 1.0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(st);
      double* g = out + c * (long long)(C / 8);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(sa),
                   "r"(C)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <class F>
double time_ms(F launch, int reps = 3) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  launch();
  CK(cudaDeviceSynchronize());
  double best = 1e30;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

int main(int argc, char** argv) {
  const double gb = argc > 1 ? atof(argv[1]) : 8.0;
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const long long bytes = (long long)(gb * 1e9) / 76800 * 76800;  // multiple of every chunk size
  double* out;
  CK(cudaMalloc(&out, bytes));
  printf("SMs %d, buffer %.2f GB\n", sms, bytes / 1e9);
  const long long rows = bytes / 1024;
  printf("A: STG.256 per-warp 1 KB stores (warps per SM, unroll -> TB/s)\n");
  for (int wps : {2, 4, 8, 12, 16, 24, 32, 48, 64}) {
    const int th = wps >= 8 ? 256 : wps * 32;
    const int nb = sms * wps * 32 / th;
    double t1 = time_ms([&] { k_stg<1><<<nb, th>>>(out, rows, 1.0); });
    double t4 = time_ms([&] { k_stg<4><<<nb, th>>>(out, rows, 1.0); });
    double t16 = time_ms([&] { k_stg<16><<<nb, th>>>(out, rows, 1.0); });
    printf("  warps/SM %2d: U1 %.3f  U4 %.3f  U16 %.3f TB/s\n", wps, bytes / t1 / 1e9,
           bytes / t4 / 1e9, bytes / t16 / 1e9);
  }
  printf("A2: STG.256, per-warp contiguous 76.8 KB groups (warps per SM -> TB/s)\n");
  for (int wps : {2, 4, 8, 16, 24, 40, 64}) {
    const int th = wps >= 8 ? 256 : wps * 32;
    const int nb = sms * wps * 32 / th;
    double t = time_ms([&] { k_stg_groups<<<nb, th>>>(out, bytes / 76800, 1.0); });
    printf("  warps/SM %2d: %.3f TB/s (%.3f ms)\n", wps, bytes / t / 1e9, t);
  }
  printf("A3: per-warp contiguous groups at 8 warps/SM, store variants -> TB/s\n");
  {
    const int nb = sms, th = 256;
    const long long groups = bytes / 76800;
    printf("  st.global        : %.3f\n", bytes / time_ms([&] { k_stg_policy<0, 9><<<nb, th>>>(out, groups, 1.0); }) / 1e9);
    printf("  st.global.cg     : %.3f\n", bytes / time_ms([&] { k_stg_policy<1, 9><<<nb, th>>>(out, groups, 1.0); }) / 1e9);
    printf("  st.global.wt     : %.3f\n", bytes / time_ms([&] { k_stg_policy<2, 9><<<nb, th>>>(out, groups, 1.0); }) / 1e9);
    printf("  st.global.cs     : %.3f\n", bytes / time_ms([&] { k_stg_policy<3, 9><<<nb, th>>>(out, groups, 1.0); }) / 1e9);
    printf("  hint evict_first : %.3f\n", bytes / time_ms([&] { k_stg_policy<4, 0><<<nb, th>>>(out, groups, 1.0); }) / 1e9);
    printf("  hint evict_last  : %.3f\n", bytes / time_ms([&] { k_stg_policy<4, 1><<<nb, th>>>(out, groups, 1.0); }) / 1e9);
    printf("  hint unchanged   : %.3f\n", bytes / time_ms([&] { k_stg_policy<4, 2><<<nb, th>>>(out, groups, 1.0); }) / 1e9);
    printf("  hint evict_normal: %.3f\n", bytes / time_ms([&] { k_stg_policy<4, 3><<<nb, th>>>(out, groups, 1.0); }) / 1e9);
    printf("  2 x st.v2.f64    : %.3f\n", bytes / time_ms([&] { k_stg_policy<5, 9><<<nb, th>>>(out, groups, 1.0); }) / 1e9);
    const long long rpb = rows / sms;
    printf("  one region per SM: %.3f\n", rpb * sms * 1024 / time_ms([&] { k_stg_sm_region<<<sms, 256>>>(out, rpb, 1.0); }) / 1e9);
    for (int val : {0, 0x5A}) {
      double t = time_ms([&] { CK(cudaMemsetAsync(out, val, bytes)); });
      printf("  cudaMemset(0x%02x)  : %.3f\n", val, bytes / t / 1e9);
    }
    for (int vary : {0, 1})
      for (int bps : {8, 16, 32}) {
        double t = time_ms([&] { k_fill128<<<sms * bps, 256>>>((double2*)out, bytes / 16, make_double2(0.0, 0.0), vary); });
        printf("  k_fill128 vary %d, %2d blocks/SM: %.3f\n", vary, bps, bytes / t / 1e9);
      }
    {
      double t = time_ms([&] { k_fill128<<<sms * 16, 256>>>((double2*)out, bytes / 16, make_double2(1.5, -2.25), 0); });
      printf("  k_fill128 constant (1.5, -2.25): %.3f\n", bytes / t / 1e9);
    }
    for (int wps : {8, 16, 32, 64}) {
      double t = time_ms([&] { k_stg_groups128<<<sms * wps / 8, 256>>>(out, bytes / 76800, 1.0); });
      printf("  groups, 128-bit stores, %2d warps/SM: %.3f\n", wps, bytes / t / 1e9);
    }
    for (int bps : {8, 16, 32}) {
      double t = time_ms([&] { k_fill256<<<sms * bps, 256>>>(out, bytes / 32, 1.0); });
      printf("  k_fill256 (linear sweep), %2d blocks/SM: %.3f\n", bps, bytes / t / 1e9);
    }
    for (int bps : {9, 10, 12, 24, 64}) {
      double t = time_ms([&] { k_fill256<<<sms * bps, 256>>>(out, bytes / 32, 1.0); });
      printf("  k_fill256 (linear sweep), %2d blocks/SM: %.3f\n", bps, bytes / t / 1e9);
    }
    unsigned long long* ctr;
    CK(cudaMalloc(&ctr, 8));
    for (int wps : {4, 8, 16, 32, 64}) {
      const int th = wps >= 8 ? 256 : wps * 32;
      double t = time_ms([&] { CK(cudaMemsetAsync(ctr, 0, 8)); k_stg_groups_dyn<<<sms * wps * 32 / th, th>>>(out, bytes / 76800, 1.0, ctr); });
      printf("  groups claimed dynamically, %2d warps/SM: %.3f\n", wps, bytes / t / 1e9);
    }
    for (int th : {64, 128, 256}) {
      const long long groups = bytes / 76800;
      double t = time_ms([&] { k_stg_groups_np<<<(unsigned)((groups * 32 + th - 1) / th), th>>>(out, groups, 1.0); });
      printf("  non-persistent, one group per warp, %3d threads/block: %.3f\n", th, bytes / t / 1e9);
    }
    CK(cudaFuncSetAttribute(k_bulk_warp_dyn<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_bulk_warp_dyn<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    {
      double t = time_ms([&] { CK(cudaMemsetAsync(ctr, 0, 8)); k_bulk_warp_dyn<6><<<sms, 128, 4 * 6 * 4800>>>(out, bytes / 76800, 1.0, ctr); });
      printf("  bulk, warp rings 6 x 4800 B, 4 warps/SM, dynamic groups: %.3f\n", bytes / t / 1e9);
      t = time_ms([&] { CK(cudaMemsetAsync(ctr, 0, 8)); k_bulk_warp_dyn<3><<<sms, 256, 8 * 3 * 4800>>>(out, bytes / 76800, 1.0, ctr); });
      printf("  bulk, warp rings 3 x 4800 B, 8 warps/SM, dynamic groups: %.3f\n", bytes / t / 1e9);
      t = time_ms([&] { CK(cudaMemsetAsync(ctr, 0, 8)); k_bulk_warp_dyn<3><<<2 * sms, 128, 4 * 3 * 4800>>>(out, bytes / 76800, 1.0, ctr); });
      printf("  bulk, warp rings 3 x 4800 B, 2 x 4 warps/SM, dynamic groups: %.3f\n", bytes / t / 1e9);
    }
    CK(cudaMemset(out, 0, 1024));
    double tm = time_ms([&] { CK(cudaMemsetAsync(out, 0, bytes)); });
    printf("  cudaMemset       : %.3f\n", bytes / tm / 1e9);
  }
  CK(cudaFuncSetAttribute(k_bulk2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(k_bulk2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(k_bulk2<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(k_bulk_warp<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(k_bulk_warp<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  printf("B: block-wide bulk copies, 1 block per SM (threads, chunk bytes, stages -> TB/s)\n");
  for (int th : {128, 256})
    for (int C : {4800, 9600, 19200, 38400}) {
      const long long chunks = bytes / C;
      double r1 = 0, r2 = 0, r3 = 0;
      if (2 * C <= 200 * 1024)
        r1 = bytes / time_ms([&] { k_bulk2<1><<<sms, th, 2 * C>>>(out, chunks, C, 2, 1.0); }) / 1e9;
      if (3 * C <= 200 * 1024)
        r2 = bytes / time_ms([&] { k_bulk2<2><<<sms, th, 3 * C>>>(out, chunks, C, 3, 1.0); }) / 1e9;
      if (4 * C <= 200 * 1024)
        r3 = bytes / time_ms([&] { k_bulk2<3><<<sms, th, 4 * C>>>(out, chunks, C, 4, 1.0); }) / 1e9;
      printf("  T %3d C %5d: D2 %.3f  D3 %.3f  D4 %.3f TB/s\n", th, C, r1, r2, r3);
    }
  printf("B': same, 2 blocks per SM\n");
  for (int C : {9600, 19200}) {
    const long long chunks = bytes / C;
    double r2 = bytes / time_ms([&] { k_bulk2<2><<<2 * sms, 128, 3 * C>>>(out, chunks, C, 3, 1.0); }) / 1e9;
    printf("  T 128 C %5d D3: %.3f TB/s\n", C, r2);
  }
  printf("B3: warp-private rings, 1 block per SM (warps, chunk bytes, in flight per warp -> TB/s)\n");
  for (int wps : {4, 8})
    for (int C : {2400, 4800, 9600}) {
      const long long chunks = bytes / C;
      double r1 = 0, r2 = 0;
      if ((size_t)wps * 2 * C <= 200 * 1024)
        r1 = bytes / time_ms([&] { k_bulk_warp<1><<<sms, wps * 32, wps * 2 * C>>>(out, chunks, C, 1.0); }) / 1e9;
      if ((size_t)wps * 3 * C <= 200 * 1024)
        r2 = bytes / time_ms([&] { k_bulk_warp<2><<<sms, wps * 32, wps * 3 * C>>>(out, chunks, C, 1.0); }) / 1e9;
      printf("  warps %d C %5d: F1 %.3f  F2 %.3f TB/s\n", wps, C, r1, r2);
    }
  return 0;
}
