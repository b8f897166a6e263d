// sm_100a kernels of the design-update pass (SURVEY.md §2 "Kernels": K0-K7).
// All FP64. Memory-bound streams use 16-byte vector stores with the
// streaming (.cs) hint; stencils stage halo tiles in shared memory; scalar
// reductions are deterministic (fixed warp/block/grid trees).
#pragma once

#include "common.cuh"
#include "control.h"

namespace topo {

constexpr int kThreads = 256;

// ============================================================================
// K0: element DOFs and lower-triangle index pairs (grid.hpp:89-153)
// ============================================================================

// DOFs of element (i, k, j) in the node order of grid.hpp:105-107 / :118-122.
// `jbase` shifts global node columns for slab-local U indexing (0 = global).
__device__ __forceinline__ void element_dofs(const Geo& G, int i, int k, int j, int jbase,
                                             int* dofs) {
  const long long ny1 = G.nely + 1;
  if (!G.is3d) {
    const int jj = j - jbase;
    const int n0 = int((long long)jj * ny1 + i + 1), n1 = int((long long)(jj + 1) * ny1 + i + 1);
    const int n2 = int((long long)(jj + 1) * ny1 + i), n3 = int((long long)jj * ny1 + i);
    const int nodes[4] = {n0, n1, n2, n3};
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      dofs[2 * a] = 2 * nodes[a];
      dofs[2 * a + 1] = 2 * nodes[a] + 1;
    }
  } else {
    const long long nz1 = G.nelz + 1;
    const int jj = j - jbase;
    auto node = [&](int ii, int kk, int jc) { return int(((long long)jc * nz1 + kk) * ny1 + ii); };
    const int nodes[8] = {node(i + 1, k, jj),     node(i + 1, k, jj + 1),
                          node(i, k, jj + 1),     node(i, k, jj),
                          node(i + 1, k + 1, jj), node(i + 1, k + 1, jj + 1),
                          node(i, k + 1, jj + 1), node(i, k + 1, jj)};
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      dofs[3 * a] = 3 * nodes[a];
      dofs[3 * a + 1] = 3 * nodes[a] + 1;
      dofs[3 * a + 2] = 3 * nodes[a] + 2;
    }
  }
}

__device__ __forceinline__ void elem_ijk(const Geo& G, long long e, int& i, int& k, int& j) {
  if (e <= 0xffffffffLL) {  // 32-bit division (all owned slabs below 2^32 elements)
    const unsigned u = unsigned(e), ny = unsigned(G.nely), nz = unsigned(G.nz);
    const unsigned r = u / ny;
    i = int(u - r * ny);
    const unsigned jj = r / nz;
    k = int(r - jj * nz);
    j = G.j0 + int(jj);
    return;
  }
  i = int(e % G.nely);
  const long long r = e / G.nely;
  k = int(r % G.nz);
  j = G.j0 + int(r / G.nz);
}

template <int D>
__global__ void __launch_bounds__(kThreads) k_connectivity(Geo G, int* __restrict__ dofs) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < G.m;
       e += (long long)gridDim.x * blockDim.x) {
    int i, k, j;
    elem_ijk(G, e, i, k, j);
    int d[24];
    element_dofs(G, i, k, j, 0, d);
#pragma unroll
    for (int a = 0; a < D; ++a) dofs[e * D + a] = d[a];
  }
}

// One block stages EB elements' DOFs in smem, then streams iK/jK as int4
// vectors (P is a multiple of 4 for Q4 and H8).
template <int D, int EB>
__global__ void __launch_bounds__(kThreads) k_index_pairs(Geo G, int* __restrict__ iK,
                                                          int* __restrict__ jK) {
  constexpr int P = D * (D + 1) / 2;
  constexpr int PV = P / 4;
  __shared__ int sd[EB][D];
  __shared__ unsigned char sil[P], sjl[P];
  for (int q = threadIdx.x; q < P; q += blockDim.x) {  // grid.hpp:143-144 pair order
    int t = q, jl = 0;
    while (t >= D - jl) {
      t -= D - jl;
      ++jl;
    }
    sil[q] = (unsigned char)(jl + t);
    sjl[q] = (unsigned char)jl;
  }
  const long long nchunks = (G.m + EB - 1) / EB;
  for (long long c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const long long e0 = c * EB;
    const int ne = int(min((long long)EB, G.m - e0));
    __syncthreads();
    for (int t = threadIdx.x; t < ne; t += blockDim.x) {
      int i, k, j;
      elem_ijk(G, e0 + t, i, k, j);
      int d[24];
      element_dofs(G, i, k, j, 0, d);
#pragma unroll
      for (int a = 0; a < D; ++a) sd[t][a] = d[a];
    }
    __syncthreads();
    const int nv = ne * PV;
    int4* oi = reinterpret_cast<int4*>(iK + e0 * P);
    int4* oj = reinterpret_cast<int4*>(jK + e0 * P);
    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
      const int el = v / PV, q0 = (v - el * PV) * 4;
      int a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int x = sd[el][sil[q0 + u]], y = sd[el][sjl[q0 + u]];
        a[u] = max(x, y);
        b[u] = min(x, y);
      }
      __stcs(oi + v, make_int4(a[0], a[1], a[2], a[3]));
      __stcs(oj + v, make_int4(b[0], b[1], b[2], b[3]));
    }
  }
}

// ============================================================================
// K1 / K4 / K7: cone convolution (filter.hpp:50-91) with smem halo tiles
// ============================================================================

enum ConvMode {
  CONV_PLAIN = 0,   // out = conv(in)                         (hs, adjoint of pre-divided input)
  CONV_FWD = 1,     // out = conv(in) / hs, optional pin      (apply_filter + pin_passives)
  CONV_ADJ_DIV = 3, // out = conv(in / hs)                    (apply_filter_adjoint)
  CONV_ADJ2_OC = 4  // dc, dV = conv(a1), conv(a2) + OC record + (sum ocP, V(0), V(inf)) partials
};

struct ConvArgs {
  const double* in0;  // storage-indexed (halo-extended) inputs
  const double* in1;
  const double* ihs;  // owned-indexed 1 / hs (CONV_FWD: xTilde = (H x) * ihs)
  const double* hs_st;  // storage-indexed hs (CONV_ADJ_DIV)
  double* out0;       // owned-indexed outputs
  double* out1;
  const uint8_t* state;
  int pin;
  double* partials;  // per block (CONV_ADJ2_OC)
  // CONV_ADJ2_OC
  const double* x;   // design (owned)
  const double* cw;  // volume weights (owned)
  double move;
  double* ocp;       // ocP per element, -1 for passives (OcRecs)
};

// eta terms are evaluated through E1 = exp(2 b t) (K2 below):
//   tanh(b (t - c)) = (E - 1) / (E + 1),  E = E1 exp(-2 b c)
//   sinh(b t) sinh(b (1 - t)) = cosh(b) / 2 - (E1 e^-b + e^b / E1) / 4
// (exact identities; rounding differs from the reference's tanh / cosh /
// sinh expression at the 1e-16 level, and eta parity is judged by the
// conditioned protocol of SURVEY.md §8(c)).

// Candidate record of oc.hpp:44-61 for one element; passives get lb = ub = x,
// which makes every candidate equal x (their xNew entries stay untouched).
__device__ __forceinline__ double4 oc_record(double x, double dc, double dV, double cw, double move,
                                             bool active) {
  if (!active) return make_double4(x, x, 0.0, cw);
  const double ocP = x * sqrt(std_max(0.0, -dc / dV));
  return make_double4(std_max(0.0, x - move), std_min(1.0, x + move), ocP, cw);
}
// The OC record (lb, ub, ocP, cw) of an element, stored as ocP only: lb and ub
// follow from the design x (oc.hpp:55-56), cw is the volume-weight field
// (null: 1), and ocP = -1 marks passives (lb = ub = x, candidate x).
struct OcRecs {
  const double* x;
  const double* ocp;
  const double* cw;
  double move;
  __device__ __forceinline__ double4 get(long long e) const {
    const double xv = x[e], p = ocp[e], w = cw ? cw[e] : 1.0;
    if (p < 0.0) return make_double4(xv, xv, 0.0, w);
    return make_double4(std_max(0.0, xv - move), std_min(1.0, xv + move), p, w);
  }
};

// oc.hpp:47-51
__device__ __forceinline__ double oc_cand(const double4& r, double s) {
  const double f = s > 0 ? r.z / s : (r.z > 0 ? INFINITY : 0.0);
  return std_min(std_max(f, r.x), r.y);
}
// the same candidate with ocP / s taken as ocP * (1 / s) (inv_s = 1 / s for
// s > 0, else +inf): within one ulp of the division, used only inside the
// volume sums of the speculative batches (the written xNew uses oc_cand)
__device__ __forceinline__ double oc_cand_rcp(const double4& r, double s, double inv_s) {
  const double f = s > 0 ? r.z * inv_s : (r.z > 0 ? INFINITY : 0.0);
  return std_min(std_max(f, r.x), r.y);
}

// Tile geometry of one conv launch. Lanes run along i (the fastest memory
// axis); each thread owns R consecutive outputs along the "run" axis (k in 3D,
// j in 2D) so that every tile value it loads feeds up to R accumulators.
// Taps are grouped in columns (fixed di and other-axis offset) whose run
// offsets form the symmetric interval [-a, a]; column weights are zero-padded
// to a multiple of R (zero-weight FMAs leave the sums unchanged). The cone is
// even in di and in the other offset, so mirrored columns share weights: only
// canonical columns (di >= 0, other >= 0) are stored, and the values of their
// 1, 2 or 4 mirrors are summed before the weights are applied.
struct ConvGeom {
  int WI, WR, WO;      // warps along i / run / other
  int TI, TR, TO;      // outputs per tile along i / run / other
  int EI, ER, EO;      // shared-memory tile extents; ER is odd (run axis contiguous)
  int reach, reach_o;  // halo along i and run / along other (0 in 2D)
  int run_n, other_n;  // owned extents of the run / other axes
  int ncol[3];         // canonical columns with 4, 2, 1 mirrors (stored in that order)
  int zb;              // k_conv3: first tile along other of this launch (chunked grids)
  unsigned magicEI;    // floor(2^32 / EI) + 1: q / EI == umulhi(q, magicEI) for q < 2^20
};

struct ConvCol {  // one canonical column of the cone stencil
  int di, dother, a, woff;
};

// accumulate the columns [c0, c1), each with NM mirrors, into acc
// Shared-memory layout [other][i][run] with the run axis contiguous: the
// values of a column are consecutive words (immediate-offset LDS), and lanes
// (consecutive i) are ER words apart, ER odd, so 64-bit accesses are
// bank-conflict free.
template <int NM, int R>
__device__ __forceinline__ void conv_columns(const double* __restrict__ tile, int sb, int sI,
                                             int sPlane, const ConvCol* __restrict__ cols, int c0,
                                             int c1, const double* __restrict__ wts,
                                             double (&acc)[R]) {
  if (c0 >= c1) return;
  // the column record and the weights of the next chunk are loaded while the
  // current chunk's FMAs run (they are global loads: exposed, they were the
  // top stall of the large-reach 2D filter)
  ConvCol col = cols[c0];
  double2 wn[R / 2];
  {
    const double2* w2 = reinterpret_cast<const double2*>(wts + col.woff);
#pragma unroll
    for (int t = 0; t < R / 2; ++t) wn[t] = __ldg(w2 + t);
  }
  for (int c = c0; c < c1; ++c) {
    const ConvCol ncol = c + 1 < c1 ? cols[c + 1] : col;
    const int base = sb - col.a;
    const int oi = col.di * sI, oo = col.dother * sPlane;
    const double* p0 = tile + base + oi + oo;
    const double* p1 = tile + base - oi - oo;  // NM == 2: the one nonzero offset flipped
    const double* p2 = tile + base - oi + oo;  // NM == 4
    const double* p3 = tile + base + oi - oo;
    auto colval = [&](int s) {
      const int o = s;
      double v = p0[o];
      if (NM == 2) v += p1[o];
      if (NM == 4) v = (v + p1[o]) + (p2[o] + p3[o]);
      return v;
    };
    const double2* w2 = reinterpret_cast<const double2*>(wts + col.woff);
    const double2* w2n = reinterpret_cast<const double2*>(wts + ncol.woff);
    const int nch = (2 * col.a + R) / R;  // ceil((2a + 1) / R)
    double v[2 * R - 1];
#pragma unroll
    for (int s = 0; s < R - 1; ++s) v[s] = colval(s);
    for (int ch = 0; ch < nch; ++ch) {
      double wv[R];
#pragma unroll
      for (int t = 0; t < R / 2; ++t) {
        wv[2 * t] = wn[t].x;
        wv[2 * t + 1] = wn[t].y;
      }
      const double2* wnext = ch + 1 < nch ? w2 + (ch + 1) * (R / 2) : w2n;
#pragma unroll
      for (int t = 0; t < R / 2; ++t) wn[t] = __ldg(wnext + t);
#pragma unroll
      for (int s = 0; s < R; ++s) v[R - 1 + s] = colval(ch * R + R - 1 + s);
#pragma unroll
      for (int t = 0; t < R; ++t)
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = fma(wv[t], v[r + t], acc[r]);
#pragma unroll
      for (int s = 0; s < R - 1; ++s) v[s] = v[R + s];
    }
    col = ncol;
  }
}

// Small-reach variant (compile-time half-width bound A): all R + 2A mirror-
// summed values of a column are loaded once into registers and every column
// applies 2A + 1 weights (zero outside its own [-a, a]; woff points at the
// centred, zero-padded 2A + 2 weights), fully unrolled.
template <int NM, int R, int A>
__device__ __forceinline__ void conv_columns_direct(const double* __restrict__ tile, int sb, int sI,
                                                    int sPlane, const ConvCol* __restrict__ cols,
                                                    int c0, int c1,
                                                    const double* __restrict__ wts,
                                                    double (&acc)[R]) {
  for (int c = c0; c < c1; ++c) {
    const ConvCol col = cols[c];
    const int base = sb - A;
    const int oi = col.di * sI, oo = col.dother * sPlane;
    const double* p0 = tile + base + oi + oo;
    const double* p1 = tile + base - oi - oo;
    const double* p2 = tile + base - oi + oo;
    const double* p3 = tile + base + oi - oo;
    double v[R + 2 * A];
#pragma unroll
    for (int q = 0; q < R + 2 * A; ++q) {
      double t = p0[q];
      if (NM == 2) t += p1[q];
      if (NM == 4) t = (t + p1[q]) + (p2[q] + p3[q]);
      v[q] = t;
    }
    const double2* w2 = reinterpret_cast<const double2*>(wts + col.woff);
    double w[2 * A + 2];
#pragma unroll
    for (int t = 0; t < A + 1; ++t) {
      const double2 ww = __ldg(w2 + t);
      w[2 * t] = ww.x;
      w[2 * t + 1] = ww.y;
    }
#pragma unroll
    for (int d = 0; d < 2 * A + 1; ++d)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = fma(w[d], v[r + d], acc[r]);
  }
}

// Shared by the conv kernels: per tile line (other, run) the source offset of
// its i = 0 element (-1: zero line) and its first smem word; per i the folded
// source i (-1: zero pad).
__device__ __forceinline__ void conv_tables(const Geo& G, const ConvGeom& T, const ConvArgs& A,
                                            int bi, int br, int bo, long long* lineSrc,
                                            int* lineDst, int* mapI) {
  const int tid = threadIdx.x, nlines = T.EO * T.ER, sPlane = T.EI * T.ER;
  auto fold = [&](int t, int n) {  // mirror (Neumann) or -1 outside (Dirichlet)
    if (t >= 0 && t < n) return t;
    return G.bc == 0 ? reflect_index(t, n) : -1;
  };
  for (int q = tid; q < T.EI; q += blockDim.x) {
    mapI[q] = fold(bi + q - T.reach, G.nely);
    TOPO_CHECK(mapI[q] >= -1 && mapI[q] < G.nely);
  }
  for (int line = tid; line < nlines; line += blockDim.x) {
    const int to = line / T.ER, tr = line - to * T.ER;
    int jo, jr;
    if (G.is3d) {
      jo = fold(G.j0 + bo + to - T.reach_o, G.nelx);
      jr = fold(br + tr - T.reach, G.nz);
    } else {
      jo = 0;
      jr = fold(G.j0 + br + tr - T.reach, G.nelx);
    }
    // -1: zero line (outside the domain, Dirichlet; or, with an input field,
    // a column this slab does not store: such values only meet zero-padded
    // weights or outputs beyond the tile, the slab setup guarantees every
    // real tap is stored). A null input is the all-ones field: any in-domain
    // line is valid (index 0 marks it).
    long long src = -1;
    const int jcol = G.is3d ? jo : jr;
    if (jo >= 0 && jr >= 0) {
      if (A.in0 == nullptr)
        src = 0;
      else if (jcol >= G.sj0 && jcol < G.sj0 + G.sjn)
        src = G.is3d ? ((long long)(jo - G.sj0) * G.nz + jr) * G.nely
                     : (long long)(jr - G.sj0) * G.nely;
    }
    TOPO_CHECK(src >= -1 && src + G.nely <= (long long)G.sjn * G.S);
    TOPO_CHECK(to * sPlane + tr < T.EI * T.ER * T.EO);
    lineSrc[line] = src;
    lineDst[line] = to * sPlane + tr;
  }
}

// tile load, flat over (line, i): coalesced along i; line = q / EI by a
// multiply-high with the host-computed magic (exact for q < 2^20)
template <int MODE>
__device__ __forceinline__ void conv_fill(const ConvGeom& T, const ConvArgs& A,
                                          const double* __restrict__ in, double* tile,
                                          const long long* lineSrc, const int* lineDst,
                                          const int* mapI) {
  const int tileN = T.EI * T.ER * T.EO, sI = T.ER;
  constexpr int U = 8;  // loads in flight per thread
  for (int q0 = threadIdx.x; q0 < tileN; q0 += U * blockDim.x) {
    double v[U];
    int dst[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = q0 + u * blockDim.x;
      v[u] = 0.0;
      dst[u] = -1;
      if (q < tileN) {
        const int line = int(__umulhi(unsigned(q), T.magicEI));
        const int ti = q - line * T.EI;
        const long long rb = lineSrc[line];
        const int ii = mapI[ti];
        dst[u] = lineDst[line] + ti * sI;
        if (rb >= 0 && ii >= 0) {
          const long long src = rb + ii;
          v[u] = in ? __ldg(in + src) : 1.0;  // null input: the all-ones field (hs)
          if (MODE == CONV_ADJ_DIV) v[u] = v[u] / __ldg(A.hs_st + src);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (dst[u] >= 0) tile[dst[u]] = v[u];
  }
}

// per-output epilogue: (v0, v1) = the filtered field(s) at element e
template <int NF, int MODE>
__device__ __forceinline__ void conv_store(const Geo& G, const ConvArgs& A, long long e, double v0,
                                           double v1, double (&red)[3]) {
  if (MODE == CONV_PLAIN || MODE == CONV_ADJ_DIV) {
    A.out0[e] = v0;
  } else if (MODE == CONV_FWD) {
    double v = v0 * A.ihs[e];  // filter.hpp:121 cwiseQuotient(hs), as a product with 1 / hs
    const int s = elem_state(A.state, e);
    if (A.pin && s == 1) v = 1.0;  // driver.hpp:130-133
    if (A.pin && s == 2) v = 0.0;
    A.out0[e] = v;
  } else if (MODE == CONV_ADJ2_OC) {
    const double dc = v0, dV = NF > 1 ? v1 : v0;
    if (A.out0) A.out0[e] = dc;
    if (A.out1) A.out1[e] = dV;
    const bool act = elem_state(A.state, e) == 0;
    const double4 rec = oc_record(A.x[e], dc, dV, A.cw ? A.cw[e] : 1.0, A.move, act);
    A.ocp[e] = act ? rec.z : -1.0;
    if (act) red[0] += rec.z;
    red[1] += rec.w * oc_cand(rec, 0.0);
    red[2] += rec.w * std_min(std_max(0.0, rec.x), rec.y);  // V(s -> inf)
  }
}

// conv_store with the per-element inputs already loaded: l0 = 1 / hs (FWD) or x
// (ADJ2_OC), l1 = cw (ADJ2_OC), st = element state
template <int NF, int MODE>
__device__ __forceinline__ void conv_store_pre(const ConvArgs& A, long long e, double v0, double v1,
                                               double l0, double l1, int st, double (&red)[3]) {
  if (MODE == CONV_PLAIN || MODE == CONV_ADJ_DIV) {
    A.out0[e] = v0;
  } else if (MODE == CONV_FWD) {
    double v = v0 * l0;  // filter.hpp:121 cwiseQuotient(hs); l0 = 1 / hs
    if (A.pin && st == 1) v = 1.0;  // driver.hpp:130-133
    if (A.pin && st == 2) v = 0.0;
    A.out0[e] = v;
  } else if (MODE == CONV_ADJ2_OC) {
    const double dc = v0, dV = NF > 1 ? v1 : v0;
    if (A.out0) A.out0[e] = dc;
    if (A.out1) A.out1[e] = dV;
    const bool act = st == 0;
    const double4 rec = oc_record(l0, dc, dV, l1, A.move, act);
    A.ocp[e] = act ? rec.z : -1.0;
    if (act) red[0] += rec.z;
    red[1] += rec.w * oc_cand(rec, 0.0);
    red[2] += rec.w * std_min(std_max(0.0, rec.x), rec.y);  // V(s -> inf)
  }
}

template <int MODE>
__device__ __forceinline__ void conv_partials(const ConvArgs& A, double (&red)[3], int zb = 0) {
  if (MODE == CONV_ADJ2_OC) {
    __shared__ double scratch[3 * 32];
    block_sum<3>(red, scratch);
    const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * (zb + blockIdx.z));
    if (threadIdx.x == 0) {
      A.partials[3 * b] = red[0];
      A.partials[3 * b + 1] = red[1];
      A.partials[3 * b + 2] = red[2];
    }
  }
}

template <int NF, int MODE, int R, int AW>
__global__ void __launch_bounds__(kThreads) k_conv(Geo G, ConvGeom T, const ConvCol* __restrict__ cols,
                                                   int ncols, const double* __restrict__ wts,
                                                   ConvArgs A) {
  extern __shared__ double tile[];
  const int tileN = T.EI * T.ER * T.EO, nlines = T.EO * T.ER;
  long long* lineSrc = reinterpret_cast<long long*>(tile + tileN);
  int* lineDst = reinterpret_cast<int*>(lineSrc + nlines);
  int* mapI = lineDst + nlines;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wi = warp % T.WI, wr = (warp / T.WI) % T.WR, wo = warp / (T.WI * T.WR);
  const int bi = blockIdx.x * T.TI, br = blockIdx.y * T.TR, bo = blockIdx.z * T.TO;
  const int sI = T.ER, sPlane = T.EI * T.ER;
  // thread base: its first output (r = 0) in tile coordinates
  const int sb = (wo + T.reach_o) * sPlane + (wi * 32 + lane + T.reach) * sI + (wr * R + T.reach);
  conv_tables(G, T, A, bi, br, bo, lineSrc, lineDst, mapI);
  __syncthreads();

  double acc[NF][R];
#pragma unroll
  for (int f = 0; f < NF; ++f)
#pragma unroll
    for (int r = 0; r < R; ++r) acc[f][r] = 0.0;

#pragma unroll
  for (int f = 0; f < NF; ++f) {
    if (f > 0) __syncthreads();
    conv_fill<MODE>(T, A, f == 0 ? A.in0 : A.in1, tile, lineSrc, lineDst, mapI);
    __syncthreads();
    if (AW > 0) {
      conv_columns_direct<4, R, AW>(tile, sb, sI, sPlane, cols, 0, T.ncol[0], wts, acc[f]);
      conv_columns_direct<2, R, AW>(tile, sb, sI, sPlane, cols, T.ncol[0], T.ncol[0] + T.ncol[1],
                                    wts, acc[f]);
      conv_columns_direct<1, R, AW>(tile, sb, sI, sPlane, cols, T.ncol[0] + T.ncol[1], ncols, wts,
                                   acc[f]);
    } else {
      conv_columns<4, R>(tile, sb, sI, sPlane, cols, 0, T.ncol[0], wts, acc[f]);
      conv_columns<2, R>(tile, sb, sI, sPlane, cols, T.ncol[0], T.ncol[0] + T.ncol[1], wts,
                         acc[f]);
      conv_columns<1, R>(tile, sb, sI, sPlane, cols, T.ncol[0] + T.ncol[1], ncols, wts, acc[f]);
    }
  }

  double red[3] = {0.0, 0.0, 0.0};
  const int gi = bi + wi * 32 + lane, go = bo + wo;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int grun = br + wr * R + r;
    if (gi >= G.nely || grun >= T.run_n || go >= T.other_n) continue;
    const long long e = ((long long)go * T.run_n + grun) * G.nely + gi;
    conv_store<NF, MODE>(G, A, e, acc[0][r], acc[NF - 1][r], red);
  }
  conv_partials<MODE>(A, red);
}

// 3D small reach (half-width AR <= 4), register-blocked: every thread owns an
// RB (run) x TB (other) block of outputs at one i. Taps are folded over +-di
// only (mirror pairs along i share the weight), so each tile row of the
// thread's (TB + 2 AR)-row window is loaded once and reused by all TB output
// rows it reaches: ~(2AR+1)(TB+2AR)(RB+2AR)/(RB TB) shared loads per output
// instead of ~(#columns)(R+2AR)/R. Weights w3[di][|do|][|dr|] (zero outside
// the cone) are uniform loads.
// Cone weights of k_conv3, passed BY VALUE as a kernel parameter: with di,
// |do| and |dr| compile-time (fully unrolled loops, 2 x 2 outputs per
// thread) every weight is a constant-bank operand of its DFMA and takes no
// register (C4 adjoint filter 0.035 vs 0.050 ms).
// w[di][|do|][|dr|] (zero outside the cone); hw[di][|do|] = largest |dr| with
// a nonzero weight (-1: none).
struct ConvW3 {
  double w[5 * 5 * 5];
  int hw[5 * 5];
};

template <int AR, int RB, int TB, bool FOLD, int DI>
__device__ __forceinline__ void conv3_di(const double* __restrict__ base, int sI, int sPlane,
                                         const ConvW3& W, double (&acc)[TB][RB]) {
  constexpr int NW = AR + 1;
  const double* p = base + DI * sI;
  const double* q = base - DI * sI;
#pragma unroll
  for (int kk = 0; kk < TB + 2 * AR; ++kk) {
    double v[RB + 2 * AR];
#pragma unroll
    for (int j = 0; j < RB + 2 * AR; ++j)
      v[j] = FOLD ? p[kk * sPlane + j] + q[kk * sPlane + j] : p[kk * sPlane + j];
    // taps outside the cone (zero weight) skipped by uniform branches on the
    // column's half-width hw (its weights vanish beyond it); the +-dr pair
    // shares its weight, so it is pre-added once per row and feeds every
    // output row t it reaches: one FMA per pair, and consecutive FMAs go to
    // different accumulators (no back-to-back dependency)
#pragma unroll
    for (int t = 0; t < TB; ++t) {
      const int dO = kk - t - AR;
      if (dO < -AR || dO > AR) continue;
      const int ao = dO < 0 ? -dO : dO;
      if (W.hw[DI * NW + ao] < 0) continue;
#pragma unroll
      for (int r = 0; r < RB; ++r) acc[t][r] = fma(W.w[(DI * NW + ao) * NW], v[r + AR], acc[t][r]);
    }
#pragma unroll
    for (int ad = 1; ad <= AR; ++ad) {
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const double pr = v[r + AR - ad] + v[r + AR + ad];
#pragma unroll
        for (int t = 0; t < TB; ++t) {
          const int dO = kk - t - AR;
          if (dO < -AR || dO > AR) continue;
          const int ao = dO < 0 ? -dO : dO;
          if (W.hw[DI * NW + ao] >= ad)
            acc[t][r] = fma(W.w[(DI * NW + ao) * NW + ad], pr, acc[t][r]);
        }
      }
    }
  }
}

// 4 x 4 outputs per thread (large grids): the weights of the di slice in
// registers and the +-dr taps as two FMAs (measured: the pre-added form
// below spills at this block size, C5 K1 0.44 vs 0.36 ms)
template <int AR, int RB, int TB, bool FOLD>
__device__ __forceinline__ void conv3_di_rw(const double* __restrict__ base, int di, int sI,
                                            int sPlane, const ConvW3& W,
                                         double (&acc)[TB][RB]) {
  constexpr int NW = AR + 1;
  double w[NW][NW];
#pragma unroll
  for (int a = 0; a < NW; ++a)
#pragma unroll
    for (int b = 0; b < NW; ++b) w[a][b] = W.w[(di * NW + a) * NW + b];
  int hw[NW];  // largest |dr| with a nonzero weight at (di, |do|), -1: none
#pragma unroll
  for (int a = 0; a < NW; ++a) {
    hw[a] = -1;
#pragma unroll
    for (int b = 0; b < NW; ++b)
      if (w[a][b] != 0.0) hw[a] = b;
  }
  const double* p = base + di * sI;
  const double* q = base - di * sI;
#pragma unroll
  for (int kk = 0; kk < TB + 2 * AR; ++kk) {
    double v[RB + 2 * AR];
#pragma unroll
    for (int j = 0; j < RB + 2 * AR; ++j)
      v[j] = FOLD ? p[kk * sPlane + j] + q[kk * sPlane + j] : p[kk * sPlane + j];
#pragma unroll
    for (int t = 0; t < TB; ++t) {
      const int dO = kk - t - AR;
      if (dO < -AR || dO > AR) continue;
      const int ao = dO < 0 ? -dO : dO;
      // taps outside the cone (zero weight) skipped by uniform branches on the
      // column's half-width hw[ao] (its weights vanish beyond it)
      const int hwa = hw[ao];
      if (hwa < 0) continue;
#pragma unroll
      for (int r = 0; r < RB; ++r) acc[t][r] = fma(w[ao][0], v[r + AR], acc[t][r]);
#pragma unroll
      for (int ad = 1; ad <= AR; ++ad) {
        if (hwa < ad) break;
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          acc[t][r] = fma(w[ao][ad], v[r + AR - ad], acc[t][r]);
          acc[t][r] = fma(w[ao][ad], v[r + AR + ad], acc[t][r]);
        }
      }
    }
  }
}

// Compile-time cone (R2 >= 0: the taps are exactly di^2 + do^2 + dr^2 <= R2,
// checked on the host from the weights): every loop bound, skip and weight
// index is a constant, so there are no branches, the weights are constant-bank
// DFMA operands, and the +-dr pair of a row is pre-added once for all output
// rows it feeds. C5 (rmin 4: AR 3, R2 14): 87 FMA + 49 DADD per output
// against 148 + 19 with the runtime-shaped loop.
__host__ __device__ constexpr int isqrt_c(int n) {
  int r = 0;
  while ((r + 1) * (r + 1) <= n) ++r;
  return r;
}
__host__ __device__ constexpr int cone_hw(int R2, int AR, int di, int ao) {
  return di * di + ao * ao > R2 ? -1 : (isqrt_c(R2 - di * di - ao * ao) < AR ? isqrt_c(R2 - di * di - ao * ao) : AR);
}

template <int AR, int R2, int RB, int TB, int DI>
__device__ __forceinline__ void conv3_cone_di(const double* __restrict__ base, int sI, int sPlane,
                                              const ConvW3& W, double (&acc)[TB][RB]) {
  constexpr int NW = AR + 1;
  const double* p = base + DI * sI;
  const double* q = base - DI * sI;
#pragma unroll
  for (int kk = 0; kk < TB + 2 * AR; ++kk) {
    // rows of this slice that reach no output row (all |do| out of the cone) are skipped
    bool any = false;
#pragma unroll
    for (int t = 0; t < TB; ++t) {
      const int dO = kk - t - AR;
      const int ao = dO < 0 ? -dO : dO;
      if (ao <= AR && cone_hw(R2, AR, DI, ao) >= 0) any = true;
    }
    if (!any) continue;
    double v[RB + 2 * AR];
#pragma unroll
    for (int j = 0; j < RB + 2 * AR; ++j)
      v[j] = DI > 0 ? p[kk * sPlane + j] + q[kk * sPlane + j] : p[kk * sPlane + j];
#pragma unroll
    for (int t = 0; t < TB; ++t) {
      const int dO = kk - t - AR;
      const int ao = dO < 0 ? -dO : dO;
      if (ao > AR || cone_hw(R2, AR, DI, ao) < 0) continue;
#pragma unroll
      for (int r = 0; r < RB; ++r) acc[t][r] = fma(W.w[(DI * NW + ao) * NW], v[r + AR], acc[t][r]);
    }
#pragma unroll
    for (int ad = 1; ad <= AR; ++ad) {
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const double pr = v[r + AR - ad] + v[r + AR + ad];
#pragma unroll
        for (int t = 0; t < TB; ++t) {
          const int dO = kk - t - AR;
          const int ao = dO < 0 ? -dO : dO;
          if (ao > AR || cone_hw(R2, AR, DI, ao) < ad) continue;
          acc[t][r] = fma(W.w[(DI * NW + ao) * NW + ad], pr, acc[t][r]);
        }
      }
    }
  }
}

template <int AR, int R2, int RB, int TB>
__device__ __forceinline__ void conv3_all(const double* __restrict__ base, int sI, int sPlane,
                                          const ConvW3& W, double (&acc)[TB][RB]) {
  if (R2 >= 0) {
    conv3_cone_di<AR, R2, RB, TB, 0>(base, sI, sPlane, W, acc);
    if (AR >= 1) conv3_cone_di<AR, R2, RB, TB, AR >= 1 ? 1 : 0>(base, sI, sPlane, W, acc);
    if (AR >= 2) conv3_cone_di<AR, R2, RB, TB, AR >= 2 ? 2 : 0>(base, sI, sPlane, W, acc);
    if (AR >= 3) conv3_cone_di<AR, R2, RB, TB, AR >= 3 ? 3 : 0>(base, sI, sPlane, W, acc);
    if (AR >= 4) conv3_cone_di<AR, R2, RB, TB, AR >= 4 ? 4 : 0>(base, sI, sPlane, W, acc);
    return;
  }
  if (RB * TB >= 16) {
    conv3_di_rw<AR, RB, TB, false>(base, 0, sI, sPlane, W, acc);
#pragma unroll 1
    for (int di = 1; di <= AR; ++di) conv3_di_rw<AR, RB, TB, true>(base, di, sI, sPlane, W, acc);
    return;
  }
  conv3_di<AR, RB, TB, false, 0>(base, sI, sPlane, W, acc);
  if (AR >= 1) conv3_di<AR, RB, TB, true, AR >= 1 ? 1 : 0>(base, sI, sPlane, W, acc);
  if (AR >= 2) conv3_di<AR, RB, TB, true, AR >= 2 ? 2 : 0>(base, sI, sPlane, W, acc);
  if (AR >= 3) conv3_di<AR, RB, TB, true, AR >= 3 ? 3 : 0>(base, sI, sPlane, W, acc);
  if (AR >= 4) conv3_di<AR, RB, TB, true, AR >= 4 ? 4 : 0>(base, sI, sPlane, W, acc);
}

template <int NF, int MODE, int AR, int RB, int TB, int R2>
__global__ void __launch_bounds__(kThreads, 2) k_conv3(Geo G, ConvGeom T, const __grid_constant__ ConvW3 W,
                                                       ConvArgs A) {
  extern __shared__ double tile[];
  const int tileN = T.EI * T.ER * T.EO, nlines = T.EO * T.ER;
  long long* lineSrc = reinterpret_cast<long long*>(tile + tileN);
  int* lineDst = reinterpret_cast<int*>(lineSrc + nlines);
  int* mapI = lineDst + nlines;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wr = warp % T.WR, wo = warp / T.WR;  // one warp along i
  const int bi = blockIdx.x * 32, br = blockIdx.y * T.TR, bo = (T.zb + blockIdx.z) * T.TO;
  const int sI = T.ER, sPlane = T.EI * T.ER;
  // window origin: tile row wo*TB (halo included), i = lane + AR, run wr*RB
  const int sb0 = (wo * TB) * sPlane + (lane + AR) * sI + wr * RB;
  conv_tables(G, T, A, bi, br, bo, lineSrc, lineDst, mapI);
  __syncthreads();
  double red[3] = {0.0, 0.0, 0.0};
  double keep[TB][RB];  // field 0 while field 1 accumulates (NF == 2)
  const int gi = bi + lane;
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    if (f > 0) __syncthreads();
    conv_fill<MODE>(T, A, f == 0 ? A.in0 : A.in1, tile, lineSrc, lineDst, mapI);
    __syncthreads();
    double acc[TB][RB];
#pragma unroll
    for (int t = 0; t < TB; ++t)
#pragma unroll
      for (int r = 0; r < RB; ++r) acc[t][r] = 0.0;
    conv3_all<AR, R2, RB, TB>(tile + sb0, sI, sPlane, W, acc);
    if (f + 1 < NF) {
#pragma unroll
      for (int t = 0; t < TB; ++t)
#pragma unroll
        for (int r = 0; r < RB; ++r) keep[t][r] = acc[t][r];
      continue;
    }
    if (MODE != CONV_FWD) {  // (measured: batching the ADJ2_OC loads costs registers)
#pragma unroll
      for (int t = 0; t < TB; ++t)
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const int grun = br + wr * RB + r, go = bo + wo * TB + t;
          if (gi >= G.nely || grun >= T.run_n || go >= T.other_n) continue;
          const long long e = ((long long)go * T.run_n + grun) * G.nely + gi;
          conv_store<NF, MODE>(G, A, e, NF > 1 ? keep[t][r] : acc[t][r], acc[t][r], red);
        }
      continue;
    }
    // FWD epilogue one output row (RB outputs) at a time, its loads issued first
#pragma unroll
    for (int t = 0; t < TB; ++t) {
      const int go = bo + wo * TB + t;
      long long eo[RB];
      double l0[RB], l1[RB];
      int sv[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int grun = br + wr * RB + r;
        const bool ok = gi < G.nely && grun < T.run_n && go < T.other_n;
        eo[r] = ok ? ((long long)go * T.run_n + grun) * G.nely + gi : -1;
        l0[r] = l1[r] = 0.0;
        sv[r] = 0;
        if (ok) {
          if (MODE == CONV_FWD) l0[r] = A.ihs[eo[r]];
          if (MODE == CONV_ADJ2_OC) {
            l0[r] = A.x[eo[r]];
            l1[r] = A.cw ? A.cw[eo[r]] : 1.0;
          }
          if (MODE == CONV_FWD || MODE == CONV_ADJ2_OC) sv[r] = elem_state(A.state, eo[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        if (eo[r] < 0) continue;
        conv_store_pre<NF, MODE>(A, eo[r], NF > 1 ? keep[t][r] : acc[t][r], acc[t][r], l0[r],
                                 l1[r], sv[r], red);
      }
    }
  }
  conv_partials<MODE>(A, red, T.zb);
}

// ============================================================================
// K2: volume-preserving eta (filter.hpp:182-228), cooperative Newton replay
// ============================================================================

struct EtaArgs {
  Geo G;
  const double* xt;
  const uint8_t* state;
  double beta, eta0, mtotal;
  double* partials;         // [gridDim][kEtaNS] + 2 control words
  double* result;           // eta, iterations (as double), g
};

// reciprocal: hardware estimate + two Newton steps (within an ulp; finite x > 0)
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// K2 from moment sums: one pass over xTilde per centre c (normally one in
// all). With T = tanh(beta (t - c)) and d = tanh(beta (eta - c)), the addition
// theorem gives tanh(beta (t - eta)) = (T - d) / (1 - T d), hence for every eta
//   sum th(eta)           = M1 - sum_{k=1..} d^k G_{k-1},   G_j = sum (1 - T^2) T^j
//   sum f sech^2(eta)     = (1 - d^2) sum_{k=0..} (k+1) d^k F_k,   F_k = sum f (1 - T^2) T^k
// with M1 = sum T and f = sinh(beta t) sinh(beta (1 - t)) (filter.hpp:157-161),
// so the mismatch g = ((n a + sum th) / den - sum t) / m (filter.hpp:187-192)
// and the slope (:194-198) of ANY eta follow from 2K + 4 sums. Truncated
// after K terms the remainder is below n |d|^(K+1) / (1 - |d|) < 1e-17 n for
// |d| <= kEtaDmax, under the rounding of the sums themselves; a Newton
// request beyond that re-centres (one more pass at that eta, where d = 0).
// The replay (EtaCtl, filter.hpp:200-226) runs on one thread. Against one
// pass per evaluation: C5 4 passes (+ an exp(2 beta t) cache written and read
// back) -> 1, and one grid-wide barrier instead of one per evaluation.
constexpr int kEtaK = 12;
constexpr int kEtaNS = 2 * kEtaK + 4;  // [0] sum t, [1] n, [2] M1, [3..3+K) G, [3+K..4+2K) F
constexpr double kEtaDmax = 0.045;     // 0.045^13 / 0.955 = 3.3e-18

struct EtaSeries {
  double beta, c, mtotal;
  const double* s;  // kEtaNS sums about c
  __host__ __device__ double dval(double eta) const { return tanh(beta * (eta - c)); }
  __host__ __device__ void eval(double eta, double d, double* g, double* gp) const {
    const double a = tanh(beta * eta);
    const double den = a + tanh(beta * (1.0 - eta));
    double acc = 0.0;
    for (int j = kEtaK - 1; j >= 0; --j) acc = fma(acc, d, s[3 + j]);
    const double sum_th = fma(-d, acc, s[2]);
    *g = ((s[1] * a + sum_th) / den - s[0]) / mtotal;
    double q = 0.0;
    for (int k = kEtaK; k >= 0; --k) q = fma(q, d, double(k + 1) * s[3 + kEtaK + k]);
    *gp = -beta / sinh(beta) * ((1.0 - d * d) * q) / mtotal;
  }
};

// this thread's share of the kEtaNS sums about centre c (active elements,
// grid-stride, 4 loads in flight)
__device__ __forceinline__ void eta_moments(const EtaArgs& A, double c, double (&red)[kEtaNS]) {
  const double kc = exp(-2.0 * A.beta * c);
  const double half_coshb = 0.5 * cosh(A.beta), eb = exp(A.beta), emb = exp(-A.beta);
#pragma unroll
  for (int q = 0; q < kEtaNS; ++q) red[q] = 0.0;
  constexpr int U = 4;
  const long long S = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < A.G.m; e += U * S) {
    double v[U];
    bool act[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long q = e + u * S;
      act[u] = q < A.G.m && elem_state(A.state, q) == 0;  // active set (filter.hpp:190)
      v[u] = act[u] ? A.xt[q] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!act[u]) continue;
      const double t = v[u];
      red[0] += t;
      red[1] += 1.0;
      const double E1 = exp(2.0 * A.beta * t);
      const double E = E1 * kc;
      double T, w;  // T = tanh(beta (t - c)) = 1 - 2 / (E + 1), w = 1 - T^2 = 4 E / (E + 1)^2
      if (E < INFINITY) {
        const double r = rcp_nr(E + 1.0);
        T = fma(-2.0, r, 1.0);
        w = 4.0 * E * r * r;
      } else {
        T = 1.0;
        w = 0.0;
      }
      const double f = half_coshb - 0.25 * fma(E1, emb, eb * rcp_nr(E1));
      red[2] += T;
      double p = w;
#pragma unroll
      for (int j = 0; j < kEtaK; ++j) {
        red[3 + j] += p;
        p *= T;
      }
      double q = w * f;
#pragma unroll
      for (int k = 0; k <= kEtaK; ++k) {
        red[3 + kEtaK + k] += q;
        q *= T;
      }
    }
  }
}

// Fixed-order sum of the kEtaNS-wide partial records of `nb` blocks into
// out[0..kEtaNS) (shared memory) by one block: 8 threads per component, each
// with all its loads in flight, then a fixed 8-lane shuffle tree (one L2 round
// trip per 8 records instead of one per component)
__device__ __forceinline__ void eta_sum_partials(const double* __restrict__ P, int nb,
                                                 double* out) {
  static_assert(kEtaNS * 8 <= kThreads, "8 threads per component");
  const int q = threadIdx.x >> 3, sub = threadIdx.x & 7;
  double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (q < kEtaNS) {
    int b = sub;
    for (; b + 56 < nb; b += 64)
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] += __ldcg(P + (long long)(b + 8 * u) * kEtaNS + q);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (b + 8 * u < nb) a[u] += __ldcg(P + (long long)(b + 8 * u) * kEtaNS + q);
  }
  double v = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  if (q < kEtaNS && sub == 0) out[q] = v;
  __syncthreads();
}

// Newton replay from the sums about `c`: feeds ctl until it finishes (returns
// false) or requests an eta too far from c (returns true, *c_next = it)
__host__ __device__ inline bool eta_replay(EtaCtl& ctl, const EtaSeries& S, double* c_next) {
  while (!ctl.done) {
    const double d = S.dval(ctl.eta);
    if (!(fabs(d) <= kEtaDmax)) {
      *c_next = ctl.eta;
      return true;
    }
    double g, gp;
    S.eval(ctl.eta, d, &g, &gp);
    ctl.feed(g, gp);
  }
  return false;
}

__global__ void __launch_bounds__(kThreads) k_eta_solve(EtaArgs A) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double scratch[kEtaNS * 32];
  __shared__ double s_c;
  __shared__ int s_go;
  EtaCtl ctl;  // block 0, thread 0
  if (threadIdx.x == 0) {
    ctl.init(A.eta0);
    s_c = ctl.eta;
  }
  __syncthreads();
  double* ctrl = A.partials + (long long)kEtaNS * gridDim.x;  // go flag, next centre
  for (int round = 0; round < 64; ++round) {
    const double c = s_c;
    double red[kEtaNS];
    eta_moments(A, c, red);
    block_sum<kEtaNS>(red, scratch);
    if (threadIdx.x == 0)
      for (int q = 0; q < kEtaNS; ++q) A.partials[(long long)kEtaNS * blockIdx.x + q] = red[q];
    grid.sync();
    if (blockIdx.x == 0) {  // one block sums in a fixed order and decides
      eta_sum_partials(A.partials, gridDim.x, scratch);
      if (threadIdx.x == 0) {
        const EtaSeries S{A.beta, c, A.mtotal, scratch};
        double cn = c;
        const bool go = eta_replay(ctl, S, &cn);
        ctrl[0] = go ? 1.0 : 0.0;
        ctrl[1] = cn;
        if (!go) {
          A.result[0] = ctl.eta;
          A.result[1] = double(ctl.it);
          A.result[2] = ctl.g;
        }
      }
    }
    grid.sync();
    if (threadIdx.x == 0) {
      s_go = __ldcg(ctrl) != 0.0;
      s_c = __ldcg(ctrl + 1);
    }
    __syncthreads();
    if (!s_go) break;
  }
}

// Multi-GPU eta: the same sums per rank -> on-device sum -> allreduce (NCCL,
// on the stream) -> one-thread replay; the host reads `go` once per round
// (normally one round: one host synchronisation per eta solve).
struct EtaDev {
  EtaCtl ctl;
  double c;
  int go;      // another round is needed
  int rounds;  // rounds that did work so far (the host adapts its speculation to it)
};

__global__ void k_eta_dev_init(EtaDev* st, double eta0) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    st->ctl.init(eta0);
    st->c = st->ctl.eta;
    st->go = 1;
    st->rounds = 0;
  }
}

__global__ void __launch_bounds__(kThreads) k_eta_moments_dev(EtaArgs A, const EtaDev* st) {
  if (!st->go) return;  // converged: a speculative round is a no-op
  __shared__ double scratch[kEtaNS * 32];
  double red[kEtaNS];
  eta_moments(A, st->c, red);
  block_sum<kEtaNS>(red, scratch);
  if (threadIdx.x == 0)
    for (int q = 0; q < kEtaNS; ++q) A.partials[(long long)kEtaNS * blockIdx.x + q] = red[q];
}

__global__ void __launch_bounds__(kThreads) k_eta_reduce(const double* __restrict__ P, int nb,
                                                         double* __restrict__ sums) {
  __shared__ double out[kEtaNS];
  eta_sum_partials(P, nb, out);
  if (threadIdx.x < kEtaNS) sums[threadIdx.x] = out[threadIdx.x];
}

// sums: the allreduced kEtaNS sums about st->c
__global__ void k_eta_dev_step(EtaDev* st, const double* __restrict__ sums, double beta,
                               double mtotal, double* __restrict__ result) {
  if (threadIdx.x != 0 || blockIdx.x != 0 || !st->go) return;
  EtaCtl ctl = st->ctl;
  const EtaSeries S{beta, st->c, mtotal, sums};
  double cn = st->c;
  st->go = eta_replay(ctl, S, &cn) ? 1 : 0;
  st->rounds += 1;
  st->c = cn;
  st->ctl = ctl;
  result[0] = ctl.eta;
  result[1] = double(ctl.it);
  result[2] = ctl.g;
}

// ============================================================================
// K3a: projection + SIMP + sensitivity + pre-adjoint fields (one element/thread)
//   filter.hpp:137-154, fea.hpp:135-146, fea.hpp:248-272, filter.hpp:170
// ============================================================================

template <int D>
struct KeFull {
  double k[D * D];  // column-major (fea.hpp ElementStiffness::full)
};

struct ElemArgs {
  const double* xt;      // owned filtered field (or xPhys when input_is_phys)
  int input_is_phys;     // 1: xt already holds xPhys (compliance_and_sensitivity API)
  const double* eta_ptr; // device scalar eta (written by K2)
  const double* U;       // slab node planes [j0, j0 + jn]
  const uint8_t* state;
  const double* ihs;     // owned 1 / hs
  double beta, e0, emin, penal, inv_m;
  double* xPhys;         // owned, may be null
  double* dcPhys;        // owned, may be null
  double* a1;            // storage-indexed pre-adjoint fields (dH dcPhys / hs, dH dV0 / hs)
  double* a2;
  double* partials;      // per block: compliance partial
  long long e_begin, e_end;  // element range of this launch (e_end 0: all)
};

__device__ __forceinline__ double simp_xp(double x, double p) {
  const double pm1 = p - 1.0;
  return pm1 == 2.0 ? x * x : pow(x, pm1);  // std::pow(x, p - 1), fea.hpp:141
}

// Each thread handles NE elements (e, e + H, ...) so every Ke coefficient
// fetched from the constant bank feeds NE FMAs.
template <int D, int NE>
__global__ void __launch_bounds__(kThreads, 4 - NE) k_elem_sens(Geo G, KeFull<D> K, ElemArgs A) {
  __shared__ double scratch[32];
  const double eta = A.input_is_phys ? 0.5 : *A.eta_ptr;
  const double a = tanh(A.beta * eta);
  const double denom = a + tanh(A.beta * (1.0 - eta));
  const double de = A.e0 - A.emin;
  const long long eb = A.e_begin, ee = A.e_end > 0 ? A.e_end : G.m;
  const long long H = (ee - eb + NE - 1) / NE;  // element stride between a thread's elements
  double csum = 0.0;
  for (long long e0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; e0 < H;
       e0 += (long long)gridDim.x * blockDim.x) {
    double ue[NE][D];
    double xphys[NE], dH[NE];
    bool ok[NE];
#pragma unroll
    for (int n = 0; n < NE; ++n) {
      const long long e = eb + e0 + n * H;
      ok[n] = e < ee;
      const long long ec = ok[n] ? e : eb + e0;
      int i, k, j;
      elem_ijk(G, ec, i, k, j);
      const double t = A.xt[ec];
      if (A.input_is_phys) {
        xphys[n] = t;
        dH[n] = 0.0;
      } else {
        const double th = tanh(A.beta * (t - eta));
        xphys[n] = (a + th) / denom;                          // filter.hpp:142
        dH[n] = A.beta * (1.0 - th * th) / denom;             // filter.hpp:151
      }
      int dofs[24];
      element_dofs(G, i, k, j, G.j0, dofs);
#pragma unroll
      for (int q = 0; q < D; ++q) {
        TOPO_CHECK(dofs[q] >= 0 && dofs[q] < G.dim * (G.jn + 1) * (G.nely + 1) * (G.is3d ? G.nz + 1 : 1));
        ue[n][q] = __ldg(A.U + dofs[q]);
      }
    }
    // quad = ue . (Ke ue) (fea.hpp:267), on the symmetric upper half
    double quad[NE];
#pragma unroll
    for (int n = 0; n < NE; ++n) quad[n] = 0.0;
#pragma unroll
    for (int r = 0; r < D; ++r) {
      const double hk = 0.5 * K.k[r * D + r];
      double s[NE];
#pragma unroll
      for (int n = 0; n < NE; ++n) s[n] = hk * ue[n][r];
#pragma unroll
      for (int c = r + 1; c < D; ++c) {
        const double kc = K.k[c * D + r];
#pragma unroll
        for (int n = 0; n < NE; ++n) s[n] = fma(kc, ue[n][c], s[n]);
      }
#pragma unroll
      for (int n = 0; n < NE; ++n) quad[n] = fma(ue[n][r], s[n], quad[n]);
    }
#pragma unroll
    for (int n = 0; n < NE; ++n) {
      if (!ok[n]) continue;
      const long long e = eb + e0 + n * H;
      const double q2 = 2.0 * quad[n];
      const double xp = simp_xp(xphys[n], A.penal);
      const double sK = A.emin + xp * xphys[n] * de;          // fea.hpp:142
      const double dsK = A.penal * xp * de;                   // fea.hpp:143
      csum = fma(sK, q2, csum);
      const int st = elem_state(A.state, e);
      const double dcp = st == 0 ? -dsK * q2 : 0.0;
      const double dv0 = st == 0 ? A.inv_m : 0.0;             // driver.hpp:155
      if (A.xPhys) A.xPhys[e] = xphys[n];
      if (A.dcPhys) A.dcPhys[e] = dcp;
      if (A.a1) {
        const double ih = A.ihs[e];
        const long long es = e + (long long)(G.j0 - G.sj0) * G.S;
        A.a1[es] = (dH[n] * dcp) * ih;                        // backfilter, filter.hpp:170, :128
        A.a2[es] = (dH[n] * dv0) * ih;
      }
    }
  }
  double red[1] = {csum};
  block_sum<1>(red, scratch);
  if (threadIdx.x == 0) A.partials[blockIdx.x] = red[0];
}

// K3a for hexahedra in Walsh coordinates. Per displacement component the 8
// nodal values are Walsh-Hadamard transformed over the element's three binary
// node coordinates (i, k, j); a mirror-symmetric Ke (every H8 Ke of an
// isotropic cube) couples only the three modes of equal reflection
// signature, so u' Ke u = sum over 8 signatures of a 3x3 quadratic form:
// 72 add/sub + 48 FMA instead of the 300-term upper-triangle sum. The host
// derives the blocks from the given Ke (Wt Ke W / 64) and uses this kernel
// only when every coupling outside them is negligible (capi.cu, walsh_blocks).
struct KeWalsh {
  double k[8][6];  // per signature: k00, 2k01, 2k02, k11, 2k12, k22
};
// component c's mode of signature sig has Walsh mask sig ^ (1 << kWalshAxis[c])
// (component 0 = x flips with j, 1 = y with i, 2 = z with k)
__host__ __device__ constexpr int walsh_axis(int c) { return c == 0 ? 2 : (c == 1 ? 0 : 1); }

// 104 registers (20 doubles spill to local memory; the kernel is gather-latency
// bound): two of its blocks and the store's block (128 x 96) fill the register
// file exactly, so the overlapped store is resident from the start instead of
// waiting for K3a's first wave to drain (C5 pass 6.05 -> 5.91 ms, C4 0.130 ->
// 0.1245 ms on the same box).
__global__ void __maxnreg__(104) k_elem_walsh(Geo G, KeWalsh K, ElemArgs A) {
  __shared__ double scratch[32];
  const double eta = A.input_is_phys ? 0.5 : *A.eta_ptr;
  const double a = tanh(A.beta * eta);
  const double denom = a + tanh(A.beta * (1.0 - eta));
  const double de = A.e0 - A.emin;
  const long long ny1 = G.nely + 1, pl = ny1 * (G.nelz + 1);
  const long long ee = A.e_end > 0 ? A.e_end : G.m;
  double csum = 0.0;
  for (long long e = A.e_begin + blockIdx.x * (long long)blockDim.x + threadIdx.x; e < ee;
       e += (long long)gridDim.x * blockDim.x) {
    int i, k, j;
    elem_ijk(G, e, i, k, j);
    // every load of the element first (latency overlap): x~, hs, state, u_e
    const double t = A.xt[e];
    const double ihv = A.a1 ? A.ihs[e] : 1.0;
    const int st = elem_state(A.state, e);
    const long long n0 = (long long)(j - G.j0) * pl + (long long)k * ny1 + i;  // node (i, k, j)
    double h[3][8];  // [component][binary node index oi + 2 ok + 4 oj]
    {
      // the element's nodes are 4 (k, j) pairs of 2 consecutive i: 6 doubles each
      const double* u0 = A.U + 3 * n0;
      const double* up[4] = {u0, u0 + 3 * ny1, u0 + 3 * pl, u0 + 3 * (pl + ny1)};
      TOPO_CHECK(n0 >= 0 && n0 + pl + ny1 + 1 < (long long)(G.jn + 1) * pl);
#pragma unroll
      for (int b = 0; b < 8; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c) h[c][b] = __ldg(up[b >> 1] + 3 * (b & 1) + c);
    }
    double xphys, dH;
    if (A.input_is_phys) {
      xphys = t;
      dH = 0.0;
    } else {
      const double th = tanh(A.beta * (t - eta));
      xphys = (a + th) / denom;               // filter.hpp:142
      dH = A.beta * (1.0 - th * th) / denom;  // filter.hpp:151
    }
    const double xp = simp_xp(xphys, A.penal);
    const double sK = A.emin + xp * xphys * de;  // fea.hpp:142
    const double dsK = A.penal * xp * de;        // fea.hpp:143
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int bit = 1; bit < 8; bit <<= 1)
#pragma unroll
        for (int b = 0; b < 8; ++b)
          if (!(b & bit)) {
            const double lo = h[c][b], hi = h[c][b | bit];
            h[c][b] = hi + lo;
            h[c][b | bit] = hi - lo;
          }
    double q2 = 0.0;  // u' Ke u (fea.hpp:267)
#pragma unroll
    for (int sig = 0; sig < 8; ++sig) {
      const double m0 = h[0][sig ^ (1 << walsh_axis(0))];
      const double m1 = h[1][sig ^ (1 << walsh_axis(1))];
      const double m2 = h[2][sig ^ (1 << walsh_axis(2))];
      const double* kk = K.k[sig];
      const double r0 = fma(kk[0], m0, fma(kk[1], m1, kk[2] * m2));
      const double r1 = fma(kk[3], m1, kk[4] * m2);
      q2 = fma(m0, r0, q2);
      q2 = fma(m1, r1, q2);
      q2 = fma(m2, kk[5] * m2, q2);
    }
    csum = fma(sK, q2, csum);
    const double dcp = st == 0 ? -dsK * q2 : 0.0;
    const double dv0 = st == 0 ? A.inv_m : 0.0;  // driver.hpp:155
    if (A.xPhys) A.xPhys[e] = xphys;
    if (A.dcPhys) A.dcPhys[e] = dcp;
    if (A.a1) {
      const double ih = ihv;
      const long long es = e + (long long)(G.j0 - G.sj0) * G.S;
      A.a1[es] = (dH * dcp) * ih;  // backfilter, filter.hpp:170, :128
      A.a2[es] = (dH * dv0) * ih;
    }
  }
  double red[1] = {csum};
  block_sum<1>(red, scratch);
  if (threadIdx.x == 0) A.partials[blockIdx.x] = red[0];
}

// ============================================================================
// K3b: lower-triangle stiffness values sK[e*P + q] = E(xPhys_e) Ke_lower[q]
//   (fea.hpp:135-146 + :162-169); the dominant HBM store stream
// ============================================================================

struct SkArgs {
  const double* xt;  // owned filtered field (null: use sKe directly)
  const double* sKe; // per-element modulus (topo_assemble_values)
  const double* ke_lower;
  const double* eta_ptr;  // device scalar eta
  double beta, e0, emin, penal;
  double* sK;
  unsigned long long* counter;  // k_sk_store_tma: {next group, finished warps}, zero between launches
  int gch;                      // groups per claim
};

// 256-bit streaming store (STG.E.EF.ENL2.256 on sm_100a): evict-first, the
// values are consumed by the solver, not by this pass.
__device__ __forceinline__ void st256_cs(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c),
               "d"(d)
               : "memory");
}

// One warp owns 32 consecutive elements: lane l computes the modulus of
// element l (one tanh + SIMP), then the warp streams the group's 32*P values
// as 32-byte vectors (fully coalesced, no block barriers), taking each value's
// modulus from its owner lane by shuffle and Ke_lower from shared memory.
constexpr int kSkUnroll = 4;
template <int P>
__global__ void __launch_bounds__(kThreads) k_sk_store(Geo G, SkArgs A) {
  constexpr int PV = P / 4;  // double4 per element
  __shared__ double4 kl[PV];
  for (int q = threadIdx.x; q < PV; q += blockDim.x)
    kl[q] = make_double4(A.ke_lower[4 * q], A.ke_lower[4 * q + 1], A.ke_lower[4 * q + 2],
                         A.ke_lower[4 * q + 3]);
  double a = 0, denom = 1, de = 0, eta = 0;
  if (A.xt) {
    eta = *A.eta_ptr;
    a = tanh(A.beta * eta);
    denom = a + tanh(A.beta * (1.0 - eta));
    de = A.e0 - A.emin;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long ngroups = (G.m + 31) >> 5;
  auto group = [&](long long g) {
    const long long e0 = g << 5;
    const int ne = int(min(32LL, G.m - e0));
    double s = 0.0;
    if (lane < ne) {
      if (A.xt) {
        const double xphys = (a + tanh(A.beta * (A.xt[e0 + lane] - eta))) / denom;  // :142
        const double xp = simp_xp(xphys, A.penal);
        s = A.emin + xp * xphys * de;  // fea.hpp:142
      } else {
        s = A.sKe[e0 + lane];
      }
    }
    double* out = A.sK + e0 * P;
    const int nv = ne * PV;
#pragma unroll kSkUnroll
    for (int base = 0; base < nv; base += 32) {
      const int v = base + lane;
      const int el = min(v / PV, 31);
      const double se = __shfl_sync(0xffffffffu, s, el);
      if (v < nv) {
        TOPO_CHECK(e0 * P + 4 * (long long)v + 3 < G.m * P && v - el * PV < PV);
        const double4 k = kl[v - el * PV];
        st256_cs(out + 4 * (long long)v, se * k.x, se * k.y, se * k.z, se * k.w);  // fea.hpp:168
      }
    }
  };
  const long long warp0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long g = warp0; g < ngroups; g += nwarps) group(g);
}

// K3b beside other kernels (the overlapped 3D pass), through the bulk-copy
// (TMA) engine. One persistent block of 4 warps per SM. A group of 32 elements
// is written as 16 element pairs (A, B) of 150 32-byte vectors; lane l owns
// vector l + 32 j of every pair, i.e. always the same five Ke_lower slices (A:
// l, 32 + l, 64 + l for l < 11; B: l - 11 for l >= 11, 21 + l, 53 + l for
// l < 22), held in registers for the kernel's lifetime. The products of a pair
// (4800 B) go to a warp-private stage in shared memory and lane 0 hands the
// stage to `cp.async.bulk` (shared -> global, L2 evict-first). D stages per
// warp, D - 1 copies in flight, no block barriers. Why not plain stores
// (scripts/store_bench.cu, profiles/r02/store_bench_*.txt): a store instruction
// keeps its source registers until its data has left the SM, microseconds
// beside a saturated write stream, so the bytes in flight (~100 KB per SM for
// the full rate) would live in registers the co-running filter and sensitivity
// kernels need; here they live in shared memory, the block takes 90 x 128
// registers, and the copies bypass the LSU queue the co-runners' loads wait
// in. Runs of `gch` groups are claimed from a counter; the claim of the run
// after next and the input of the next group are in flight while a group is
// written, so no read latency sits in front of the copies. Same products as
// k_sk_store: bitwise equal.
template <int D>
__global__ void __launch_bounds__(128) k_sk_store_tma(Geo G, SkArgs A) {
  constexpr int P = 300, PV = 75, CH = 2 * P * 8;  // bytes per element pair
  extern __shared__ __align__(128) unsigned char sk_ring[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* mine = sk_ring + (size_t)wib * D * CH;
  const double4* kl = reinterpret_cast<const double4*>(A.ke_lower);
  const double4 k0 = kl[lane], k1 = kl[32 + lane];
  const double4 k2 = kl[lane < 11 ? 64 + lane : lane - 11];
  const double4 k3 = kl[21 + lane], k4 = kl[min(53 + lane, PV - 1)];
  double a = 0, denom = 1, de = 0, eta = 0;
  if (A.xt) {
    eta = *A.eta_ptr;
    a = tanh(A.beta * eta);
    denom = a + tanh(A.beta * (1.0 - eta));
    de = A.e0 - A.emin;
  }
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const long long ngroups = (G.m + 31) >> 5;
  const double* src = A.xt ? A.xt : A.sKe;
  auto ldx = [&](long long g) {
    const long long e = (g << 5) + lane;
    return g < ngroups && e < G.m ? __ldg(src + e) : 0.0;
  };
  auto modulus = [&](double v) {
    if (!A.xt) return v;
    const double xphys = (a + tanh(A.beta * (v - eta))) / denom;  // filter.hpp:142
    const double xp = simp_xp(xphys, A.penal);
    return A.emin + xp * xphys * de;  // fea.hpp:142
  };
  const int GCH = A.gch;
  auto claim = [&]() {
    return lane == 0 ? atomicAdd(A.counter, (unsigned long long)GCH) : 0ull;
  };
  unsigned long long pend = claim();
  long long g0 = (long long)__shfl_sync(0xffffffffu, pend, 0);
  pend = claim();
  int stage = 0;
  if (g0 < ngroups) {
    double xv = ldx(g0);
    for (;;) {
      const long long ng0 = (long long)__shfl_sync(0xffffffffu, pend, 0);
      pend = claim();
      const long long g1 = min(g0 + GCH, ngroups);
      for (long long g = g0; g < g1; ++g) {
        const double s = modulus(xv);
        xv = ldx(g + 1 < g1 ? g + 1 : ng0);
        const long long e0 = g << 5;
        const int ne = int(min(32LL, G.m - e0));
        if (ne == 32) {
          TOPO_CHECK((e0 + 32) * P <= G.m * P);
#pragma unroll 2
          for (int k = 0; k < 16; ++k) {
            const double sa = __shfl_sync(0xffffffffu, s, 2 * k);
            const double sb = __shfl_sync(0xffffffffu, s, 2 * k + 1);
            const double sm = lane < 11 ? sa : sb;
            // the copy that read this stage D pairs ago has finished reading
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(D - 1) : "memory");
            __syncwarp();
            double2* st = reinterpret_cast<double2*>(mine + (size_t)stage * CH) + 2 * lane;
            st[0] = make_double2(sa * k0.x, sa * k0.y);  // fea.hpp:168
            st[1] = make_double2(sa * k0.z, sa * k0.w);
            st[64] = make_double2(sa * k1.x, sa * k1.y);
            st[65] = make_double2(sa * k1.z, sa * k1.w);
            st[128] = make_double2(sm * k2.x, sm * k2.y);
            st[129] = make_double2(sm * k2.z, sm * k2.w);
            st[192] = make_double2(sb * k3.x, sb * k3.y);
            st[193] = make_double2(sb * k3.z, sb * k3.w);
            if (lane < 22) {
              st[256] = make_double2(sb * k4.x, sb * k4.y);
              st[257] = make_double2(sb * k4.z, sb * k4.w);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              const unsigned sa32 = (unsigned)__cvta_generic_to_shared(mine + (size_t)stage * CH);
              double* gp = A.sK + (e0 + 2 * k) * P;
              asm volatile(
                  "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gp),
                  "r"(sa32), "n"(CH), "l"(pol)
                  : "memory");
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            stage = stage + 1 == D ? 0 : stage + 1;
          }
        } else {  // ragged last group: element by element, direct stores
          for (int el = 0; el < ne; ++el) {
            const double se = __shfl_sync(0xffffffffu, s, el);
            for (int v = lane; v < PV; v += 32) {
              const double4 k = kl[v];
              st256_cs(A.sK + (e0 + el) * P + 4 * v, se * k.x, se * k.y, se * k.z, se * k.w);
            }
          }
        }
      }
      g0 = ng0;
      if (g0 >= ngroups) break;
    }
  }
  // the copies must have completed (shared memory read, global memory
  // written) before the warp retires
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  // the last warp to finish re-arms the counters for the next launch (no
  // memset node on the critical path between K2 and the store)
  if (lane == 0) {
    __threadfence();
    const unsigned long long nw = (unsigned long long)gridDim.x * (blockDim.x >> 5);
    if (atomicAdd(A.counter + 1, 1ull) == nw - 1) {
      A.counter[0] = 0;
      A.counter[1] = 0;
      __threadfence();
    }
  }
}

// ============================================================================
// elementwise helpers for the stage-level API
// ============================================================================

__global__ void k_project(long long m, const double* __restrict__ xt, double eta, double beta,
                          double* __restrict__ out, int derivative) {
  const double a = tanh(beta * eta);
  const double denom = a + tanh(beta * (1.0 - eta));
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x) {
    const double th = tanh(beta * (xt[e] - eta));
    out[e] = derivative ? beta * (1.0 - th * th) / denom : (a + th) / denom;
  }
}

__global__ void k_recip(long long m, const double* __restrict__ a, double* __restrict__ out) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = 1.0 / a[e];
}

__global__ void k_simp(long long m, const double* __restrict__ x, double e0, double emin,
                       double p, double* __restrict__ sK, double* __restrict__ dsK) {
  const double de = e0 - emin;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x) {
    const double xp = simp_xp(x[e], p);
    if (sK) sK[e] = emin + xp * x[e] * de;
    if (dsK) dsK[e] = p * xp * de;
  }
}

// out_storage[e] = (dH[e] * g[e]) (projection on) or g[e]; already divided by
// hs when `div_hs` (backfilter pre-adjoint field)
__global__ void k_prescale(Geo G, const double* __restrict__ g, const double* __restrict__ xt,
                           double eta, double beta, int proj_on, const double* __restrict__ ihs,
                           double* __restrict__ out_st) {
  const double denom = tanh(beta * eta) + tanh(beta * (1.0 - eta));
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < G.m;
       e += (long long)gridDim.x * blockDim.x) {
    double v = g[e];
    if (proj_on) {
      const double th = tanh(beta * (xt[e] - eta));
      v = (beta * (1.0 - th * th) / denom) * v;
    }
    out_st[e + (long long)(G.j0 - G.sj0) * G.S] = v * ihs[e];
  }
}

__global__ void k_copy_to_storage(Geo G, const double* __restrict__ in, double* __restrict__ out_st) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < G.m;
       e += (long long)gridDim.x * blockDim.x)
    out_st[e + (long long)(G.j0 - G.sj0) * G.S] = in[e];
}

// compact active gathers (oc.hpp:63-67 take) are done on the host side of the
// API; the OC kernels below work on full-length element arrays.

// OC record + (sum ocP, V(0), V(inf)) partials from full-length x, dc, dV
__global__ void __launch_bounds__(kThreads) k_oc_prep(long long m, const double* __restrict__ x,
                                                      const double* __restrict__ dc,
                                                      const double* __restrict__ dV,
                                                      const uint8_t* __restrict__ state,
                                                      const double* __restrict__ cw, double move,
                                                      double* __restrict__ ocp,
                                                      double* __restrict__ partials) {
  __shared__ double scratch[3 * 32];
  double red[3] = {0.0, 0.0, 0.0};
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x) {
    const bool act = elem_state(state, e) == 0;
    const double4 r = oc_record(x[e], dc[e], dV[e], cw ? cw[e] : 1.0, move, act);
    ocp[e] = act ? r.z : -1.0;
    if (act) red[0] += r.z;
    red[1] += r.w * oc_cand(r, 0.0);
    red[2] += r.w * std_min(std_max(0.0, r.x), r.y);
  }
  block_sum<3>(red, scratch);
  if (threadIdx.x == 0) {
    partials[3 * blockIdx.x] = red[0];
    partials[3 * blockIdx.x + 1] = red[1];
    partials[3 * blockIdx.x + 2] = red[2];
  }
}

// ============================================================================
// K5 + K6: OC bisection (oc.hpp:93-174), cooperative; volume of a candidate
// from the exact identity mean(pin(H xc)) = (|P1| + c . xc) / m with
// c = H' 1_notP (ft = 3) or c = 1, |P1| -> 0 (ft = 1). Speculative batches
// evaluate every multiplier the replay can request in the next kDepth steps.
// ============================================================================

constexpr int kOcK = 16;

struct OcArgs {
  long long m;
  OcRecs R;
  const double* prep_partials;  // stride 3, count n_prep
  int n_prep;
  double volfrac, rel_tol, vol_tol, abs_tol, lambda_max, mtotal, add_const;
  int lambda_space;
  double margin;      // bound-shortcut margin
  double* partials;   // [2][kOcK][gridDim]
  double* xNew;       // full length (passives = x via their records)
  double* result;     // lambda, bisections, evaluations, status, batches, shortcut
  long long* dbg;     // optional clock64 trace of block 0 (profiling aid)
};

template <int KK>  // requests per batch: 16 (4 levels) or 32 (5 levels)
__global__ void __launch_bounds__(kThreads) k_oc_bisect(OcArgs A) {
  cg::grid_group grid = cg::this_grid();
  OcCtl ctl;  // replayed by thread 0 of every block (registers, not shared memory)
  int mode = 0, nbatch = 0;
  __shared__ double sreq[KK], sinv[KK];
  __shared__ double sval[KK];
  __shared__ int nreq;
  __shared__ double scratch[KK * 32];
  int ndbg = 0;
  auto mark = [&]() {
    if (A.dbg && blockIdx.x == 0 && threadIdx.x == 0 && ndbg < 120) A.dbg[ndbg++] = clock64();
  };
  mark();
  if (threadIdx.x < 32) {
    double s[3];
    warp_sum_partials<3>(A.prep_partials, A.n_prep, 3, s);
    if (threadIdx.x == 0) {
      // oc.hpp:112-116 lambda# = [sum x sqrt(-dc/dV) / (m volfrac)]^2
      double lamMax = A.lambda_max;
      if (!(A.lambda_max > 0)) {
        const double root = s[0] / (A.mtotal * A.volfrac);
        lamMax = root * root;
      }
      ctl.init(lamMax, A.volfrac, A.rel_tol, A.vol_tol, A.lambda_space, A.abs_tol);
      const double V0 = (A.add_const + s[1]) / A.mtotal;
      const double Vinf = (A.add_const + s[2]) / A.mtotal;
      // every candidate volume lies in [V(inf), V(0)] (monotone, c >= 0):
      // when the whole interval is decisively on one side, every decision of
      // the reference is known without evaluating (SURVEY.md §7 hard part 2)
      mode = 0;
      if (Vinf > A.volfrac + 0.5 * A.vol_tol + A.margin) mode = 1;
      if (V0 < A.volfrac - 0.5 * A.vol_tol - A.margin) mode = -1;
      nbatch = 0;
    }
  }
  __syncthreads();
  int buf = 0;
  for (;;) {
    if (threadIdx.x == 0) {
      nreq = 0;
      if (mode != 0) {
        ctl.replay_known(mode > 0 ? INFINITY : -INFINITY);
      } else if (ctl.pending()) {
        nreq = oc_speculate<KK>(ctl, sreq);
        for (int q = 0; q < KK; ++q) {  // reciprocals for the batch sums (1/0 = inf)
          if (q >= nreq) sreq[q] = 1.0;
          sinv[q] = 1.0 / sreq[q];
        }
      }
    }
    __syncthreads();
    mark();
    if (nreq == 0) break;
    const int K = nreq;
    double acc[KK];
#pragma unroll
    for (int q = 0; q < KK; ++q) acc[q] = 0.0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < A.m;
         e += (long long)gridDim.x * blockDim.x) {
      const double4 r = A.R.get(e);
#pragma unroll
      for (int q = 0; q < KK; ++q)
        if (q < K) acc[q] = fma(r.w, oc_cand_rcp(r, sreq[q], sinv[q]), acc[q]);
    }
    mark();
    block_sum<KK>(acc, scratch);
    double* P = A.partials + (long long)buf * KK * gridDim.x;
    if (threadIdx.x == 0)
      for (int q = 0; q < K; ++q) P[(long long)q * gridDim.x + blockIdx.x] = acc[q];
    mark();
    grid.sync();
    mark();
    // every block reduces the same partials in the same fixed order: 16
    // threads per request, all requests in parallel
    {
      constexpr int G = kThreads / KK;  // threads per request (16 or 8)
      const int q = threadIdx.x / G, sub = threadIdx.x % G;
      double sum = 0.0;
      if (q < K) sum = strided_sum_l2(P + (long long)q * gridDim.x, gridDim.x, sub, G);
#pragma unroll
      for (int off = G / 2; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
      if (sub == 0 && q < K) sval[q] = (A.add_const + sum) / A.mtotal;
    }
    __syncthreads();
    mark();
    if (threadIdx.x == 0) {
      ++nbatch;
      while (ctl.pending()) {
        int hit = -1;
        for (int q = 0; q < K; ++q)
          if (sreq[q] == ctl.s_req) hit = q;
        if (hit < 0) break;
        ctl.feed(sval[hit]);
      }
    }
    buf ^= 1;
    __syncthreads();
  }
  // K6 (xNew at the final multiplier) runs as k_oc_final with full occupancy
  // (measured: inside this grid, beside the sK stream, C4 OC 0.128 vs 0.04 ms;
  // the prep and compliance sums folded in here: C4 pass 0.23 vs 0.195 ms)
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.result[0] = ctl.lam_result;
    A.result[1] = ctl.bis;
    A.result[2] = ctl.evals;
    A.result[3] = ctl.status;
    A.result[4] = nbatch;
    A.result[5] = mode;
    A.result[6] = ctl.s_final;
    if (A.dbg) A.dbg[127] = ndbg;
  }
}

// K6: xNew at the final multiplier s = result[6] (oc.hpp:108, :171), skipped
// when the bisection reported an error (result[3])
__global__ void __launch_bounds__(kThreads) k_oc_final(long long m, OcRecs R,
                                                       const double* __restrict__ result,
                                                       double* __restrict__ out) {
  if (result[3] != 0.0) return;
  const double s = result[6];
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = oc_cand(R.get(e), s);
}


// oc.hpp:209-222: block partial (sumClamped, sumMid, numMid) of the
// primal-dual iteration at the sqrt multiplier lm, over active elements
__global__ void __launch_bounds__(kThreads) k_oc_pd_sums(long long m, OcRecs R, double lm,
                                                         double* __restrict__ partials) {
  __shared__ double scratch[3 * 32];
  double red[3] = {0.0, 0.0, 0.0};
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x) {
    if (R.ocp[e] < 0.0) continue;  // passive
    const double4 r = R.get(e);
    const double f = r.z / lm;
    if (f > r.y)
      red[0] += r.y;
    else if (f < r.x)
      red[0] += r.x;
    else {
      red[1] += r.z;
      red[2] += 1.0;
    }
  }
  block_sum<3>(red, scratch);
  if (threadIdx.x == 0)
    for (int q = 0; q < 3; ++q) partials[3 * blockIdx.x + q] = red[q];
}

// row q of a [rows][count] partial table summed in a fixed order by block q
__global__ void k_reduce_rows(const double* __restrict__ p, int count, double* __restrict__ out) {
  __shared__ double scratch[32];
  double v[1] = {0.0};
  const double* row = p + (long long)blockIdx.x * count;
  for (int i = threadIdx.x; i < count; i += blockDim.x) v[0] += row[i];
  block_sum<1>(v, scratch);
  if (threadIdx.x == 0) out[blockIdx.x] = v[0];
}

// ---------------------------------------------------------------------------
// Multi-rank OC (identity volumes) with the bisection state in device memory:
// every rank replays the same decisions from allreduced sums, batches of
// speculative volume sums are allreduced on the stream (NCCL), and no host
// round trip is needed until the pass ends (oc.hpp:93-174 via OcCtl).
struct OcDev {
  OcCtl ctl;
  int K;     // requests to evaluate in the next round (0: none)
  int done;  // the replay has finished
  double req[kOcK];
};

struct OcDevParams {
  double volfrac, rel_tol, vol_tol, abs_tol, lambda_max, mtotal, add_const, margin;
  int lambda_space;
};

// sums3: the allreduced (sum ocP, V(0) sum, V(inf) sum) of K4
__global__ void k_oc_dev_init(OcDev* st, const double* __restrict__ sums3, OcDevParams P) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  OcCtl ctl;
  double lamMax = P.lambda_max;
  if (!(P.lambda_max > 0)) {  // oc.hpp:112-116
    const double root = sums3[0] / (P.mtotal * P.volfrac);
    lamMax = root * root;
  }
  ctl.init(lamMax, P.volfrac, P.rel_tol, P.vol_tol, P.lambda_space, P.abs_tol);
  const double V0 = (P.add_const + sums3[1]) / P.mtotal;
  const double Vinf = (P.add_const + sums3[2]) / P.mtotal;
  int mode = 0;  // the bound shortcut (k_oc_bisect)
  if (Vinf > P.volfrac + 0.5 * P.vol_tol + P.margin) mode = 1;
  if (V0 < P.volfrac - 0.5 * P.vol_tol - P.margin) mode = -1;
  if (mode != 0) ctl.replay_known(mode > 0 ? INFINITY : -INFINITY);
  st->K = ctl.pending() ? oc_speculate<kOcK>(ctl, st->req) : 0;
  st->done = !ctl.pending();
  st->ctl = ctl;
}

// K speculative volume sums over this rank's elements (no-op when K == 0)
__global__ void __launch_bounds__(kThreads) k_oc_batch_dev(long long m, OcRecs R,
                                                           const OcDev* __restrict__ st,
                                                           double* __restrict__ partials) {
  const int K = st->K;
  if (K == 0) return;
  __shared__ double scratch[kOcK * 32];
  double acc[kOcK], sq[kOcK], iq[kOcK];
#pragma unroll
  for (int q = 0; q < kOcK; ++q) {
    acc[q] = 0.0;
    sq[q] = q < K ? st->req[q] : 1.0;
    iq[q] = 1.0 / sq[q];
  }
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x) {
    const double4 r = R.get(e);
#pragma unroll
    for (int q = 0; q < kOcK; ++q)
      if (q < K) acc[q] = fma(r.w, oc_cand_rcp(r, sq[q], iq[q]), acc[q]);
  }
  block_sum<kOcK>(acc, scratch);
  if (threadIdx.x == 0)
    for (int q = 0; q < kOcK; ++q) partials[(long long)q * gridDim.x + blockIdx.x] = acc[q];
}

// sums: the allreduced volume sums of the round's requests
__global__ void k_oc_dev_feed(OcDev* st, const double* __restrict__ sums, double add_const,
                              double mtotal) {
  if (threadIdx.x != 0 || blockIdx.x != 0 || st->K == 0) return;
  OcCtl ctl = st->ctl;
  const int K = st->K;
  while (ctl.pending()) {
    int hit = -1;
    for (int q = 0; q < K; ++q)
      if (st->req[q] == ctl.s_req) hit = q;
    if (hit < 0) break;
    ctl.feed((add_const + sums[hit]) / mtotal);
  }
  st->K = ctl.pending() ? oc_speculate<kOcK>(ctl, st->req) : 0;
  st->done = !ctl.pending();
  st->ctl = ctl;
}

// xNew at the final multiplier once the replay is done (oc.hpp:171)
__global__ void k_oc_dev_final(long long m, OcRecs R, const OcDev* __restrict__ st,
                               double* __restrict__ out) {
  if (!st->done || st->ctl.status != OcCtl::ST_OK) return;
  const double s = st->ctl.s_final;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = oc_cand(R.get(e), s);
}

// res[0..3] lambda, bisections, evaluations, status; res[7] done
__global__ void k_oc_dev_result(const OcDev* __restrict__ st, double* __restrict__ res) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  res[0] = st->ctl.lam_result;
  res[1] = st->ctl.bis;
  res[2] = st->ctl.evals;
  res[3] = st->ctl.status;
  res[7] = st->done;
}

// ---------------------------------------------------------------------------
// Redesign-loop helpers (SURVEY.md §8(f) row 3, driver.hpp:189, :235-263)

// per block: sum (xPhys - xPrev)^2, sum xPhys, sum x (1 - x); xPrev <- xPhys
__global__ void __launch_bounds__(kThreads) k_loop_records(long long m, const double* __restrict__ xp,
                                                           double* __restrict__ xprev,
                                                           const double* __restrict__ x,
                                                           double* __restrict__ partials) {
  __shared__ double scratch[3 * 32];
  double red[3] = {0.0, 0.0, 0.0};
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x) {
    const double v = xp[e], d = v - xprev[e], xv = x[e];
    red[0] = fma(d, d, red[0]);
    red[1] += v;
    red[2] = fma(xv, 1.0 - xv, red[2]);
    xprev[e] = v;
  }
  block_sum<3>(red, scratch);
  if (threadIdx.x == 0)
    for (int q = 0; q < 3; ++q) partials[3 * blockIdx.x + q] = red[q];
}

// Anderson extrapolation (accel.hpp:21-95) over the active elements of the
// device design: column `slot` of the cyclic difference window, then prevX /
// prevR <- (x_before, x_new - x_before); passives hold zeros throughout
__global__ void k_and_hist(long long m, const uint8_t* __restrict__ state,
                           const double* __restrict__ xb, const double* __restrict__ xn,
                           double* __restrict__ dx, double* __restrict__ dr,
                           double* __restrict__ px, double* __restrict__ pr, int slot,
                           int has_prev) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x) {
    const bool act = elem_state(state, e) == 0;
    const double xa = act ? xb[e] : 0.0, ra = act ? xn[e] - xb[e] : 0.0;
    if (has_prev) {
      dx[(long long)slot * m + e] = xa - px[e];
      dr[(long long)slot * m + e] = ra - pr[e];
    }
    px[e] = xa;
    pr[e] = ra;
  }
}

constexpr int kAndMax = 8;  // window columns supported on the device

// per block: the upper triangle of R'R (cols (cols+1)/2) then R'r (cols)
__global__ void __launch_bounds__(kThreads) k_and_gram(long long m, int cols,
                                                       const double* __restrict__ dr,
                                                       const double* __restrict__ pr,
                                                       double* __restrict__ partials) {
  constexpr int NQ = kAndMax * (kAndMax + 1) / 2 + kAndMax;
  __shared__ double scratch[NQ * 32];
  double red[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) red[q] = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x) {
    double c[kAndMax];
#pragma unroll
    for (int i = 0; i < kAndMax; ++i) c[i] = i < cols ? dr[(long long)i * m + e] : 0.0;
    const double r = pr[e];
    int q = 0;
#pragma unroll
    for (int i = 0; i < kAndMax; ++i)
#pragma unroll
      for (int j = i; j < kAndMax; ++j, ++q) red[q] = fma(c[i], c[j], red[q]);
#pragma unroll
    for (int i = 0; i < kAndMax; ++i, ++q) red[q] = fma(c[i], r, red[q]);
  }
  block_sum<NQ>(red, scratch);
  if (threadIdx.x == 0)
    for (int q = 0; q < NQ; ++q) partials[(long long)NQ * blockIdx.x + q] = red[q];
}

// gamma = sum over eigenpairs of R'R with ev > 1e-13 max|ev| of v (v'R'r) / ev
// (accel.hpp:76-92): the partial records summed in a fixed order, then cyclic
// Jacobi on the cols x cols Gram matrix (one thread), eigenvalues ascending
__global__ void k_and_solve(const double* __restrict__ partials, int nblocks, int cols,
                            double* __restrict__ gamma) {
  constexpr int NQ = kAndMax * (kAndMax + 1) / 2 + kAndMax;
  __shared__ double tot[NQ];
  for (int q = threadIdx.x; q < NQ; q += blockDim.x)
    tot[q] = strided_sum_l2(partials, nblocks, 0, 1, NQ, q);
  __syncthreads();
  if (threadIdx.x != 0) return;
  double G[kAndMax][kAndMax], V[kAndMax][kAndMax], rhs[kAndMax];
  int q = 0;
  for (int i = 0; i < kAndMax; ++i)
    for (int j = i; j < kAndMax; ++j) {
      G[i][j] = G[j][i] = tot[q++];
    }
  for (int i = 0; i < kAndMax; ++i) rhs[i] = tot[q++];
  for (int i = 0; i < kAndMax; ++i)
    for (int j = 0; j < kAndMax; ++j) V[i][j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < cols; ++i) {
      diag += G[i][i] * G[i][i];
      for (int j = i + 1; j < cols; ++j) off += G[i][j] * G[i][j];
    }
    if (!(off > 1e-32 * diag)) break;
    for (int p = 0; p < cols; ++p)
      for (int r = p + 1; r < cols; ++r) {
        if (G[p][r] == 0.0) continue;
        const double theta = (G[r][r] - G[p][p]) / (2.0 * G[p][r]);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < cols; ++k) {  // G <- J' G J
          const double gkp = G[k][p], gkr = G[k][r];
          G[k][p] = c * gkp - s * gkr;
          G[k][r] = s * gkp + c * gkr;
        }
        for (int k = 0; k < cols; ++k) {
          const double gpk = G[p][k], grk = G[r][k];
          G[p][k] = c * gpk - s * grk;
          G[r][k] = s * gpk + c * grk;
        }
        for (int k = 0; k < cols; ++k) {  // V <- V J
          const double vkp = V[k][p], vkr = V[k][r];
          V[k][p] = c * vkp - s * vkr;
          V[k][r] = s * vkp + c * vkr;
        }
      }
  }
  int ord[kAndMax];
  for (int i = 0; i < cols; ++i) ord[i] = i;
  for (int i = 1; i < cols; ++i)  // ascending eigenvalues (SelfAdjointEigenSolver order)
    for (int j = i; j > 0 && G[ord[j]][ord[j]] < G[ord[j - 1]][ord[j - 1]]; --j) {
      const int t = ord[j];
      ord[j] = ord[j - 1];
      ord[j - 1] = t;
    }
  double amax = 0.0;
  for (int i = 0; i < cols; ++i) amax = fmax(amax, fabs(G[i][i]));
  const double cutoff = amax * 1e-13;
  double g[kAndMax];
  for (int i = 0; i < kAndMax; ++i) g[i] = 0.0;
  if (cutoff > 0) {
    for (int ii = 0; ii < cols; ++ii) {
      const int i = ord[ii];
      const double ev = G[i][i];
      if (!(ev > cutoff)) continue;
      double vr = 0.0;
      for (int k = 0; k < cols; ++k) vr += V[k][i] * rhs[k];
      const double f = vr / ev;
      for (int k = 0; k < cols; ++k) g[k] += V[k][i] * f;
    }
  }
  for (int i = 0; i < kAndMax; ++i) gamma[i] = g[i];
}

// xn[e] <- clamp(x + mix r - (X + mix R) gamma, 0, 1) on the active elements
// (accel.hpp:64-71, driver.hpp:240-243)
__global__ void k_and_apply(long long m, const uint8_t* __restrict__ state,
                            const double* __restrict__ xb, double* __restrict__ xn,
                            const double* __restrict__ dx, const double* __restrict__ dr,
                            const double* __restrict__ gamma, int cols, double mix) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x) {
    if (elem_state(state, e) != 0) continue;
    const double xa = xb[e], ra = xn[e] - xa;
    double out = xa + mix * ra;
    if (cols > 0) {
      double corr = 0.0;
      for (int j = 0; j < cols; ++j)
        corr += (dx[(long long)j * m + e] + mix * dr[(long long)j * m + e]) * gamma[j];
      out -= corr;
    }
    xn[e] = fmin(fmax(out, 0.0), 1.0);
  }
}

// candidate at one multiplier (host-driven OC modes and final write)
__global__ void k_oc_candidates(long long m, OcRecs R, double s, double* __restrict__ out) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = oc_cand(R.get(e), s);
}

// block partial sums of v (optionally projected: mean(H(v)))
__global__ void __launch_bounds__(kThreads) k_sum(long long m, const double* __restrict__ v,
                                                  int project, double eta, double beta,
                                                  double* __restrict__ partials) {
  __shared__ double scratch[32];
  double a = 0, denom = 1;
  if (project) {
    a = tanh(beta * eta);
    denom = a + tanh(beta * (1.0 - eta));
  }
  double red[1] = {0.0};
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x)
    red[0] += project ? (a + tanh(beta * (v[e] - eta))) / denom : v[e];
  block_sum<1>(red, scratch);
  if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
}

// fixed-order final reduction of `count` partials (stride) into out[0..N)
// oc.hpp:195-236 on the device (single rank): the whole dual fixed-point
// iteration lm <- sumMid(lm) / (budget - sumClamped(lm)) in one cooperative
// launch, one grid barrier per iteration. Every block sums the per-block
// records in the same fixed order (warp_sum_partials, the order of the
// host-driven loop's reductions) and takes the same decisions, so the
// multiplier sequence is bitwise that of the host-driven loop.
// result: {lm, iterations, fell_back}.
struct OcPdArgs {
  long long m;
  OcRecs R;
  const double* prep;  // K4-style prep records (stride 3): [0] = sum ocP
  int n_prep;
  double budget, pd_tol, mtotal, volfrac;
  double* partials;    // [2][3 * gridDim]
  double* result;
};

__global__ void __launch_bounds__(kThreads) k_oc_pd(OcPdArgs A) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double scratch[3 * 32];
  __shared__ double s_lm;
  __shared__ int s_state;  // 0: iterate, 1: converged, 2: fall back
  if (threadIdx.x < 32) {
    double s[3];
    warp_sum_partials<3>(A.prep, A.n_prep, 3, s);
    if (threadIdx.x == 0) {
      s_lm = s[0] / (A.mtotal * A.volfrac);  // oc.hpp:204
      s_state = s_lm > 0 ? 0 : 2;
    }
  }
  __syncthreads();
  double lm = s_lm;
  int it = 0, fb = s_state == 2, buf = 0;
  for (; !fb; ++it) {
    if (it >= 1000) {
      fb = 1;
      break;
    }
    double red[3] = {0.0, 0.0, 0.0};
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < A.m;
         e += (long long)gridDim.x * blockDim.x) {
      if (A.R.ocp[e] < 0.0) continue;  // passive
      const double4 r = A.R.get(e);
      const double f = r.z / lm;
      if (f > r.y)
        red[0] += r.y;
      else if (f < r.x)
        red[0] += r.x;
      else {
        red[1] += r.z;
        red[2] += 1.0;
      }
    }
    block_sum<3>(red, scratch);
    double* P = A.partials + (long long)buf * 3 * gridDim.x;
    if (threadIdx.x == 0)
      for (int q = 0; q < 3; ++q) P[3 * blockIdx.x + q] = red[q];
    grid.sync();
    if (threadIdx.x < 32) {
      double s[3];
      warp_sum_partials<3>(P, gridDim.x, 3, s);
      if (threadIdx.x == 0) {
        const double sumClamped = s[0], sumMid = s[1], numMid = s[2];
        const double den = A.budget - sumClamped;
        const double lmNext = sumMid / den;
        if (numMid == 0 || den <= 0 || !(lmNext > 0) || !isfinite(lmNext)) {
          s_state = 2;
        } else {
          s_state = fabs(lmNext - lm) <= A.pd_tol ? 1 : 0;
          s_lm = lmNext;
        }
      }
    }
    __syncthreads();
    const int state = s_state;
    if (state == 2) {
      fb = 1;
      break;
    }
    lm = s_lm;
    buf ^= 1;
    __syncthreads();  // (s_state / s_lm are rewritten in the next iteration)
    if (state == 1) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.result[0] = lm;
    A.result[1] = double(it);
    A.result[2] = double(fb);
  }
}

template <int N>
__global__ void k_reduce_partials(const double* __restrict__ p, int count, int stride,
                                  double* __restrict__ out) {
  double s[N];
  warp_sum_partials<N>(p, count, stride, s);
  if (threadIdx.x == 0)
    for (int q = 0; q < N; ++q) out[q] = s[q];
}

// fixed-order reduction of `count` partial records with one block (any size)
template <int N>
__global__ void k_reduce_block(const double* __restrict__ p, int count, int stride,
                               double* __restrict__ out) {
  __shared__ double scratch[N * 32];
  double v[N];
#pragma unroll
  for (int q = 0; q < N; ++q) v[q] = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x)
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] += p[(long long)i * stride + q];
  block_sum<N>(v, scratch);
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < N; ++q) out[q] = v[q];
}

// oc.hpp:31-39 / :72-79 on compact arrays
__global__ void k_oc_compact(long long n, const double* __restrict__ x,
                             const double* __restrict__ dc, const double* __restrict__ dV,
                             double sqrt_lambda, double move, double* __restrict__ out,
                             double* __restrict__ partials) {
  __shared__ double scratch[32];
  double red[1] = {0.0};
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const double4 r = oc_record(x[e], dc[e], dV[e], 1.0, move, true);
    red[0] += r.z;
    if (out) out[e] = oc_cand(r, sqrt_lambda);
  }
  block_sum<1>(red, scratch);
  if (threadIdx.x == 0 && partials) partials[blockIdx.x] = red[0];
}

// ============================================================================
// Duplicate-summed lower-triangle CSC of K: the
// matrix assemble_lower builds with setFromTriplets (fea.hpp:154-176), values
// summed per slot in triplet order (ascending element), no atomics.
//   Column c = dim * node + cc. Its rows are the lower-triangle DOFs of the
//   nodes one step away in x, z, y (ascending node order = lexicographic
//   (dx, dz, dy)); table entry (cc, j) is candidate row j of such a column and
//   the elements shared by the two nodes, in ascending element order, with
//   the lower-triangle index q of the pair in each (grid.hpp:143-150).
// ============================================================================
struct CscTab {
  int ncand[3];
  int cand[3][42];    // (dx + 1) | (dz + 1) << 2 | (dy + 1) << 4 | cr << 6
  int ncon[3][42];
  int con[3][42][8];  // (ex + 1) | (ez + 1) << 1 | (ey + 1) << 2 | q << 3
};

// Interior nodes (all 8 surrounding elements and all neighbours exist) share
// one slot layout: slot s of the node's run sums, over the elements in
// ascending order k (element code kOrd[k]), E_k * klt[k][s] where pmask[s]
// has bit k set.
struct CscInterior {
  int nslot;
  int branchless;           // no Ke_lower entry is -0: absent terms may add +0 (exact)
  int code[128];            // candidate code of slot s (cand packing)
  unsigned char pmask[128];
  double klt[8][128];
};
// ascending element order of the codes (ex + 1) | (ez + 1) << 1 | (ey + 1) << 2
__host__ __device__ constexpr int csc_ord(int k) {
  return (k >> 2 & 1) | (k >> 1 & 1) << 1 | (k & 1) << 2;  // ex slowest, then ez, then ey
}

struct CscGeo {
  int dim, nelx, nely, nz;  // element extents (nz = 1 in 2D)
  long long ny1, pl;        // node strides: y 1, z ny1, x pl = nz1 * ny1
  int nz1;                  // node extent along z (1 in 2D)
  long long n;              // DOFs (full columns)
  const int* map;           // reduced mode (EquilibriumSolver, fea.hpp:188-199, :316-336):
                            // DOF -> free index or -1; null = the full matrix
  const unsigned char* clean;  // reduced mode: node whose 27-neighbourhood is all free
};

__device__ __forceinline__ void csc_col(const CscGeo& C, long long c, int& cc, long long& nc, int& ix,
                                        int& iz, int& iy) {
  nc = c / C.dim;
  cc = int(c - nc * C.dim);
  iy = int(nc % C.ny1);
  const long long t = nc / C.ny1;
  iz = int(t % C.nz1);
  ix = int(t / C.nz1);
}

__device__ __forceinline__ bool csc_valid(const CscGeo& C, int code, int ix, int iz, int iy) {
  const int dx = (code & 3) - 1, dz = ((code >> 2) & 3) - 1, dy = ((code >> 4) & 3) - 1;
  return ix + dx >= 0 && ix + dx <= C.nelx && iz + dz >= 0 && iz + dz < C.nz1 && iy + dy >= 0 &&
         iy + dy <= C.nely;
}

__device__ __forceinline__ long long csc_row(const CscGeo& C, long long nc, int code) {
  const int dx = (code & 3) - 1, dz = ((code >> 2) & 3) - 1, dy = ((code >> 4) & 3) - 1;
  return C.dim * (nc + dx * C.pl + dz * C.ny1 + dy) + (code >> 6);
}

// slots per (free) column; cnt is indexed by the (reduced) column number
__global__ void k_csc_count(CscGeo C, const CscTab* __restrict__ T, long long* __restrict__ cnt) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < C.n;
       c += (long long)gridDim.x * blockDim.x) {
    if (C.map && C.map[c] < 0) continue;
    int cc, ix, iz, iy;
    long long nc;
    csc_col(C, c, cc, nc, ix, iz, iy);
    int k = 0;
    for (int j = 0; j < T->ncand[cc]; ++j) {
      const int code = T->cand[cc][j];
      k += csc_valid(C, code, ix, iz, iy) && (!C.map || C.map[csc_row(C, nc, code)] >= 0);
    }
    cnt[C.map ? C.map[c] : c] = k;
  }
}

// reduced mode: node flags, 1 when every DOF of its 27-neighbourhood is free
__global__ void k_csc_clean(CscGeo C, unsigned char* __restrict__ clean) {
  const long long nn = C.n / C.dim;
  for (long long nc = blockIdx.x * (long long)blockDim.x + threadIdx.x; nc < nn;
       nc += (long long)gridDim.x * blockDim.x) {
    const int iy = int(nc % C.ny1);
    const long long t = nc / C.ny1;
    const int iz = int(t % C.nz1), ix = int(t / C.nz1);
    bool ok = true;
    for (int dx = -1; dx <= 1; ++dx)
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy) {
          const int jx = ix + dx, jz = iz + dz, jy = iy + dy;
          if (jx < 0 || jx > C.nelx || jz < 0 || jz >= C.nz1 || jy < 0 || jy > C.nely) continue;
          const long long nr = ((long long)jx * C.nz1 + jz) * C.ny1 + jy;
          for (int c = 0; c < C.dim; ++c) ok = ok && C.map[C.dim * nr + c] >= 0;
        }
    clean[nc] = ok;
  }
}

// one warp per node: its dim columns are consecutive, so the node's slots are
// one contiguous run of the value array. Lanes take the node's candidate rows
// (flattened over (cc, j)); a ballot per round compacts them in slot order.
// The <= 8 elements around the node (all the elements any of its slots sums
// over) have their moduli staged once per warp in shared memory; the tables
// and Ke_lower live in shared memory.
template <bool ROWS, bool VALS>
__global__ void __launch_bounds__(kThreads) k_csc_fill(CscGeo C, const CscTab* __restrict__ T,
                                                        const CscInterior* __restrict__ TI,
                                                        const long long* __restrict__ col_ptr,
                                                        const double* __restrict__ E,
                                                        const double* __restrict__ kl,
                                                        int* __restrict__ rows,
                                                        double* __restrict__ vals) {
  __shared__ CscTab st;
  __shared__ double skl[300];
  __shared__ double sE[kThreads / 32][8];
  __shared__ unsigned char sflat[128][2];  // (cc, j) of flattened candidate k
  __shared__ int snflat;
  __shared__ CscInterior si;
  {
    const int* srci = reinterpret_cast<const int*>(TI);
    int* dsti = reinterpret_cast<int*>(&si);
    for (int q = threadIdx.x; q < int(sizeof(CscInterior) / sizeof(int)); q += blockDim.x)
      dsti[q] = srci[q];
    const int* src = reinterpret_cast<const int*>(T);
    int* dst = reinterpret_cast<int*>(&st);
    for (int q = threadIdx.x; q < int(sizeof(CscTab) / sizeof(int)); q += blockDim.x) dst[q] = src[q];
    if (VALS)
      for (int q = threadIdx.x; q < (C.dim == 3 ? 300 : 36); q += blockDim.x) skl[q] = kl[q];
    if (threadIdx.x == 0) {
      int k = 0;
      for (int cc = 0; cc < C.dim; ++cc)
        for (int j = 0; j < T->ncand[cc]; ++j, ++k) {
          sflat[k][0] = (unsigned char)cc;
          sflat[k][1] = (unsigned char)j;
        }
      snflat = k;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long nnodes = C.n / C.dim;
  const int nflat = snflat;
  const bool fast = !VALS || si.branchless;
  for (long long nc = w0; nc < nnodes; nc += nw) {
    int iy, iz, ix;
    if (nc <= 0xffffffffLL) {  // 32-bit division
      const unsigned u = unsigned(nc), ny1 = unsigned(C.ny1), nz1 = unsigned(C.nz1);
      const unsigned t = u / ny1;
      iy = int(u - t * ny1);
      ix = int(t / nz1);
      iz = int(t - unsigned(ix) * nz1);
    } else {
      iy = int(nc % C.ny1);
      const long long t = nc / C.ny1;
      iz = int(t % C.nz1);
      ix = int(t / C.nz1);
    }
    // the node's first (free) column and its slot run
    long long c0 = nc * C.dim;
    if (C.map) {
      int q = 0;
      while (q < C.dim && C.map[c0 + q] < 0) ++q;
      if (q == C.dim) continue;  // every DOF of the node is fixed: no columns
      c0 = C.map[c0 + q];
    }
    const long long base0 = col_ptr[c0];
    const bool interior = ix >= 1 && ix < C.nelx && iy >= 1 && iy < C.nely &&
                          (C.nz1 == 1 || (iz >= 1 && iz < C.nz1 - 1)) && (!C.map || C.clean[nc]);
    unsigned emask = 0;  // elements (ex, ez, ey) around the node that exist
    if (interior) {
      emask = C.nz1 == 1 ? 0xCCu : 0xFFu;  // 2D: only ez = 0 (code bit 1 set)
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int ex = ix + (q & 1) - 1, ez = iz + ((q >> 1) & 1) - 1, ey = iy + ((q >> 2) & 1) - 1;
        if (ex >= 0 && ex < C.nelx && ez >= 0 && ez < C.nz && ey >= 0 && ey < C.nely)
          emask |= 1u << q;
      }
    }
    if (VALS) {
      __syncwarp();
      if (lane < 8 && (emask >> lane & 1u)) {
        const int ex = ix + (lane & 1) - 1, ez = iz + ((lane >> 1) & 1) - 1,
                  ey = iy + ((lane >> 2) & 1) - 1;
        sE[wib][lane] = E[((long long)ex * C.nz + ez) * C.nely + ey];
      }
      __syncwarp();
    }
    if (interior && fast) {  // fixed layout: every candidate valid, every element present
      double Ek[8];
      if (VALS) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          Ek[k] = (emask >> csc_ord(k) & 1u) ? sE[wib][csc_ord(k)] : 0.0;
      }
      for (int s0 = 0; s0 < si.nslot; s0 += 32) {
        const int sl = s0 + lane;
        if (sl >= si.nslot) continue;
        if (ROWS) {
          const long long r = csc_row(C, nc, si.code[sl]);
          rows[base0 + sl] = C.map ? C.map[r] : int(r);
        }
        if (VALS) {
          // absent terms carry weight +0: acc + E * 0 = acc and 0 + v1 = v1, so
          // the sum is the reference's v1 + v2 + ... bit for bit (no -0 in Ke)
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < 8; ++k) acc = __dadd_rn(acc, __dmul_rn(Ek[k], si.klt[k][sl]));
          vals[base0 + sl] = acc;
        }
      }
      continue;
    }
    long long base = base0;
    for (int k0 = 0; k0 < nflat; k0 += 32) {
      const int k = k0 + lane;
      int cc = 0, j = 0, code = 0;
      bool ok = false;
      if (k < nflat) {
        cc = sflat[k][0];
        j = sflat[k][1];
        code = st.cand[cc][j];
        ok = csc_valid(C, code, ix, iz, iy) &&
             (!C.map || (C.map[nc * C.dim + cc] >= 0 && C.map[csc_row(C, nc, code)] >= 0));
      }
      const unsigned bal = __ballot_sync(0xffffffffu, ok);
      if (ok) {
        const long long slot = base + __popc(bal & ((1u << lane) - 1u));
        if (ROWS) {
          const long long r = csc_row(C, nc, code);
          rows[slot] = C.map ? C.map[r] : int(r);
        }
        if (VALS) {
          double acc = 0.0;
          bool first = true;
          const int ncon = st.ncon[cc][j];
          for (int q = 0; q < ncon; ++q) {  // ascending element = triplet order
            const int w = st.con[cc][j][q];
            if (!(emask >> (w & 7) & 1u)) continue;
            const double v = sE[wib][w & 7] * skl[w >> 3];  // fea.hpp:168
            acc = first ? v : acc + v;                       // setFromTriplets duplicate sum
            first = false;
          }
          vals[slot] = acc;
        }
      }
      base += __popc(bal);
    }
  }
}

// per-element modulus E(xPhys) from the filtered field and eta (fea.hpp:142)
__global__ void k_modulus(long long m, const double* __restrict__ xt, const double* __restrict__ eta_ptr,
                          double beta, double e0, double emin, double penal, double* __restrict__ E) {
  const double eta = *eta_ptr;
  const double a = tanh(beta * eta);
  const double denom = a + tanh(beta * (1.0 - eta));
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x) {
    const double xphys = (a + tanh(beta * (xt[e] - eta))) / denom;  // filter.hpp:142
    const double xp = simp_xp(xphys, penal);
    E[e] = emin + xp * xphys * (e0 - emin);
  }
}

// ============================================================================
// State solve K u = f (fea.hpp:205-239 solve_equilibrium
// on the free DOFs): matrix-free Jacobi-preconditioned conjugate gradients on
// the structured grid. K x is gathered per node (no atomics, fixed order):
// y[dof] = sum over the elements around the node of E_e (Ke x_e)[local dof].
// ============================================================================
struct StateGeo {
  int dim, nelx, nely, nz, nz1;  // elements along x, y, z (nz = 1 in 2D); node layers nz1
  long long ny1, pl, nn;          // node strides, node count
  const double* E;                // per-element modulus
  const unsigned char* fixed;     // per DOF: 1 = fixed (u = 0)
};

// local node index of binary offsets (oi, ok, oj) in the element_dofs order
__device__ __forceinline__ int local_node(int dim, int oi, int ok, int oj) {
  return dim == 3 ? ((ok << 2) | (oi ? (oj ? 1 : 0) : (oj ? 2 : 3)))
                  : (oi ? (oj ? 1 : 0) : (oj ? 2 : 3));
}

__device__ __forceinline__ void node_xyz(const StateGeo& S, long long nd, int& ix, int& iz, int& iy) {
  const long long t = nd / S.ny1;
  iy = int(nd - t * S.ny1);
  ix = int(t / S.nz1);
  iz = int(t - (long long)ix * S.nz1);
}

// y = K x over the free DOFs (fixed rows zeroed; x is zero on fixed DOFs) and
// block partials of x . y; Ke (full, column-major) staged in shared memory
template <int DIM>
__global__ void __launch_bounds__(kThreads) k_state_matvec(StateGeo S, const double* __restrict__ ke,
                                                           const double* __restrict__ x,
                                                           double* __restrict__ y,
                                                           double* __restrict__ partials) {
  constexpr int D = 4 * (DIM == 3 ? 2 : 1) * DIM;  // 8 or 24 element DOFs
  __shared__ double sk[D * D];
  __shared__ double scratch[32];
  for (int q = threadIdx.x; q < D * D; q += blockDim.x) sk[q] = ke[q];
  __syncthreads();
  double dot = 0.0;
  for (long long nd = blockIdx.x * (long long)blockDim.x + threadIdx.x; nd < S.nn;
       nd += (long long)gridDim.x * blockDim.x) {
    int ix, iz, iy;
    node_xyz(S, nd, ix, iz, iy);
    double acc[DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c) acc[c] = 0.0;
#pragma unroll
    for (int q = 0; q < (DIM == 3 ? 8 : 4); ++q) {  // elements around the node, ascending
      const int ex = ix - 1 + (q >> (DIM == 3 ? 2 : 1) & 1);
      const int ez = DIM == 3 ? iz - 1 + (q >> 1 & 1) : 0;
      const int ey = iy - 1 + (q & 1);
      if (ex < 0 || ex >= S.nelx || ez < 0 || ez >= S.nz || ey < 0 || ey >= S.nely) continue;
      const double Ee = S.E[((long long)ex * S.nz + ez) * S.nely + ey];
      const int a = local_node(DIM, iy - ey, iz - ez, ix - ex);
      const long long n0 = ((long long)ex * S.nz1 + ez) * S.ny1 + ey;  // element corner node
      double part[DIM];
#pragma unroll
      for (int c = 0; c < DIM; ++c) part[c] = 0.0;
#pragma unroll
      for (int b = 0; b < (DIM == 3 ? 8 : 4); ++b) {
        // local node b's binary offsets (inverse of local_node)
        const int oi = (b & 3) == 0 || (b & 3) == 1 ? 1 : 0;
        const int oj = (b & 3) == 1 || (b & 3) == 2 ? 1 : 0;
        const int ok = DIM == 3 ? (b >> 2) : 0;
        const long long nb = n0 + oi + (long long)ok * S.ny1 + (long long)oj * S.pl;
#pragma unroll
        for (int cc = 0; cc < DIM; ++cc) {
          const double xv = x[DIM * nb + cc];
#pragma unroll
          for (int c = 0; c < DIM; ++c)
            part[c] = fma(sk[(DIM * b + cc) * D + DIM * a + c], xv, part[c]);  // Ke(row, col)
        }
      }
#pragma unroll
      for (int c = 0; c < DIM; ++c) acc[c] = fma(Ee, part[c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      const long long d = DIM * nd + c;
      const double v = S.fixed[d] ? 0.0 : acc[c];
      y[d] = v;
      dot = fma(x[d], v, dot);
    }
  }
  double red[1] = {dot};
  block_sum<1>(red, scratch);
  if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
}

// Jacobi diagonal of K (1 on fixed DOFs)
template <int DIM>
__global__ void k_state_diag(StateGeo S, const double* __restrict__ ke, double* __restrict__ diag) {
  constexpr int D = 4 * (DIM == 3 ? 2 : 1) * DIM;
  for (long long nd = blockIdx.x * (long long)blockDim.x + threadIdx.x; nd < S.nn;
       nd += (long long)gridDim.x * blockDim.x) {
    int ix, iz, iy;
    node_xyz(S, nd, ix, iz, iy);
    double acc[DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c) acc[c] = 0.0;
    for (int q = 0; q < (DIM == 3 ? 8 : 4); ++q) {
      const int ex = ix - 1 + (q >> (DIM == 3 ? 2 : 1) & 1);
      const int ez = DIM == 3 ? iz - 1 + (q >> 1 & 1) : 0;
      const int ey = iy - 1 + (q & 1);
      if (ex < 0 || ex >= S.nelx || ez < 0 || ez >= S.nz || ey < 0 || ey >= S.nely) continue;
      const double Ee = S.E[((long long)ex * S.nz + ez) * S.nely + ey];
      const int a = local_node(DIM, iy - ey, iz - ez, ix - ex);
#pragma unroll
      for (int c = 0; c < DIM; ++c) acc[c] = fma(Ee, ke[(DIM * a + c) * D + DIM * a + c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      const long long d = DIM * nd + c;
      diag[d] = S.fixed[d] ? 1.0 : acc[c];
    }
  }
}

// CG scalars (device): [0] rz, [1] pq, [2] rr, [3] rz_new, [5] rz0, [6] ff
// u += a p, r -= a q, z = r / diag; partials (r.r, r.z); a = rz / pq
__global__ void __launch_bounds__(kThreads) k_cg_update(long long n, const double* __restrict__ sc,
                                                        const double* __restrict__ p,
                                                        const double* __restrict__ q,
                                                        const double* __restrict__ diag,
                                                        double* __restrict__ u, double* __restrict__ r,
                                                        double* __restrict__ z,
                                                        double* __restrict__ partials) {
  __shared__ double scratch[2 * 32];
  const double a = sc[0] / sc[1];
  double red[2] = {0.0, 0.0};
  for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < n;
       d += (long long)gridDim.x * blockDim.x) {
    u[d] = fma(a, p[d], u[d]);
    const double rv = fma(-a, q[d], r[d]);
    r[d] = rv;
    const double zv = rv / diag[d];
    z[d] = zv;
    red[0] = fma(rv, rv, red[0]);
    red[1] = fma(rv, zv, red[1]);
  }
  block_sum<2>(red, scratch);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = red[0];
    partials[2 * blockIdx.x + 1] = red[1];
  }
}

// p = z + (rz_new / rz) p; then rz = rz_new (one thread, after the grid)
__global__ void k_cg_direction(long long n, const double* __restrict__ sc, const double* __restrict__ z,
                               double* __restrict__ p) {
  const double b = sc[3] / sc[0];
  for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < n;
       d += (long long)gridDim.x * blockDim.x)
    p[d] = fma(b, p[d], z[d]);
}

// initial residual: r = f (0 on fixed), z = r / diag, p = z, u = 0; partials (r.z, f.f)
__global__ void __launch_bounds__(kThreads) k_cg_init(long long n, const double* __restrict__ f,
                                                      const unsigned char* __restrict__ fixed,
                                                      const double* __restrict__ diag,
                                                      double* __restrict__ u, double* __restrict__ r,
                                                      double* __restrict__ z, double* __restrict__ p,
                                                      double* __restrict__ partials) {
  __shared__ double scratch[2 * 32];
  double red[2] = {0.0, 0.0};
  for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < n;
       d += (long long)gridDim.x * blockDim.x) {
    const double rv = fixed[d] ? 0.0 : f[d];
    const double zv = rv / diag[d];
    u[d] = 0.0;
    r[d] = rv;
    z[d] = zv;
    p[d] = zv;
    red[0] = fma(rv, zv, red[0]);
    red[1] = fma(rv, rv, red[1]);
  }
  block_sum<2>(red, scratch);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = red[0];
    partials[2 * blockIdx.x + 1] = red[1];
  }
}

// u += a p, r -= a q (a = rz / pq); partials of r.r (PCG with an external preconditioner)
__global__ void __launch_bounds__(kThreads) k_cg_update_ur(long long n, const double* __restrict__ sc,
                                                           const double* __restrict__ p,
                                                           const double* __restrict__ q,
                                                           double* __restrict__ u,
                                                           double* __restrict__ r,
                                                           double* __restrict__ partials) {
  __shared__ double scratch[32];
  const double a = sc[0] / sc[1];
  double red[1] = {0.0};
  for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < n;
       d += (long long)gridDim.x * blockDim.x) {
    u[d] = fma(a, p[d], u[d]);
    const double rv = fma(-a, q[d], r[d]);
    r[d] = rv;
    red[0] = fma(rv, rv, red[0]);
  }
  block_sum<1>(red, scratch);
  if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
}

// block partials of a . b
__global__ void __launch_bounds__(kThreads) k_dot(long long n, const double* __restrict__ a,
                                                  const double* __restrict__ b,
                                                  double* __restrict__ partials) {
  __shared__ double scratch[32];
  double red[1] = {0.0};
  for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < n;
       d += (long long)gridDim.x * blockDim.x)
    red[0] = fma(a[d], b[d], red[0]);
  block_sum<1>(red, scratch);
  if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
}

__global__ void k_copy_scalar(const double* __restrict__ src, double* __restrict__ dst) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *dst = *src;
}

// FP64 peak probe: 8 independent FMA chains per thread (topo_fp64_peak)
__global__ void __launch_bounds__(kThreads) k_dfma_peak(int iters, double seed, double* out) {
  double a[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) a[q] = seed + threadIdx.x * 1e-9 + q;
  const double b = 0.999999999, c = 1e-12;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = fma(a[q], b, c);
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += a[q];
  if (s == 12345.678) out[0] = s;  // keeps the loop alive
}

}  // namespace topo
