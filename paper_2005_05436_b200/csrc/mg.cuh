// Geometric multigrid preconditioner for the state solve (SURVEY.md §8(f)
// row 2; the MGCG variant of top3D125). Levels coarsen the
// structured grid by 2 per axis; level l >= 1 stores one Galerkin element
// matrix per coarse element, Kc = sum_p Q_p' K_child(p) Q_p over its 2^dim
// children, with Q_p the (tri)linear interpolation from the coarse element's
// nodes to child p's nodes (level 1: K_child = E_f Ke, so Kc = sum_p E_p Kp
// with Kp = Q_p' Ke Q_p precomputed). The element operator is applied by
// colour (elements of one colour share no node), so y = K x is accumulated
// without atomics in a fixed order. Restriction (full weighting = P') and
// prolongation are node gathers. Damped Jacobi smoothing, a fixed number of
// Jacobi sweeps on the coarsest level: the V-cycle is a fixed symmetric
// linear operator, used inside plain PCG.
#pragma once

#include "common.cuh"
#include "kernels.cuh"

namespace topo {

struct MgGeo {         // one level
  int nelx, nely, nz;  // elements along x, y, z (nz = 1 in 2D)
  int nz1;             // node layers along z (1 in 2D)
  long long ny1, pl;   // node strides
  long long nn, n, m;  // nodes, DOFs, elements
  const unsigned char* fixed;
};

template <int DIM>
struct MgT {
  static constexpr int NN = DIM == 3 ? 8 : 4;  // nodes per element
  static constexpr int D = NN * DIM;           // DOFs per element
};

// local node of binary offsets (oi, ok, oj) in the element_dofs order
__host__ __device__ inline int mg_local(int dim, int oi, int ok, int oj) {
  const int base = oi ? (oj ? 1 : 0) : (oj ? 2 : 3);
  return dim == 3 ? (ok << 2) | base : base;
}
__host__ __device__ inline void mg_offsets(int b, int& oi, int& ok, int& oj) {
  oi = (b & 3) == 0 || (b & 3) == 1;
  oj = (b & 3) == 1 || (b & 3) == 2;
  ok = b >> 2;
}

__device__ __forceinline__ void mg_elem(const MgGeo& L, long long e, int& ex, int& ez, int& ey) {
  ey = int(e % L.nely);
  const long long t = e / L.nely;
  ez = int(t % L.nz);
  ex = int(t / L.nz);
}

// global DOF of local DOF q of element (ex, ez, ey)
template <int DIM>
__device__ __forceinline__ long long mg_dof(const MgGeo& L, int ex, int ez, int ey, int q) {
  const int b = q / DIM, c = q - b * DIM;
  int oi, ok, oj;
  mg_offsets(b, oi, ok, oj);
  const long long node = ((long long)(ex + oj) * L.nz1 + (ez + ok)) * L.ny1 + (ey + oi);
  return DIM * node + c;
}

// Kc[e] = sum over children p of E(child) * Kp[p] (level 1)
template <int DIM>
__global__ void k_mg_galerkin1(MgGeo C, MgGeo F, const double* __restrict__ E,
                               const double* __restrict__ Kp, double* __restrict__ Kc) {
  constexpr int NN = MgT<DIM>::NN, D = MgT<DIM>::D, DD = D * D;
  const long long tot = C.m * DD;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    const long long e = t / DD;
    int q = int(t - e * DD);
    if (q % D < q / D) q = (q % D) * D + q / D;  // exactly symmetric: (i < j) takes (j, i)
    int ex, ez, ey;
    mg_elem(C, e, ex, ez, ey);
    double acc = 0.0;
#pragma unroll
    for (int p = 0; p < NN; ++p) {
      int pi, pk, pj;
      mg_offsets(p, pi, pk, pj);
      const long long ef = ((long long)(2 * ex + pj) * F.nz + (2 * ez + pk)) * F.nely + (2 * ey + pi);
      acc = fma(E[ef], Kp[p * DD + q], acc);
    }
    Kc[t] = acc;
  }
}

// Level-2 Galerkin matrices straight from the fine moduli (level 1 is not
// stored): Kc[e] = sum over the (2^dim)^2 fine grandchildren g = p1 * NN + p2 of
// E_g M[g], M[g] = (Q_p2 Q_p1)' Ke (Q_p2 Q_p1) precomputed (exactly symmetric).
// A block takes NE coarse elements: their E in shared memory, each M entry
// read once per block and used NE times.
template <int DIM, int NE>
__global__ void __launch_bounds__(192) k_mg_galerkin2e(MgGeo C, const double* __restrict__ E,
                                                       const double* __restrict__ M,
                                                       double* __restrict__ Kc) {
  constexpr int NN = MgT<DIM>::NN, D = MgT<DIM>::D, DD = D * D, NG = NN * NN;
  __shared__ double sE[NE][NG];
  const long long fny = 4LL * C.nely, fnz = DIM == 3 ? 4LL * C.nz : 1;
  for (long long e0 = (long long)blockIdx.x * NE; e0 < C.m; e0 += (long long)gridDim.x * NE) {
    __syncthreads();
    for (int i = threadIdx.x; i < NE * NG; i += blockDim.x) {
      const int n = i / NG, g = i - n * NG;
      const long long e = e0 + n;
      double v = 0.0;
      if (e < C.m) {
        int ex, ez, ey;
        mg_elem(C, e, ex, ez, ey);
        int i1, k1, j1, i2, k2, j2;
        mg_offsets(g / NN, i1, k1, j1);
        mg_offsets(g % NN, i2, k2, j2);
        const long long fx = 4LL * ex + 2 * j1 + j2, fy = 4LL * ey + 2 * i1 + i2;
        const long long fz = DIM == 3 ? 4LL * ez + 2 * k1 + k2 : 0;
        v = E[(fx * fnz + fz) * fny + fy];
      }
      sE[n][g] = v;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < DD; q += blockDim.x) {
      double acc[NE];
#pragma unroll
      for (int n = 0; n < NE; ++n) acc[n] = 0.0;
#pragma unroll 4
      for (int g = 0; g < NG; ++g) {
        const double m = __ldg(M + (long long)g * DD + q);
#pragma unroll
        for (int n = 0; n < NE; ++n) acc[n] = fma(sE[n][g], m, acc[n]);
      }
#pragma unroll
      for (int n = 0; n < NE; ++n)
        if (e0 + n < C.m) Kc[(e0 + n) * DD + q] = acc[n];
    }
  }
}

// Kc[e] = sum_p Qp' Kf[child p] Qp (levels >= 2); one block per coarse element
// FROM_E: the children's matrices are level-1 Galerkin matrices built on the
// fly, K_child = sum_p' E(grandchild p') Kp[p'] (Kf = fine E, Kp: the 8 Qp' Ke Qp)
template <int DIM, bool FROM_E = false>
__global__ void __launch_bounds__(256) k_mg_galerkin(MgGeo C, MgGeo F, const double* __restrict__ Kf,
                                                     const double* __restrict__ Q,
                                                     double* __restrict__ Kc,
                                                     const double* __restrict__ Kp = nullptr) {
  constexpr int NN = MgT<DIM>::NN, D = MgT<DIM>::D, DD = D * D;
  __shared__ double sK[DD], sT[DD], sQ[DD];
  for (long long e = blockIdx.x; e < C.m; e += gridDim.x) {
    int ex, ez, ey;
    mg_elem(C, e, ex, ez, ey);
    double acc[(DD + 255) / 256];
#pragma unroll
    for (int r = 0; r < (DD + 255) / 256; ++r) acc[r] = 0.0;
    for (int p = 0; p < NN; ++p) {
      int pi, pk, pj;
      mg_offsets(p, pi, pk, pj);
      const long long ef = ((long long)(2 * ex + pj) * F.nz + (2 * ez + pk)) * F.nely + (2 * ey + pi);
      __syncthreads();
      for (int q = threadIdx.x; q < DD; q += blockDim.x) {
        if (FROM_E) {
          // child ef = (fx, fz, fy) of level F; its children on the finest grid
          const int fy = 2 * ey + pi, fz = 2 * ez + pk, fx = 2 * ex + pj;
          const int qs = q % D < q / D ? (q % D) * D + q / D : q;  // symmetric (as galerkin1)
          double acc1 = 0.0;
#pragma unroll
          for (int p2 = 0; p2 < NN; ++p2) {
            int qi, qk, qj;
            mg_offsets(p2, qi, qk, qj);
            const long long eg =
                ((long long)(2 * fx + qj) * (DIM == 3 ? 2 * F.nz : 1) + (DIM == 3 ? 2 * fz + qk : 0)) *
                    (2 * F.nely) + (2 * fy + qi);
            acc1 = fma(Kf[eg], Kp[p2 * DD + qs], acc1);
          }
          sK[q] = acc1;
        } else {
          sK[q] = Kf[ef * DD + q];
        }
        sQ[q] = Q[p * DD + q];
      }
      __syncthreads();
      for (int q = threadIdx.x; q < DD; q += blockDim.x) {  // T = Kf Qp (column-major)
        const int i = q % D, j = q / D;
        double s = 0.0;
        for (int k = 0; k < D; ++k) s = fma(sK[k * D + i], sQ[j * D + k], s);
        sT[q] = s;
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < (DD + 255) / 256; ++r) {  // acc += Qp' T
        const int q = threadIdx.x + 256 * r;
        if (q >= DD) continue;
        const int i = q % D, j = q / D;
        double s = 0.0;
        for (int k = 0; k < D; ++k) s = fma(sQ[i * D + k], sT[j * D + k], s);
        acc[r] += s;
      }
    }
    // stored exactly symmetric: entry (i, j) with i < j takes (j, i)'s value
    __syncthreads();
#pragma unroll
    for (int r = 0; r < (DD + 255) / 256; ++r) {
      const int q = threadIdx.x + 256 * r;
      if (q < DD) sT[q] = acc[r];
    }
    __syncthreads();
    for (int q = threadIdx.x; q < DD; q += blockDim.x) {
      const int i = q % D, j = q / D;
      Kc[e * DD + q] = i >= j ? sT[q] : sT[i * D + j];
    }
  }
}

// y += K x over the elements of one colour (FINE: K_e = E_e Ke)
template <int DIM, bool FINE>
__global__ void __launch_bounds__(256) k_mg_apply(MgGeo L, const double* __restrict__ K,
                                                  const double* __restrict__ E, int color,
                                                  const double* __restrict__ x, double* __restrict__ y) {
  constexpr int D = MgT<DIM>::D;
  __shared__ double sKe[FINE ? D * D : 1];
  if (FINE) {
    for (int q = threadIdx.x; q < D * D; q += blockDim.x) sKe[q] = K[q];
    __syncthreads();
  }
  const int cx = color & 1, cz = (color >> 1) & 1, cy = (color >> 2) & 1;
  const long long hx = (L.nelx - cx + 1) / 2, hz = (L.nz - cz + 1) / 2, hy = (L.nely - cy + 1) / 2;
  const long long tot = hx * hz * hy;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    const int ey = cy + 2 * int(t % hy);
    const long long u = t / hy;
    const int ez = cz + 2 * int(u % hz), ex = cx + 2 * int(u / hz);
    const long long e = ((long long)ex * L.nz + ez) * L.nely + ey;
    long long dof[D];
    double xe[D];
#pragma unroll
    for (int q = 0; q < D; ++q) {
      dof[q] = mg_dof<DIM>(L, ex, ez, ey, q);
      xe[q] = x[dof[q]];
    }
    const double* Km = FINE ? sKe : K + e * (long long)(D * D);
    const double s = FINE ? E[e] : 1.0;
#pragma unroll 4
    for (int i = 0; i < D; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) acc = fma(Km[j * D + i], xe[j], acc);
      y[dof[i]] += s * acc;
    }
  }
}

// y += K x over the elements of one colour, stored element matrices: one
// warp per element, lane i computes row i (the matrix column j is read by the
// lanes contiguously), x_e broadcast by shuffles
template <int DIM>
__global__ void __launch_bounds__(256) k_mg_apply_warp(MgGeo L, const double* __restrict__ K, int color,
                                                       const double* __restrict__ x,
                                                       double* __restrict__ y) {
  constexpr int D = MgT<DIM>::D;
  const int lane = threadIdx.x & 31;
  const int cx = color & 1, cz = (color >> 1) & 1, cy = (color >> 2) & 1;
  const long long hx = (L.nelx - cx + 1) / 2, hz = (L.nz - cz + 1) / 2, hy = (L.nely - cy + 1) / 2;
  const long long tot = hx * hz * hy;
  const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long t = w0; t < tot; t += nw) {
    const int ey = cy + 2 * int(t % hy);
    const long long u = t / hy;
    const int ez = cz + 2 * int(u % hz), ex = cx + 2 * int(u / hz);
    const long long e = ((long long)ex * L.nz + ez) * L.nely + ey;
    long long dof = 0;
    double xv = 0.0;
    if (lane < D) {
      dof = mg_dof<DIM>(L, ex, ez, ey, lane);
      xv = x[dof];
    }
    const double* Km = K + e * (long long)(D * D);
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double xj = __shfl_sync(0xffffffffu, xv, j);
      if (lane < D) acc = fma(Km[j * D + lane], xj, acc);
    }
    if (lane < D) y[dof] += acc;
  }
}

// E_e Ke x_e for one hexahedron in Walsh coordinates (Ke = W Kt W', the
// blocks of k_elem_walsh): per component an 8-point Walsh-Hadamard transform
// of x_e, the 8 signature blocks (3x3), the inverse transform; 216 flops per
// element instead of 576. h holds x_e on entry ([component][binary node index
// oi + 2 ok + 4 oj]) and the element's output on exit. sk: per signature k00,
// k01, k02, k11, k12, k22 (plain, not doubled).
// h <- H h per component (H[m][b] = prod over the axes a in m of (bit a of b ? 1 : -1))
__device__ __forceinline__ void wh_butterfly(double (&h)[3][8]) {
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
}
// h <- S h, S = diag((-1)^popcount(b))
__device__ __forceinline__ void wh_signs(double (&h)[3][8]) {
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int b = 0; b < 8; ++b)
      if (__popc(b) & 1) h[c][b] = -h[c][b];
}
// the 8 signature blocks (3 x 3) times Ee, on Walsh coefficients
__device__ __forceinline__ void wh_blocks(const double* sk, double Ee, double (&h)[3][8]) {
#pragma unroll
  for (int sig = 0; sig < 8; ++sig) {
    const int i0 = sig ^ (1 << walsh_axis(0)), i1 = sig ^ (1 << walsh_axis(1)),
              i2 = sig ^ (1 << walsh_axis(2));
    const double m0 = h[0][i0], m1 = h[1][i1], m2 = h[2][i2];
    const double* k = sk + 6 * sig;
    h[0][i0] = Ee * fma(k[0], m0, fma(k[1], m1, k[2] * m2));
    h[1][i1] = Ee * fma(k[1], m0, fma(k[3], m1, k[4] * m2));
    h[2][i2] = Ee * fma(k[2], m0, fma(k[4], m1, k[5] * m2));
  }
}

// E_e Ke x_e for one hexahedron in Walsh coordinates (Ke = W Kt W', the
// blocks of k_elem_walsh): per component an 8-point Walsh-Hadamard transform
// of x_e, the 8 signature blocks (3x3), the inverse transform (S H S = H',
// H H' = 8 I); 216 flops per element instead of 576. h holds x_e on entry
// ([component][binary node index oi + 2 ok + 4 oj]) and the element's output
// on exit. sk: per signature k00, k01, k02, k11, k12, k22 (plain, not doubled).
__device__ __forceinline__ void walsh_elem_apply(const double* sk, double Ee, double (&h)[3][8]) {
  wh_butterfly(h);
  wh_blocks(sk, Ee, h);
  wh_signs(h);
  wh_butterfly(h);
  wh_signs(h);
}

// y += E_e Ke x_e over one colour for hexahedra in Walsh coordinates
__global__ void __launch_bounds__(256) k_mg_apply_walsh(MgGeo L, const double* __restrict__ kw,
                                                        const double* __restrict__ E, int color,
                                                        const double* __restrict__ x,
                                                        double* __restrict__ y) {
  __shared__ double sk[48];
  if (threadIdx.x < 48) sk[threadIdx.x] = kw[threadIdx.x];
  __syncthreads();
  const int cx = color & 1, cz = (color >> 1) & 1, cy = (color >> 2) & 1;
  const long long hx = (L.nelx - cx + 1) / 2, hz = (L.nz - cz + 1) / 2, hy = (L.nely - cy + 1) / 2;
  const long long tot = hx * hz * hy;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    const int ey = cy + 2 * int(t % hy);
    const long long u = t / hy;
    const int ez = cz + 2 * int(u % hz), ex = cx + 2 * int(u / hz);
    const long long e = ((long long)ex * L.nz + ez) * L.nely + ey;
    const long long n0 = ((long long)ex * L.nz1 + ez) * L.ny1 + ey;  // node (ey, ez, ex)
    double h[3][8];  // [component][binary node index oi + 2 ok + 4 oj]
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const long long nd = n0 + (b & 1) + ((b >> 1) & 1) * L.ny1 + ((b >> 2) & 1) * L.pl;
#pragma unroll
      for (int c = 0; c < 3; ++c) h[c][b] = x[3 * nd + c];
    }
    walsh_elem_apply(sk, E[e], h);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const long long nd = n0 + (b & 1) + ((b >> 1) & 1) * L.ny1 + ((b >> 2) & 1) * L.pl;
#pragma unroll
      for (int c = 0; c < 3; ++c) y[3 * nd + c] += h[c][b];
    }
  }
}

// y = K x for hexahedra in Walsh form, one launch, node-centric output: a block
// owns a tile of kTY x kTZ nodes in (y, z) and marches along x over a range
// of node layers. Per step it stages the next node layer of x in shared
// memory, computes one element layer (kTY+1 x kTZ+1 = 256 elements, one per
// thread), keeps the element outputs in shared memory, and gathers node layer
// ex from the element layers ex - 1 and ex. Every node sums its (up to) 8
// element contributions in colour order, exactly as the 8 colour launches of
// k_mg_apply_walsh do from y = 0, so the result is bitwise the same, with x and
// y touched once (the colour launches read and rewrite y 8 times).
// CG: y = 0 on fixed DOFs and per-block partials of x . y (k_state_matvec's
// contract).
// Level-1 Galerkin element operator applied on the fly (H8): Kc x_c =
// sum_p Q_p' (E_p Ke) Q_p x_c over the 8 children p of the coarse element, Q_p
// the trilinear interpolation to child p's nodes. Everything stays in Walsh
// coefficients: with h^ = H x_c, Q_p = H' T_p H / 8 where T_p is, per axis a,
// the pair map (u0, u1) -> (u0 + c_a u1, u1 / 2), c_a = +-1/2 the child's
// offset (a linear coarse mode restricted to a half cell); Ke = H' Kt H / 8
// gives Kc x_c = H' sum_p T_p' (E_p Kt T_p h^): one transform in and one out
// per coarse element, 72 + 105 + 72 flops per child. Algebraically the stored
// Kc = sum_p E_p Kp, without its 4.6 KB per coarse element. h: x_c in, Kc x_c
// out. Eb: the modulus of child (0, 0, 0), children at + (p & 1) + ((p >> 1) & 1)
// sz + (p >> 2) sx (null: an element outside the grid, all moduli 0).
__device__ __forceinline__ void mg_c1_elem(const double* sk, const double* __restrict__ Eb,
                                           long long sz, long long sx, double (&h)[3][8]) {
  wh_butterfly(h);
  double acc[3][8];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[c][b] = 0.0;
#pragma unroll 1
  for (int p = 0; p < 8; ++p) {
    const double* skp = sk;
    asm volatile("" : "+l"(skp));  // re-read the blocks per child: no 48 registers held
    const double Ep = Eb ? Eb[(p & 1) + ((p >> 1) & 1) * sz + (p >> 2) * sx] : 0.0;
    double g[3][8];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int b = 0; b < 8; ++b) g[c][b] = h[c][b];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double ca = ((p >> a) & 1) ? 0.5 : -0.5;
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int b = 0; b < 8; ++b)
          if (!(b & (1 << a))) {
            const double u1 = g[c][b | (1 << a)];
            g[c][b] = fma(ca, u1, g[c][b]);
            g[c][b | (1 << a)] = 0.5 * u1;
          }
    }
    wh_blocks(skp, Ep, g);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double ca = ((p >> a) & 1) ? 0.5 : -0.5;
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int b = 0; b < 8; ++b)
          if (!(b & (1 << a))) g[c][b | (1 << a)] = fma(ca, g[c][b], 0.5 * g[c][b | (1 << a)]);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int b = 0; b < 8; ++b) acc[c][b] += g[c][b];
  }
  wh_signs(acc);
  wh_butterfly(acc);
  wh_signs(acc);
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int b = 0; b < 8; ++b) h[c][b] = acc[c][b];
}

constexpr int kTY = 31, kTZ = 7;             // owned nodes per tile
constexpr int kEY = kTY + 1, kEZ = kTZ + 1;  // elements per layer (256)
constexpr int kNY = kTY + 2, kNZ = kTZ + 2;  // element nodes per layer
constexpr int kLX = kNY * kNZ * 3;           // doubles per staged node layer
constexpr int kCS = kEY * kEZ + 4;  // contribution row stride: rows r*3+c land 8 banks apart
constexpr int kTileSmem = (2 * kLX + 3 * 12 * kCS) * int(sizeof(double));

__host__ __device__ inline int tile_ny(const MgGeo& L) { return int((L.ny1 + kTY - 1) / kTY); }
__host__ __device__ inline int tile_nz(const MgGeo& L) { return (L.nz1 + kTZ - 1) / kTZ; }

// C1: level 1 of the hierarchy, elements by mg_c1_elem from the fine moduli E
// Epilogues (EPI): y = A x; CG: y = A x masked + dot partials; JACOBI: y = x +
// w (b - A x) / diag (0 on fixed; y must not alias x); RESIDUAL: y = b - A x
// (0 on fixed).
enum { kEpiApply = 0, kEpiCG = 1, kEpiJacobi = 2, kEpiResidual = 3 };
struct TileEpi {
  const double* b;
  const double* diag;
  double w;
  double* partials;
};

template <int EPI, bool C1 = false>
__global__ void __launch_bounds__(256, C1 ? 1 : 2) k_mg_apply_tile(MgGeo L, const double* __restrict__ kw,
                                                          const double* __restrict__ E,
                                                          const double* __restrict__ x,
                                                          double* __restrict__ y, int xchunk,
                                                          TileEpi ep) {
  constexpr bool CG = EPI == kEpiCG;
  static_assert(kEY * kEZ == 256, "one element per thread");
  extern __shared__ double smem[];
  double* xs = smem;             // [2][kLX] node layers (parity of the layer index)
  double* c0 = xs + 2 * kLX;     // [12][256] oj = 0 outputs of the current element layer
  double* c1 = c0 + 12 * kCS;    // [2][12][kCS] oj = 1 outputs (parity of the element layer)
  __shared__ double sk[48];
  __shared__ double scratch[32];
  if (threadIdx.x < 48) sk[threadIdx.x] = kw[threadIdx.x];
  const int nty = tile_ny(L), ntz = tile_nz(L);
  const int by = blockIdx.x % nty, bz = (blockIdx.x / nty) % ntz, bx = blockIdx.x / (nty * ntz);
  const int y0 = by * kTY, z0 = bz * kTZ;
  const int nx1 = L.nelx + 1;
  const int ix0 = bx * xchunk, ix1 = min(nx1, ix0 + xchunk);
  const int t = threadIdx.x;
  // node layers are staged through registers one step ahead (the global loads
  // of layer ex + 2 are in flight while element layer ex + 1 is computed)
  constexpr int kPer = (kLX + 255) / 256;
  double pre[kPer];
  auto fetch = [&](int lx) {
    const bool okx = lx >= 0 && lx < nx1;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int i = t + 256 * j;
      const int row = i / (3 * kNY), k = i - row * (3 * kNY);
      const int iz = z0 - 1 + row, iy = y0 - 1 + k / 3;
      double v = 0.0;
      if (i < kLX && okx && iz >= 0 && iz < L.nz1 && iy >= 0 && iy < L.ny1)
        v = x[3 * (((long long)lx * L.nz1 + iz) * L.ny1 + (y0 - 1)) + k];
      pre[j] = v;
    }
  };
  auto commit = [&](int lx) {
    double* dst = xs + (lx & 1) * kLX;
#pragma unroll
    for (int j = 0; j < kPer; ++j)
      if (t + 256 * j < kLX) dst[t + 256 * j] = pre[j];
  };
  const int ly = t % kEY, lz = t / kEY;  // this thread's element in the layer
  const int ey = y0 - 1 + ly, ez = z0 - 1 + lz;
  const bool okyz = ey >= 0 && ey < L.nely && ez >= 0 && ez < L.nz;
  auto fetchE = [&](int ex) {
    return okyz && ex >= 0 && ex < L.nelx ? E[((long long)ex * L.nz + ez) * L.nely + ey] : 0.0;
  };
  const int ony = t % kTY, onz = t / kTY;  // this thread's node (t < kTY * kTZ)
  const int iy = y0 + ony, iz = z0 + onz;
  const bool own = t < kTY * kTZ && iy < L.ny1 && iz < L.nz1;
  double dot = 0.0;
  fetch(ix0 - 1);
  commit(ix0 - 1);
  fetch(ix0);
  commit(ix0);
  fetch(ix0 + 1);
  double Enext = C1 ? 0.0 : fetchE(ix0 - 1);
  for (int ex = ix0 - 1; ex < ix1; ++ex) {
    __syncthreads();
    {  // element layer ex
      double h[3][8];
      const double* xa = xs + (ex & 1) * kLX;
      const double* xb = xs + ((ex + 1) & 1) * kLX;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const double* src = (b & 4) ? xb : xa;
        const int o = ((lz + ((b >> 1) & 1)) * kNY + ly + (b & 1)) * 3;
#pragma unroll
        for (int c = 0; c < 3; ++c) h[c][b] = src[o + c];
      }
      const bool ok = okyz && ex >= 0 && ex < L.nelx;
      if (C1) {
        const long long fny = 2 * L.nely, fnz = 2 * L.nz;
        const double* Eb = ok ? E + ((long long)(2 * ex) * fnz + 2 * ez) * fny + 2 * ey : nullptr;
        mg_c1_elem(sk, Eb, fny, fnz * fny, h);
      } else {
        const double Ee = Enext;
        Enext = fetchE(ex + 1);
        walsh_elem_apply(sk, Ee, h);
      }
      double* h1 = c1 + (ex & 1) * 12 * kCS;
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          c0[(r * 3 + c) * kCS + t] = ok ? h[c][r] : 0.0;
          h1[(r * 3 + c) * kCS + t] = ok ? h[c][r + 4] : 0.0;
        }
    }
    __syncthreads();
    if (ex >= ix0 && own) {  // node layer ix = ex
      const int ix = ex;
      const double* h1p = c1 + ((ex - 1) & 1) * 12 * kCS;
      double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int col = 0; col < 8; ++col) {
        const int cx = col & 1, cz = (col >> 1) & 1, cy = (col >> 2) & 1;
        const int oj = ((ix - 1) & 1) == cx ? 1 : 0;  // element layer ix - oj
        const int ok = ((iz - 1) & 1) == cz ? 1 : 0;
        const int oi = ((iy - 1) & 1) == cy ? 1 : 0;
        const int le = (onz + 1 - ok) * kEY + (ony + 1 - oi);  // element (ly, lz) in the tile
        const double* src = oj ? h1p : c0;
        const int r = oi + 2 * ok;
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c] += src[(r * 3 + c) * kCS + le];
      }
      const long long nd = ((long long)ix * L.nz1 + iz) * L.ny1 + iy;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const long long d = 3 * nd + c;
        if (CG) {
          const double v = L.fixed[d] ? 0.0 : acc[c];
          y[d] = v;
          dot = fma(x[d], v, dot);
        } else if (EPI == kEpiJacobi) {
          y[d] = L.fixed[d] ? 0.0 : x[d] + ep.w * (ep.b[d] - acc[c]) / ep.diag[d];
        } else if (EPI == kEpiResidual) {
          y[d] = L.fixed[d] ? 0.0 : ep.b[d] - acc[c];
        } else {
          y[d] = acc[c];
        }
      }
    }
    commit(ex + 2);  // (layer ex's buffer: read by the compute above, before the barrier)
    fetch(ex + 3);
  }
  if (CG) {
    double red[1] = {dot};
    block_sum<1>(red, scratch);
    if (threadIdx.x == 0) ep.partials[blockIdx.x] = red[0];
  }
}

// Node-centric operator on a level with stored (symmetric) element matrices,
// one launch instead of 8 colour launches: each node gathers its rows of the
// (up to 2^dim) elements around it, in ascending element order, so every
// matrix entry is read once per apply and y is written once. Rows are read as
// columns (the Galerkin matrices are stored exactly symmetric), contiguous.
// MODE 0: y = A x. MODE 1: damped Jacobi, y = x + w (b - A x) / diag (0 on
// fixed DOFs; y must not alias x). MODE 2: y = b - A x (0 on fixed DOFs).
// ROWS = DIM: all rows of node nd; ROWS = 1: row c0 only (small levels: 3x
// the threads, shorter dependency chains)
template <int DIM, int MODE, int ROWS = DIM>
__device__ __forceinline__ void mg_node_rows(const MgGeo& L, const double* __restrict__ K,
                                             const double* __restrict__ x,
                                             const double* __restrict__ b,
                                             const double* __restrict__ diag, double w,
                                             double* __restrict__ y, long long nd, int c0 = 0) {
  constexpr int NN = MgT<DIM>::NN, D = MgT<DIM>::D;
  const int iy = int(nd % L.ny1);
  const long long t = nd / L.ny1;
  const int iz = int(t % L.nz1), ix = int(t / L.nz1);
  double acc[ROWS];
#pragma unroll
  for (int c = 0; c < ROWS; ++c) acc[c] = 0.0;
#pragma unroll 1
  for (int q = 0; q < NN; ++q) {  // elements around the node, ascending
    const int ex = ix - 1 + (q >> (DIM == 3 ? 2 : 1) & 1);
    const int ez = DIM == 3 ? iz - 1 + (q >> 1 & 1) : 0;
    const int ey = iy - 1 + (q & 1);
    if (ex < 0 || ex >= L.nelx || ez < 0 || ez >= L.nz || ey < 0 || ey >= L.nely) continue;
    const long long e = ((long long)ex * L.nz + ez) * L.nely + ey;
    const int a = mg_local(DIM, iy - ey, iz - ez, ix - ex);
    double xe[D];
#pragma unroll
    for (int j = 0; j < D; ++j) xe[j] = __ldg(x + mg_dof<DIM>(L, ex, ez, ey, j));
#pragma unroll
    for (int c = 0; c < ROWS; ++c) {
      const double2* row = reinterpret_cast<const double2*>(K + e * (long long)(D * D) +
                                                            (DIM * a + c + c0) * D);
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < D / 2; ++j) {
        const double2 k = __ldg(row + j);
        s = fma(k.x, xe[2 * j], s);
        s = fma(k.y, xe[2 * j + 1], s);
      }
      acc[c] += s;
    }
  }
#pragma unroll
  for (int c = 0; c < ROWS; ++c) {
    const long long d = DIM * nd + c + c0;
    if (MODE == 0) {
      y[d] = acc[c];
    } else if (MODE == 1) {
      y[d] = L.fixed[d] ? 0.0 : x[d] + w * (b[d] - acc[c]) / diag[d];
    } else {
      y[d] = L.fixed[d] ? 0.0 : b[d] - acc[c];
    }
  }
}

template <int DIM, int MODE>
__global__ void __launch_bounds__(256) k_mg_node(MgGeo L, const double* __restrict__ K,
                                                 const double* __restrict__ x,
                                                 const double* __restrict__ b,
                                                 const double* __restrict__ diag, double w,
                                                 double* __restrict__ y) {
  for (long long nd = blockIdx.x * (long long)blockDim.x + threadIdx.x; nd < L.nn;
       nd += (long long)gridDim.x * blockDim.x)
    mg_node_rows<DIM, MODE>(L, K, x, b, diag, w, y, nd);
}

// One damped-Jacobi row of a small stored level by NN lanes (lane q takes the
// q-th element around the node; a fixed shuffle tree sums them): short
// dependency chains for the latency-bound coarsest level. All lanes of the
// group must call it (the shuffles); returns the new value on lane 0.
template <int DIM>
__device__ __forceinline__ double mg_row_lanes(const MgGeo& L, const double* __restrict__ K,
                                               const double* __restrict__ x, long long d, int q,
                                               bool valid) {
  constexpr int NN = MgT<DIM>::NN, D = MgT<DIM>::D;
  double s = 0.0;
  if (valid) {
    const long long nd = d / DIM;
    const int c = int(d - nd * DIM);
    const int iy = int(nd % L.ny1);
    const long long t = nd / L.ny1;
    const int iz = int(t % L.nz1), ix = int(t / L.nz1);
    const int ex = ix - 1 + (q >> (DIM == 3 ? 2 : 1) & 1);
    const int ez = DIM == 3 ? iz - 1 + (q >> 1 & 1) : 0;
    const int ey = iy - 1 + (q & 1);
    if (ex >= 0 && ex < L.nelx && ez >= 0 && ez < L.nz && ey >= 0 && ey < L.nely) {
      const long long e = ((long long)ex * L.nz + ez) * L.nely + ey;
      const int a = mg_local(DIM, iy - ey, iz - ez, ix - ex);
      const double2* row =
          reinterpret_cast<const double2*>(K + e * (long long)(D * D) + (DIM * a + c) * D);
#pragma unroll
      for (int j = 0; j < D / 2; ++j) {
        const double2 k = __ldg(row + j);
        const long long d0 = mg_dof<DIM>(L, ex, ez, ey, 2 * j), d1 = mg_dof<DIM>(L, ex, ez, ey, 2 * j + 1);
        s = fma(k.x, __ldg(x + d0), s);
        s = fma(k.y, __ldg(x + d1), s);
      }
    }
  }
#pragma unroll
  for (int o = NN / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, NN);
  return s;
}

// k_mg_node with NN lanes per row (stored levels: short dependency chains,
// NN x the threads). MODE as k_mg_node.
template <int DIM, int MODE>
__global__ void __launch_bounds__(256) k_mg_node_lanes(MgGeo L, const double* __restrict__ K,
                                                       const double* __restrict__ x,
                                                       const double* __restrict__ b,
                                                       const double* __restrict__ diag, double w,
                                                       double* __restrict__ y) {
  constexpr int NN = MgT<DIM>::NN;
  const int q = threadIdx.x % NN;
  const long long S = (long long)gridDim.x * blockDim.x / NN;
  const long long nrounds = (L.n + S - 1) / S;
  for (long long r = 0; r < nrounds; ++r) {  // uniform trip count: the shuffles need all lanes
    const long long d = r * S + (blockIdx.x * (long long)blockDim.x + threadIdx.x) / NN;
    const bool valid = d < L.n;
    const double ax = mg_row_lanes<DIM>(L, K, x, d, q, valid);
    if (!valid || q != 0) continue;
    if (MODE == 0)
      y[d] = ax;
    else if (MODE == 1)
      y[d] = L.fixed[d] ? 0.0 : x[d] + w * (b[d] - ax) / diag[d];
    else
      y[d] = L.fixed[d] ? 0.0 : b[d] - ax;
  }
}

// Exact solve on a small coarsest level (n <= kCoarseDenseMax): the dense
// matrix is gathered from the element matrices (fixed DOFs: identity rows and
// columns), inverted once per solve by blocked Gauss-Jordan (k_dense_inverse,
// SPD, no pivoting), and each V-cycle applies x = A^-1 b with one warp per row.
constexpr int kCoarseDenseMax = 4096;

// A[i][j] = sum over the elements holding both DOFs (ascending) of K_e(li, lj)
template <int DIM>
__global__ void k_mg_dense_gather(MgGeo L, const double* __restrict__ K, double* __restrict__ A) {
  constexpr int NN = MgT<DIM>::NN, D = MgT<DIM>::D;
  const long long n = L.n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n * n;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / n, j = t - i * n;
    if (L.fixed[i] || L.fixed[j]) {
      A[t] = i == j ? 1.0 : 0.0;
      continue;
    }
    const long long ni = i / DIM, nj = j / DIM;
    const int ci = int(i - ni * DIM), cj = int(j - nj * DIM);
    const int iy = int(ni % L.ny1), iz = int((ni / L.ny1) % L.nz1), ix = int(ni / L.pl);
    const int jy = int(nj % L.ny1), jz = int((nj / L.ny1) % L.nz1), jx = int(nj / L.pl);
    double a = 0.0;
    for (int q = 0; q < NN; ++q) {  // elements around node i, ascending
      const int ex = ix - 1 + (q >> (DIM == 3 ? 2 : 1) & 1);
      const int ez = DIM == 3 ? iz - 1 + (q >> 1 & 1) : 0;
      const int ey = iy - 1 + (q & 1);
      if (ex < 0 || ex >= L.nelx || ez < 0 || ez >= L.nz || ey < 0 || ey >= L.nely) continue;
      const int oj = jx - ex, ok = jz - ez, oi = jy - ey;  // node j inside this element?
      if (oj < 0 || oj > 1 || oi < 0 || oi > 1 || ok < 0 || ok > (DIM == 3 ? 1 : 0)) continue;
      const long long e = ((long long)ex * L.nz + ez) * L.nely + ey;
      const int li = DIM * mg_local(DIM, iy - ey, iz - ez, ix - ex) + ci;
      const int lj = DIM * mg_local(DIM, oi, ok, oj) + cj;
      a += K[e * (long long)(D * D) + (long long)lj * D + li];
    }
    A[t] = a;
  }
}

// In-place inverse of the SPD coarsest-grid matrix (row-major n x n) by
// blocked Gauss-Jordan (the sweep operator on panels of kGjB pivots), one
// cooperative launch, three grid barriers per panel (n = 1911 for C4 / C5:
// 60 panels). For pivot block P = A[K,K] and the rest R:
//   A[K,K] <- P^-1, A[K,R] <- W = P^-1 A[K,R], A[R,K] <- -A[R,K] P^-1,
//   A[R,R] <- A[R,R] - A[R,K] W
// (the column panel is copied to C first: its old values feed the update).
// No pivoting (SPD); a non-positive or non-finite pivot sets *bad (the caller
// then falls back to Jacobi sweeps on the coarsest grid).
constexpr int kGjB = 32, kGjT = 64;  // panel width, update tile (measured: 64-wide
                                     // panels are slower, C1 solve 55 vs 37 ms)
constexpr int kGjThreads = 128;
__global__ void __launch_bounds__(kGjThreads) k_dense_inverse(int n, double* __restrict__ A,
                                                              double* __restrict__ W,
                                                              double* __restrict__ Cp,
                                                              double* __restrict__ Pinv,
                                                              int* __restrict__ bad) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sP[kGjB][kGjB + 1];
  __shared__ double sC[kGjT][kGjB + 1];
  __shared__ double sW[kGjB][kGjT + 1];
  __shared__ double rowk[kGjB], colk[kGjB];
  const int tid = threadIdx.x;
  const long long S = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + tid;
  const int ntile = (n + kGjT - 1) / kGjT;
  for (int k0 = 0; k0 < n; k0 += kGjB) {
    const int b = min(kGjB, n - k0);
    // phase 1: block 0 inverts the pivot block; everyone copies the column panel
    if (blockIdx.x == 0) {
      for (int q = tid; q < b * b; q += blockDim.x) sP[q / b][q % b] = A[(long long)(k0 + q / b) * n + k0 + q % b];
      __syncthreads();
      for (int kk = 0; kk < b; ++kk) {
        if (tid < b) {
          rowk[tid] = sP[kk][tid];
          colk[tid] = sP[tid][kk];
        }
        __syncthreads();
        double piv = rowk[kk];
        if (!(piv > 0.0) || !(piv < INFINITY)) {
          if (tid == 0) *bad = 1;
          piv = 1.0;
        }
        const double inv = 1.0 / piv;
        for (int q = tid; q < b * b; q += blockDim.x) {
          const int i = q / b, j = q % b;
          double v;
          if (i == kk)
            v = j == kk ? inv : rowk[j] * inv;
          else
            v = j == kk ? -colk[i] * inv : fma(-colk[i], rowk[j] * inv, sP[i][j]);
          sP[i][j] = v;
        }
        __syncthreads();
      }
      for (int q = tid; q < b * b; q += blockDim.x) Pinv[q] = sP[q / b][q % b];
    }
    for (long long t = t0; t < (long long)n * b; t += S) {
      const int i = int(t / b), c = int(t % b);
      Cp[t] = A[(long long)i * n + k0 + c];
    }
    grid.sync();
    // phase 2: W = P^-1 A[K, :]
    for (long long t = t0; t < (long long)b * n; t += S) {
      const int r = int(t / n), j = int(t % n);
      double pv[kGjB], av[kGjB];  // every load of the row issued before the FMAs
#pragma unroll
      for (int q = 0; q < kGjB; ++q) {
        pv[q] = q < b ? __ldcg(Pinv + r * b + q) : 0.0;
        av[q] = q < b ? A[(long long)(k0 + q) * n + j] : 0.0;
      }
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < kGjB; ++q) acc = fma(pv[q], av[q], acc);
      W[t] = acc;
    }
    grid.sync();
    // phase 3: every 64 x 64 tile of A, 8 x 4 outputs per thread
    for (int tile = blockIdx.x; tile < ntile * ntile; tile += gridDim.x) {
      const int I0 = (tile / ntile) * kGjT, J0 = (tile % ntile) * kGjT;
      __syncthreads();
      {  // tile fill: all 2 x 16 loads of a thread in flight at once
        constexpr int NL = kGjT * kGjB / kGjThreads;
        double lc[NL], lw[NL];
#pragma unroll
        for (int it = 0; it < NL; ++it) {
          const int q = tid + kGjThreads * it;
          const int i = q / kGjB, c = q % kGjB;
          lc[it] = (I0 + i < n && c < b) ? __ldcg(Cp + (long long)(I0 + i) * b + c) : 0.0;
          const int r = q / kGjT, j = q % kGjT;
          lw[it] = (J0 + j < n && r < b) ? __ldcg(W + (long long)r * n + J0 + j) : 0.0;
        }
#pragma unroll
        for (int it = 0; it < NL; ++it) {
          const int q = tid + kGjThreads * it;
          sC[q / kGjB][q % kGjB] = lc[it];
          sW[q / kGjT][q % kGjT] = lw[it];
        }
      }
      for (int q = tid; q < b * b; q += blockDim.x)  // (block-local copy of P^-1)
        sP[q / b][q % b] = __ldcg(Pinv + q);
      __syncthreads();
      const int ti = (tid / 16) * 8, tj = (tid % 16) * 4;
      double acc[8][4] = {};
      for (int c = 0; c < b; ++c) {
        double cv[8], wv[4];
#pragma unroll
        for (int u = 0; u < 8; ++u) cv[u] = sC[ti + u][c];
#pragma unroll
        for (int v = 0; v < 4; ++v) wv[v] = sW[c][tj + v];
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fma(cv[u], wv[v], acc[u][v]);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int i = I0 + ti + u, j = J0 + tj + v;
          if (i >= n || j >= n) continue;
          const bool iK = i >= k0 && i < k0 + b, jK = j >= k0 && j < k0 + b;
          double* a = A + (long long)i * n + j;
          if (iK && jK) {
            *a = sP[i - k0][j - k0];
          } else if (iK) {
            *a = sW[i - k0][tj + v];
          } else if (jK) {
            double s2 = 0.0;
            for (int c = 0; c < b; ++c) s2 = fma(sC[ti + u][c], sP[c][j - k0], s2);
            *a = -s2;
          } else {
            *a -= acc[u][v];
          }
        }
    }
    grid.sync();
  }
}

// x = A^-1 b, one warp per row (fixed-order lane sums + shuffle tree)
__global__ void k_dense_matvec(int n, const double* __restrict__ Ainv, const double* __restrict__ b,
                               double* __restrict__ x) {
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += (gridDim.x * blockDim.x) >> 5) {
    const double* r = Ainv + (long long)i * n;
    double s = 0.0;
    for (int j = lane; j < n; j += 32) s = fma(__ldg(r + j), __ldg(b + j), s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) x[i] = s;
  }
}

// The coarsest level's Jacobi sweeps in one cooperative launch: x = w b / diag,
// then sweeps - 1 damped-Jacobi sweeps ping-ponging x <-> y with a grid
// barrier between sweeps; the result ends in x.
template <int DIM>
__global__ void __launch_bounds__(256) k_mg_coarse_sweeps(MgGeo L, const double* __restrict__ K,
                                                          const double* __restrict__ b,
                                                          const double* __restrict__ diag, double w,
                                                          double* __restrict__ x,
                                                          double* __restrict__ y, int sweeps) {
  cg::grid_group grid = cg::this_grid();
  const long long S = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (long long d = t0; d < L.n; d += S) x[d] = L.fixed[d] ? 0.0 : w * b[d] / diag[d];
  double *src = x, *dst = y;
  constexpr int NN = MgT<DIM>::NN;
  const int q = threadIdx.x % NN;
  const long long ng = S / NN;  // lane groups in the grid (blockDim is a multiple of NN)
  const long long nrounds = (L.n + ng - 1) / ng;
  for (int s = 1; s < sweeps; ++s) {
    grid.sync();
    for (long long r = 0; r < nrounds; ++r) {  // uniform trip count: the shuffles need all lanes
      const long long d = r * ng + t0 / NN;
      const bool valid = d < L.n;
      const double ax = mg_row_lanes<DIM>(L, K, src, d, q, valid);
      if (valid && q == 0) dst[d] = L.fixed[d] ? 0.0 : src[d] + w * (b[d] - ax) / diag[d];
    }
    double* tmp = src;
    src = dst;
    dst = tmp;
  }
  if (src != x) {
    grid.sync();
    for (long long d = t0; d < L.n; d += S) x[d] = src[d];
  }
}

// level-1 Jacobi diagonal from the fine moduli: sum_p E_p Kp[p](l, l)
template <int DIM>
__global__ void k_mg_diag_c1(MgGeo L, const double* __restrict__ Kp, const double* __restrict__ E,
                             double* __restrict__ diag) {
  constexpr int NN = MgT<DIM>::NN, D = MgT<DIM>::D;
  for (long long nd = blockIdx.x * (long long)blockDim.x + threadIdx.x; nd < L.nn;
       nd += (long long)gridDim.x * blockDim.x) {
    const int iy = int(nd % L.ny1);
    const long long t = nd / L.ny1;
    const int iz = int(t % L.nz1), ix = int(t / L.nz1);
    double acc[DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c) acc[c] = 0.0;
    for (int q = 0; q < NN; ++q) {
      const int ex = ix - 1 + (q >> (DIM == 3 ? 2 : 1) & 1);
      const int ez = DIM == 3 ? iz - 1 + (q >> 1 & 1) : 0;
      const int ey = iy - 1 + (q & 1);
      if (ex < 0 || ex >= L.nelx || ez < 0 || ez >= L.nz || ey < 0 || ey >= L.nely) continue;
      const int a = mg_local(DIM, iy - ey, iz - ez, ix - ex);
      for (int c = 0; c < DIM; ++c) {
        const int l = DIM * a + c;
        double s = 0.0;
        for (int p = 0; p < NN; ++p) {
          int pi, pk, pj;
          mg_offsets(p, pi, pk, pj);
          const long long ef =
              ((long long)(2 * ex + pj) * (DIM == 3 ? 2 * L.nz : 1) + (DIM == 3 ? 2 * ez + pk : 0)) *
                  (2 * L.nely) + (2 * ey + pi);
          s = fma(E[ef], Kp[p * D * D + l * D + l], s);
        }
        acc[c] += s;
      }
    }
    for (int c = 0; c < DIM; ++c) {
      const long long d = DIM * nd + c;
      diag[d] = L.fixed[d] ? 1.0 : acc[c];
    }
  }
}

// Point-block Jacobi (H8 levels 0 and 1): the inverse of each node's 3 x 3
// diagonal block, from E and Ke (level 0) or from the fine moduli and the 8
// Kp = Qp' Ke Qp (level 1, on the fly like the operator); fixed DOFs get
// identity rows / columns. Stored as 9 doubles per node (row-major).
template <bool C1>
__global__ void k_mg_bdiag(MgGeo L, const double* __restrict__ K, const double* __restrict__ E,
                           double* __restrict__ Binv) {
  constexpr int D = 24, DD = D * D;
  for (long long nd = blockIdx.x * (long long)blockDim.x + threadIdx.x; nd < L.nn;
       nd += (long long)gridDim.x * blockDim.x) {
    const int iy = int(nd % L.ny1);
    const long long t = nd / L.ny1;
    const int iz = int(t % L.nz1), ix = int(t / L.nz1);
    double B[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int q = 0; q < 8; ++q) {  // elements around the node, ascending
      const int ex = ix - 1 + (q >> 2 & 1), ez = iz - 1 + (q >> 1 & 1), ey = iy - 1 + (q & 1);
      if (ex < 0 || ex >= L.nelx || ez < 0 || ez >= L.nz || ey < 0 || ey >= L.nely) continue;
      const int a = mg_local(3, iy - ey, iz - ez, ix - ex);
      if (!C1) {
        const double Ee = E[((long long)ex * L.nz + ez) * L.nely + ey];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) B[i][j] = fma(Ee, K[(3 * a + j) * D + 3 * a + i], B[i][j]);
      } else {
        for (int p = 0; p < 8; ++p) {
          int pi, pk, pj;
          mg_offsets(p, pi, pk, pj);
          const long long ef = ((long long)(2 * ex + pj) * (2 * L.nz) + 2 * ez + pk) * (2 * L.nely) +
                               (2 * ey + pi);
          const double Ep = E[ef];
          for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
              B[i][j] = fma(Ep, K[p * DD + (3 * a + j) * D + 3 * a + i], B[i][j]);
        }
      }
    }
    for (int c = 0; c < 3; ++c)
      if (L.fixed[3 * nd + c])
        for (int k = 0; k < 3; ++k) B[c][k] = B[k][c] = (k == c ? 1.0 : 0.0);
    // symmetric 3 x 3 inverse by cofactors
    const double c00 = B[1][1] * B[2][2] - B[1][2] * B[2][1];
    const double c01 = B[1][2] * B[2][0] - B[1][0] * B[2][2];
    const double c02 = B[1][0] * B[2][1] - B[1][1] * B[2][0];
    const double det = B[0][0] * c00 + B[0][1] * c01 + B[0][2] * c02;
    const double id = 1.0 / det;
    double* o = Binv + 9 * nd;
    o[0] = c00 * id;
    o[1] = (B[0][2] * B[2][1] - B[0][1] * B[2][2]) * id;
    o[2] = (B[0][1] * B[1][2] - B[0][2] * B[1][1]) * id;
    o[3] = c01 * id;
    o[4] = (B[0][0] * B[2][2] - B[0][2] * B[2][0]) * id;
    o[5] = (B[0][2] * B[1][0] - B[0][0] * B[1][2]) * id;
    o[6] = c02 * id;
    o[7] = (B[0][1] * B[2][0] - B[0][0] * B[2][1]) * id;
    o[8] = (B[0][0] * B[1][1] - B[0][1] * B[1][0]) * id;
  }
}

// point-block Jacobi step per node: MODE 0: x = x + w Binv (b - Ax) (Ax null:
// x = w Binv b), 0 on fixed DOFs; MODE 1: out = Binv (Ax) with Ax masked to 0
// on fixed DOFs (power iteration for lambda_max(Binv A))
template <int MODE>
__global__ void k_mg_jacobi_b(long long nn, const unsigned char* __restrict__ fixed,
                              const double* __restrict__ b, const double* __restrict__ Ax,
                              const double* __restrict__ Binv, double w, double* __restrict__ x) {
  for (long long nd = blockIdx.x * (long long)blockDim.x + threadIdx.x; nd < nn;
       nd += (long long)gridDim.x * blockDim.x) {
    double r[3];
    bool fx[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const long long d = 3 * nd + c;
      fx[c] = fixed[d] != 0;
      const double v = MODE == 1 ? Ax[d] : (Ax ? b[d] - Ax[d] : b[d]);
      r[c] = fx[c] ? 0.0 : v;
    }
    const double* m = Binv + 9 * nd;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const long long d = 3 * nd + c;
      const double z = fma(m[3 * c], r[0], fma(m[3 * c + 1], r[1], m[3 * c + 2] * r[2]));
      if (MODE == 1)
        x[d] = fx[c] ? 0.0 : z;
      else
        x[d] = fx[c] ? 0.0 : (Ax ? x[d] : 0.0) + w * z;
    }
  }
}

// Jacobi diagonal (fixed DOFs: 1), node-centric
template <int DIM, bool FINE>
__global__ void k_mg_diag(MgGeo L, const double* __restrict__ K, const double* __restrict__ E,
                          double* __restrict__ diag) {
  constexpr int NN = MgT<DIM>::NN, D = MgT<DIM>::D;
  for (long long nd = blockIdx.x * (long long)blockDim.x + threadIdx.x; nd < L.nn;
       nd += (long long)gridDim.x * blockDim.x) {
    const int iy = int(nd % L.ny1);
    const long long t = nd / L.ny1;
    const int iz = int(t % L.nz1), ix = int(t / L.nz1);
    double acc[DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c) acc[c] = 0.0;
    for (int q = 0; q < NN; ++q) {  // elements around the node, ascending
      const int ex = ix - 1 + (q >> (DIM == 3 ? 2 : 1) & 1);
      const int ez = DIM == 3 ? iz - 1 + (q >> 1 & 1) : 0;
      const int ey = iy - 1 + (q & 1);
      if (ex < 0 || ex >= L.nelx || ez < 0 || ez >= L.nz || ey < 0 || ey >= L.nely) continue;
      const long long e = ((long long)ex * L.nz + ez) * L.nely + ey;
      const int a = mg_local(DIM, iy - ey, iz - ez, ix - ex);
      for (int c = 0; c < DIM; ++c) {
        const int l = DIM * a + c;
        acc[c] += FINE ? E[e] * K[l * D + l] : K[e * (long long)(D * D) + l * D + l];
      }
    }
    for (int c = 0; c < DIM; ++c) {
      const long long d = DIM * nd + c;
      diag[d] = L.fixed[d] ? 1.0 : acc[c];
    }
  }
}

// r_c = P' r_f (full weighting), zero on fixed coarse DOFs
template <int DIM>
__global__ void k_mg_restrict(MgGeo C, MgGeo F, const double* __restrict__ rf, double* __restrict__ rc) {
  for (long long N = blockIdx.x * (long long)blockDim.x + threadIdx.x; N < C.nn;
       N += (long long)gridDim.x * blockDim.x) {
    const int iy = int(N % C.ny1);
    const long long t = N / C.ny1;
    const int iz = int(t % C.nz1), ix = int(t / C.nz1);
    double acc[DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c) acc[c] = 0.0;
    for (int dx = -1; dx <= 1; ++dx)
      for (int dz = (DIM == 3 ? -1 : 0); dz <= (DIM == 3 ? 1 : 0); ++dz)
        for (int dy = -1; dy <= 1; ++dy) {
          const int fx = 2 * ix + dx, fz = 2 * iz + dz, fy = 2 * iy + dy;
          if (fx < 0 || fx > F.nelx || fz < 0 || fz >= F.nz1 || fy < 0 || fy > F.nely) continue;
          const double w = (dx ? 0.5 : 1.0) * (dz ? 0.5 : 1.0) * (dy ? 0.5 : 1.0);
          const long long n = ((long long)fx * F.nz1 + fz) * F.ny1 + fy;
          for (int c = 0; c < DIM; ++c) acc[c] = fma(w, rf[DIM * n + c], acc[c]);
        }
    for (int c = 0; c < DIM; ++c) {
      const long long d = DIM * N + c;
      rc[d] = C.fixed[d] ? 0.0 : acc[c];
    }
  }
}

// x_f += P e_c (linear interpolation), fixed fine DOFs untouched
template <int DIM>
__global__ void k_mg_prolong_add(MgGeo C, MgGeo F, const double* __restrict__ ec,
                                 double* __restrict__ xf) {
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < F.nn;
       n += (long long)gridDim.x * blockDim.x) {
    const int fy = int(n % F.ny1);
    const long long t = n / F.ny1;
    const int fz = int(t % F.nz1), fx = int(t / F.nz1);
    double acc[DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c) acc[c] = 0.0;
    const int x0 = fx >> 1, x1 = (fx + 1) >> 1, z0 = fz >> 1, z1 = (fz + 1) >> 1, y0 = fy >> 1,
              y1 = (fy + 1) >> 1;
    for (int X = x0; X <= x1; ++X)
      for (int Z = z0; Z <= z1; ++Z)
        for (int Y = y0; Y <= y1; ++Y) {
          const double w = (x1 > x0 ? 0.5 : 1.0) * (z1 > z0 ? 0.5 : 1.0) * (y1 > y0 ? 0.5 : 1.0);
          const long long N = ((long long)X * C.nz1 + Z) * C.ny1 + Y;
          for (int c = 0; c < DIM; ++c) acc[c] = fma(w, ec[DIM * N + c], acc[c]);
        }
    for (int c = 0; c < DIM; ++c) {
      const long long d = DIM * n + c;
      if (!F.fixed[d]) xf[d] += acc[c];
    }
  }
}

// x += w (b - Ax) / diag on free DOFs (Ax null: x = 0 before, x = w b / diag)
__global__ void k_mg_jacobi(long long n, const unsigned char* __restrict__ fixed,
                            const double* __restrict__ b, const double* __restrict__ Ax,
                            const double* __restrict__ diag, double w, double* __restrict__ x) {
  for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < n;
       d += (long long)gridDim.x * blockDim.x) {
    if (fixed[d]) {
      x[d] = 0.0;
      continue;
    }
    const double r = Ax ? b[d] - Ax[d] : b[d];
    x[d] = (Ax ? x[d] : 0.0) + w * r / diag[d];
  }
}

// r = b - Ax (0 on fixed)
__global__ void k_mg_residual(long long n, const unsigned char* __restrict__ fixed,
                              const double* __restrict__ b, const double* __restrict__ Ax,
                              double* __restrict__ r) {
  for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < n;
       d += (long long)gridDim.x * blockDim.x)
    r[d] = fixed[d] ? 0.0 : b[d] - Ax[d];
}

// power-iteration step for lambda_max(D^-1 A): x <- (D^-1 A x) / ||D^-1 A x|| is
// done on the host side from w = D^-1 (A x) (0 on fixed DOFs)
__global__ void k_mg_dinv(long long n, const unsigned char* __restrict__ fixed,
                          const double* __restrict__ Ax, const double* __restrict__ diag,
                          double* __restrict__ w) {
  for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < n;
       d += (long long)gridDim.x * blockDim.x)
    w[d] = fixed[d] ? 0.0 : Ax[d] / diag[d];
}
// x = s * w, and x = 1 on free DOFs when init
__global__ void k_mg_scale(long long n, const unsigned char* __restrict__ fixed, int init, double s,
                           const double* __restrict__ w, double* __restrict__ x) {
  for (long long d = blockIdx.x * (long long)blockDim.x + threadIdx.x; d < n;
       d += (long long)gridDim.x * blockDim.x)
    x[d] = fixed[d] ? 0.0 : (init ? 1.0 + 1e-3 * double(d % 7) : s * w[d]);
}

// coarse fixed mask: coarse DOF fixed when its coinciding fine DOF is fixed
template <int DIM>
__global__ void k_mg_fixed(MgGeo C, MgGeo F, const unsigned char* __restrict__ ff,
                           unsigned char* __restrict__ fc) {
  for (long long N = blockIdx.x * (long long)blockDim.x + threadIdx.x; N < C.nn;
       N += (long long)gridDim.x * blockDim.x) {
    const int iy = int(N % C.ny1);
    const long long t = N / C.ny1;
    const int iz = int(t % C.nz1), ix = int(t / C.nz1);
    const long long n = ((long long)(2 * ix) * F.nz1 + 2 * iz) * F.ny1 + 2 * iy;
    for (int c = 0; c < DIM; ++c) fc[DIM * N + c] = ff[DIM * n + c];
  }
}

}  // namespace topo
