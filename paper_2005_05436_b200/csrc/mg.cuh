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
    const int q = int(t - e * DD);
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

// Kc[e] = sum_p Qp' Kf[child p] Qp (levels >= 2); one block per coarse element
template <int DIM>
__global__ void __launch_bounds__(256) k_mg_galerkin(MgGeo C, MgGeo F, const double* __restrict__ Kf,
                                                     const double* __restrict__ Q,
                                                     double* __restrict__ Kc) {
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
        sK[q] = Kf[ef * DD + q];
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
#pragma unroll
    for (int r = 0; r < (DD + 255) / 256; ++r) {
      const int q = threadIdx.x + 256 * r;
      if (q < DD) Kc[e * DD + q] = acc[r];
    }
    __syncthreads();
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

// y += E_e Ke x_e over one colour for hexahedra in Walsh coordinates
// (Ke = W Kt W', the blocks of k_elem_walsh): per component an 8-point
// Walsh-Hadamard transform of x_e, the 8 signature blocks (3x3), the inverse
// transform; 216 flops per element instead of 576. kw: per signature k00,
// k01, k02, k11, k12, k22 (plain, not doubled).
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
    const double Ee = E[e];
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
    // W g = D B(D g): the butterfly B is W' = D H (H symmetric Sylvester,
    // D = (-1)^popcount on the index), so the inverse needs the sign flips
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int b = 0; b < 8; ++b)
        if (__popc(b) & 1) h[c][b] = -h[c][b];
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
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const long long nd = n0 + (b & 1) + ((b >> 1) & 1) * L.ny1 + ((b >> 2) & 1) * L.pl;
      const double sg = (__popc(b) & 1) ? -1.0 : 1.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) y[3 * nd + c] += sg * h[c][b];
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
