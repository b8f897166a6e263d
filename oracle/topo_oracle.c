/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle (plain C restatement) of the
 * design-update hot path of arxiv/paper_2005_05436. See topo_oracle.h for the
 * usage rules and how it is pinned. References "grid.hpp:N" etc. are to
 * /root/reference/proj/include/topopt/.
 *
 * Floating-point statements keep the reference's operation order; the
 * reference is built without FMA contraction (proj/CMakeLists.txt has no
 * -march), so this file is compiled with -ffp-contract=off.
 * OpenMP parallelises only over output elements of the convolution
 * (per-element summation order preserved, bitwise equal to one thread);
 * every scalar reduction stays sequential.
 */
#include "topo_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static __thread char g_err[512];
static void set_err(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}
const char* orc_last_error(void) { return g_err; }

int orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

/* the benchmark input generator (not a reference
 * function; both sides consume identical arrays) */
static inline uint64_t orc_splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void orc_generate(uint64_t seed, uint64_t stream, int kind, double a, double b, int64_t offset,
                  int64_t count, double* out) {
  const uint64_t key = orc_splitmix64(seed ^ orc_splitmix64(stream + 0x632BE59BD9B4E019ull));
  const double two53 = 1.0 / 9007199254740992.0;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < count; ++t) {
    const uint64_t idx = (uint64_t)(offset + t);
    if (kind == 0) {
      out[t] = a + (b - a) * ((double)(orc_splitmix64(key + idx) >> 11) * two53);
    } else {
      const uint64_t k = idx >> 1;
      const double u1 = ((double)(orc_splitmix64(key + 2 * k) >> 11) + 1.0) * two53;
      const double u2 = (double)(orc_splitmix64(key + 2 * k + 1) >> 11) * two53;
      const double rad = sqrt(-2.0 * log(u1));
      const double ang = 6.283185307179586 * u2;
      out[t] = a + b * ((idx & 1) ? rad * sin(ang) : rad * cos(ang));
    }
  }
}

/* std::max / std::min semantics (return the first argument unless the second
 * compares strictly greater / smaller), used by oc.hpp:36,49-51,59 */
static inline double std_max(double a, double b) { return (a < b) ? b : a; }
static inline double std_min(double a, double b) { return (b < a) ? b : a; }

/* ------------------------------------------------------------------ grid.hpp */

static int is3d(orc_grid g) { return g.nelz > 0; }

/* grid.hpp:26-33 */
int64_t orc_num_elements(orc_grid g) {
  return (int64_t)g.nelx * g.nely * (is3d(g) ? g.nelz : 1);
}
int64_t orc_num_dofs(orc_grid g) {
  int64_t nn = (int64_t)(g.nelx + 1) * (g.nely + 1);
  if (is3d(g)) nn *= (g.nelz + 1);
  return (is3d(g) ? 3 : 2) * nn;
}

/* grid.hpp:82-85 */
static int validate_grid(orc_grid g) {
  if (g.nelx < 1 || g.nely < 1 || g.nelz < 0) {
    set_err("grid: element counts must be >= 1 per active axis");
    return ORC_EINVAL;
  }
  return ORC_OK;
}

/* grid.hpp:36-41 */
static inline int64_t node2(orc_grid g, int i, int j) { return (int64_t)j * (g.nely + 1) + i; }
static inline int64_t node3(orc_grid g, int i, int k, int j) {
  return ((int64_t)j * (g.nelz + 1) + k) * (g.nely + 1) + i;
}

/* grid.hpp:89-131 */
int orc_build_connectivity(orc_grid g, int32_t* dofs) {
  int st = validate_grid(g);
  if (st) return st;
  if (orc_num_dofs(g) > INT32_MAX) {
    set_err("grid: DOF count %lld exceeds 32-bit index range", (long long)orc_num_dofs(g));
    return ORC_EOVERFLOW;
  }
  int32_t* out = dofs;
  if (!is3d(g)) {
    for (int j = 0; j < g.nelx; ++j)
      for (int i = 0; i < g.nely; ++i) {
        const int32_t nodes[4] = {(int32_t)node2(g, i + 1, j), (int32_t)node2(g, i + 1, j + 1),
                                  (int32_t)node2(g, i, j + 1), (int32_t)node2(g, i, j)};
        for (int a = 0; a < 4; ++a) {
          *out++ = 2 * nodes[a];
          *out++ = 2 * nodes[a] + 1;
        }
      }
  } else {
    for (int j = 0; j < g.nelx; ++j)
      for (int k = 0; k < g.nelz; ++k)
        for (int i = 0; i < g.nely; ++i) {
          const int32_t nodes[8] = {
              (int32_t)node3(g, i + 1, k, j),     (int32_t)node3(g, i + 1, k, j + 1),
              (int32_t)node3(g, i, k, j + 1),     (int32_t)node3(g, i, k, j),
              (int32_t)node3(g, i + 1, k + 1, j), (int32_t)node3(g, i + 1, k + 1, j + 1),
              (int32_t)node3(g, i, k + 1, j + 1), (int32_t)node3(g, i, k + 1, j)};
          for (int a = 0; a < 8; ++a) {
            *out++ = 3 * nodes[a];
            *out++ = 3 * nodes[a] + 1;
            *out++ = 3 * nodes[a] + 2;
          }
        }
  }
  return ORC_OK;
}

/* grid.hpp:133-153 */
int orc_build_index_pairs(orc_grid g, int32_t* iK, int32_t* jK) {
  const int64_t m = orc_num_elements(g);
  const int d = is3d(g) ? 24 : 8;
  int32_t* conn = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m * d));
  if (!conn) {
    set_err("oracle: out of memory");
    return ORC_EINVAL;
  }
  int st = orc_build_connectivity(g, conn);
  if (st) {
    free(conn);
    return st;
  }
  int64_t t = 0;
  for (int64_t e = 0; e < m; ++e) {
    const int32_t* row = conn + e * d;
    for (int jl = 0; jl < d; ++jl)
      for (int il = jl; il < d; ++il) {
        const int32_t a = row[il], b = row[jl];
        iK[t] = a > b ? a : b;
        jK[t] = a < b ? a : b;
        ++t;
      }
  }
  free(conn);
  return ORC_OK;
}

static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* grid.hpp:155-188 -> per-element state 0 act / 1 pasS / 2 pasV */
int orc_partition(orc_grid g, const int32_t* pasS, int64_t nS, const int32_t* pasV, int64_t nV,
                  uint8_t* state) {
  int st = validate_grid(g);
  if (st) return st;
  const int64_t m = orc_num_elements(g);
  int32_t* s = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nS + 1));
  int32_t* v = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nV + 1));
  if (nS) memcpy(s, pasS, sizeof(int32_t) * (size_t)nS);
  if (nV) memcpy(v, pasV, sizeof(int32_t) * (size_t)nV);
  qsort(s, (size_t)nS, sizeof(int32_t), cmp_i32);
  qsort(v, (size_t)nV, sizeof(int32_t), cmp_i32);
  if ((nS && (s[0] < 0 || s[nS - 1] >= m))) {
    set_err("partition: pasS contains an element index outside [0, m)");
    st = ORC_EINVAL;
  } else if (nV && (v[0] < 0 || v[nV - 1] >= m)) {
    set_err("partition: pasV contains an element index outside [0, m)");
    st = ORC_EINVAL;
  }
  if (!st) {
    memset(state, 0, (size_t)m);
    for (int64_t q = 0; q < nS; ++q) state[s[q]] = 1;
    for (int64_t q = 0; q < nV; ++q) {
      if (q > 0 && v[q] == v[q - 1]) continue; /* unique */
      if (state[v[q]] != 0) {
        set_err("partition: passive solid and void sets overlap at element %d", v[q]);
        st = ORC_EINVAL;
        break;
      }
      state[v[q]] = 2;
    }
  }
  free(s);
  free(v);
  return st;
}

/* ------------------------------------------------------------------- fea.hpp */

/* fea.hpp:33-40 */
static void lower_cm(const double* full, int d, double* lower) {
  int64_t t = 0;
  for (int j = 0; j < d; ++j)
    for (int i = j; i < d; ++i) lower[t++] = full[j * d + i];
}

/* fea.hpp:51-68 (Q4) and fea.hpp:73-121 (H8). `full` is column-major d x d.
 * The H8 accumulation 0.125 * B' * D * B is evaluated left to right
 * ((0.125 B') D) B with sequential inner sums. */
int orc_element_stiffness(int dim, double nu, double* full, double* lower) {
  if (!(nu > -1.0 && nu < 0.5)) {
    set_err("element stiffness: Poisson ratio must lie in (-1, 0.5)");
    return ORC_EINVAL;
  }
  if (dim == 2) {
    const double k[8] = {0.5 - nu / 6.0,          0.125 + nu / 8.0,  -0.25 - nu / 12.0,
                         -0.125 + 3.0 * nu / 8.0, -0.25 + nu / 12.0, -0.125 - nu / 8.0,
                         nu / 6.0,                0.125 - 3.0 * nu / 8.0};
    static const int pattern[8][8] = {
        {0, 1, 2, 3, 4, 5, 6, 7}, {1, 0, 7, 6, 5, 4, 3, 2}, {2, 7, 0, 5, 6, 3, 4, 1},
        {3, 6, 5, 0, 7, 2, 1, 4}, {4, 5, 6, 7, 0, 1, 2, 3}, {5, 4, 3, 2, 1, 0, 7, 6},
        {6, 3, 4, 1, 2, 7, 0, 5}, {7, 2, 1, 4, 3, 6, 5, 0}};
    const double scale = 1.0 / (1.0 - nu * nu);
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) full[j * 8 + i] = scale * k[pattern[i][j]];
    lower_cm(full, 8, lower);
    return ORC_OK;
  }
  if (dim != 3) {
    set_err("element stiffness: dim must be 2 or 3");
    return ORC_EINVAL;
  }
  const double lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  const double mu = 1.0 / (2.0 * (1.0 + nu));
  static const double cx[8] = {0, 1, 1, 0, 0, 1, 1, 0};
  static const double cy[8] = {0, 0, 1, 1, 0, 0, 1, 1};
  static const double cz[8] = {0, 0, 0, 0, 1, 1, 1, 1};
  double D[6][6];
  memset(D, 0, sizeof D);
  D[0][0] = D[1][1] = D[2][2] = lam + 2.0 * mu;
  D[0][1] = D[0][2] = D[1][0] = D[1][2] = D[2][0] = D[2][1] = lam;
  D[3][3] = D[4][4] = D[5][5] = mu;
  const double gp[2] = {0.5 - 0.5 / sqrt(3.0), 0.5 + 0.5 / sqrt(3.0)};
  double kfull[24][24]; /* kfull[i][j] */
  memset(kfull, 0, sizeof kfull);
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b)
      for (int c = 0; c < 2; ++c) {
        const double x = gp[a], y = gp[b], z = gp[c];
        double B[6][24];
        memset(B, 0, sizeof B);
        for (int node = 0; node < 8; ++node) {
          const double lx = cx[node] > 0.5 ? x : 1.0 - x;
          const double ly = cy[node] > 0.5 ? y : 1.0 - y;
          const double lz = cz[node] > 0.5 ? z : 1.0 - z;
          const double sx = cx[node] > 0.5 ? 1.0 : -1.0;
          const double sy = cy[node] > 0.5 ? 1.0 : -1.0;
          const double sz = cz[node] > 0.5 ? 1.0 : -1.0;
          const double dNdx = sx * ly * lz;
          const double dNdy = lx * sy * lz;
          const double dNdz = lx * ly * sz;
          const int col = 3 * node;
          B[0][col] = dNdx;
          B[1][col + 1] = dNdy;
          B[2][col + 2] = dNdz;
          B[3][col + 1] = dNdz;
          B[3][col + 2] = dNdy;
          B[4][col] = dNdz;
          B[4][col + 2] = dNdx;
          B[5][col] = dNdy;
          B[5][col + 1] = dNdx;
        }
        double T2[24][6];
        for (int i = 0; i < 24; ++i)
          for (int l = 0; l < 6; ++l) {
            double s = 0;
            for (int k = 0; k < 6; ++k) s += (B[k][i] * 0.125) * D[k][l];
            T2[i][l] = s;
          }
        for (int j = 0; j < 24; ++j)
          for (int i = 0; i < 24; ++i) {
            double s = 0;
            for (int l = 0; l < 6; ++l) s += T2[i][l] * B[l][j];
            kfull[i][j] += s;
          }
      }
  for (int j = 0; j < 24; ++j)
    for (int i = 0; i < 24; ++i) full[j * 24 + i] = (kfull[i][j] + kfull[j][i]) * 0.5;
  lower_cm(full, 24, lower);
  return ORC_OK;
}

/* fea.hpp:135-146 */
void orc_simp(int64_t m, const double* xhat, double e0, double emin, double p, double* sK,
              double* dsK) {
  const double de = e0 - emin;
  for (int64_t e = 0; e < m; ++e) {
    const double xp = pow(xhat[e], p - 1.0);
    if (sK) sK[e] = emin + xp * xhat[e] * de;
    if (dsK) dsK[e] = p * xp * de;
  }
}

/* fea.hpp:162-169: value[t = e*P + q] = sK_e * Ke_lower[q] */
void orc_assemble_values(int64_t m, int P, const double* sK, const double* ke_lower,
                         double* vals) {
  int64_t t = 0;
  for (int64_t e = 0; e < m; ++e) {
    const double s = sK[e];
    for (int q = 0; q < P; ++q, ++t) vals[t] = s * ke_lower[q];
  }
}

/* fea.hpp:154-176 assemble_lower: the triplets (iK[t], jK[t], sK[e] * Ke_lower[q])
 * of t = e*P + q through Eigen's setFromTriplets (restated from its published
 * algorithm, Eigen 3.x SparseMatrix::setFromTriplets): triplets are bucketed
 * by outer index (column, ColMajor) in input order, duplicates summed in that
 * order (collapseDuplicates, scalar_sum_op), inner (row) indices ascending.
 * Two calls: col_ptr/row_idx/values NULL returns nnz only. */
int orc_assemble_lower(orc_grid g, double nu, const double* sK, int32_t* col_ptr,
                       int32_t* row_idx, double* values, int64_t* nnz) {
  const int dim = g.nelz > 0 ? 3 : 2, d = dim == 3 ? 24 : 8, P = d * (d + 1) / 2;
  const int64_t m = (int64_t)g.nelx * g.nely * (g.nelz > 0 ? g.nelz : 1);
  const int64_t n = (int64_t)dim * (g.nelx + 1) * (g.nely + 1) * (g.nelz > 0 ? g.nelz + 1 : 1);
  const int64_t T = m * P;
  double kf[576], kl[300];
  if (orc_element_stiffness(dim, nu, kf, kl)) return 1;
  int32_t* iK = malloc(sizeof(int32_t) * T);
  int32_t* jK = malloc(sizeof(int32_t) * T);
  int64_t* start = calloc((size_t)n + 1, sizeof(int64_t));
  int64_t* order = malloc(sizeof(int64_t) * T);
  int rc = orc_build_index_pairs(g, iK, jK);
  if (!rc) {
    for (int64_t t = 0; t < T; ++t) ++start[jK[t] + 1];
    for (int64_t c = 0; c < n; ++c) start[c + 1] += start[c];
    int64_t* fill = malloc(sizeof(int64_t) * n);
    for (int64_t c = 0; c < n; ++c) fill[c] = start[c];
    for (int64_t t = 0; t < T; ++t) order[fill[jK[t]]++] = t; /* input order per column */
    free(fill);
    /* per column: distinct rows ascending, each summed over its triplets in input order */
    int64_t k = 0;
    if (col_ptr) col_ptr[0] = 0;
    for (int64_t c = 0; c < n; ++c) {
      const int64_t a = start[c], b = start[c + 1];
      /* stable insertion sort of this column's triplets by row (input order kept on ties) */
      for (int64_t i = a + 1; i < b; ++i) {
        const int64_t v = order[i];
        int64_t j = i - 1;
        while (j >= a && iK[order[j]] > iK[v]) {
          order[j + 1] = order[j];
          --j;
        }
        order[j + 1] = v;
      }
      for (int64_t i = a; i < b; ++i) {
        const int64_t t = order[i];
        const double v = sK[t / P] * kl[t % P]; /* fea.hpp:168 */
        if (i == a || iK[t] != iK[order[i - 1]]) {
          if (row_idx) row_idx[k] = iK[t];
          if (values) values[k] = v;
          ++k;
        } else if (values) {
          values[k - 1] += v;
        }
      }
      if (col_ptr) col_ptr[c + 1] = (int32_t)k;
    }
    *nnz = k;
  }
  free(iK);
  free(jK);
  free(start);
  free(order);
  return rc;
}

/* fea.hpp:248-272 */
int orc_compliance_sensitivity(orc_grid g, const double* ke_full, const double* u,
                               const double* xhat, double e0, double emin, double p,
                               const uint8_t* state, double* c, double* dc) {
  const int64_t m = orc_num_elements(g);
  const int d = is3d(g) ? 24 : 8;
  int32_t* conn = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m * d));
  int st = orc_build_connectivity(g, conn);
  if (st) {
    free(conn);
    return st;
  }
  const double de = e0 - emin;
  double csum = 0;
  for (int64_t e = 0; e < m; ++e) {
    const int32_t* row = conn + e * d;
    double ue[24], ku[24];
    for (int a = 0; a < d; ++a) ue[a] = u[row[a]];
    for (int i = 0; i < d; ++i) { /* ke.full * ue, fea.hpp:267 */
      double s = 0;
      for (int k = 0; k < d; ++k) s += ke_full[k * d + i] * ue[k];
      ku[i] = s;
    }
    double quad = 0;
    for (int i = 0; i < d; ++i) quad += ue[i] * ku[i];
    const double xp = pow(xhat[e], p - 1.0); /* simp_interpolate, fea.hpp:256 */
    const double sK = emin + xp * xhat[e] * de;
    const double dsK = p * xp * de;
    csum += sK * quad;
    dc[e] = (!state || state[e] == 0) ? -dsK * quad : 0.0;
  }
  *c = csum;
  free(conn);
  return ORC_OK;
}

/* ---------------------------------------------------------------- filter.hpp */

struct orc_filter {
  orc_grid g;
  double rmin;
  int bc; /* 0 Neumann (mirror), 1 Dirichlet (zero) */
  int ntaps;
  int32_t *di, *dj, *dk;
  double* w;
  double* hs;
};

/* filter.hpp:43-48 */
static inline int reflect_index(int t, int n) {
  const int period = 2 * n;
  t %= period;
  if (t < 0) t += period;
  return t < n ? t : period - 1 - t;
}

/* filter.hpp:50-91 */
void orc_cone_convolve(const orc_filter* f, const double* v, double* out) {
  const int nx = f->g.nelx, ny = f->g.nely, nz = f->g.nelz;
  const int mirror = f->bc == 0;
  const int T = f->ntaps;
  if (!is3d(f->g)) {
#pragma omp parallel for schedule(static)
    for (int j = 0; j < nx; ++j)
      for (int i = 0; i < ny; ++i) {
        double acc = 0;
        for (int t = 0; t < T; ++t) {
          int ii = i + f->di[t], jj = j + f->dj[t];
          if (mirror) {
            ii = reflect_index(ii, ny);
            jj = reflect_index(jj, nx);
          } else if (ii < 0 || ii >= ny || jj < 0 || jj >= nx) {
            continue;
          }
          acc += f->w[t] * v[(int64_t)jj * ny + ii];
        }
        out[(int64_t)j * ny + i] = acc;
      }
  } else {
#pragma omp parallel for collapse(2) schedule(static)
    for (int j = 0; j < nx; ++j)
      for (int k = 0; k < nz; ++k)
        for (int i = 0; i < ny; ++i) {
          double acc = 0;
          for (int t = 0; t < T; ++t) {
            int ii = i + f->di[t], jj = j + f->dj[t], kk = k + f->dk[t];
            if (mirror) {
              ii = reflect_index(ii, ny);
              jj = reflect_index(jj, nx);
              kk = reflect_index(kk, nz);
            } else if (ii < 0 || ii >= ny || jj < 0 || jj >= nx || kk < 0 || kk >= nz) {
              continue;
            }
            acc += f->w[t] * v[((int64_t)jj * nz + kk) * ny + ii];
          }
          out[((int64_t)j * nz + k) * ny + i] = acc;
        }
  }
}

/* filter.hpp:95-117 */
orc_filter* orc_filter_create(orc_grid g, double rmin, int bc) {
  if (validate_grid(g)) return NULL;
  if (rmin < 1.0) {
    set_err("filter: rmin must be >= 1 element");
    return NULL;
  }
  orc_filter* f = (orc_filter*)calloc(1, sizeof *f);
  f->g = g;
  f->rmin = rmin;
  f->bc = bc;
  const int reach = (int)ceil(rmin) - 1;
  const int dkMax = is3d(g) ? reach : 0;
  const int64_t cap = (int64_t)(2 * reach + 1) * (2 * reach + 1) * (2 * dkMax + 1);
  f->di = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap);
  f->dj = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap);
  f->dk = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap);
  f->w = (double*)malloc(sizeof(double) * (size_t)cap);
  int n = 0;
  for (int dj = -reach; dj <= reach; ++dj)
    for (int dk = -dkMax; dk <= dkMax; ++dk)
      for (int di = -reach; di <= reach; ++di) {
        const double dist = sqrt((double)di * di + (double)dj * dj + (double)dk * dk);
        const double w = rmin - dist;
        if (w > 0) {
          f->di[n] = di;
          f->dj[n] = dj;
          f->dk[n] = dk;
          f->w[n] = w;
          ++n;
        }
      }
  f->ntaps = n;
  const int64_t m = orc_num_elements(g);
  double* ones = (double*)malloc(sizeof(double) * (size_t)m);
  for (int64_t e = 0; e < m; ++e) ones[e] = 1.0;
  f->hs = (double*)malloc(sizeof(double) * (size_t)m);
  orc_cone_convolve(f, ones, f->hs);
  free(ones);
  return f;
}

void orc_filter_destroy(orc_filter* f) {
  if (!f) return;
  free(f->di);
  free(f->dj);
  free(f->dk);
  free(f->w);
  free(f->hs);
  free(f);
}
int orc_filter_ntaps(const orc_filter* f) { return f->ntaps; }
void orc_filter_taps(const orc_filter* f, int32_t* di, int32_t* dj, int32_t* dk, double* w) {
  for (int t = 0; t < f->ntaps; ++t) {
    di[t] = f->di[t];
    dj[t] = f->dj[t];
    dk[t] = f->dk[t];
    w[t] = f->w[t];
  }
}
const double* orc_filter_hs(const orc_filter* f) { return f->hs; }

/* filter.hpp:119-122 */
void orc_apply_filter(const orc_filter* f, const double* x, double* out) {
  const int64_t m = orc_num_elements(f->g);
  orc_cone_convolve(f, x, out);
  for (int64_t e = 0; e < m; ++e) out[e] = out[e] / f->hs[e];
}

/* filter.hpp:126-129 */
void orc_apply_filter_adjoint(const orc_filter* f, const double* g, double* out) {
  const int64_t m = orc_num_elements(f->g);
  double* tmp = (double*)malloc(sizeof(double) * (size_t)m);
  for (int64_t e = 0; e < m; ++e) tmp[e] = g[e] / f->hs[e];
  orc_cone_convolve(f, tmp, out);
  free(tmp);
}

/* filter.hpp:137-144 */
void orc_project(int64_t m, const double* xt, double eta, double beta, double* out) {
  const double a = tanh(beta * eta);
  const double denom = a + tanh(beta * (1.0 - eta));
  for (int64_t e = 0; e < m; ++e) out[e] = (a + tanh(beta * (xt[e] - eta))) / denom;
}

/* filter.hpp:146-154 */
void orc_project_derivative(int64_t m, const double* xt, double eta, double beta, double* out) {
  const double denom = tanh(beta * eta) + tanh(beta * (1.0 - eta));
  for (int64_t e = 0; e < m; ++e) {
    const double th = tanh(beta * (xt[e] - eta));
    out[e] = beta * (1.0 - th * th) / denom;
  }
}

/* filter.hpp:157-161 */
double orc_project_eta_derivative(double xt, double eta, double b) {
  const double sech = 1.0 / cosh(b * (xt - eta));
  return -b / sinh(b) * sech * sech * sinh(b * xt) * sinh(b * (1.0 - xt));
}

/* filter.hpp:166-171 */
void orc_backfilter(const orc_filter* f, const double* g, const double* xt, double eta,
                    double beta, int proj_on, double* out) {
  if (!proj_on) {
    orc_apply_filter_adjoint(f, g, out);
    return;
  }
  const int64_t m = orc_num_elements(f->g);
  double* tmp = (double*)malloc(sizeof(double) * (size_t)m);
  orc_project_derivative(m, xt, eta, beta, tmp);
  for (int64_t e = 0; e < m; ++e) tmp[e] = tmp[e] * g[e];
  orc_apply_filter_adjoint(f, tmp, out);
  free(tmp);
}

/* filter.hpp:187-196 */
double orc_eta_mismatch(int64_t m, const double* xt, double beta, double eta,
                        const uint8_t* state) {
  const double a = tanh(beta * eta);
  const double denom = a + tanh(beta * (1.0 - eta));
  double g = 0;
  for (int64_t e = 0; e < m; ++e) {
    if (state && state[e]) continue;
    const double t = xt[e];
    g += (a + tanh(beta * (t - eta))) / denom - t;
  }
  return g / (double)m;
}

/* filter.hpp:197-201 */
static double eta_slope(int64_t m, const double* xt, double beta, double eta,
                        const uint8_t* state) {
  double gp = 0;
  for (int64_t e = 0; e < m; ++e) {
    if (state && state[e]) continue;
    gp += orc_project_eta_derivative(xt[e], eta, beta);
  }
  return gp / (double)m;
}

/* filter.hpp:182-228 */
int orc_solve_eta(int64_t m, const double* xt, double beta, double eta0, const uint8_t* state,
                  double* eta_out, int* iters) {
  if (!(beta > 0)) {
    set_err("eta solve: beta must be positive");
    return ORC_EINVAL;
  }
  double lo = 0.0, hi = 1.0;
  double eta = eta0 < 0.0 ? 0.0 : (eta0 > 1.0 ? 1.0 : eta0); /* std::clamp */
  const double tol = 1e-6;
  const int maxIter = 50;
  int it_done = 0;
  double g = orc_eta_mismatch(m, xt, beta, eta, state);
  double step = INFINITY;
  for (int it = 0; it < maxIter && (fabs(g) > tol || step > 1e-8); ++it) {
    if (g > 0)
      lo = eta;
    else
      hi = eta;
    const double gp = eta_slope(m, xt, beta, eta, state);
    double next = eta - g / gp;
    if (!isfinite(next) || next <= lo || next >= hi) next = 0.5 * (lo + hi);
    step = fabs(next - eta);
    eta = next;
    g = orc_eta_mismatch(m, xt, beta, eta, state);
    it_done = it + 1;
  }
  *eta_out = eta;
  if (iters) *iters = it_done;
  return ORC_OK;
}

/* -------------------------------------------------------------------- oc.hpp */

/* oc.hpp:31-39 */
double orc_lambda_upper(int64_t n, const double* xAct, const double* dcAct, const double* dVAct,
                        double volfrac, int64_t mTotal) {
  double s = 0;
  for (int64_t e = 0; e < n; ++e) s += xAct[e] * sqrt(std_max(0.0, -dcAct[e] / dVAct[e]));
  const double root = s / ((double)mTotal * volfrac);
  return root * root;
}

/* oc.hpp:44-53 */
static void oc_candidate_into(int64_t n, const double* xAct, const double* ocP,
                              double sqrtLambda, double move, double* out) {
  for (int64_t e = 0; e < n; ++e) {
    const double f = sqrtLambda > 0 ? ocP[e] / sqrtLambda : (ocP[e] > 0 ? INFINITY : 0.0);
    const double lowerBound = std_max(0.0, xAct[e] - move);
    const double upperBound = std_min(1.0, xAct[e] + move);
    out[e] = std_min(std_max(f, lowerBound), upperBound);
  }
}

/* oc.hpp:55-61 */
static void oc_constant(int64_t n, const double* xAct, const double* dcAct, const double* dVAct,
                        double* ocP) {
  for (int64_t e = 0; e < n; ++e) ocP[e] = xAct[e] * sqrt(std_max(0.0, -dcAct[e] / dVAct[e]));
}

/* oc.hpp:72-79 */
int orc_oc_candidate(int64_t n, const double* xAct, const double* dcAct, const double* dVAct,
                     double lambda, double move, double* out) {
  if (!(lambda > 0)) {
    set_err("oc: multiplier must be positive");
    return ORC_EINVAL;
  }
  double* ocP = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  oc_constant(n, xAct, dcAct, dVAct, ocP);
  oc_candidate_into(n, xAct, ocP, sqrt(lambda), move, out);
  free(ocP);
  return ORC_OK;
}

/* oc.hpp:108 */
static void scatter_act(int64_t nact, const int32_t* act, const double* cand, double* xNew) {
  for (int64_t q = 0; q < nact; ++q) xNew[act[q]] = cand[q];
}

typedef struct {
  int64_t m, nact;
  const int32_t* act;
  const uint8_t* state;
  const orc_filter* f;
  double eta, beta;
  int mode;
  orc_volume_fn cb;
  void* user;
  double* xNew;
  double* tmp;
  const double* cw; /* identity weights */
  double pinnedS;   /* |P1| */
} vol_ctx;

/* the volume callbacks of driver.hpp:214-229 plus the identity mode */
static double phys_volume(vol_ctx* v) {
  const int64_t m = v->m;
  switch (v->mode) {
    case ORC_VOL_CALLBACK:
      return v->cb(v->user, v->xNew, m);
    case ORC_VOL_MEAN: { /* driver.hpp:216 */
      double s = 0;
      for (int64_t e = 0; e < m; ++e) s += v->xNew[e];
      return s / (double)m;
    }
    case ORC_VOL_PROJECTED:   /* driver.hpp:218-222 */
    case ORC_VOL_FILTERED: {  /* driver.hpp:224-228 */
      orc_apply_filter(v->f, v->xNew, v->tmp);
      if (v->state)
        for (int64_t e = 0; e < m; ++e) {
          if (v->state[e] == 1) v->tmp[e] = 1.0;
          else if (v->state[e] == 2) v->tmp[e] = 0.0;
        }
      if (v->mode == ORC_VOL_PROJECTED) orc_project(m, v->tmp, v->eta, v->beta, v->tmp);
      double s = 0;
      for (int64_t e = 0; e < m; ++e) s += v->tmp[e];
      return s / (double)m;
    }
    case ORC_VOL_IDENTITY: { /* mean(pin(H xc)) = (|P1| + c . xc) / m, c = H' 1_notP */
      double s = 0;
      for (int64_t e = 0; e < m; ++e) s += v->cw[e] * v->xNew[e];
      return (v->pinnedS + s) / (double)m;
    }
  }
  return NAN;
}

/* oc.hpp:93-174 */
/* oc.hpp:181-241 primal_dual_update: the clamped resize alternated with the
 * closed-form dual map over the unclamped set until the multiplier stagnates
 * (|lm' - lm| <= pdTol); falls back to bisect_update with the mean volume
 * (oc.hpp:190-193) when the budget, the sums or the map degenerate, or after
 * 1000 iterations. *fell_back = 1 then, and *iterations is the bisection count. */
int orc_primal_dual_update(int64_t m, const double* x, const double* dc, const double* dV,
                           const uint8_t* state, const orc_oc_params* prm, double pd_tol,
                           double* xNew, double* lambda_out, int* iterations_out,
                           int* fell_back) {
  int64_t nact = 0, nS = 0;
  for (int64_t e = 0; e < m; ++e) {
    nact += (!state || state[e] == 0);
    nS += (state && state[e] == 1);
  }
  int32_t* act = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nact + 1));
  double* xAct = (double*)malloc(sizeof(double) * (size_t)(nact + 1));
  double* dcAct = (double*)malloc(sizeof(double) * (size_t)(nact + 1));
  double* dVAct = (double*)malloc(sizeof(double) * (size_t)(nact + 1));
  double* ocP = (double*)malloc(sizeof(double) * (size_t)(nact + 1));
  double* upper = (double*)malloc(sizeof(double) * (size_t)(nact + 1));
  double* lower = (double*)malloc(sizeof(double) * (size_t)(nact + 1));
  {
    int64_t q = 0;
    for (int64_t e = 0; e < m; ++e)
      if (!state || state[e] == 0) act[q++] = (int32_t)e;
  }
  for (int64_t q = 0; q < nact; ++q) {
    xAct[q] = x[act[q]];
    dcAct[q] = dc[act[q]];
    dVAct[q] = dV[act[q]];
  }
  oc_constant(nact, xAct, dcAct, dVAct, ocP);
  int fb = 0, it = 0;
  double lm = 0;
  const double budget = prm->volfrac * (double)m - (double)nS; /* oc.hpp:195 */
  if (budget <= 0) fb = 1;
  if (!fb) {
    for (int64_t q = 0; q < nact; ++q) {
      upper[q] = std_min(1.0, xAct[q] + prm->move); /* oc.hpp:199-202 */
      lower[q] = std_max(0.0, xAct[q] - prm->move);
    }
    double s = 0;
    for (int64_t q = 0; q < nact; ++q) s += ocP[q];
    lm = s / ((double)m * prm->volfrac); /* oc.hpp:204 */
    if (!(lm > 0)) fb = 1;
  }
  for (; !fb; ++it) {
    if (it >= 1000) {
      fb = 1;
      break;
    }
    double sumClamped = 0, sumMid = 0;
    int64_t numMid = 0;
    for (int64_t q = 0; q < nact; ++q) {
      const double f = ocP[q] / lm;
      if (f > upper[q])
        sumClamped += upper[q];
      else if (f < lower[q])
        sumClamped += lower[q];
      else {
        sumMid += ocP[q];
        ++numMid;
      }
    }
    if (numMid == 0) {
      fb = 1;
      break;
    }
    const double den = budget - sumClamped;
    if (den <= 0) {
      fb = 1;
      break;
    }
    const double lmNext = sumMid / den;
    if (!(lmNext > 0) || !isfinite(lmNext)) {
      fb = 1;
      break;
    }
    const int done = fabs(lmNext - lm) <= pd_tol;
    lm = lmNext;
    if (done) break;
  }
  int rc = ORC_OK;
  if (fb) {
    orc_oc_params bp = *prm;
    int evals = 0;
    rc = orc_bisect_update(m, x, dc, dV, state, &bp, ORC_VOL_MEAN, NULL, 0.0, 0.0, NULL, NULL, xNew,
                           lambda_out, iterations_out, &evals);
  } else {
    memcpy(xNew, x, sizeof(double) * (size_t)m); /* oc.hpp:233-236 */
    oc_candidate_into(nact, xAct, ocP, lm, prm->move, upper);
    for (int64_t q = 0; q < nact; ++q) xNew[act[q]] = upper[q];
    *lambda_out = lm * lm;
    *iterations_out = it;
  }
  if (fell_back) *fell_back = fb;
  free(act);
  free(xAct);
  free(dcAct);
  free(dVAct);
  free(ocP);
  free(upper);
  free(lower);
  return rc;
}

int orc_bisect_update(int64_t m, const double* x, const double* dc, const double* dV,
                      const uint8_t* state, const orc_oc_params* prm, int volume_mode,
                      const orc_filter* f, double eta, double beta, orc_volume_fn cb, void* user,
                      double* xNew, double* lambda_out, int* bisections_out, int* evals_out) {
  int st = ORC_OK;
  int64_t nact = 0;
  for (int64_t e = 0; e < m; ++e) nact += (!state || state[e] == 0);
  int32_t* act = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nact + 1));
  double* xAct = (double*)malloc(sizeof(double) * (size_t)(nact + 1));
  double* dcAct = (double*)malloc(sizeof(double) * (size_t)(nact + 1));
  double* dVAct = (double*)malloc(sizeof(double) * (size_t)(nact + 1));
  double* ocP = (double*)malloc(sizeof(double) * (size_t)(nact + 1));
  double* cand = (double*)malloc(sizeof(double) * (size_t)(nact + 1));
  {
    int64_t q = 0;
    for (int64_t e = 0; e < m; ++e)
      if (!state || state[e] == 0) act[q++] = (int32_t)e;
  }
  for (int64_t q = 0; q < nact; ++q) { /* detail::take, oc.hpp:63-67 */
    xAct[q] = x[act[q]];
    dcAct[q] = dc[act[q]];
    dVAct[q] = dV[act[q]];
  }
  oc_constant(nact, xAct, dcAct, dVAct, ocP);
  memcpy(xNew, x, sizeof(double) * (size_t)m); /* res.xNew = x */

  vol_ctx vc;
  memset(&vc, 0, sizeof vc);
  vc.m = m;
  vc.nact = nact;
  vc.act = act;
  vc.state = state;
  vc.f = f;
  vc.eta = eta;
  vc.beta = beta;
  vc.mode = volume_mode;
  vc.cb = cb;
  vc.user = user;
  vc.xNew = xNew;
  vc.tmp = (double*)malloc(sizeof(double) * (size_t)m);
  double* cw = NULL;
  if (volume_mode == ORC_VOL_IDENTITY) {
    double* notP = (double*)malloc(sizeof(double) * (size_t)m);
    cw = (double*)malloc(sizeof(double) * (size_t)m);
    double pS = 0;
    for (int64_t e = 0; e < m; ++e) {
      notP[e] = (!state || state[e] == 0) ? 1.0 : 0.0;
      if (state && state[e] == 1) pS += 1.0;
    }
    orc_apply_filter_adjoint(f, notP, cw);
    free(notP);
    vc.cw = cw;
    vc.pinnedS = pS;
  }
  int evals = 0;
#define VOLUME_AT(s_)                                                        \
  (oc_candidate_into(nact, xAct, ocP, (s_), prm->move, cand),                \
   scatter_act(nact, act, cand, xNew), ++evals, phys_volume(&vc))

  int bis = 0;
  double lam_res = 0;
  double lamMax = prm->lambda_max > 0
                      ? prm->lambda_max
                      : orc_lambda_upper(nact, xAct, dcAct, dVAct, prm->volfrac, m);
  if (!(lamMax > 0)) {
    (void)VOLUME_AT(1.0);
    lam_res = 0;
    goto done;
  }
  {
    double vHi = VOLUME_AT(sqrt(lamMax));
    int widenings = 0;
    while (vHi > prm->volfrac && widenings++ < 40) {
      lamMax *= 4.0;
      vHi = VOLUME_AT(sqrt(lamMax));
    }
    double vLo = VOLUME_AT(0.0);
    const double monoSlack = 1e-9;

    if (prm->lambda_space) {
      double lo = 0.0, hi = lamMax, lam = lamMax;
      while (hi - lo > prm->abs_tol && bis < 4000) {
        lam = 0.5 * (lo + hi);
        const double v = VOLUME_AT(sqrt(lam));
        if (v > vLo + monoSlack || v < vHi - monoSlack) {
          set_err("oc: candidate volume is not monotone in the multiplier");
          st = ORC_ENONMONO;
          goto done;
        }
        if (v > prm->volfrac) {
          lo = lam;
          vLo = v;
        } else {
          hi = lam;
          vHi = v;
        }
        ++bis;
      }
      lam_res = lam;
      goto done;
    }

    double lo = 0.0, hi = sqrt(lamMax), mid = hi;
    double v = vLo;
    while ((hi - lo) / (hi + lo) > prm->bisect_rel_tol ||
           (fabs(v - prm->volfrac) > 0.5 * prm->volume_tol && bis < 200)) {
      mid = 0.5 * (lo + hi);
      v = VOLUME_AT(mid);
      if (v > vLo + monoSlack || v < vHi - monoSlack) {
        set_err("oc: candidate volume is not monotone in the multiplier");
        st = ORC_ENONMONO;
        goto done;
      }
      if (v > prm->volfrac) {
        lo = mid;
        vLo = v;
      } else {
        hi = mid;
        vHi = v;
      }
      if (++bis >= 500) break;
    }
    (void)VOLUME_AT(mid);
    lam_res = mid * mid;
  }
done:
#undef VOLUME_AT
  if (lambda_out) *lambda_out = lam_res;
  if (bisections_out) *bisections_out = bis;
  if (evals_out) *evals_out = evals;
  free(act);
  free(xAct);
  free(dcAct);
  free(dVAct);
  free(ocP);
  free(cand);
  free(vc.tmp);
  free(cw);
  return st;
}

/* ---------------------------------------------------------------- driver.hpp */

/* driver.hpp:130-133 */
static void pin_passives(int64_t m, double* field, const uint8_t* state) {
  if (!state) return;
  for (int64_t e = 0; e < m; ++e) {
    if (state[e] == 1) field[e] = 1.0;
    else if (state[e] == 2) field[e] = 0.0;
  }
}

/* driver.hpp:183-231 (ft = 3); the state solve is skipped: u is an input */
int orc_design_pass(orc_grid g, const orc_filter* f, const double* ke_full,
                    const uint8_t* state, const double* x, const double* u,
                    const orc_pass_params* prm, orc_pass_out* out) {
  const int64_t m = orc_num_elements(g);
  int st;
  /* RL.1 */
  orc_apply_filter(f, x, out->xTilde);
  pin_passives(m, out->xTilde, state);
  if (isnan(prm->eta_override)) {
    st = orc_solve_eta(m, out->xTilde, prm->beta, prm->eta0, state, &out->eta, &out->eta_iters);
    if (st) return st;
  } else {
    out->eta = prm->eta_override;
    out->eta_iters = 0;
  }
  orc_project(m, out->xTilde, out->eta, prm->beta, out->xPhys);
  /* RL.2 (material law only) */
  orc_simp(m, out->xPhys, prm->e0, prm->emin, prm->penal, out->sKe, NULL);
  /* RL.3 */
  st = orc_compliance_sensitivity(g, ke_full, u, out->xPhys, prm->e0, prm->emin, prm->penal,
                                  state, &out->c, out->dcPhys);
  if (st) return st;
  orc_backfilter(f, out->dcPhys, out->xTilde, out->eta, prm->beta, 1, out->dc);
  double* dV0 = (double*)malloc(sizeof(double) * (size_t)m); /* driver.hpp:154-155 */
  for (int64_t e = 0; e < m; ++e) dV0[e] = (!state || state[e] == 0) ? 1.0 / (double)m : 0.0;
  orc_backfilter(f, dV0, out->xTilde, out->eta, prm->beta, 1, out->dV);
  free(dV0);
  /* RL.4 */
  orc_oc_params oc = {prm->move, prm->volfrac, 1e-4, 1e-3, 0, 1e-8, 0.0};
  return orc_bisect_update(m, x, out->dc, out->dV, state, &oc, prm->volume_mode, f, out->eta,
                           prm->beta, NULL, NULL, out->xNew, &out->lambda, &out->bisections,
                           &out->evaluations);
}
