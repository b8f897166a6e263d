// Host-side setup helpers of the C-ABI (no device work): the unit-modulus
// element matrices (fea.hpp:51-121) and the counter-based input generator of
// SURVEY.md Appendix B.
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "../../include/topo_capi.h"

namespace {

void lower_cm(const double* full, int d, double* lower) {  // fea.hpp:33-40
  int64_t t = 0;
  for (int j = 0; j < d; ++j)
    for (int i = j; i < d; ++i) lower[t++] = full[j * d + i];
}

inline uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace

extern "C" {

// fea.hpp:51-68 (Q4, closed form) and fea.hpp:73-121 (H8, 2x2x2 Gauss). The
// H8 product 0.125 B' D B is accumulated ((0.125 B') D) B with sequential
// inner sums; full = 0.5 (K + K') as fea.hpp:118.
topo_status topo_element_stiffness(int dim, double nu, double* full, double* lower) {
  if (!(nu > -1.0 && nu < 0.5)) return TOPO_EINVAL;
  if (dim == 2) {
    const double k[8] = {0.5 - nu / 6.0,          0.125 + nu / 8.0,  -0.25 - nu / 12.0,
                         -0.125 + 3.0 * nu / 8.0, -0.25 + nu / 12.0, -0.125 - nu / 8.0,
                         nu / 6.0,                0.125 - 3.0 * nu / 8.0};
    static const int pat[8][8] = {{0, 1, 2, 3, 4, 5, 6, 7}, {1, 0, 7, 6, 5, 4, 3, 2},
                                  {2, 7, 0, 5, 6, 3, 4, 1}, {3, 6, 5, 0, 7, 2, 1, 4},
                                  {4, 5, 6, 7, 0, 1, 2, 3}, {5, 4, 3, 2, 1, 0, 7, 6},
                                  {6, 3, 4, 1, 2, 7, 0, 5}, {7, 2, 1, 4, 3, 6, 5, 0}};
    const double scale = 1.0 / (1.0 - nu * nu);
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) full[j * 8 + i] = scale * k[pat[i][j]];
    lower_cm(full, 8, lower);
    return TOPO_OK;
  }
  if (dim != 3) return TOPO_EINVAL;
  const double lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  const double mu = 1.0 / (2.0 * (1.0 + nu));
  static const double cx[8] = {0, 1, 1, 0, 0, 1, 1, 0};
  static const double cy[8] = {0, 0, 1, 1, 0, 0, 1, 1};
  static const double cz[8] = {0, 0, 0, 0, 1, 1, 1, 1};
  double D[6][6] = {};
  D[0][0] = D[1][1] = D[2][2] = lam + 2.0 * mu;
  D[0][1] = D[0][2] = D[1][0] = D[1][2] = D[2][0] = D[2][1] = lam;
  D[3][3] = D[4][4] = D[5][5] = mu;
  const double gp[2] = {0.5 - 0.5 / sqrt(3.0), 0.5 + 0.5 / sqrt(3.0)};
  double K[24][24] = {};
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b)
      for (int c = 0; c < 2; ++c) {
        const double x = gp[a], y = gp[b], z = gp[c];
        double B[6][24] = {};
        for (int node = 0; node < 8; ++node) {
          const double lx = cx[node] > 0.5 ? x : 1.0 - x;
          const double ly = cy[node] > 0.5 ? y : 1.0 - y;
          const double lz = cz[node] > 0.5 ? z : 1.0 - z;
          const double sx = cx[node] > 0.5 ? 1.0 : -1.0;
          const double sy = cy[node] > 0.5 ? 1.0 : -1.0;
          const double sz = cz[node] > 0.5 ? 1.0 : -1.0;
          const double dx = sx * ly * lz, dy = lx * sy * lz, dz = lx * ly * sz;
          const int col = 3 * node;
          B[0][col] = dx;
          B[1][col + 1] = dy;
          B[2][col + 2] = dz;
          B[3][col + 1] = dz;
          B[3][col + 2] = dy;
          B[4][col] = dz;
          B[4][col + 2] = dx;
          B[5][col] = dy;
          B[5][col + 1] = dx;
        }
        double T[24][6];
        for (int i = 0; i < 24; ++i)
          for (int l = 0; l < 6; ++l) {
            double s = 0;
            for (int q = 0; q < 6; ++q) s += (B[q][i] * 0.125) * D[q][l];
            T[i][l] = s;
          }
        for (int j = 0; j < 24; ++j)
          for (int i = 0; i < 24; ++i) {
            double s = 0;
            for (int l = 0; l < 6; ++l) s += T[i][l] * B[l][j];
            K[i][j] += s;
          }
      }
  for (int j = 0; j < 24; ++j)
    for (int i = 0; i < 24; ++i) full[j * 24 + i] = (K[i][j] + K[j][i]) * 0.5;
  lower_cm(full, 24, lower);
  return TOPO_OK;
}

// counter-based splitmix64 on (seed, stream, index), so
// any rank or the CPU reproduces any element independently.
//   uniform: a + (b - a) * u, u = (r >> 11) * 2^-53
//   normal : a + b * z, Box-Muller on the index pair (2k, 2k + 1)
void topo_generate(uint64_t seed, uint64_t stream, int kind, double a, double b, int64_t offset,
                   int64_t count, double* out) {
  const uint64_t key = splitmix64(seed ^ splitmix64(stream + 0x632BE59BD9B4E019ull));
  const double two53 = 1.0 / 9007199254740992.0;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < count; ++t) {
    const uint64_t idx = uint64_t(offset + t);
    if (kind == 0) {
      const double u = double(splitmix64(key + idx) >> 11) * two53;
      out[t] = a + (b - a) * u;
    } else {
      const uint64_t k = idx >> 1;
      const double u1 = (double(splitmix64(key + 2 * k) >> 11) + 1.0) * two53;  // (0, 1]
      const double u2 = double(splitmix64(key + 2 * k + 1) >> 11) * two53;
      const double rad = sqrt(-2.0 * log(u1));
      const double ang = 6.283185307179586 * u2;
      const double z = (idx & 1) ? rad * sin(ang) : rad * cos(ang);
      out[t] = a + b * z;
    }
  }
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Host replays of the device control state machines (control.h), driven by
// caller-supplied scalar functions. The multi-GPU path runs exactly these
// replays on the host; the CPU test suite checks them against the oracle's
// bisect_update / solve_volume_preserving_eta on the same volume functions.
#include "control.h"

extern "C" {

typedef double (*topo_sfun)(void* user, double s);
typedef void (*topo_gfun)(void* user, double eta, double* g, double* gp);

// oc.hpp:93-174 replay; V(s) from `vol`. speculative = 1 evaluates requests
// in the batches the device kernel uses (oc_speculate; 1: 16 requests per
// batch, 2: 32) and replays them.
int topo_host_oc_replay(const topo_oc_params* prm, double lamMax, topo_sfun vol, void* user,
                        int speculative, double* lambda, int32_t* bisections,
                        int32_t* evaluations, double* s_final, int32_t* batches) {
  topo::OcCtl c;
  c.init(lamMax, prm->volfrac, prm->bisect_rel_tol, prm->volume_tol, prm->lambda_space,
         prm->abs_tol);
  int nb = 0;
  if (speculative < 0) {  // known outcome: vol's first value (+-inf) for every evaluation
    c.replay_known(vol(user, c.s_req));
  } else if (!speculative) {
    while (c.pending()) c.feed(vol(user, c.s_req));
  } else {
    double req[32], val[32];
    while (c.pending()) {
      const int n = speculative >= 2 ? topo::oc_speculate<32>(c, req) : topo::oc_speculate<16>(c, req);
      for (int q = 0; q < n; ++q) val[q] = vol(user, req[q]);
      ++nb;
      while (c.pending()) {
        int hit = -1;
        for (int q = 0; q < n; ++q)
          if (req[q] == c.s_req) hit = q;
        if (hit < 0) break;
        c.feed(val[hit]);
      }
    }
  }
  if (lambda) *lambda = c.lam_result;
  if (bisections) *bisections = c.bis;
  if (evaluations) *evaluations = c.evals;
  if (s_final) *s_final = c.s_final;
  if (batches) *batches = nb;
  return c.status;
}

// filter.hpp:182-228 replay; (g, g') at eta from `gf` (already divided by m)
int topo_host_eta_replay(double eta0, topo_gfun gf, void* user, double* eta, int32_t* iters) {
  topo::EtaCtl c;
  c.init(eta0);
  for (;;) {
    double g, gp;
    gf(user, c.eta, &g, &gp);
    if (!c.feed(g, gp)) break;
  }
  if (eta) *eta = c.eta;
  if (iters) *iters = c.it;
  return 0;
}

}  // extern "C"
