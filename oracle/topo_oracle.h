/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the design-update hot path.
 *
 * A plain-C restatement of the reference's algorithm (arxiv/paper_2005_05436,
 * /root/reference/proj/include/topopt/{grid,fea,filter,oc,driver}.hpp). Every
 * function cites the reference file:line it follows. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library, and only as the checker or the timed CPU baseline —
 * never as the product path.
 *
 * Pinning: the restatement is checked against (1) the reference's own
 * known-answer tests (tests/golden/reference_kat.json, values copied from
 * proj/tests/test_*.cpp) and (2) the reference headers themselves, compiled
 * verbatim against oracle/eigen_shim into oracle/_ref/libtopo_ref.so
 * (tests/test_oracle_vs_reference.py, fixtures in tests/golden/).
 *
 * Element / node numbering follows grid.hpp:35-45 (y fastest, then z, then x).
 * Status codes match include/topo_capi.h.
 */
#ifndef TOPO_ORACLE_H
#define TOPO_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_EOVERFLOW = 2, ORC_ENONMONO = 3 };

typedef struct {
  int32_t nelx, nely, nelz;
} orc_grid;

const char* orc_last_error(void);
int orc_set_threads(int n);

/* SURVEY.md Appendix B input generator (counter-based splitmix64; kind 0
 * uniform [a, b), 1 normal(a, b) by Box-Muller on index pairs). Lets the CPU
 * reference arm build the benchmark inputs without the product library. */
void orc_generate(uint64_t seed, uint64_t stream, int kind, double a, double b, int64_t offset,
                  int64_t count, double* out);

/* grid.hpp */
int64_t orc_num_elements(orc_grid g);
int64_t orc_num_dofs(orc_grid g);
int orc_build_connectivity(orc_grid g, int32_t* dofs);
int orc_build_index_pairs(orc_grid g, int32_t* iK, int32_t* jK);
int orc_partition(orc_grid g, const int32_t* pasS, int64_t nS, const int32_t* pasV, int64_t nV,
                  uint8_t* state);

/* fea.hpp */
int orc_element_stiffness(int dim, double nu, double* full, double* lower);
void orc_simp(int64_t m, const double* xhat, double e0, double emin, double p, double* sK,
              double* dsK);
void orc_assemble_values(int64_t m, int P, const double* sK, const double* ke_lower, double* vals);
int orc_assemble_lower(orc_grid g, double nu, const double* sK, int32_t* col_ptr,
                       int32_t* row_idx, double* values, int64_t* nnz);
int orc_compliance_sensitivity(orc_grid g, const double* ke_full, const double* u,
                               const double* xhat, double e0, double emin, double p,
                               const uint8_t* state, double* c, double* dc);

/* filter.hpp */
typedef struct orc_filter orc_filter;
orc_filter* orc_filter_create(orc_grid g, double rmin, int bc);
void orc_filter_destroy(orc_filter* f);
int orc_filter_ntaps(const orc_filter* f);
void orc_filter_taps(const orc_filter* f, int32_t* di, int32_t* dj, int32_t* dk, double* w);
const double* orc_filter_hs(const orc_filter* f);
void orc_cone_convolve(const orc_filter* f, const double* v, double* out);
void orc_apply_filter(const orc_filter* f, const double* x, double* out);
void orc_apply_filter_adjoint(const orc_filter* f, const double* g, double* out);
void orc_project(int64_t m, const double* xt, double eta, double beta, double* out);
void orc_project_derivative(int64_t m, const double* xt, double eta, double beta, double* out);
double orc_project_eta_derivative(double xt, double eta, double beta);
void orc_backfilter(const orc_filter* f, const double* g, const double* xt, double eta,
                    double beta, int proj_on, double* out);
int orc_solve_eta(int64_t m, const double* xt, double beta, double eta0, const uint8_t* state,
                  double* eta, int* iters);
double orc_eta_mismatch(int64_t m, const double* xt, double beta, double eta,
                        const uint8_t* state);

/* oc.hpp */
double orc_lambda_upper(int64_t n, const double* xAct, const double* dcAct, const double* dVAct,
                        double volfrac, int64_t mTotal);
int orc_oc_candidate(int64_t n, const double* xAct, const double* dcAct, const double* dVAct,
                     double lambda, double move, double* out);

typedef double (*orc_volume_fn)(void* user, const double* xNew, int64_t m);

typedef struct {
  double move, volfrac, bisect_rel_tol, volume_tol;
  int lambda_space;
  double abs_tol, lambda_max;
} orc_oc_params;

/* volume modes of driver.hpp:214-229, plus 4 = the c = H'1_notP identity of
 * SURVEY.md §8(a) A15 and 0 = user callback */
enum { ORC_VOL_CALLBACK = 0, ORC_VOL_MEAN = 1, ORC_VOL_PROJECTED = 2, ORC_VOL_FILTERED = 3,
       ORC_VOL_IDENTITY = 4 };

int orc_bisect_update(int64_t m, const double* x, const double* dc, const double* dV,
                      const uint8_t* state, const orc_oc_params* prm, int volume_mode,
                      const orc_filter* f, double eta, double beta, orc_volume_fn cb, void* user,
                      double* xNew, double* lambda, int* bisections, int* evaluations);
int orc_primal_dual_update(int64_t m, const double* x, const double* dc, const double* dV,
                           const uint8_t* state, const orc_oc_params* prm, double pd_tol,
                           double* xNew, double* lambda, int* iterations, int* fell_back);

/* driver.hpp:183-231 (ft = 3 branch) — one design-update pass */
typedef struct {
  double e0, emin, penal, beta, eta0, move, volfrac;
  double eta_override; /* NaN: solve eta; else use it (conditioned protocol) */
  int volume_mode;     /* ORC_VOL_FILTERED (literal) or ORC_VOL_IDENTITY */
} orc_pass_params;

typedef struct {
  double* xTilde; /* m */
  double* xPhys;  /* m */
  double* sKe;    /* m, per-element modulus */
  double* dcPhys; /* m */
  double* dc;     /* m */
  double* dV;     /* m */
  double* xNew;   /* m */
  double eta, c, lambda;
  int eta_iters, bisections, evaluations;
} orc_pass_out;

int orc_design_pass(orc_grid g, const orc_filter* f, const double* ke_full,
                    const uint8_t* state, const double* x, const double* u,
                    const orc_pass_params* prm, orc_pass_out* out);

#ifdef __cplusplus
}
#endif
#endif
