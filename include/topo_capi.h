/*
 * topo_capi.h — C-ABI of the B200-native design-update hot path
 * (density filter -> volume-preserving Heaviside projection -> SIMP +
 * lower-triangle stiffness values -> element compliance sensitivity from a
 * supplied U -> chain-rule back-filter -> OC bisection update).
 *
 * The reference (arxiv/paper_2005_05436, /root/reference/proj/include/topopt)
 * exposes this path as free inline C++ functions; each entry point below names
 * the reference function it replaces (file:line). Plain pointers and sizes
 * only. Every array argument may be a HOST pointer (copied through the
 * context's device buffers) or a DEVICE pointer (used in place); the kind is
 * detected per call with cudaPointerGetAttributes. Calls are stream-ordered on
 * the context's stream and synchronous at return.
 *
 * Error model: a non-zero topo_status; topo_last_error(ctx) has the message.
 * The C++ adapter (include/topopt_gpu.hpp) maps TOPO_EINVAL ->
 * std::invalid_argument, TOPO_EOVERFLOW -> std::overflow_error, TOPO_ENONMONO
 * / TOPO_ECUDA / TOPO_ENCCL -> std::runtime_error, as the reference throws
 * (grid.hpp:92, fea.hpp:159-160, filter.hpp:96,120,127,184, oc.hpp:74,140,161).
 *
 * Multi-GPU: one context per GPU/rank, x-slab decomposition.
 * With nranks > 1 every per-element array is the rank's slab
 * (columns [j0, j1) of the global grid, element order of grid.hpp:42-45) and
 * U is the rank's node planes [j0, j1] inclusive.
 */
#ifndef TOPO_CAPI_H
#define TOPO_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TOPO_CAPI_VERSION 1

typedef struct topo_ctx topo_ctx;

typedef enum {
  TOPO_OK = 0,
  TOPO_EINVAL = 1,    /* std::invalid_argument in the reference */
  TOPO_EOVERFLOW = 2, /* std::overflow_error (grid.hpp:91-93) */
  TOPO_ENONMONO = 3,  /* std::runtime_error  (oc.hpp:139-140, :160-161) */
  TOPO_ECUDA = 4,
  TOPO_ENCCL = 5,
  TOPO_ENOMEM = 6
} topo_status;

/* filter.hpp:14 FilterBC */
enum { TOPO_BC_NEUMANN = 0, TOPO_BC_DIRICHLET = 1 };
/* grid.hpp:73-78 DomainPartition as a per-element state byte */
enum { TOPO_ACTIVE = 0, TOPO_PASSIVE_SOLID = 1, TOPO_PASSIVE_VOID = 2 };
/* the physical-volume callback of bisect_update (oc.hpp:96), built by
 * driver.hpp:214-229 per filter mode ft; a std::function cannot cross the
 * C-ABI, so the callback becomes an enum (plus an optional C callback) */
enum {
  TOPO_VOL_CALLBACK = 0,  /* user C callback on the host copy of xNew */
  TOPO_VOL_MEAN = 1,      /* ft = 1: mean(xc)                    driver.hpp:216     */
  TOPO_VOL_PROJECTED = 2, /* ft = 2: mean(H(pin(filter(xc))))    driver.hpp:218-222 */
  TOPO_VOL_FILTERED = 3   /* ft = 3: mean(pin(filter(xc)))       driver.hpp:224-228 */
};

typedef struct {
  int32_t nelx, nely, nelz; /* grid.hpp:17-46; nelz = 0 selects 2D Q4 */
  double rmin;              /* filter.hpp:95 build_filter */
  int32_t bc;               /* TOPO_BC_* */
  double nu;                /* Poisson ratio for the element stiffness (fea.hpp:51,73) */
  int32_t device;           /* CUDA ordinal; -1 = current device */
  int32_t rank, nranks;     /* x-slab decomposition; single GPU: 0, 1 */
  int32_t j0, j1;           /* slab columns [j0, j1); j1 <= j0 -> even split by rank */
} topo_grid_desc;

typedef struct { /* fea.hpp:124-128 SimpParams */
  double e0, emin, penal;
} topo_simp;

typedef struct { /* oc.hpp:14-20 OcParams + oc.hpp:81-85 BisectOptions */
  double move, volfrac, bisect_rel_tol, volume_tol;
  int32_t lambda_space;
  double abs_tol, lambda_max;
} topo_oc_params;

typedef double (*topo_volume_fn)(void* user, const double* xNew, int64_t m);

typedef struct { /* driver.hpp:56-75 RunConfig fields the pass reads (ft = 3) */
  topo_simp simp;
  double beta, eta0;
  double move, volfrac;
  double eta_override; /* NaN: solve eta (filter.hpp:182); else use it as given */
  int32_t volume_mode; /* TOPO_VOL_FILTERED for ft = 3 */
  int32_t write_sk;    /* 1: produce the m*P lower-triangle values (fea.hpp:162-169) */
} topo_pass_params;

typedef struct {
  /* caller buffers (host or device, length m unless noted) or NULL to skip */
  double *xTilde, *xPhys, *dcPhys, *dc, *dV, *xNew;
  double* sK; /* m*P; NULL keeps the values in the context (topo_device_buffer) */
  double eta, c, lambda;
  int32_t eta_iters, bisections, evaluations;
  /* duplicate-summed lower-triangle CSC values of K (topo_csc_pattern order,
   * nnz entries), or NULL; single-rank contexts */
  double* Kval;
} topo_pass_out;

/* device buffers owned by the context, for zero-copy consumers (the state
 * solve). xPhys is written by the fused pass only
 * once TOPO_BUF_XPHYS has been requested (from then on, every pass); xNew
 * holds the last pass's result when that pass got no device xNew array (a
 * device output array is written in place instead of through the context). */
enum { TOPO_BUF_SK = 0, TOPO_BUF_IK = 1, TOPO_BUF_JK = 2, TOPO_BUF_XNEW = 3, TOPO_BUF_XPHYS = 4 };

/* ---- lifecycle ---------------------------------------------------------- */
/* ke_full (d*d, column-major) / ke_lower (d(d+1)/2, fea.hpp:33-40 order) are
 * the host-built element matrices (fea.hpp:51-121); NULL builds them from
 * desc->nu with topo_element_stiffness. elem_state: m_local bytes of
 * TOPO_ACTIVE/..., or NULL (all active). */
topo_status topo_ctx_create(const topo_grid_desc* desc, const double* ke_full,
                            const double* ke_lower, const uint8_t* elem_state, topo_ctx** out);
void topo_ctx_destroy(topo_ctx* ctx);
const char* topo_last_error(const topo_ctx* ctx);
/* run on an external stream (e.g. torch.cuda.current_stream().cuda_stream) */
topo_status topo_set_stream(topo_ctx* ctx, void* cuda_stream);
topo_status topo_sync(topo_ctx* ctx);
/* order the context's stream after the work already queued on cuda_stream
 * (the stream that produced device inputs or last used device output blocks;
 * NULL = legacy default stream). Entry points are synchronous at return, so
 * outputs need no fence the other way. */
topo_status topo_wait_stream(topo_ctx* ctx, void* cuda_stream);
topo_status topo_device_buffer(topo_ctx* ctx, int which, void** ptr, int64_t* count);
/* device memory for callers without a CUDA runtime of their own (the C++
 * adapter's device-resident redesign loop): allocate / free on the context's
 * device, and a copy in any direction ordered on the context stream
 * (synchronous at return) */
topo_status topo_device_alloc(topo_ctx* ctx, int64_t bytes, void** ptr);
topo_status topo_device_free(topo_ctx* ctx, void* ptr);
topo_status topo_copy(topo_ctx* ctx, void* dst, const void* src, int64_t bytes);
/* sizes: m (local elements), n (local DOFs), P (pairs/element), ntaps, reach,
 * j0, j1 */
topo_status topo_ctx_info(const topo_ctx* ctx, int64_t* m, int64_t* n, int32_t* P,
                          int32_t* ntaps, int32_t* reach, int32_t* j0, int32_t* j1);
/* multi-GPU: join an NCCL clique (nccl_unique_id = 128 bytes from rank 0's
 * topo_nccl_unique_id, broadcast by the caller); halos and scalar sums then
 * travel over NCCL (NVLink) on the context's stream */
topo_status topo_nccl_unique_id(void* out128);
topo_status topo_comm_init_nccl(topo_ctx* ctx, const void* nccl_unique_id);
/* ...or through host callbacks (the caller moves host buffers, e.g. with
 * torch.distributed); `exchange` sends n_send_left / n_send_right doubles to
 * rank - 1 / rank + 1 and fills the receive buffers from them */
typedef struct {
  void* user;
  int (*exchange)(void* user, const double* send_left, int64_t n_send_left,
                  const double* send_right, int64_t n_send_right, double* recv_left,
                  int64_t n_recv_left, double* recv_right, int64_t n_recv_right);
  int (*allreduce_sum)(void* user, double* values, int n);
} topo_host_comm;
topo_status topo_comm_init_host(topo_ctx* ctx, const topo_host_comm* comm);
/* host-only slab plan of a rank: out[0..8) = j0, j1, sj0, sj1 (owned and
 * stored columns) and the columns sent to / received from the left and right
 * neighbours; TOPO_EINVAL if the slab is narrower than the filter reach */
topo_status topo_slab_plan(const topo_grid_desc* desc, int64_t* out);

/* ---- host setup helpers (no device work) -------------------------------- */
/* fea.hpp:51-68 (dim 2) / fea.hpp:73-121 (dim 3) */
topo_status topo_element_stiffness(int dim, double nu, double* ke_full, double* ke_lower);
/* SURVEY.md Appendix B counter-based generator (splitmix64):
 * kind 0 uniform [a, b), kind 1 normal(a, b) via Box-Muller on pairs */
void topo_generate(uint64_t seed, uint64_t stream, int kind, double a, double b, int64_t offset,
                   int64_t count, double* out);

/* host replays of the scalar control flow (no device work): oc.hpp:93-174
 * driven by V(s) = vol(user, sqrt-multiplier), optionally in the speculative
 * batches of the device kernel (speculative 1: 4 levels, 2: 5 levels; -1: the
 * bound-shortcut replay, vol's first value taken for every evaluation);
 * filter.hpp:182-228 driven by (g, g')(eta) */
typedef double (*topo_sfun)(void* user, double s);
typedef void (*topo_gfun)(void* user, double eta, double* g, double* gp);
int topo_host_oc_replay(const topo_oc_params* prm, double lamMax, topo_sfun vol, void* user,
                        int speculative, double* lambda, int32_t* bisections,
                        int32_t* evaluations, double* s_final, int32_t* batches);
int topo_host_eta_replay(double eta0, topo_gfun gf, void* user, double* eta, int32_t* iters);

/* ---- K0: grid.hpp:89-153 ------------------------------------------------ */
topo_status topo_build_connectivity(topo_ctx* ctx, int32_t* dofs);          /* m*d */
topo_status topo_build_index_pairs(topo_ctx* ctx, int32_t* iK, int32_t* jK); /* m*P; NULL=keep */

/* ---- fea.hpp ------------------------------------------------------------ */
/* fea.hpp:135-146 simp_interpolate */
topo_status topo_simp_interpolate(topo_ctx* ctx, const double* xhat, const topo_simp* prm,
                                  double* sK, double* dsK);
/* fea.hpp:154-176 assemble_lower, value generation (:162-169): vals[e*P+q] =
 * sK[e] * Ke_lower[q] (duplicates are summed by the consumer) */
topo_status topo_assemble_values(topo_ctx* ctx, const double* sK, double* vals);
/* the matrix assemble_lower returns (fea.hpp:154-176): setFromTriplets of the
 * (iK, jK, vals) triplets, i.e. the n x n lower triangle of K in compressed
 * column form with ascending rows and duplicates summed in triplet order
 * (ascending element). topo_csc_pattern: col_ptr n+1 (int64), row_idx nnz;
 * any pointer may be NULL (query nnz first). topo_csc_values: values[nnz]
 * from the per-element modulus sK (m), bitwise equal to the reference's sums.
 * Built on the device without the m*P triplets; single-rank contexts. */
topo_status topo_csc_pattern(topo_ctx* ctx, int64_t* col_ptr, int32_t* row_idx, int64_t* nnz);
/* reduced mode (EquilibriumSolver, fea.hpp:316-361; solve_equilibrium :206-239):
 * with the load case's fixed DOFs (host, any order, duplicates allowed), the
 * CSC covers only the free DOFs, renumbered by detail::free_dof_map
 * (fea.hpp:186-199); col_ptr then has num_free+1 entries. nfixed = 0 returns
 * to the full matrix. Values accumulate per slot in triplet order starting
 * from 0 (fea.hpp:352-361), bitwise equal to the reference's. */
topo_status topo_csc_set_fixed(topo_ctx* ctx, const int32_t* fixed, int64_t nfixed,
                               int64_t* num_free);
topo_status topo_csc_values(topo_ctx* ctx, const double* sK, double* values);
/* fea.hpp:248-272 compliance_and_sensitivity (c is the rank-local partial) */
topo_status topo_sensitivity(topo_ctx* ctx, const double* U, const double* xhat,
                             const topo_simp* prm, double* c, double* dc);

/* ---- filter.hpp --------------------------------------------------------- */
topo_status topo_filter(topo_ctx* ctx, const double* x, double* xTilde, int pin); /* :119-122 */
topo_status topo_filter_adjoint(topo_ctx* ctx, const double* g, double* out);      /* :126-129 */
topo_status topo_project(topo_ctx* ctx, const double* xt, double eta, double beta,
                         double* out); /* :137-144 */
topo_status topo_project_derivative(topo_ctx* ctx, const double* xt, double eta, double beta,
                                    double* out); /* :146-154 */
topo_status topo_backfilter(topo_ctx* ctx, const double* g, const double* xt, double eta,
                            double beta, int proj_on, double* out); /* :166-171 */
topo_status topo_solve_eta(topo_ctx* ctx, const double* xTilde, double beta, double eta0,
                           double* eta, int32_t* iters); /* :182-228 (active set from ctx) */
/* filter taps in reference order (filter.hpp:107-113) and hs */
topo_status topo_filter_taps(topo_ctx* ctx, int32_t* di, int32_t* dj, int32_t* dk, double* w);
topo_status topo_filter_hs(topo_ctx* ctx, double* hs);

/* ---- oc.hpp ------------------------------------------------------------- */
/* oc.hpp:31-39, compact active arrays of length nact */
topo_status topo_lambda_upper(topo_ctx* ctx, int64_t nact, const double* xAct,
                              const double* dcAct, const double* dVAct, double volfrac,
                              int64_t mTotal, double* lambda);
/* oc.hpp:72-79 */
topo_status topo_oc_candidate(topo_ctx* ctx, int64_t nact, const double* xAct,
                              const double* dcAct, const double* dVAct, double lambda,
                              double move, double* out);
/* oc.hpp:93-174 bisect_update over full-length x, dc, dV (passives from ctx).
 * eta/beta are used by TOPO_VOL_PROJECTED; cb/user by TOPO_VOL_CALLBACK. */
topo_status topo_oc_bisect(topo_ctx* ctx, const double* x, const double* dc, const double* dV,
                           const topo_oc_params* prm, int volume_mode, double eta, double beta,
                           topo_volume_fn cb, void* user, double* xNew, double* lambda,
                           int32_t* bisections, int32_t* evaluations);

/* oc.hpp:181-241 primal_dual_update (driver.hpp:211-212, ft = 1): explicit
 * dual-map iteration to |lm' - lm| <= pd_tol (OcParams::pdTol, 1e-10), with
 * the reference's fallback to bisect_update on the mean volume (*fell_back =
 * 1; *iterations then counts bisections, as UpdateResult::bisections does) */
topo_status topo_oc_primal_dual(topo_ctx* ctx, const double* x, const double* dc,
                                const double* dV, const topo_oc_params* prm, double pd_tol,
                                double* xNew, double* lambda, int32_t* iterations,
                                int32_t* fell_back);

/* ---- state solve: fea.hpp:205-239 solve_equilibrium
 * K(sK) u = f on the free DOFs (u = 0 on `fixed`, LoadCase, fea.hpp:178-182),
 * matrix-free Jacobi-preconditioned CG on the structured grid to
 * ||r|| <= rtol ||f|| (the reference factorises; solutions agree to the solver
 * tolerance). sK: per-element modulus (m); f, u: n. Single-rank contexts. */
topo_status topo_solve_state(topo_ctx* ctx, const double* sK, const double* f,
                             const int32_t* fixed, int64_t nfixed, double rtol, int32_t maxit,
                             double* u, int32_t* iterations, double* relres);
/* the same solve with a geometric multigrid V-cycle as the preconditioner
 * (the MGCG variant of top3D125): Galerkin element matrices on grids halved
 * per axis while every element count stays even, damped-Jacobi smoothing,
 * Jacobi sweeps on the coarsest grid; the Jacobi-PCG solve when the grid
 * cannot be coarsened */
topo_status topo_solve_state_mg(topo_ctx* ctx, const double* sK, const double* f,
                                const int32_t* fixed, int64_t nfixed, double rtol, int32_t maxit,
                                double* u, int32_t* iterations, double* relres);

/* y = K(sK) x, the matrix-free stiffness operator of the solves (no fixed
 * DOFs; K = sum_e sK_e Ke over the grid, fea.hpp:162-174 assembled in full).
 * variant 0: the solver's default (one-launch Walsh-form node tiles for H8,
 * else the node-centric gather); 1: per-colour element launches (H8, Walsh);
 * 2: node-centric gather with the dense Ke. 0 and 1 are bitwise equal. */
topo_status topo_apply_stiffness(topo_ctx* ctx, const double* sK, const double* x, double* y,
                                 int32_t variant);

/* ---- redesign-loop helpers on device arrays (driver.hpp:189, :235-263) ---
 * topo_loop_records: out3 = {ch = ||xPhys - xPrev|| / sqrt(m) (driver.hpp:189),
 * v = mean(xPhys) (:249), mnd = nondiscreteness(x) (:39-43, :251)}; xPrev is
 * overwritten with xPhys. Fixed-order device reductions, one 24-byte read. */
topo_status topo_loop_records(topo_ctx* ctx, const double* xPhys, double* xPrev,
                              const double* x, double* out3);
/* AndersonAccelerator (accel.hpp:21-95) applied as driver.hpp:235-244 does:
 * over the active elements, x_before = the design before the update and
 * x_inout = the updated design on entry, the extrapolated design clamped to
 * [0, 1] on return (passives untouched). The difference window lives in the
 * context (depth <= 8 columns of m doubles each); reset clears it. */
typedef struct { /* AndersonOptions (accel.hpp:9-14) */
  int32_t depth, period;
  double mix_plain, mix_accel;
} topo_anderson;
topo_status topo_anderson_step(topo_ctx* ctx, const topo_anderson* opt, const double* x_before,
                               double* x_inout);
topo_status topo_anderson_reset(topo_ctx* ctx);

/* ---- fused pass: driver.hpp:183-231 (ft = 3) minus the state solve ------ */
topo_status topo_design_pass(topo_ctx* ctx, const double* x, const double* U,
                             const topo_pass_params* prm, topo_pass_out* out);
/* The same pass in two halves, for callers that overlap host work with it or
 * time it on the device: _begin validates, enqueues everything on the
 * context's stream(s) and returns without waiting (x, U and the arrays in
 * `out` must stay valid and untouched until _end); _end waits for the stream,
 * completes the host-side parts (multi-rank OC / eta completion) and fills the
 * scalars of `out` (pass the same `out`). topo_design_pass = _begin + _end.
 * One pass in flight per context, and no other call on the context between
 * the two halves (they share its scratch buffers and result words). */
topo_status topo_design_pass_begin(topo_ctx* ctx, const double* x, const double* U,
                                   const topo_pass_params* prm, topo_pass_out* out);
topo_status topo_design_pass_end(topo_ctx* ctx, topo_pass_out* out);
/* number of this library's kernel launches issued by the last call */
int64_t topo_last_launch_count(const topo_ctx* ctx);
/* per-stage CUDA-event timing of topo_design_pass (off by default). times_ms
 * receives TOPO_NSTAGES values for the last pass, each measured with events
 * on the stream its kernel runs on: K1 filter, K2 eta, K3a element, K4
 * adjoint+OC prep, K5/K6 OC, K3b sK store (aux stream), whole pass. */
enum { TOPO_STAGE_FILTER = 0, TOPO_STAGE_ETA, TOPO_STAGE_ELEM, TOPO_STAGE_ADJOINT, TOPO_STAGE_OC,
       TOPO_STAGE_SK, TOPO_STAGE_PASS, TOPO_NSTAGES };
topo_status topo_set_timing(topo_ctx* ctx, int on);
topo_status topo_stage_times(topo_ctx* ctx, double* times_ms);
/* repeated single-rank topo_design_pass calls over the same device arrays and
 * parameters are captured into a CUDA graph (second call) and replayed;
 * replays = passes served by the graph so far (TOPO_PASS_GRAPH=0 disables) */
topo_status topo_pass_graph_replays(const topo_ctx* ctx, int64_t* replays);

/* ---- measurement helper (not part of the reference API) ------------------
 * FP64 FMA throughput of `device` in TFLOP/s (2 flops per DFMA), measured
 * with a dependent-chain-free DFMA loop over the whole GPU (SURVEY.md §8(d):
 * the FP64 roof of the filter-bound configs C2/C3). */
topo_status topo_fp64_peak(int device, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* TOPO_CAPI_H */
