// TEST INFRASTRUCTURE ONLY — a C API over the reference's OWN hot-path
// headers (/root/reference/proj/include/topopt/{grid,fea,filter,oc}.hpp),
// compiled verbatim against oracle/eigen_shim by oracle/Makefile into
// oracle/_ref/libtopo_ref.so. Nothing here reimplements the reference's
// arithmetic: every numeric result comes from the reference functions. The
// only restated code is the ft = 3 pass glue of driver.hpp:183-231 (the
// driver cannot run without the out-of-path state solve, and U is an input
// of this path) and driver.hpp:130-133 pin_passives (in namespace detail).
//
// Used (1) to pin the C restatement in topo_oracle.c, (2) to generate the
// fixtures under tests/golden/, and (3) as the timed CPU reference arm of
// bench.py (--impl reference, cpu_baseline.kind = "reference").
#include <cmath>
#include <cstdint>
#include <algorithm>
#include <cstring>
#include <exception>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "topopt/fea.hpp"
#include "topopt/filter.hpp"
#include "topopt/grid.hpp"
#include "topopt/oc.hpp"

using namespace topopt;

namespace {
thread_local std::string g_err;

// status codes of include/topo_capi.h / oracle/topo_oracle.h
enum { OK = 0, EINVAL_ = 1, EOVERFLOW_ = 2, ENONMONO = 3, EOTHER = 9 };

template <typename F>
int guard(F&& f) {
  try {
    f();
    return OK;
  } catch (const std::overflow_error& e) {
    g_err = e.what();
    return EOVERFLOW_;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return EINVAL_;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return ENONMONO;
  } catch (const std::exception& e) {
    g_err = e.what();
    return EOTHER;
  }
}

Eigen::VectorXd vec(const double* p, int64_t n) {
  Eigen::VectorXd v(n);
  std::memcpy(v.data(), p, sizeof(double) * size_t(n));
  return v;
}
void out(const Eigen::VectorXd& v, double* p) {
  std::memcpy(p, v.data(), sizeof(double) * size_t(v.size()));
}

DomainPartition partition_from_state(const StructuredGrid& g, const uint8_t* state) {
  std::vector<std::int32_t> s, v;
  if (state)
    for (int64_t e = 0; e < g.numElements(); ++e) {
      if (state[e] == 1) s.push_back(std::int32_t(e));
      if (state[e] == 2) v.push_back(std::int32_t(e));
    }
  return partition_domain(g, s, v);
}

// driver.hpp:130-133
void pin_passives(Eigen::VectorXd& field, const DomainPartition& part) {
  for (auto e : part.pasS) field[e] = 1.0;
  for (auto e : part.pasV) field[e] = 0.0;
}
}  // namespace

extern "C" {

typedef struct {
  int32_t nelx, nely, nelz;
} ref_grid;

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_build_connectivity(ref_grid g, int32_t* dofs) {
  return guard([&] {
    const Connectivity c = build_connectivity({g.nelx, g.nely, g.nelz});
    std::memcpy(dofs, c.dofs.data(), sizeof(int32_t) * c.dofs.size());
  });
}

int ref_build_index_pairs(ref_grid g, int32_t* iK, int32_t* jK) {
  return guard([&] {
    const IndexPairs p = build_symmetric_index_pairs(build_connectivity({g.nelx, g.nely, g.nelz}));
    std::memcpy(iK, p.iK.data(), sizeof(int32_t) * p.iK.size());
    std::memcpy(jK, p.jK.data(), sizeof(int32_t) * p.jK.size());
  });
}

int ref_partition(ref_grid g, const int32_t* pasS, int64_t nS, const int32_t* pasV, int64_t nV,
                  uint8_t* state) {
  return guard([&] {
    const StructuredGrid grid{g.nelx, g.nely, g.nelz};
    const DomainPartition p = partition_domain(grid, std::vector<std::int32_t>(pasS, pasS + nS),
                                               std::vector<std::int32_t>(pasV, pasV + nV));
    std::memset(state, 0, size_t(grid.numElements()));
    for (auto e : p.pasS) state[e] = 1;
    for (auto e : p.pasV) state[e] = 2;
  });
}

int ref_element_stiffness(int dim, double nu, double* full, double* lower) {
  return guard([&] {
    const ElementStiffness ke = dim == 3 ? element_stiffness_h8(nu) : element_stiffness_q4(nu);
    std::memcpy(full, ke.full.data(), sizeof(double) * size_t(ke.full.size()));
    out(ke.lower, lower);
  });
}

void ref_simp(int64_t m, const double* xhat, double e0, double emin, double p, double* sK,
              double* dsK) {
  const SimpField f = simp_interpolate(vec(xhat, m), {e0, emin, p});
  out(f.sK, sK);
  out(f.dsK, dsK);
}

// assemble_lower (fea.hpp:154-176) -> duplicate-summed lower CSC. Two calls:
// first with col_ptr only (returns nnz), then with all arrays.
int ref_assemble_lower(ref_grid g, double nu, const double* sK, int32_t* col_ptr,
                       int32_t* row_idx, double* values, int64_t* nnz) {
  return guard([&] {
    const StructuredGrid grid{g.nelx, g.nely, g.nelz};
    const ElementStiffness ke = grid.is3d() ? element_stiffness_h8(nu) : element_stiffness_q4(nu);
    const IndexPairs pairs = build_symmetric_index_pairs(build_connectivity(grid));
    const SymmetricSparseMatrix K =
        assemble_lower(pairs, ke, vec(sK, grid.numElements()), grid.numDofs());
    *nnz = K.lower.nonZeros();
    if (col_ptr)
      std::memcpy(col_ptr, K.lower.outerIndexPtr(), sizeof(int32_t) * size_t(grid.numDofs() + 1));
    if (row_idx) std::memcpy(row_idx, K.lower.innerIndexPtr(), sizeof(int32_t) * size_t(*nnz));
    if (values) std::memcpy(values, K.lower.valuePtr(), sizeof(double) * size_t(*nnz));
  });
}

int ref_compliance_sensitivity(ref_grid g, double nu, const double* u, const double* xhat,
                               double e0, double emin, double p, const uint8_t* state, double* c,
                               double* dc) {
  return guard([&] {
    const StructuredGrid grid{g.nelx, g.nely, g.nelz};
    const ElementStiffness ke = grid.is3d() ? element_stiffness_h8(nu) : element_stiffness_q4(nu);
    const ComplianceResult r =
        compliance_and_sensitivity(vec(u, grid.numDofs()), build_connectivity(grid),
                                   vec(xhat, grid.numElements()), {e0, emin, p}, ke,
                                   partition_from_state(grid, state));
    *c = r.c;
    out(r.dc, dc);
  });
}

// ---------------------------------------------------------------- filter.hpp
void* ref_filter_create(ref_grid g, double rmin, int bc) {
  FilterOperator* op = nullptr;
  const int st = guard([&] {
    op = new FilterOperator(build_filter({g.nelx, g.nely, g.nelz}, rmin,
                                         bc == 0 ? FilterBC::Neumann : FilterBC::Dirichlet));
  });
  return st == OK ? op : nullptr;
}
void ref_filter_destroy(void* h) { delete static_cast<FilterOperator*>(h); }
int ref_filter_ntaps(void* h) { return int(static_cast<FilterOperator*>(h)->taps.size()); }
void ref_filter_taps(void* h, int32_t* di, int32_t* dj, int32_t* dk, double* w) {
  const auto& t = static_cast<FilterOperator*>(h)->taps;
  for (size_t q = 0; q < t.size(); ++q) {
    di[q] = t[q].di;
    dj[q] = t[q].dj;
    dk[q] = t[q].dk;
    w[q] = t[q].w;
  }
}
void ref_filter_hs(void* h, double* hs) { out(static_cast<FilterOperator*>(h)->hs, hs); }
int ref_apply_filter(void* h, const double* x, double* o) {
  auto* op = static_cast<FilterOperator*>(h);
  return guard([&] { out(apply_filter(vec(x, op->numElements()), *op), o); });
}
int ref_apply_filter_adjoint(void* h, const double* x, double* o) {
  auto* op = static_cast<FilterOperator*>(h);
  return guard([&] { out(apply_filter_adjoint(vec(x, op->numElements()), *op), o); });
}
void ref_project(int64_t m, const double* xt, double eta, double beta, double* o) {
  out(project(vec(xt, m), {eta, beta}), o);
}
void ref_project_derivative(int64_t m, const double* xt, double eta, double beta, double* o) {
  out(project_derivative(vec(xt, m), {eta, beta}), o);
}
double ref_project_eta_derivative(double xt, double eta, double beta) {
  return project_eta_derivative(xt, {eta, beta});
}
int ref_backfilter(void* h, const double* g, const double* xt, double eta, double beta, int on,
                   double* o) {
  auto* op = static_cast<FilterOperator*>(h);
  const int64_t m = op->numElements();
  return guard(
      [&] { out(backfilter(vec(g, m), vec(xt, m), *op, {eta, beta}, on != 0), o); });
}
int ref_solve_eta(ref_grid g, const double* xt, double beta, double eta0, const uint8_t* state,
                  double* eta, int* iters) {
  return guard([&] {
    const StructuredGrid grid{g.nelx, g.nely, g.nelz};
    const EtaSolveResult r = solve_volume_preserving_eta(vec(xt, grid.numElements()), beta, eta0,
                                                         partition_from_state(grid, state));
    *eta = r.eta;
    *iters = r.iterations;
  });
}

// -------------------------------------------------------------------- oc.hpp
double ref_lambda_upper(int64_t n, const double* x, const double* dc, const double* dV,
                        double volfrac, int64_t mTotal) {
  return lambda_upper_estimate(vec(x, n), vec(dc, n), vec(dV, n), volfrac, mTotal);
}
int ref_oc_candidate(int64_t n, const double* x, const double* dc, const double* dV,
                     double lambda, double move, double* o) {
  return guard([&] { out(oc_candidate(vec(x, n), vec(dc, n), vec(dV, n), lambda, move), o); });
}

typedef double (*ref_volume_fn)(void* user, const double* xNew, int64_t m);
typedef struct {
  double move, volfrac, bisect_rel_tol, volume_tol;
  int lambda_space;
  double abs_tol, lambda_max;
} ref_oc_params;

// volume modes: 0 callback, 1 mean (driver.hpp:216), 2 projected (:218-222),
// 3 filtered (:224-228)
int ref_bisect_update(ref_grid g, const double* x, const double* dc, const double* dV,
                      const uint8_t* state, const ref_oc_params* p, int mode, void* filter,
                      double eta, double beta, ref_volume_fn cb, void* user, double* xNew,
                      double* lambda, int* bisections, int* evaluations) {
  int evals = 0;
  return guard([&] {
    const StructuredGrid grid{g.nelx, g.nely, g.nelz};
    const int64_t m = grid.numElements();
    const DomainPartition part = partition_from_state(grid, state);
    const FilterOperator* flt = static_cast<FilterOperator*>(filter);
    const ProjectionParams prj{eta, beta};
    std::function<double(const Eigen::VectorXd&)> vol;
    switch (mode) {
      case 0:
        vol = [&](const Eigen::VectorXd& xc) { return cb(user, xc.data(), m); };
        break;
      case 1:
        vol = [](const Eigen::VectorXd& xc) { return xc.mean(); };
        break;
      case 2:
        vol = [&](const Eigen::VectorXd& xc) {
          Eigen::VectorXd xf = apply_filter(xc, *flt);
          pin_passives(xf, part);
          return project(xf, prj).mean();
        };
        break;
      default:
        vol = [&](const Eigen::VectorXd& xc) {
          Eigen::VectorXd xf = apply_filter(xc, *flt);
          pin_passives(xf, part);
          return xf.mean();
        };
    }
    auto counted = [&](const Eigen::VectorXd& xc) {
      ++evals;
      return vol(xc);
    };
    OcParams oc;
    oc.move = p->move;
    oc.volfrac = p->volfrac;
    oc.bisectRelTol = p->bisect_rel_tol;
    oc.volumeTol = p->volume_tol;
    BisectOptions opt;
    opt.lambdaSpace = p->lambda_space != 0;
    opt.absTol = p->abs_tol;
    opt.lambdaMax = p->lambda_max;
    const UpdateResult r =
        bisect_update(vec(x, m), vec(dc, m), vec(dV, m), part, oc, counted, opt);
    out(r.xNew, xNew);
    *lambda = r.lambda;
    *bisections = r.bisections;
    if (evaluations) *evaluations = evals;
  });
}

// oc.hpp:181-241 primal_dual_update (ft = 1); *fell_back is not observable in
// the reference's result and is reported as -1 here
int ref_primal_dual_update(ref_grid g, const double* x, const double* dc, const double* dV,
                           const uint8_t* state, const ref_oc_params* p, double pd_tol,
                           double* xNew, double* lambda, int* iterations) {
  return guard([&] {
    const StructuredGrid grid{g.nelx, g.nely, g.nelz};
    const int64_t m = grid.numElements();
    const DomainPartition part = partition_from_state(grid, state);
    OcParams oc;
    oc.move = p->move;
    oc.volfrac = p->volfrac;
    oc.bisectRelTol = p->bisect_rel_tol;
    oc.volumeTol = p->volume_tol;
    oc.pdTol = pd_tol;
    const UpdateResult r = primal_dual_update(vec(x, m), vec(dc, m), vec(dV, m), part, oc);
    out(r.xNew, xNew);
    *lambda = r.lambda;
    *iterations = r.bisections;
  });
}

// fea.hpp:205-239 solve_equilibrium(assemble_lower(...), LoadCase{f, fixed})
int ref_solve_state(ref_grid g, double nu, const double* sK, const double* f,
                    const int32_t* fixed, int64_t nfixed, double* u) {
  return guard([&] {
    const StructuredGrid grid{g.nelx, g.nely, g.nelz};
    const ElementStiffness ke = grid.is3d() ? element_stiffness_h8(nu) : element_stiffness_q4(nu);
    const IndexPairs pairs = build_symmetric_index_pairs(build_connectivity(grid));
    const SymmetricSparseMatrix K =
        assemble_lower(pairs, ke, vec(sK, grid.numElements()), grid.numDofs());
    LoadCase load;
    load.f = vec(f, grid.numDofs());
    load.fixed.assign(fixed, fixed + nfixed);
    std::sort(load.fixed.begin(), load.fixed.end());
    load.fixed.erase(std::unique(load.fixed.begin(), load.fixed.end()), load.fixed.end());
    out(solve_equilibrium(K, load), u);
  });
}

// ---------------------------------------------------------- pass (driver glue)
typedef struct {
  double e0, emin, penal, beta, eta0, move, volfrac;
  double eta_override;  // NaN: solve eta
  int volume_mode;      // 3 literal ft=3 callback (anything else is treated as 3)
} ref_pass_params;

typedef struct {
  double *xTilde, *xPhys, *sKe, *dcPhys, *dc, *dV, *xNew;
  double eta, c, lambda;
  int eta_iters, bisections, evaluations;
} ref_pass_out;

struct RefProblem {
  StructuredGrid grid;
  Connectivity conn;
  ElementStiffness ke;
  FilterOperator flt;
  DomainPartition part;
};

void* ref_problem_create(ref_grid g, double rmin, int bc, double nu, const uint8_t* state) {
  RefProblem* p = nullptr;
  const int st = guard([&] {
    auto* q = new RefProblem;
    q->grid = {g.nelx, g.nely, g.nelz};
    q->conn = build_connectivity(q->grid);
    q->ke = q->grid.is3d() ? element_stiffness_h8(nu) : element_stiffness_q4(nu);
    q->flt = build_filter(q->grid, rmin, bc == 0 ? FilterBC::Neumann : FilterBC::Dirichlet);
    q->part = partition_from_state(q->grid, state);
    p = q;
  });
  return st == OK ? p : nullptr;
}
void ref_problem_destroy(void* h) { delete static_cast<RefProblem*>(h); }

// driver.hpp:183-231 with cfg.ft == 3; the equilibrium solve is replaced by
// the supplied displacement u.
int ref_design_pass(void* h, const double* x_in, const double* u_in, const ref_pass_params* prm,
                    ref_pass_out* o) {
  auto* P = static_cast<RefProblem*>(h);
  return guard([&] {
    const int64_t m = P->grid.numElements();
    const DomainPartition& part = P->part;
    const Eigen::VectorXd x = vec(x_in, m);
    const Eigen::VectorXd u = vec(u_in, P->grid.numDofs());
    Eigen::VectorXd dV0 = Eigen::VectorXd::Zero(m);  // driver.hpp:154-155
    for (auto e : part.act) dV0[e] = 1.0 / double(m);

    // RL.1
    Eigen::VectorXd xTilde = apply_filter(x, P->flt);
    pin_passives(xTilde, part);
    double eta = prm->eta0;
    int etaIters = 0;
    if (std::isnan(prm->eta_override)) {
      const EtaSolveResult r = solve_volume_preserving_eta(xTilde, prm->beta, eta, part);
      eta = r.eta;
      etaIters = r.iterations;
    } else {
      eta = prm->eta_override;
    }
    const ProjectionParams prj{eta, prm->beta};
    const Eigen::VectorXd xPhys = project(xTilde, prj);
    // RL.2
    const SimpParams simp{prm->e0, prm->emin, prm->penal};
    const SimpField law = simp_interpolate(xPhys, simp);
    // RL.3
    const ComplianceResult comp = compliance_and_sensitivity(u, P->conn, xPhys, simp, P->ke, part);
    const Eigen::VectorXd dc = backfilter(comp.dc, xTilde, P->flt, prj, true);
    const Eigen::VectorXd dV = backfilter(dV0, xTilde, P->flt, prj, true);
    // RL.4
    OcParams oc;
    oc.move = prm->move;
    oc.volfrac = prm->volfrac;
    int evals = 0;
    auto physVolume = [&](const Eigen::VectorXd& xc) {
      ++evals;
      Eigen::VectorXd xf = apply_filter(xc, P->flt);
      pin_passives(xf, part);
      return xf.mean();
    };
    const UpdateResult up = bisect_update(x, dc, dV, part, oc, physVolume);

    if (o->xTilde) out(xTilde, o->xTilde);
    if (o->xPhys) out(xPhys, o->xPhys);
    if (o->sKe) out(law.sK, o->sKe);
    if (o->dcPhys) out(comp.dc, o->dcPhys);
    if (o->dc) out(dc, o->dc);
    if (o->dV) out(dV, o->dV);
    if (o->xNew) out(up.xNew, o->xNew);
    o->eta = eta;
    o->eta_iters = etaIters;
    o->c = comp.c;
    o->lambda = up.lambda;
    o->bisections = up.bisections;
    o->evaluations = evals;
  });
}

}  // extern "C"
