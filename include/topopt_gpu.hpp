// topopt_gpu.hpp — drop-in C++ adapter for the reference's design-update
// operator API (arxiv/paper_2005_05436, proj/include/topopt/*.hpp) on top of
// the B200 C-ABI (topo_capi.h). Same function names, argument meaning and
// exception types as the reference; the setup objects the reference passes
// around (StructuredGrid, FilterOperator, ElementStiffness, DomainPartition)
// are bound once into a gpu::Device, which owns the device buffers.
//
// Include after the reference headers (it uses their types):
//     #include "topopt/grid.hpp"  "topopt/fea.hpp"  "topopt/filter.hpp"  "topopt/oc.hpp"
//     #include "topopt_gpu.hpp"
// and link libtopo_b200.so. See INTEGRATION.md.
#pragma once

#include <chrono>
#include <cstring>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "topo_capi.h"

namespace topopt {
namespace gpu {

/// Throws the reference's exception type for a C-ABI status (grid.hpp:92,
/// fea.hpp:159-160, filter.hpp:96,120,127,184, oc.hpp:74,140,161).
inline void check(topo_status s, const topo_ctx* ctx) {
  if (s == TOPO_OK) return;
  const std::string msg = ctx ? topo_last_error(ctx) : "topo: error";
  switch (s) {
    case TOPO_EINVAL: throw std::invalid_argument(msg);
    case TOPO_EOVERFLOW: throw std::overflow_error(msg);
    default: throw std::runtime_error(msg);
  }
}

/// One GPU bound to the reference's immutable setup objects.
class Device {
 public:
  Device(const StructuredGrid& grid, const FilterOperator& flt, const ElementStiffness& ke,
         const DomainPartition& part, int device = -1) {
    topo_grid_desc d{};
    d.nelx = grid.nelx;
    d.nely = grid.nely;
    d.nelz = grid.nelz;
    d.rmin = flt.rmin;
    d.bc = flt.bc == FilterBC::Neumann ? TOPO_BC_NEUMANN : TOPO_BC_DIRICHLET;
    d.nu = 0.3;  // unused: ke is passed explicitly
    d.device = device;
    d.rank = 0;
    d.nranks = 1;
    m_ = grid.numElements();
    n_ = grid.numDofs();
    std::vector<uint8_t> state(size_t(m_), TOPO_ACTIVE);
    for (auto e : part.pasS) state[size_t(e)] = TOPO_PASSIVE_SOLID;
    for (auto e : part.pasV) state[size_t(e)] = TOPO_PASSIVE_VOID;
    const topo_status s = topo_ctx_create(&d, ke.full.data(), ke.lower.data(), state.data(), &h_);
    if (s != TOPO_OK) {
      topo_ctx* bad = h_;
      h_ = nullptr;
      try {
        check(s, bad);
      } catch (...) {
        topo_ctx_destroy(bad);
        throw;
      }
    }
    act_ = part.act;
  }
  ~Device() { topo_ctx_destroy(h_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;

  topo_ctx* handle() const { return h_; }
  std::int64_t numElements() const { return m_; }
  std::int64_t numDofs() const { return n_; }
  const std::vector<std::int32_t>& active() const { return act_; }

 private:
  topo_ctx* h_ = nullptr;
  std::int64_t m_ = 0, n_ = 0;
  std::vector<std::int32_t> act_;
};

namespace detail {
inline void need(Eigen::Index got, std::int64_t want, const char* what) {
  if (got != want) throw std::invalid_argument(std::string(what) + ": field length mismatch");
}
}  // namespace detail

// ---------------------------------------------------------------- grid.hpp
/// grid.hpp:133-153 (built on the device, copied back)
inline IndexPairs build_symmetric_index_pairs(Device& dev) {
  IndexPairs p;
  std::int64_t m = 0, n = 0;
  std::int32_t P = 0;
  check(topo_ctx_info(dev.handle(), &m, &n, &P, nullptr, nullptr, nullptr, nullptr), dev.handle());
  p.iK.resize(size_t(m * P));
  p.jK.resize(size_t(m * P));
  check(topo_build_index_pairs(dev.handle(), p.iK.data(), p.jK.data()), dev.handle());
  return p;
}

// ------------------------------------------------------------------ fea.hpp
/// fea.hpp:135-146
inline SimpField simp_interpolate(const Eigen::VectorXd& xhat, const SimpParams& prm, Device& dev) {
  detail::need(xhat.size(), dev.numElements(), "simp");
  SimpField f;
  f.sK.resize(xhat.size());
  f.dsK.resize(xhat.size());
  const topo_simp s{prm.e0, prm.eMin, prm.p};
  check(topo_simp_interpolate(dev.handle(), xhat.data(), &s, f.sK.data(), f.dsK.data()),
        dev.handle());
  return f;
}

/// fea.hpp:162-169: the triplet values of assemble_lower, t = e * P + q
/// (aligned with build_symmetric_index_pairs; duplicates summed by the consumer)
inline std::vector<double> assemble_lower_values(const Eigen::VectorXd& sK, Device& dev) {
  if (sK.size() != dev.numElements())
    throw std::invalid_argument("assemble: index pairs do not match element count");
  std::int64_t m = 0;
  std::int32_t P = 0;
  check(topo_ctx_info(dev.handle(), &m, nullptr, &P, nullptr, nullptr, nullptr, nullptr),
        dev.handle());
  std::vector<double> vals(size_t(m * P));
  check(topo_assemble_values(dev.handle(), sK.data(), vals.data()), dev.handle());
  return vals;
}

/// fea.hpp:154-176 assemble_lower: the duplicate-summed lower triangle of K
/// (setFromTriplets order), built on the device from the per-element modulus
/// without the m*P triplets; filled through Eigen's public compressed-storage
/// API (resize + resizeNonZeros + outer/inner/value pointers).
inline SymmetricSparseMatrix assemble_lower(const Eigen::VectorXd& sK, Device& dev) {
  if (sK.size() != dev.numElements())
    throw std::invalid_argument("assemble: index pairs do not match element count");
  std::int64_t nnz = 0, m = 0, n = 0;
  check(topo_ctx_info(dev.handle(), &m, &n, nullptr, nullptr, nullptr, nullptr, nullptr),
        dev.handle());
  check(topo_csc_pattern(dev.handle(), nullptr, nullptr, &nnz), dev.handle());
  std::vector<std::int64_t> cp(size_t(n + 1));
  SymmetricSparseMatrix mat;
  mat.n = n;
  mat.lower.resize(n, n);
  mat.lower.resizeNonZeros(nnz);
  static_assert(sizeof(*mat.lower.innerIndexPtr()) == sizeof(std::int32_t), "int32 rows");
  check(topo_csc_pattern(dev.handle(), cp.data(),
                         reinterpret_cast<std::int32_t*>(mat.lower.innerIndexPtr()), nullptr),
        dev.handle());
  for (std::int64_t c = 0; c <= n; ++c) mat.lower.outerIndexPtr()[c] = int(cp[size_t(c)]);
  check(topo_csc_values(dev.handle(), sK.data(), mat.lower.valuePtr()), dev.handle());
  return mat;
}

/// fea.hpp:205-239 solve_equilibrium with the modulus field instead of the
/// assembled matrix: K(sK) u = f on the free DOFs, u = 0 on load.fixed, by
/// the device's matrix-free PCG (geometric-multigrid V-cycle preconditioner,
/// Jacobi when the grid cannot be coarsened) to ||r|| <= rtol ||f|| (the
/// reference factorises; the two agree to the solver tolerance)
/// per-thread totals of solve_state calls (wall seconds incl. host copies,
/// PCG iterations); reset by the caller
struct SolveStats {
  double seconds = 0.0;
  long long iterations = 0, calls = 0;
};
inline SolveStats& solve_stats() {
  static thread_local SolveStats s;
  return s;
}

inline Eigen::VectorXd solve_state(const Eigen::VectorXd& sK, const LoadCase& load, Device& dev,
                                   double rtol = 1e-12, int maxit = 1000000) {
  detail::need(sK.size(), dev.numElements(), "solve");
  if (load.f.size() != dev.numDofs())
    throw std::invalid_argument("solve: load vector length mismatch");
  Eigen::VectorXd u(dev.numDofs());
  std::int32_t it = 0;
  double rr = 0;
  const auto t0 = std::chrono::steady_clock::now();
  check(topo_solve_state_mg(dev.handle(), sK.data(), load.f.data(), load.fixed.data(),
                            std::int64_t(load.fixed.size()), rtol, maxit, u.data(), &it, &rr),
        dev.handle());
  SolveStats& st = solve_stats();
  st.seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  st.iterations += it;
  ++st.calls;
  if (!(rr <= rtol)) throw std::runtime_error("solve: CG did not reach the tolerance");
  return u;
}

/// fea.hpp:248-272
inline ComplianceResult compliance_and_sensitivity(const Eigen::VectorXd& u,
                                                   const Eigen::VectorXd& xhat,
                                                   const SimpParams& prm, Device& dev) {
  detail::need(u.size(), dev.numDofs(), "sensitivity");
  detail::need(xhat.size(), dev.numElements(), "sensitivity");
  ComplianceResult r;
  r.dc.resize(xhat.size());
  const topo_simp s{prm.e0, prm.eMin, prm.p};
  check(topo_sensitivity(dev.handle(), u.data(), xhat.data(), &s, &r.c, r.dc.data()),
        dev.handle());
  return r;
}

// --------------------------------------------------------------- filter.hpp
/// filter.hpp:119-122
inline Eigen::VectorXd apply_filter(const Eigen::VectorXd& x, Device& dev) {
  detail::need(x.size(), dev.numElements(), "filter");
  Eigen::VectorXd out(x.size());
  check(topo_filter(dev.handle(), x.data(), out.data(), 0), dev.handle());
  return out;
}

/// filter.hpp:126-129
inline Eigen::VectorXd apply_filter_adjoint(const Eigen::VectorXd& g, Device& dev) {
  detail::need(g.size(), dev.numElements(), "filter");
  Eigen::VectorXd out(g.size());
  check(topo_filter_adjoint(dev.handle(), g.data(), out.data()), dev.handle());
  return out;
}

/// filter.hpp:137-144 / :146-154
inline Eigen::VectorXd project(const Eigen::VectorXd& xt, const ProjectionParams& prm, Device& dev) {
  detail::need(xt.size(), dev.numElements(), "project");
  Eigen::VectorXd out(xt.size());
  check(topo_project(dev.handle(), xt.data(), prm.eta, prm.beta, out.data()), dev.handle());
  return out;
}
inline Eigen::VectorXd project_derivative(const Eigen::VectorXd& xt, const ProjectionParams& prm,
                                          Device& dev) {
  detail::need(xt.size(), dev.numElements(), "project");
  Eigen::VectorXd out(xt.size());
  check(topo_project_derivative(dev.handle(), xt.data(), prm.eta, prm.beta, out.data()),
        dev.handle());
  return out;
}

/// filter.hpp:166-171
inline Eigen::VectorXd backfilter(const Eigen::VectorXd& gradXhat, const Eigen::VectorXd& xTilde,
                                  Device& dev, const ProjectionParams& prm, bool projectionOn) {
  detail::need(gradXhat.size(), dev.numElements(), "filter");
  Eigen::VectorXd out(gradXhat.size());
  check(topo_backfilter(dev.handle(), gradXhat.data(), xTilde.data(), prm.eta, prm.beta,
                        projectionOn ? 1 : 0, out.data()),
        dev.handle());
  return out;
}

/// filter.hpp:182-228 (active set bound in the Device)
inline EtaSolveResult solve_volume_preserving_eta(const Eigen::VectorXd& xTilde, double beta,
                                                  double eta0, Device& dev) {
  detail::need(xTilde.size(), dev.numElements(), "eta solve");
  EtaSolveResult r;
  std::int32_t it = 0;
  check(topo_solve_eta(dev.handle(), xTilde.data(), beta, eta0, &r.eta, &it), dev.handle());
  r.iterations = it;
  return r;
}

// ------------------------------------------------------------------- oc.hpp
/// oc.hpp:31-39
inline double lambda_upper_estimate(const Eigen::VectorXd& xAct, const Eigen::VectorXd& dcAct,
                                    const Eigen::VectorXd& dVAct, double volfrac,
                                    std::int64_t mTotal, Device& dev) {
  double lam = 0;
  check(topo_lambda_upper(dev.handle(), xAct.size(), xAct.data(), dcAct.data(), dVAct.data(),
                          volfrac, mTotal, &lam),
        dev.handle());
  return lam;
}

/// oc.hpp:72-79
inline Eigen::VectorXd oc_candidate(const Eigen::VectorXd& xAct, const Eigen::VectorXd& dcAct,
                                    const Eigen::VectorXd& dVAct, double lambda, double move,
                                    Device& dev) {
  Eigen::VectorXd out(xAct.size());
  check(topo_oc_candidate(dev.handle(), xAct.size(), xAct.data(), dcAct.data(), dVAct.data(),
                          lambda, move, out.data()),
        dev.handle());
  return out;
}

/// The physical-volume callback of oc.hpp:96 as the built-in volume of a
/// filter mode (driver.hpp:214-229): device-resident, no host round trips.
enum class VolumeMode { Mean = TOPO_VOL_MEAN, Projected = TOPO_VOL_PROJECTED,
                        Filtered = TOPO_VOL_FILTERED };

namespace detail {
inline double volume_trampoline(void* user, const double* x, int64_t m) {
  auto* f = static_cast<const std::function<double(const Eigen::VectorXd&)>*>(user);
  Eigen::VectorXd v(m);
  std::memcpy(v.data(), x, sizeof(double) * size_t(m));
  return (*f)(v);
}
inline UpdateResult bisect(const Eigen::VectorXd& x, const Eigen::VectorXd& dc,
                           const Eigen::VectorXd& dV, const OcParams& prm, const BisectOptions& opt,
                           int mode, double eta, double beta, topo_volume_fn cb, void* user,
                           Device& dev) {
  need(x.size(), dev.numElements(), "oc");
  UpdateResult r;
  r.xNew.resize(x.size());
  const topo_oc_params p{prm.move, prm.volfrac, prm.bisectRelTol, prm.volumeTol,
                         opt.lambdaSpace ? 1 : 0, opt.absTol, opt.lambdaMax};
  std::int32_t bis = 0;
  check(topo_oc_bisect(dev.handle(), x.data(), dc.data(), dV.data(), &p, mode, eta, beta, cb, user,
                       r.xNew.data(), &r.lambda, &bis, nullptr),
        dev.handle());
  r.bisections = bis;
  return r;
}
}  // namespace detail

/// oc.hpp:93-174 with a host callback (the reference's std::function form)
inline UpdateResult bisect_update(const Eigen::VectorXd& x, const Eigen::VectorXd& dc,
                                  const Eigen::VectorXd& dV, const OcParams& prm,
                                  const std::function<double(const Eigen::VectorXd&)>& physicalVolume,
                                  Device& dev, const BisectOptions& opt = {}) {
  return detail::bisect(x, dc, dV, prm, opt, TOPO_VOL_CALLBACK, 0.5, 1.0,
                        detail::volume_trampoline,
                        const_cast<std::function<double(const Eigen::VectorXd&)>*>(&physicalVolume),
                        dev);
}

/// oc.hpp:93-174 with a device-resident volume (ft = 1 / 2 / 3)
inline UpdateResult bisect_update(const Eigen::VectorXd& x, const Eigen::VectorXd& dc,
                                  const Eigen::VectorXd& dV, const OcParams& prm, VolumeMode mode,
                                  Device& dev, const ProjectionParams& prj = {},
                                  const BisectOptions& opt = {}) {
  return detail::bisect(x, dc, dV, prm, opt, int(mode), prj.eta, prj.beta, nullptr, nullptr, dev);
}

/// oc.hpp:181-241 primal_dual_update (ft = 1), with the reference's fallback
/// to the mean-volume bisection
inline UpdateResult primal_dual_update(const Eigen::VectorXd& x, const Eigen::VectorXd& dc,
                                       const Eigen::VectorXd& dV, const OcParams& prm,
                                       Device& dev) {
  detail::need(x.size(), dev.numElements(), "oc");
  detail::need(dc.size(), dev.numElements(), "oc");
  detail::need(dV.size(), dev.numElements(), "oc");
  topo_oc_params p{prm.move, prm.volfrac, prm.bisectRelTol, prm.volumeTol, 0, 1e-8, 0.0};
  UpdateResult r;
  r.xNew.resize(x.size());
  std::int32_t it = 0, fb = 0;
  check(topo_oc_primal_dual(dev.handle(), x.data(), dc.data(), dV.data(), &p, prm.pdTol,
                            r.xNew.data(), &r.lambda, &it, &fb),
        dev.handle());
  r.bisections = it;
  return r;
}

// ----------------------------------------------------------- fused pass
/// driver.hpp:183-231 (ft = 3) with the displacement supplied
struct PassResult {
  Eigen::VectorXd xTilde, xPhys, dcPhys, dc, dV, xNew;
  double eta = 0, c = 0, lambda = 0;
  int etaIterations = 0, bisections = 0;
};

inline PassResult design_pass(const Eigen::VectorXd& x, const Eigen::VectorXd& u,
                              const SimpParams& simp, double beta, double eta0, double move,
                              double volfrac, Device& dev) {
  detail::need(x.size(), dev.numElements(), "pass");
  detail::need(u.size(), dev.numDofs(), "pass");
  PassResult r;
  for (auto* v : {&r.xTilde, &r.xPhys, &r.dcPhys, &r.dc, &r.dV, &r.xNew}) v->resize(x.size());
  topo_pass_params p{};
  p.simp = {simp.e0, simp.eMin, simp.p};
  p.beta = beta;
  p.eta0 = eta0;
  p.move = move;
  p.volfrac = volfrac;
  p.eta_override = std::numeric_limits<double>::quiet_NaN();
  p.volume_mode = TOPO_VOL_FILTERED;
  p.write_sk = 1;
  topo_pass_out o{};
  o.xTilde = r.xTilde.data();
  o.xPhys = r.xPhys.data();
  o.dcPhys = r.dcPhys.data();
  o.dc = r.dc.data();
  o.dV = r.dV.data();
  o.xNew = r.xNew.data();
  check(topo_design_pass(dev.handle(), x.data(), u.data(), &p, &o), dev.handle());
  r.eta = o.eta;
  r.c = o.c;
  r.lambda = o.lambda;
  r.etaIterations = o.eta_iters;
  r.bisections = o.bisections;
  return r;
}

}  // namespace gpu
}  // namespace topopt
