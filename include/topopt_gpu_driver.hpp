// topopt_gpu_driver.hpp — the reference's run_optimization (driver.hpp:137-265)
// on the B200 operators of topopt_gpu.hpp: every hot-path stage, the state
// solve, the Anderson extrapolation (accel.hpp) and the record reductions on
// the device; the scalar control (continuation, loop exit) on the host exactly
// as the reference does it. TOPO_LOOP_DEVICE=0 runs the stage-by-stage loop
// over host Eigen vectors instead (the reference's own AndersonAccelerator).
// Include after "topopt/driver.hpp" and "topopt_gpu.hpp".
// SURVEY.md §8(f) row 3 (the full redesign loop).
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>

namespace topopt {
namespace gpu {

namespace detail {
// device buffer through the C-ABI (the header has no CUDA runtime of its own)
struct DevVec {
  topo_ctx* h = nullptr;
  double* p = nullptr;
  DevVec(topo_ctx* ctx, std::int64_t n) : h(ctx) {
    void* q = nullptr;
    check(topo_device_alloc(h, std::int64_t(sizeof(double)) * n, &q), h);
    p = static_cast<double*>(q);
  }
  ~DevVec() { topo_device_free(h, p); }
  DevVec(const DevVec&) = delete;
  DevVec& operator=(const DevVec&) = delete;
};
}  // namespace detail

/// The device-resident form of driver.hpp:179-265: design, filtered and
/// physical fields, moduli, displacements, sensitivities and the updated
/// design stay in device memory for every filter type (ft = 1 / 2 / 3), both
/// update strategies and the Anderson extrapolation (accel.hpp on the device,
/// topo_anderson_step); per iteration only scalars come back (eta, c, lambda,
/// the three records of topo_loop_records: residual ch, volume, nondiscreteness).
/// ft = 3 with bisection runs the fused pass at the solved eta (sensitivity,
/// back-filters, OC in one call); the other modes call the stage kernels on
/// device arrays. A probe, when given, receives host copies of x, dc and dV
/// (the only per-iteration transfers, made because the caller asked).
inline void run_loop_device(const RunConfig& cfg, const Problem& prob, Device& dev,
                            Eigen::VectorXd& x, double& penal, double& beta, double& eta,
                            double& ch, Eigen::VectorXd& xPrevPhys, RunResult& result,
                            const RecordSink& sink, const OcProbe& probe, double solve_rtol) {
  topo_ctx* h = dev.handle();
  const std::int64_t m = dev.numElements(), n = dev.numDofs();
  const DomainPartition& part = prob.part;
  const std::int64_t bm = std::int64_t(sizeof(double)) * m;
  detail::DevVec x_d(h, m), xn_d(h, m), xt_d(h, m), xp_d(h, m), xprev_d(h, m), e_d(h, m),
      f_d(h, n), u_d(h, n), dcp_d(h, m), dc_d(h, m), dv_d(h, m), dv0_d(h, m);
  check(topo_copy(h, x_d.p, x.data(), bm), h);
  check(topo_copy(h, xprev_d.p, xPrevPhys.data(), bm), h);
  check(topo_copy(h, f_d.p, prob.load.f.data(), std::int64_t(sizeof(double)) * n), h);
  {
    Eigen::VectorXd dV0 = Eigen::VectorXd::Zero(m);  // driver.hpp:155-156
    for (auto e : part.act) dV0[e] = 1.0 / double(m);
    check(topo_copy(h, dv0_d.p, dV0.data(), bm), h);
  }
  const bool fused = cfg.ft == 3 && cfg.update != UpdateStrategy::PrimalDual && !probe;
  const bool projecting = cfg.ft >= 2;
  const int vmode = cfg.ft == 1 ? TOPO_VOL_MEAN : cfg.ft == 2 ? TOPO_VOL_PROJECTED : TOPO_VOL_FILTERED;
  const topo_anderson aopt{cfg.accel.depth, cfg.accel.q, cfg.accel.alpha, cfg.accel.zeta};
  check(topo_anderson_reset(h), h);
  double* xcur = x_d.p;
  double* xnext = xn_d.p;
  for (int loop = 1; loop <= cfg.maxit && ch > cfg.tol; ++loop) {
    const auto iterStart = std::chrono::steady_clock::now();
    // RL.1 physical density field (driver.hpp:182-190)
    check(topo_filter(h, xcur, xt_d.p, 1), h);
    if (cfg.ft == 3) {
      double etaNew = eta;
      std::int32_t etaIts = 0;
      check(topo_solve_eta(h, xt_d.p, beta, eta, &etaNew, &etaIts), h);
      eta = etaNew;
    }
    const double* xphys = xt_d.p;
    if (projecting) {
      check(topo_project(h, xt_d.p, eta, beta, xp_d.p), h);
      xphys = xp_d.p;
    }
    // RL.2 equilibrium
    const topo_simp simp{cfg.e0, cfg.eMin, penal};
    check(topo_simp_interpolate(h, xphys, &simp, e_d.p, nullptr), h);
    std::int32_t its = 0;
    double rr = 0.0;
    const auto t0 = std::chrono::steady_clock::now();
    check(topo_solve_state_mg(h, e_d.p, f_d.p, prob.load.fixed.data(),
                              std::int64_t(prob.load.fixed.size()), solve_rtol, 1000000, u_d.p,
                              &its, &rr),
          h);
    if (!(rr <= solve_rtol)) throw std::runtime_error("solve: CG did not reach the tolerance");
    SolveStats& st = solve_stats();
    st.seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    st.iterations += its;
    ++st.calls;
    // RL.3 + RL.4 sensitivities, back-filters, redesign
    double c = 0.0;
    int bisections = 0;
    if (fused) {  // one pass at this eta (driver.hpp:192-231)
      topo_pass_params pp{};
      pp.simp = simp;
      pp.beta = beta;
      pp.eta0 = eta;
      pp.move = cfg.move;
      pp.volfrac = cfg.volfrac;
      pp.eta_override = eta;
      pp.volume_mode = TOPO_VOL_FILTERED;
      pp.write_sk = 0;
      topo_pass_out po{};
      po.xNew = xnext;
      check(topo_design_pass(h, xcur, u_d.p, &pp, &po), h);
      c = po.c;
      bisections = po.bisections;
    } else {
      check(topo_sensitivity(h, u_d.p, xphys, &simp, &c, dcp_d.p), h);  // driver.hpp:192
      check(topo_backfilter(h, dcp_d.p, xt_d.p, eta, beta, projecting ? 1 : 0, dc_d.p), h);
      check(topo_backfilter(h, dv0_d.p, xt_d.p, eta, beta, projecting ? 1 : 0, dv_d.p), h);
      if (probe) {
        Eigen::VectorXd xh(m), dch(m), dvh(m);
        check(topo_copy(h, xh.data(), xcur, bm), h);
        check(topo_copy(h, dch.data(), dc_d.p, bm), h);
        check(topo_copy(h, dvh.data(), dv_d.p, bm), h);
        probe(loop, xh, dch, dvh);
      }
      double lam = 0.0;
      if (cfg.update == UpdateStrategy::PrimalDual && cfg.ft == 1) {  // driver.hpp:211-212
        const OcParams prm{};
        topo_oc_params p{cfg.move, cfg.volfrac, prm.bisectRelTol, prm.volumeTol, 0, 1e-8, 0.0};
        std::int32_t it = 0, fb = 0;
        check(topo_oc_primal_dual(h, xcur, dc_d.p, dv_d.p, &p, prm.pdTol, xnext, &lam, &it, &fb),
              h);
        bisections = it;
      } else {  // oc.hpp:93-174 with the ft's volume (driver.hpp:213-230)
        const OcParams prm{};
        const BisectOptions bo{};
        topo_oc_params p{cfg.move, cfg.volfrac, prm.bisectRelTol, prm.volumeTol,
                         bo.lambdaSpace ? 1 : 0, bo.absTol, bo.lambdaMax};
        std::int32_t bis = 0;
        check(topo_oc_bisect(h, xcur, dc_d.p, dv_d.p, &p, vmode, eta, beta, nullptr, nullptr,
                             xnext, &lam, &bis, nullptr),
              h);
        bisections = bis;
      }
    }
    // optional extrapolation on the active design (driver.hpp:235-244)
    if (cfg.accel.enabled && loop >= cfg.accel.q0 && !part.act.empty())
      check(topo_anderson_step(h, &aopt, xcur, xnext), h);
    std::swap(xcur, xnext);
    const double penalUsed = penal, betaUsed = beta;
    if (cfg.penalCont) penal = apply_continuation(penal, *cfg.penalCont, loop);
    if (cfg.betaCont) beta = apply_continuation(beta, *cfg.betaCont, loop);
    // RL.5 record: ch (driver.hpp:189), v, mnd -- device reductions
    double rec3[3];
    check(topo_loop_records(h, xphys, xprev_d.p, xcur, rec3), h);
    ch = rec3[0];
    IterationRecord rec;
    rec.loop = loop;
    rec.c = c;
    rec.v = rec3[1];
    rec.resnorm = ch;
    rec.mnd = rec3[2];
    rec.penal = penalUsed;
    rec.beta = betaUsed;
    rec.eta = eta;
    rec.bisections = bisections;
    rec.seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - iterStart).count();
    if (sink) sink(rec);
    result.history.push_back(rec);
  }
  check(topo_copy(h, x.data(), xcur, bm), h);
  check(topo_copy(h, xPrevPhys.data(), xprev_d.p, bm), h);
}

/// driver.hpp:137-265 with the equilibrium solved by solve_state (rtol
/// solve_rtol) instead of the Cholesky factorisation.
inline RunResult run_optimization(const RunConfig& cfg, const Problem& prob,
                                  const RecordSink& sink = {}, const OcProbe& probe = {},
                                  double solve_rtol = 1e-12, int device = -1) {
  topopt::detail::validate_config(cfg, prob);
  const auto start = std::chrono::steady_clock::now();
  const StructuredGrid& grid = prob.grid;
  const std::int64_t m = grid.numElements();
  const DomainPartition& part = prob.part;
  const ElementStiffness ke =
      grid.is3d() ? element_stiffness_h8(cfg.nu) : element_stiffness_q4(cfg.nu);
  FilterOperator flt;  // the device builds its own taps / hs from (rmin, bc)
  flt.nelx = grid.nelx;
  flt.nely = grid.nely;
  flt.nelz = grid.nelz;
  flt.rmin = cfg.rmin;
  flt.bc = cfg.ftBC;
  Device dev(grid, flt, ke, part, device);

  Eigen::VectorXd dV0 = Eigen::VectorXd::Zero(m);
  for (auto e : part.act) dV0[e] = 1.0 / double(m);
  Eigen::VectorXd x = Eigen::VectorXd::Zero(m);  // driver.hpp:161-165
  const double x0 = part.act.empty() ? 0.0
                                     : (cfg.volfrac * double(m) - double(part.pasS.size())) /
                                           double(part.act.size());
  for (auto e : part.act) x[e] = std::clamp(x0, 0.0, 1.0);
  topopt::detail::pin_passives(x, part);

  double penal = cfg.penal, beta = cfg.beta, eta = cfg.eta;
  AndersonAccelerator accel(
      AndersonOptions{cfg.accel.depth, cfg.accel.q, cfg.accel.alpha, cfg.accel.zeta});
  Eigen::VectorXd xPrevPhys = Eigen::VectorXd::Ones(m);
  RunResult result;
  result.history.reserve(size_t(cfg.maxit));
  double ch = 1.0;
  const VolumeMode vmode = cfg.ft == 1 ? VolumeMode::Mean
                           : cfg.ft == 2 ? VolumeMode::Projected
                                         : VolumeMode::Filtered;

  const char* dl = std::getenv("TOPO_LOOP_DEVICE");  // 0: the stage-by-stage host loop below
  const bool device_loop = !(dl && dl[0] == '0');
  if (device_loop)
    run_loop_device(cfg, prob, dev, x, penal, beta, eta, ch, xPrevPhys, result, sink, probe,
                    solve_rtol);
  for (int loop = 1; !device_loop && loop <= cfg.maxit && ch > cfg.tol; ++loop) {
    const auto iterStart = std::chrono::steady_clock::now();
    // RL.1 physical density field
    Eigen::VectorXd xTilde = apply_filter(x, dev);
    topopt::detail::pin_passives(xTilde, part);
    if (cfg.ft == 3) eta = solve_volume_preserving_eta(xTilde, beta, eta, dev).eta;
    const ProjectionParams prj{eta, beta};
    Eigen::VectorXd xPhys = cfg.ft >= 2 ? project(xTilde, prj, dev) : xTilde;
    ch = (xPhys - xPrevPhys).norm() / std::sqrt(double(m));
    xPrevPhys = xPhys;
    // RL.2 equilibrium
    const SimpParams simp{cfg.e0, cfg.eMin, penal};
    const SimpField law = simp_interpolate(xPhys, simp, dev);
    const Eigen::VectorXd u = solve_state(law.sK, prob.load, dev, solve_rtol);
    // RL.3 sensitivities, backfiltered
    const ComplianceResult comp = compliance_and_sensitivity(u, xPhys, simp, dev);
    const bool projecting = cfg.ft >= 2;
    const Eigen::VectorXd dc = backfilter(comp.dc, xTilde, dev, prj, projecting);
    const Eigen::VectorXd dV = backfilter(dV0, xTilde, dev, prj, projecting);
    if (probe) probe(loop, x, dc, dV);
    // RL.4 redesign, optional extrapolation, continuation
    OcParams oc;
    oc.move = cfg.move;
    oc.volfrac = cfg.volfrac;
    UpdateResult up = cfg.update == UpdateStrategy::PrimalDual && cfg.ft == 1
                          ? primal_dual_update(x, dc, dV, oc, dev)
                          : bisect_update(x, dc, dV, oc, vmode, dev, prj);
    const Eigen::VectorXd xBefore = std::move(x);
    x = std::move(up.xNew);
    if (cfg.accel.enabled && loop >= cfg.accel.q0 && !part.act.empty()) {
      Eigen::VectorXd xT(Eigen::Index(part.act.size())), r(Eigen::Index(part.act.size()));
      for (size_t i = 0; i < part.act.size(); ++i) {
        xT[Eigen::Index(i)] = xBefore[part.act[i]];
        r[Eigen::Index(i)] = x[part.act[i]] - xT[Eigen::Index(i)];
      }
      const Eigen::VectorXd xNext = accel.step(xT, r);
      for (size_t i = 0; i < part.act.size(); ++i)
        x[part.act[i]] = std::clamp(xNext[Eigen::Index(i)], 0.0, 1.0);
    }
    const double penalUsed = penal, betaUsed = beta;
    if (cfg.penalCont) penal = apply_continuation(penal, *cfg.penalCont, loop);
    if (cfg.betaCont) beta = apply_continuation(beta, *cfg.betaCont, loop);
    // RL.5 record
    IterationRecord rec;
    rec.loop = loop;
    rec.c = comp.c;
    rec.v = xPhys.mean();
    rec.resnorm = ch;
    rec.mnd = nondiscreteness(x);
    rec.penal = penalUsed;
    rec.beta = betaUsed;
    rec.eta = eta;
    rec.bisections = up.bisections;
    rec.seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - iterStart).count();
    if (sink) sink(rec);
    result.history.push_back(rec);
  }
  if (!result.history.empty()) {  // driver.hpp:252-258
    Eigen::VectorXd xTilde = apply_filter(x, dev);
    topopt::detail::pin_passives(xTilde, part);
    if (cfg.ft == 3) eta = solve_volume_preserving_eta(xTilde, beta, eta, dev).eta;
    Eigen::VectorXd xPhys = cfg.ft >= 2 ? project(xTilde, {eta, beta}, dev) : xTilde;
    result.field = {std::move(x), std::move(xTilde), std::move(xPhys)};
    result.converged = ch <= cfg.tol;
  } else {
    result.field = {x, x, x};
  }
  result.wallSeconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
  return result;
}

}  // namespace gpu
}  // namespace topopt
