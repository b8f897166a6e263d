// TEST: gpu::run_optimization (include/topopt_gpu_driver.hpp) against the
// reference's run_optimization (driver.hpp:137-265, compiled from the reference
// headers with the oracle's Eigen shim): the same redesign loop with every
// stage and the state solve on the device. The reference factorises K and the
// device iterates CG to 1e-12, so histories agree to ~1e-9, not bitwise.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "topopt/driver.hpp"
#include "topopt_gpu.hpp"
#include "topopt_gpu_driver.hpp"

using namespace topopt;

static int failures = 0;
static void expect(bool ok, const char* what, double err = 0) {
  std::printf("%-52s %s  (%.3g)\n", what, ok ? "ok" : "FAIL", err);
  if (!ok) ++failures;
}

static void compare(const char* name, const RunConfig& cfg, const Problem& prob) {
  const RunResult r = run_optimization(cfg, prob);
  const RunResult g = gpu::run_optimization(cfg, prob);
  bool same = r.history.size() == g.history.size() && r.converged == g.converged;
  double dc = 0;
  for (size_t i = 0; same && i < r.history.size(); ++i) {
    const auto &a = r.history[i], &b = g.history[i];
    same = same && a.bisections == b.bisections && a.beta == b.beta && a.penal == b.penal;
    dc = std::max(dc, std::abs(a.c - b.c) / std::abs(a.c));
    dc = std::max(dc, std::abs(a.eta - b.eta));
  }
  double dx = 0;
  for (Eigen::Index e = 0; same && e < r.field.xPhys.size(); ++e)
    dx = std::max(dx, std::abs(r.field.xPhys[e] - g.field.xPhys[e]));
  char what[128];
  std::snprintf(what, sizeof what, "%s: %zu loops, history", name, r.history.size());
  expect(same && dc <= 1e-7, what, dc);
  std::snprintf(what, sizeof what, "%s: final xPhys", name);
  expect(same && dx <= 1e-6, what, dx);
}

// --bench nelx nely nelz maxit: the device loop alone on the 3D cantilever
// preset (top3D125 defaults: ft = 3, rmin = 1.5), per-iteration records
static int bench(int nelx, int nely, int nelz, int maxit) {
  RunConfig cfg;
  cfg.nelx = nelx, cfg.nely = nely, cfg.nelz = nelz, cfg.maxit = maxit;
  cfg.ft = 3, cfg.rmin = 1.5, cfg.volfrac = 0.12, cfg.move = 0.1;
  const RunResult g = gpu::run_optimization(
      cfg, preset_cantilever_3d(nelx, nely, nelz), [](const IterationRecord& r) {
        gpu::SolveStats& st = gpu::solve_stats();
        std::printf("it %3d  c %.6e  v %.4f  ch %.3e  eta %.6f  bis %3d  %.3f s  (solve %.3f s, "
                    "%lld MGCG its)\n",
                    r.loop, r.c, r.v, r.resnorm, r.eta, r.bisections, r.seconds, st.seconds,
                    st.iterations);
        st = gpu::SolveStats{};
      }, {}, 1e-6);
  std::printf("total %.2f s for %zu iterations\n", g.wallSeconds, g.history.size());
  return 0;
}

int main(int argc, char** argv) {
  if (argc == 6 && std::string(argv[1]) == "--bench")
    return bench(std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4]), std::atoi(argv[5]));
  {  // ft = 3 volume-preserving projection, MBB (top99neo defaults)
    RunConfig cfg;
    cfg.nelx = 30, cfg.nely = 10, cfg.rmin = 2.4, cfg.ft = 3, cfg.maxit = 8;
    compare("MBB 30x10 ft=3", cfg, preset_mbb_2d(30, 10));
  }
  {  // 3D cantilever, ft = 3, beta continuation
    RunConfig cfg;
    cfg.nelx = 8, cfg.nely = 4, cfg.nelz = 4, cfg.rmin = 1.5, cfg.ft = 3, cfg.maxit = 5;
    cfg.volfrac = 0.3;
    cfg.move = 0.1;
    cfg.betaCont = ContinuationSchedule{2, 8.0, 2, 2.0};
    compare("cantilever 8x4x4 ft=3 + beta continuation", cfg, preset_cantilever_3d(8, 4, 4));
  }
  {  // ft = 1 with the primal-dual update and Anderson extrapolation
    RunConfig cfg;
    cfg.nelx = 24, cfg.nely = 12, cfg.rmin = 2.0, cfg.ft = 1, cfg.maxit = 12;
    cfg.update = UpdateStrategy::PrimalDual;
    cfg.accel.enabled = true;
    cfg.accel.q0 = 3;
    compare("MBB 24x12 ft=1 primal-dual + Anderson", cfg, preset_mbb_2d(24, 12));
  }
  {  // ft = 2 fixed-threshold projection with penal continuation
    RunConfig cfg;
    cfg.nelx = 20, cfg.nely = 10, cfg.rmin = 1.8, cfg.ft = 2, cfg.maxit = 6;
    cfg.penalCont = ContinuationSchedule{1, 4.0, 2, 0.5};
    compare("MBB 20x10 ft=2 + penal continuation", cfg, preset_mbb_2d(20, 10));
  }
  {  // frame reinforcement preset: passive solid frame and void opening (driver.hpp:306-341),
     // 5202 DOFs (the smallest size the preset accepts; the shim's envelope Cholesky)
    RunConfig cfg;
    cfg.nelx = 50, cfg.nely = 50, cfg.rmin = 2.5, cfg.ft = 3, cfg.maxit = 3;
    cfg.volfrac = 0.4;
    compare("frame 50x50 ft=3 (passives)", cfg, preset_frame_2d(50, 50, 1));
  }
  {  // ft = 3 with Anderson extrapolation (device accel.hpp) and the frame's passives
    RunConfig cfg;
    cfg.nelx = 50, cfg.nely = 50, cfg.rmin = 2.5, cfg.ft = 3, cfg.maxit = 10;
    cfg.volfrac = 0.4;
    cfg.accel.enabled = true;
    cfg.accel.q0 = 2;
    cfg.accel.q = 3;
    compare("frame 50x50 ft=3 + Anderson", cfg, preset_frame_2d(50, 50, -1));
  }
  {  // ft = 2 with Anderson, bisection on the projected volume
    RunConfig cfg;
    cfg.nelx = 24, cfg.nely = 12, cfg.rmin = 2.0, cfg.ft = 2, cfg.maxit = 9;
    cfg.accel.enabled = true;
    cfg.accel.q0 = 1;
    cfg.accel.depth = 3;
    compare("MBB 24x12 ft=2 + Anderson", cfg, preset_mbb_2d(24, 12));
  }
  std::printf("%d failure(s)\n", failures);
  return failures ? 1 : 0;
}
