// TEST: the C++ drop-in adapter (include/topopt_gpu.hpp) against the
// reference's own functions (proj/include/topopt, compiled against
// oracle/eigen_shim), on small grids. Built by __graft_entry__.build() in the
// container that has /root/reference; run on a GPU by
// tests/test_gpu_adapter.py. Exit code 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <random>

#include "topopt/fea.hpp"
#include "topopt/filter.hpp"
#include "topopt/grid.hpp"
#include "topopt/oc.hpp"
#include "topopt_gpu.hpp"

using namespace topopt;

static int failures = 0;
static void expect(bool ok, const char* what, double err = 0) {
  std::printf("%-52s %s  (%.3g)\n", what, ok ? "ok" : "FAIL", err);
  if (!ok) ++failures;
}
static double rel(const Eigen::VectorXd& a, const Eigen::VectorXd& b) {
  double num = 0, den = 0;
  for (Eigen::Index i = 0; i < a.size(); ++i) {
    num = std::max(num, std::abs(a[i] - b[i]));
    den = std::max(den, std::abs(b[i]));
  }
  return den > 0 ? num / den : num;
}

int main() {
  std::mt19937 rng(11);
  std::uniform_real_distribution<double> U(0.01, 1.0);
  std::normal_distribution<double> N(0.0, 1.0);
  for (StructuredGrid grid : {StructuredGrid{30, 12, 0}, StructuredGrid{10, 7, 6}}) {
    const double rmin = grid.is3d() ? 2.3 : 3.5;
    const DomainPartition part = partition_domain(grid, {0, 1, 2}, {5, 6});
    const FilterOperator flt = build_filter(grid, rmin, FilterBC::Neumann);
    const ElementStiffness ke = grid.is3d() ? element_stiffness_h8(0.3) : element_stiffness_q4(0.3);
    gpu::Device dev(grid, flt, ke, part);
    const auto m = grid.numElements();
    Eigen::VectorXd x(m), u(grid.numDofs());
    for (Eigen::Index i = 0; i < m; ++i) x[i] = U(rng);
    for (Eigen::Index i = 0; i < u.size(); ++i) u[i] = N(rng);
    for (auto e : part.pasS) x[e] = 1.0;
    for (auto e : part.pasV) x[e] = 0.0;

    const IndexPairs pr = build_symmetric_index_pairs(build_connectivity(grid));
    const IndexPairs pg = gpu::build_symmetric_index_pairs(dev);
    expect(pr.iK == pg.iK && pr.jK == pg.jK, "index pairs bit-exact");

    const Eigen::VectorXd xt = apply_filter(x, flt), xtg = gpu::apply_filter(x, dev);
    expect(rel(xtg, xt) <= 1e-12, "apply_filter", rel(xtg, xt));
    const Eigen::VectorXd at = apply_filter_adjoint(x, flt), atg = gpu::apply_filter_adjoint(x, dev);
    expect(rel(atg, at) <= 1e-12, "apply_filter_adjoint", rel(atg, at));
    const ProjectionParams prj{0.45, 3.0};
    expect(rel(gpu::project(xt, prj, dev), project(xt, prj)) <= 1e-14, "project");
    const Eigen::VectorXd bf = backfilter(x, xt, flt, prj, true);
    expect(rel(gpu::backfilter(x, xt, dev, prj, true), bf) <= 1e-12, "backfilter");
    const EtaSolveResult er = solve_volume_preserving_eta(xt, 2.0, 0.5, part);
    const EtaSolveResult eg = gpu::solve_volume_preserving_eta(xt, 2.0, 0.5, dev);
    expect(std::abs(er.eta - eg.eta) <= 5e-8, "solve_volume_preserving_eta", er.eta - eg.eta);
    const SimpParams simp{1.0, 1e-9, 3.0};
    const SimpField sr = simp_interpolate(x, simp), sg = gpu::simp_interpolate(x, simp, dev);
    expect(rel(sg.sK, sr.sK) <= 1e-12 && rel(sg.dsK, sr.dsK) <= 1e-12, "simp_interpolate");
    const SymmetricSparseMatrix Kr = assemble_lower(pr, ke, sr.sK, grid.numDofs());
    const SymmetricSparseMatrix Kg = gpu::assemble_lower(sr.sK, dev);
    const auto nz = Kr.lower.nonZeros();
    expect(Kg.lower.nonZeros() == nz &&
               std::equal(Kr.lower.outerIndexPtr(), Kr.lower.outerIndexPtr() + grid.numDofs() + 1,
                          Kg.lower.outerIndexPtr()) &&
               std::equal(Kr.lower.innerIndexPtr(), Kr.lower.innerIndexPtr() + nz,
                          Kg.lower.innerIndexPtr()) &&
               std::memcmp(Kr.lower.valuePtr(), Kg.lower.valuePtr(), sizeof(double) * nz) == 0,
           "assemble_lower (CSC bit-exact)");
    const ComplianceResult cr = compliance_and_sensitivity(u, build_connectivity(grid), x, simp, ke, part);
    const ComplianceResult cg = gpu::compliance_and_sensitivity(u, x, simp, dev);
    expect(std::abs(cr.c - cg.c) <= 1e-12 * std::abs(cr.c) && rel(cg.dc, cr.dc) <= 1e-12,
           "compliance_and_sensitivity", rel(cg.dc, cr.dc));
    // OC with the reference's std::function callback, through the adapter
    Eigen::VectorXd dc = -cr.dc.cwiseAbs(), dV = Eigen::VectorXd::Constant(m, 1.0 / m);
    for (auto e : part.act) dc[e] -= 0.01;
    auto mean = [](const Eigen::VectorXd& v) { return v.mean(); };
    OcParams oc;
    const UpdateResult ur = bisect_update(x, dc, dV, part, oc, mean);
    const UpdateResult ug = gpu::bisect_update(x, dc, dV, oc, mean, dev);
    expect(ur.bisections == ug.bisections && std::abs(ur.lambda - ug.lambda) <= 1e-10 * ur.lambda &&
               rel(ug.xNew, ur.xNew) <= 1e-12,
           "bisect_update (std::function volume)", ur.lambda - ug.lambda);
    const UpdateResult um = gpu::bisect_update(x, dc, dV, oc, gpu::VolumeMode::Mean, dev);
    expect(um.bisections == ur.bisections && rel(um.xNew, ur.xNew) <= 1e-12,
           "bisect_update (device mean volume)");
    const UpdateResult pr_ = primal_dual_update(x, dc, dV, part, oc);
    const UpdateResult pg_ = gpu::primal_dual_update(x, dc, dV, oc, dev);
    expect(pr_.bisections == pg_.bisections &&
               std::abs(pr_.lambda - pg_.lambda) <= 1e-10 * pr_.lambda &&
               rel(pg_.xNew, pr_.xNew) <= 1e-12,
           "primal_dual_update", pr_.lambda - pg_.lambda);
    // error mapping
    bool threw = false;
    try {
      gpu::apply_filter(Eigen::VectorXd::Zero(m + 1), dev);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    expect(threw, "length mismatch -> std::invalid_argument");
  }
  std::printf("%d failure(s)\n", failures);
  return failures ? 1 : 0;
}
