// Host/device state machines that replay the reference's scalar control flow
// exactly, fed with reductions computed elsewhere (one GPU: a cooperative
// kernel; several GPUs: per-rank partial sums + an allreduce). Every scalar
// statement keeps the reference's operation order, so identical inputs give
// identical decisions on host and device.
#pragma once

#include <math.h>

#ifndef __CUDACC__
#define __host__
#define __device__
#endif

namespace topo {

/// filter.hpp:182-228 solve_volume_preserving_eta, driven by (g, g') values.
/// Usage: init(eta0); feed(g(eta), g'(eta)) at the current eta while it
/// returns 1 (a new eta to evaluate); done when it returns 0.
struct EtaCtl {
  double lo, hi, eta, g, step;
  int it, done;

  __host__ __device__ void init(double eta0) {
    lo = 0.0;
    hi = 1.0;
    eta = eta0 < 0.0 ? 0.0 : (eta0 > 1.0 ? 1.0 : eta0);  // std::clamp, filter.hpp:204
    step = INFINITY;
    it = 0;
    done = 0;
  }
  // g_cur = mismatch(eta) (already / m), gp_cur = slope(eta) (/ m)
  __host__ __device__ int feed(double g_cur, double gp_cur) {
    g = g_cur;
    const double tol = 1e-6;  // filter.hpp:206-207
    const int maxIter = 50;
    if (!(it < maxIter && (fabs(g) > tol || step > 1e-8))) {  // filter.hpp:213
      done = 1;
      return 0;
    }
    if (g > 0)
      lo = eta;
    else
      hi = eta;
    double next = eta - g / gp_cur;
    if (!isfinite(next) || next <= lo || next >= hi) next = 0.5 * (lo + hi);  // :220
    step = fabs(next - eta);
    eta = next;
    ++it;
    return 1;
  }
};

/// oc.hpp:93-174 bisect_update, driven by volume values V(s) at the requested
/// square-root multipliers s. The caller evaluates V(s_req) and calls feed()
/// while pending(); s_final is the multiplier whose candidate the reference
/// leaves in xNew, lam_result its returned lambda.
struct OcCtl {
  enum { P_WIDEN0 = 0, P_WIDEN, P_VLO, P_BIS, P_LSBIS, P_DONE };
  enum { ST_OK = 0, ST_NONMONO = 3 };
  double volfrac, relTol, volTol, absTol;
  int lambdaSpace;
  int check_mono;
  int phase, status;
  double lamMax, vHi, vLo, lo, hi, mid, v, lam;
  double s_req, s_final, lam_result;
  int widenings, bis, evals;

  __host__ __device__ void init(double lamMax0, double volfrac_, double relTol_, double volTol_,
                                int lambdaSpace_, double absTol_) {
    volfrac = volfrac_;
    relTol = relTol_;
    volTol = volTol_;
    lambdaSpace = lambdaSpace_;
    absTol = absTol_;
    check_mono = 1;
    status = ST_OK;
    widenings = bis = evals = 0;
    lo = hi = mid = v = lam = vHi = vLo = 0.0;
    lamMax = lamMax0;
    if (!(lamMax > 0)) {  // oc.hpp:117-121: volumeAt(1.0), lambda = 0
      phase = P_DONE;
      s_final = 1.0;
      lam_result = 0.0;
      evals = 1;
      return;
    }
    phase = P_WIDEN0;
    s_req = sqrt(lamMax);  // oc.hpp:125
  }
  __host__ __device__ bool pending() const { return phase != P_DONE; }
  // Every evaluation returns vv (+inf or -inf: the bound shortcut, all the
  // reference's decisions known). The same transitions as feeding vv until
  // done with check_mono off, but the bisection steps skip the next request
  // and test the cheap operand of oc.hpp:156-157 first (the same decision).
  __host__ __device__ void replay_known(double vv) {
    check_mono = 0;
    if ((phase == P_WIDEN0 || phase == P_WIDEN) && vv > volfrac && widenings <= 40) {
      // every remaining widening happens (oc.hpp:127-130): lamMax *= 4 each time,
      // i.e. an exact power-of-two scaling, then the vLo request
      const int k = 40 - widenings;
      evals += k + 1;
      lamMax = ldexp(lamMax, 2 * k);
      widenings = 41;
      vHi = vv;
      phase = P_VLO;
      s_req = 0.0;
    }
    while (phase == P_WIDEN0 || phase == P_WIDEN || phase == P_VLO) feed(vv);
    while (phase == P_BIS) {
      ++evals;
      v = vv;
      if (v > volfrac) {
        lo = mid;
        vLo = v;
      } else {
        hi = mid;
        vHi = v;
      }
      if (++bis >= 500) {
        finish_bis();
        break;
      }
      const bool far = fabs(v - volfrac) > 0.5 * volTol;
      if ((far && bis < 200) || (hi - lo) / (hi + lo) > relTol) {
        const double prev = mid;
        mid = 0.5 * (lo + hi);
        s_req = mid;
        if (mid == prev && far && !((hi - lo) / (hi + lo) > relTol)) {
          // fixed point (the bracket end moved to mid is mid again): each
          // remaining step only counts until bis = 200 ends the loop
          evals += 200 - bis;
          bis = 200;
          finish_bis();
        }
      } else {
        finish_bis();
      }
    }
    while (phase == P_LSBIS) feed(vv);
  }
  // whether the next request depends on the value fed for the current one
  __host__ __device__ bool branching() const { return phase != P_VLO; }

  __host__ __device__ void feed(double vv) {
    const double monoSlack = 1e-9;  // oc.hpp:132
    ++evals;
    switch (phase) {
      case P_WIDEN0:
      case P_WIDEN:
        vHi = vv;
        if (vHi > volfrac && widenings++ < 40) {  // oc.hpp:127-130
          lamMax *= 4.0;
          s_req = sqrt(lamMax);
          phase = P_WIDEN;
        } else {
          phase = P_VLO;  // oc.hpp:131 vLo = volumeAt(0.0)
          s_req = 0.0;
        }
        return;
      case P_VLO:
        vLo = vv;
        s_final = 0.0;
        if (lambdaSpace) {  // oc.hpp:134-152
          lo = 0.0;
          hi = lamMax;
          lam = lamMax;
          ls_next();
        } else {  // oc.hpp:154-155
          lo = 0.0;
          hi = sqrt(lamMax);
          mid = hi;
          v = vLo;
          bis_next();
        }
        return;
      case P_BIS:  // oc.hpp:158-169
        v = vv;
        if (check_mono && (v > vLo + monoSlack || v < vHi - monoSlack)) {
          status = ST_NONMONO;
          phase = P_DONE;
          return;
        }
        if (v > volfrac) {
          lo = mid;
          vLo = v;
        } else {
          hi = mid;
          vHi = v;
        }
        if (++bis >= 500) {
          finish_bis();
          return;
        }
        bis_next();
        return;
      case P_LSBIS:  // oc.hpp:137-148
        v = vv;
        s_final = s_req;
        if (check_mono && (v > vLo + monoSlack || v < vHi - monoSlack)) {
          status = ST_NONMONO;
          phase = P_DONE;
          return;
        }
        if (v > volfrac) {
          lo = lam;
          vLo = v;
        } else {
          hi = lam;
          vHi = v;
        }
        ++bis;
        ls_next();
        return;
      default:
        return;
    }
  }

 private:
  __host__ __device__ void bis_next() {  // oc.hpp:156-157
    if ((hi - lo) / (hi + lo) > relTol || (fabs(v - volfrac) > 0.5 * volTol && bis < 200)) {
      mid = 0.5 * (lo + hi);
      s_req = mid;
      phase = P_BIS;
    } else {
      finish_bis();
    }
  }
  __host__ __device__ void finish_bis() {  // oc.hpp:171-172
    s_final = mid;
    lam_result = mid * mid;
    ++evals;
    phase = P_DONE;
  }
  __host__ __device__ void ls_next() {  // oc.hpp:136, :150
    if (hi - lo > absTol && bis < 4000) {
      lam = 0.5 * (lo + hi);
      s_req = sqrt(lam);
      phase = P_LSBIS;
    } else {
      lam_result = lam;
      phase = P_DONE;
    }
  }
};

/// Speculative request set: every multiplier the controller can request in
/// the next few feeds, generated with the controller's own arithmetic (so
/// the values compare bit-equal with the replayed requests):
///   widening: sqrt(lamMax * 4^k) for the next 4 widenings, then 0 (vLo),
///             then the first 3 bisection levels under hi = sqrt(lamMax);
///   vLo:      0, then 4 bisection levels;
///   bisection (sqrt or lambda space): the full tree of the next 4 levels.
// Breadth-first midpoints of [lo, hi] for DEPTH levels (2^DEPTH - 1 values),
// fully unrolled so the arrays stay in registers on the device.
template <int DEPTH>
__host__ __device__ inline int oc_tree(double lo, double hi, bool lambda_space, double* out) {
  constexpr int W = 1 << DEPTH;  // interval endpoints of the deepest level
  double b[W + 1];               // endpoints in order: b[0] = lo, b[W] = hi
  b[0] = lo;
  b[W] = hi;
  int n = 0;
#pragma unroll
  for (int d = 0; d < DEPTH; ++d) {
    const int stride = W >> d, half = stride >> 1;
#pragma unroll
    for (int q = 0; q < (1 << d); ++q) {
      const double mid = 0.5 * (b[q * stride] + b[q * stride + stride]);  // oc.hpp:158
      b[q * stride + half] = mid;
      out[n++] = lambda_space ? sqrt(mid) : mid;
    }
  }
  return n;
}

/// Speculative request set: every multiplier the controller can request in
/// the next few feeds, generated with the controller's own arithmetic (so
/// the values compare bit-equal with the replayed requests):
///   widening: sqrt(lamMax * 4^k) for the next 4 widenings, then 0 (vLo),
///             then the first 3 bisection levels under hi = sqrt(lamMax);
///   vLo:      0, then 4 bisection levels;
///   bisection (sqrt or lambda space): the full tree of the next 4 levels.
/// KMAX 16: 4 levels per batch; KMAX >= 32: 5 levels (fewer grid-wide
/// rounds when evaluating is cheap).
template <int KMAX>
__host__ __device__ inline int oc_speculate(const OcCtl& c, double* out) {
  static_assert(KMAX >= 16, "request buffer too small");
  constexpr int L = KMAX >= 32 ? 5 : 4;
  int n = 0;
  switch (c.phase) {
    case OcCtl::P_WIDEN0:
    case OcCtl::P_WIDEN: {
      double lm = c.lamMax;
      out[n++] = sqrt(lm);  // the pending request
      for (int k = 0; k < 3; ++k) {
        lm *= 4.0;
        out[n++] = sqrt(lm);
      }
      out[n++] = 0.0;
      n += c.lambdaSpace ? oc_tree<L - 1>(0.0, c.lamMax, true, out + n)
                         : oc_tree<L - 1>(0.0, sqrt(c.lamMax), false, out + n);
      break;
    }
    case OcCtl::P_VLO:
      out[n++] = 0.0;
      n += c.lambdaSpace ? oc_tree<L>(0.0, c.lamMax, true, out + n)
                         : oc_tree<L>(0.0, sqrt(c.lamMax), false, out + n);
      break;
    case OcCtl::P_BIS:
      n = oc_tree<L>(c.lo, c.hi, false, out);
      break;
    case OcCtl::P_LSBIS:
      n = oc_tree<L>(c.lo, c.hi, true, out);
      break;
    default:
      break;
  }
  return n;
}

}  // namespace topo
