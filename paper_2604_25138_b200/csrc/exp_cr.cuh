// Correctly rounded binary64 exp for the kernel entries K_ij = exp(arg_ij)
// (Eq. sc-exp-kernel; reading R18 of DESIGN.md).
//
// Ziv-style two-phase evaluation:
//  * range reduction x = k ln2/64 + r, |r| <= ln2/128, with a 3-part Cody-Waite
//    constant (k*L1, k*L2 exact; x - k*L1 exact by Sterbenz) -> r = rh + rl;
//  * fast phase: e^r = 1 + rh + (rl + rh^2 P(rh)), degree-7 Taylor in double,
//    times 2^(j/64) held as a double-double; relative error < 2^-62;
//  * rounding test: h = RN(result) is accepted iff |l| + err < ulp(h)/2
//    (ulp(h)/4 when h is a power of two, where the binade below is finer);
//  * accurate phase (~0.2% of arguments): double-double Taylor to degree 14,
//    error < 2^-100, same test with err = 2^-96.  If that test also fails
//    (probability ~2^-44) the result is still returned and counted in
//    `inconclusive` so the caller can report it.
// exp(0) = 1 exactly; exp is otherwise never exact nor a midpoint (Lindemann).
// Arguments beyond |x| > 708 (never reached by the configs' embeddings) take
// CUDA's exp and are counted as inconclusive; x > ln(DBL_MAX) also sets
// `overflow`.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dot2.cuh"
#include "exp_cr_table.h"

namespace laker {

struct dd_num {
  double h, l;
};

__device__ __forceinline__ dd_num dd_mul(dd_num a, dd_num b) {
  double p, e;
  two_prod(a.h, b.h, p, e);
  e = __fma_rn(a.h, b.l, e);
  e = __fma_rn(a.l, b.h, e);
  dd_num r;
  fast_two_sum(p, e, r.h, r.l);
  return r;
}

__device__ __forceinline__ dd_num dd_add(dd_num a, dd_num b) {
  double s, e;
  two_sum(a.h, b.h, s, e);
  e = __dadd_rn(e, __dadd_rn(a.l, b.l));
  dd_num r;
  fast_two_sum(s, e, r.h, r.l);
  return r;
}

// ulp-based acceptance test: true iff RN(h + l + delta) == h for all |delta| <= err
__device__ __forceinline__ bool exp_round_ok(double h, double l, double err) {
  long long bits = __double_as_longlong(h);
  int ex = (int)((bits >> 52) & 0x7ff);
  double ulp = __longlong_as_double((long long)(ex - 52) << 52);  // 2^(e-52), h normal
  bool pow2 = (bits & 0x000fffffffffffffLL) == 0;
  double half = pow2 ? 0.25 * ulp : 0.5 * ulp;
  return __dadd_rn(fabs(l), err) < half;
}

__device__ __forceinline__ double exp_cr(double x, unsigned int &inconclusive, unsigned int &overflow) {
  if (x == 0.0) return 1.0;
  if (!(fabs(x) <= 708.0)) {
    if (x > 709.782712893383973096) overflow++;
    inconclusive++;
    return exp(x);
  }
  const double kf = rint(__dmul_rn(x, LAKER_EXP_INV_L));
  const double r1 = __fma_rn(-kf, LAKER_EXP_L1, x);  // exact
  const double t2 = __dmul_rn(kf, LAKER_EXP_L2);     // exact (17 + 32 bits)
  double rh, rl;
  two_sum(r1, -t2, rh, rl);
  rl = __fma_rn(-kf, LAKER_EXP_L3, rl);
  fast_two_sum(rh, rl, rh, rl);
  const int k = (int)kf;
  const int j = k & 63;
  const int m = k >> 6;  // floor division for negative k
  const dd_num T = {laker_exp_T[j][0], laker_exp_T[j][1]};

  // ---- fast phase
  double p = __fma_rn(rh, 1.0 / 5040.0, 1.0 / 720.0);
  p = __fma_rn(rh, p, 1.0 / 120.0);
  p = __fma_rn(rh, p, 1.0 / 24.0);
  p = __fma_rn(rh, p, 1.0 / 6.0);
  p = __fma_rn(rh, p, 0.5);
  p = __dmul_rn(__dmul_rn(rh, rh), p);              // rh^2/2 + ... + rh^7/5040
  double lo = __dadd_rn(__fma_rn(rh, rl, rl), p);     // rl (1 + rh) + p
  double sh, sl;
  two_sum(1.0, rh, sh, sl);
  sl = __dadd_rn(sl, lo);
  double ph, pe;
  two_prod(T.h, sh, ph, pe);
  pe = __fma_rn(T.h, sl, pe);
  pe = __fma_rn(T.l, sh, pe);
  double h, l;
  fast_two_sum(ph, pe, h, l);
  if (!exp_round_ok(h, l, __dmul_rn(fabs(h), 0x1p-62))) {
    // ---- accurate phase: e^r = sum_{i<=14} r^i / i! in double-double
    dd_num r = {rh, rl};
    dd_num s = {laker_exp_F[14][0], laker_exp_F[14][1]};
#pragma unroll 1
    for (int i = 13; i >= 0; --i) {
      s = dd_mul(s, r);
      s = dd_add(s, dd_num{laker_exp_F[i][0], laker_exp_F[i][1]});
    }
    dd_num v = dd_mul(T, s);
    h = v.h;
    l = v.l;
    if (!exp_round_ok(h, l, __dmul_rn(fabs(h), 0x1p-96))) inconclusive++;
  }
  // scale by 2^m: exact, result normal for |x| <= 708
  return __dmul_rn(h, __longlong_as_double((long long)(m + 1023) << 52));
}

}  // namespace laker
