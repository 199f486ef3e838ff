// Error-free transformations and Dot2 accumulation (Ogita, Rump & Oishi,
// "Accurate sum and dot product", SIAM J. Sci. Comput. 26(6), 2005, Alg. 5.3)
// for the fp64 reductions of the PCG (DESIGN.md §5 K5; reading R17).
//
// A Dot2 accumulator is an unevaluated pair (s, c): the running float sum and
// the running sum of its rounding errors.  Pairs combine with TwoSum, so any
// tree order gives a result within ~n u^2 cond of the exact value and the
// final RN(s + c) is the correctly rounded dot product in practice -- which is
// what makes the GPU's tree order agree bitwise with the oracle's sequential
// order (tests/test_gpu_*.py).
//
// The library is compiled with --fmad=false: a contraction of s + a*b into an
// fma would silently break TwoSum's exactness.  Every fma below is explicit.
#pragma once
#include <cuda_runtime.h>

namespace laker {

struct dd_pair {
  double s, c;
};

__device__ __forceinline__ void two_sum(double a, double b, double &s, double &e) {
  double x = __dadd_rn(a, b);
  double z = __dsub_rn(x, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(x, z)), __dsub_rn(b, z));
  s = x;
}

__device__ __forceinline__ void fast_two_sum(double a, double b, double &s, double &e) {
  // requires |a| >= |b| (or a == 0)
  double x = __dadd_rn(a, b);
  e = __dsub_rn(b, __dsub_rn(x, a));
  s = x;
}

__device__ __forceinline__ void two_prod(double a, double b, double &p, double &e) {
  double x = __dmul_rn(a, b);
  e = __fma_rn(a, b, -x);
  p = x;
}

// acc += a * b   (one Dot2 step)
__device__ __forceinline__ void dot2_step(dd_pair &acc, double a, double b) {
  double p, pe, s, se;
  two_prod(a, b, p, pe);
  two_sum(acc.s, p, s, se);
  acc.s = s;
  acc.c = __dadd_rn(acc.c, __dadd_rn(pe, se));
}

// acc += a * b with acc.s carrying a power-of-two offset C >= 2 sum|a b| over the whole
// accumulation (so |acc.s| >= C/2 >= |a b| and Fast2Sum is error-free): 7 fp64 ops
// instead of Dot2's 10.  The caller subtracts C (exactly, Sterbenz) at the end; the
// rounding errors are still captured exactly, they are just O(u C) instead of
// O(u |partial sum|) before the compensation sum (symv.cu).
__device__ __forceinline__ void dot2_step_off(dd_pair &acc, double a, double b) {
  double p, pe, s, se;
  two_prod(a, b, p, pe);
  fast_two_sum(acc.s, p, s, se);
  acc.s = s;
  acc.c = __dadd_rn(acc.c, __dadd_rn(pe, se));
}

// the smallest power of two above v (v >= 0 finite); 0 for v == 0
__device__ __forceinline__ double pow2_above(double v) {
  const long long b = __double_as_longlong(v);
  if (b == 0) return 0.0;
  const long long e = ((b >> 52) & 0x7ff) + 1;
  return __longlong_as_double((e < 2046 ? e : 2046) << 52);
}

// acc += (o.s + o.c)  without rounding the incoming pair first
__device__ __forceinline__ void pair_add(dd_pair &acc, const dd_pair &o) {
  double s, e;
  two_sum(acc.s, o.s, s, e);
  acc.s = s;
  acc.c = __dadd_rn(acc.c, __dadd_rn(o.c, e));
}

__device__ __forceinline__ double pair_value(const dd_pair &a) { return __dadd_rn(a.s, a.c); }

__device__ __forceinline__ dd_pair warp_reduce_pair(dd_pair v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    dd_pair o;
    o.s = __shfl_xor_sync(0xffffffffu, v.s, off);
    o.c = __shfl_xor_sync(0xffffffffu, v.c, off);
    pair_add(v, o);
  }
  return v;  // use lane 0's pair: lanes may differ in the last bit of c
}

}  // namespace laker
