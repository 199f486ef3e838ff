// On-the-fly kernel matvec  out_a = RN([lambda x_a +] sum_i exp(scale <eq_a, e_i>) w_i)
// -- the radio-map reconstruction r_hat(x) = sum_i G(x, x_i) alpha_i
// (Eq. sc-radio-map-reconstruction; Alg. 1 l.24; row a12)
// and, with Eq = E and the lambda term, the matrix-free operator apply
// (lambda I + K) p of P:517-519 (row a11).
//
// EXACT: every entry exactly as in assembly (the compensated dot over k with the
// emax offsets of assemble.cu, then the correctly rounded exp), accumulated as Dot2 pairs; the pairs of the 16
// threads sharing a query row are combined in a fixed butterfly order.  The
// result equals the oracle's Dot2 row sum in practice (R16: same-alpha map
// parity), and the on-the-fly apply equals the materialized one (T19).
// 64 queries x 64 training points per step, 4 x 4 entries per thread.
#include "exp_cr.cuh"
#include "laker_internal.h"

namespace laker {
namespace {

constexpr int kT = 64;
constexpr int kKC = 32;

__global__ void __launch_bounds__(256) kernel_matvec_exact_kernel(
    const double *__restrict__ Eq, int64_t m, const double *__restrict__ E, int64_t n, int d,
    double scale, const double *__restrict__ w, double lambda, const double *__restrict__ xdiag,
    double *__restrict__ out, unsigned long long *flags, const int32_t *done,
    const double *__restrict__ emq, const double *__restrict__ emE) {
  if (done != nullptr && *(volatile const int32_t *)done) return;
  __shared__ double Ea[kT][kKC + 1];
  __shared__ double Eb[kT][kKC + 1];
  __shared__ double ws[kT];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t A0 = (int64_t)blockIdx.x * kT;

  dd_pair row[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) row[i] = dd_pair{0.0, 0.0};
  if (tx == 0 && lambda != 0.0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t a = A0 + ty + 16 * i;
      if (a < m) dot2_step(row[i], lambda, xdiag[a]);
    }
  }
  unsigned int inc = 0, ovf = 0;
  const bool single_chunk = d <= kKC;
  if (single_chunk) {  // query tile loaded once
    for (int idx = tid; idx < kT * kKC; idx += 256) {
      const int r = idx / kKC, c = idx % kKC;
      Ea[r][c] = (A0 + r < m && c < d) ? Eq[(A0 + r) * d + c] : 0.0;
    }
  }
  double eq[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) eq[i] = A0 + ty + 16 * i < m ? emq[A0 + ty + 16 * i] * (2.0 * d) : 0.0;
  for (int64_t J0 = 0; J0 < n; J0 += kT) {
    // the compensated dots carry offsets C >= 2 d max|eq_a| max|e_j| (dot2_step_off, assemble.cu)
    double ee[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) ee[j] = J0 + tx + 16 * j < n ? emE[J0 + tx + 16 * j] : 0.0;
    dd_pair acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = dd_pair{pow2_above(eq[i] * ee[j]), 0.0};
    for (int k0 = 0; k0 < d; k0 += kKC) {
      const int kc = min(kKC, d - k0);
      __syncthreads();
      for (int idx = tid; idx < kT * kKC; idx += 256) {
        const int r = idx / kKC, c = idx % kKC;
        if (!single_chunk) Ea[r][c] = (A0 + r < m && c < kc) ? Eq[(A0 + r) * d + k0 + c] : 0.0;
        Eb[r][c] = (J0 + r < n && c < kc) ? E[(J0 + r) * d + k0 + c] : 0.0;
      }
      if (k0 == 0 && tid < kT) ws[tid] = (J0 + tid < n) ? w[J0 + tid] : 0.0;
      __syncthreads();
      for (int kk = 0; kk < kc; ++kk) {
        double av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = Ea[ty + 16 * i][kk];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Eb[tx + 16 * j][kk];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dot2_step_off(acc[i][j], av[i], bv[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (J0 + tx + 16 * j >= n) continue;
      const double wj = ws[tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        dd_pair a = acc[i][j];
        a.s = __dsub_rn(a.s, pow2_above(eq[i] * ee[j]));  // exact (Sterbenz)
        const double kv = exp_cr(__dmul_rn(scale, pair_value(a)), inc, ovf);
        dot2_step(row[i], kv, wj);
      }
    }
  }
  if (inc) atomicAdd(&flags[0], (unsigned long long)inc);
  if (ovf) atomicAdd(&flags[1], (unsigned long long)ovf);
  // combine the 16 column-threads of each query row (lanes tx = 0..15 of a half warp)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    dd_pair v = row[i];
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) {
      dd_pair o;
      o.s = __shfl_xor_sync(0xffffffffu, v.s, off);
      o.c = __shfl_xor_sync(0xffffffffu, v.c, off);
      pair_add(v, o);
    }
    const int64_t a = A0 + ty + 16 * i;
    if (tx == 0 && a < m) out[a] = pair_value(v);
  }
}

}  // namespace

void launch_kernel_matvec_exact(const double *Eq, int64_t m, const double *E, int64_t n, int32_t d,
                                double scale, const double *w, double lambda, const double *xdiag,
                                double *out, unsigned long long *flags, const int32_t *done,
                                cudaStream_t s, const double *emq, const double *emE) {
  const unsigned grid = (unsigned)((m + kT - 1) / kT);
  kernel_matvec_exact_kernel<<<grid, 256, 0, s>>>(Eq, m, E, n, d, scale, w, lambda, xdiag, out, flags,
                                                  done, emq, emE);
}

}  // namespace laker
