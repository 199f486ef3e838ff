// FAST-mode on-the-fly kernel matvec:
//   out_a = [lambda x_a +] sum_i exp(scale <eq_a, e_i>) w_i
// K is never stored: per CTA a 64-query tile of E_q stays in shared memory
// while 64-point tiles of E stream through a 2-stage cp.async ring; the
// 64 x 64 x d dot products run on the fp64 tensor cores (mma.sync m8n8k4 .f64,
// SASS DMMA), the scale + exp + weight epilogue is fused, and row sums are
// kept in fp64 registers (flash-attention-like, without softmax
// normalization -- P:517-519's matvec-only access).  Entries are within ~1 ulp
// of the EXACT ones; row sums are plain fp64 (FAST parity = envelope).
#include "laker_internal.h"

namespace laker {
namespace {

constexpr int kT = 64;

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src, bool ok) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
}

// dynamic smem: Aq [64][S], B[2][64][S] with S = dpad + 4 (dpad = d rounded up to 4)
__global__ void __launch_bounds__(128) otf_fast_kernel(const double *__restrict__ Eq, int64_t m,
                                                       const double *__restrict__ E, int64_t n, int d,
                                                       double scale, const double *__restrict__ w, double lambda,
                                                       const double *__restrict__ xdiag, double *__restrict__ out,
                                                       const int32_t *done) {
  if (done != nullptr && *(volatile const int32_t *)done) return;
  extern __shared__ __align__(16) double sm[];
  const int dp = (d + 3) & ~3;
  const int S = dp + 4 + ((dp + 4) % 16 == 4 ? 0 : (20 - (dp + 4) % 16) % 16);  // stride = 4 mod 16 doubles
  double *Aq = sm;
  double *Bt = sm + kT * S;
  __shared__ double wt[2][kT];
  __shared__ double red[2][kT];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wr = (warp >> 1) * 32, wc = (warp & 1) * 32;
  const int fr = lane >> 2, fk = lane & 3;
  const int64_t A0 = (int64_t)blockIdx.x * kT;

  for (int e = tid; e < kT * dp; e += 128) {
    const int r = e / dp, c = e % dp;
    Aq[r * S + c] = (A0 + r < m && c < d) ? Eq[(A0 + r) * d + c] : 0.0;
  }
  auto load_tile = [&](int st, int64_t J0) {
    double *b = Bt + st * kT * S;
    for (int e = tid; e < kT * dp; e += 128) {
      const int r = e / dp, c = e % dp;
      const bool ok = (J0 + r < n) && (c < d);
      cp_async8(&b[r * S + c], ok ? &E[(J0 + r) * d + c] : E, ok);
    }
    if (tid < kT) wt[st][tid] = (J0 + tid < n) ? w[J0 + tid] : 0.0;
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double rows[4] = {0.0, 0.0, 0.0, 0.0};
  const int64_t ntiles = (n + kT - 1) / kT;
  load_tile(0, 0);
  for (int64_t t = 0; t < ntiles; ++t) {
    const int st = (int)(t & 1);
    if (t + 1 < ntiles) {
      load_tile(st ^ 1, (t + 1) * kT);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double *b = Bt + st * kT * S;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kk = 0; kk < dp; kk += 4) {
      double a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Aq[(wr + 8 * i + fr) * S + kk + fk];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = b[(wc + 8 * j + fr) * S + kk + fk];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j], a[i], bb[j]);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double w0 = wt[st][wc + 8 * j + 2 * fk], w1 = wt[st][wc + 8 * j + 2 * fk + 1];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        rows[i] = fma(exp(scale * acc[i][j][0]), w0, rows[i]);
        rows[i] = fma(exp(scale * acc[i][j][1]), w1, rows[i]);
      }
    }
    __syncthreads();
  }
  // lanes fk = 0..3 share a row; then the two column halves
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double v = rows[i];
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    if (fk == 0) red[warp & 1][wr + 8 * i + fr] = v;
  }
  __syncthreads();
  if (tid < kT && A0 + tid < m) {
    double v = red[0][tid] + red[1][tid];
    if (lambda != 0.0) v = fma(lambda, xdiag[A0 + tid], v);
    out[A0 + tid] = v;
  }
}

int stride_for(int d) {
  const int dp = (d + 3) & ~3;
  return dp + 4 + ((dp + 4) % 16 == 4 ? 0 : (20 - (dp + 4) % 16) % 16);
}

}  // namespace

size_t otf_fast_smem(int d) { return (size_t)3 * kT * stride_for(d) * sizeof(double); }

void otf_fast_init() {
  cudaFuncSetAttribute(otf_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)otf_fast_smem(128));
}

void launch_kernel_matvec_fast(const double *Eq, int64_t m, const double *E, int64_t n, int32_t d, double scale,
                               const double *w, double lambda, const double *xdiag, double *out,
                               const int32_t *done, cudaStream_t s) {
  const unsigned grid = (unsigned)((m + kT - 1) / kT);
  otf_fast_kernel<<<grid, 128, otf_fast_smem(d), s>>>(Eq, m, E, n, d, scale, w, lambda, xdiag, out, done);
}

}  // namespace laker
