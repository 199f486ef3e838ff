// FAST-mode on-the-fly kernel matvec with the QK^T contraction on the 5th-gen
// tensor cores (BASELINE north star:
// "a QK^T dense contraction on tensor cores, with a fused exp epilogue"):
//
//   out_a = [lambda x_a +] sum_i exp(scale <eq_a, e_i>) w_i
//
// fp64 inner products emulated on tcgen05 kind::i8 (Ozaki scheme, ozaki.cu):
// the query rows and the points are pre-split into S int8 digit slices with
// power-of-two row scales; one CTA owns 128 query rows, keeps their S slices
// resident in shared memory, and streams the points in 128-row tiles.  For
// every point tile J and digit level h = S-1 .. 0 one thread issues the
// (h+1) x 4 MMAs (M = N = 128, K = 32) of the slice pairs (c, h-c) into a TMEM
// buffer (two, alternating); 8 epilogue warps add level h as v 2^(-12-7h) to fp64
// registers and, after level 0, form exp(scale 2^(ea+eb) acc) w_j and the row
// sums -- flash-attention-like, K never stored.
#include <cuda.h>

#include <cstdlib>

#include "laker_internal.h"
#include "tc_int8.cuh"

namespace laker {
bool make_tmap_s8(CUtensorMap *tm, const int8_t *base, int64_t rows, int64_t K, int64_t ld, int box_rows);
namespace {

constexpr int kOM = 128, kON = 128, kOK = 128;
constexpr int kOSmax = 7;                      // digit slices (smem: 7 query + 7 point slices)
constexpr uint32_t kOChunk = kOM * kOK;  // 16 KiB: 128 rows x 128 int8 (one 128B-swizzled box)
constexpr size_t kOSmem = 1024 + 2 * kOSmax * kOChunk + 512;
constexpr int kOEpiWarps = 16;                  // 4 per TMEM lane quadrant, 32 columns each
constexpr int kOThreads = (2 + kOEpiWarps) * 32;

// out-of-line exp: the 64 call sites of the unrolled epilogue would otherwise inline
// 64 copies of exp and overflow the instruction cache (ncu: "no_instruction" stalls)
__device__ __noinline__ double exp_ool(double x) { return exp(x); }

// exp for the FAST entries: x = k ln2 + r (|r| <= ln2/2, two-part ln2), Taylor
// polynomial of degree 13 (truncation < 2e-17 relative), times 2^k built from
// bits; no special cases (|x| <= 700 guaranteed by the overflow-free kernel
// arguments, |scale <e_i,e_j>| is small for the embeddings of R3).  <= 2 ulp.
__device__ __forceinline__ double exp_fast(double x) {
  const double k = rint(x * 1.4426950408889634);
  double r = fma(-k, 6.93147180369123816490e-01, x);
  r = fma(-k, 1.90821492927058770002e-10, r);
  double p = 1.0 / 6227020800.0;            // 1/13!
  p = fma(p, r, 1.0 / 479001600.0);         // 1/12!
  p = fma(p, r, 1.0 / 39916800.0);
  p = fma(p, r, 1.0 / 3628800.0);
  p = fma(p, r, 1.0 / 362880.0);
  p = fma(p, r, 1.0 / 40320.0);
  p = fma(p, r, 1.0 / 5040.0);
  p = fma(p, r, 1.0 / 720.0);
  p = fma(p, r, 1.0 / 120.0);
  p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  return p * __longlong_as_double((long long)((int)k + 1023) << 52);
}

// 2^k as a double (k in the normal range), else scalbn
__device__ __forceinline__ double pow2i(int k) {
  return (k >= -1022 && k <= 1023) ? __longlong_as_double((long long)(k + 1023) << 52) : scalbn(1.0, k);
}

struct OtfArgs {
  int64_t a0, m, n;
  int S;
  const int32_t *ea, *eb;
  double scale, lambda;
  const double *w, *xdiag;
  double *out;
  const int32_t *done;
};

template <bool MATERIALIZE>
__global__ void __launch_bounds__(kOThreads, 1)
    otf_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const OtfArgs f) {
  if (f.done != nullptr && *(volatile const int32_t *)f.done) return;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t base_s = smem_u32(smem_raw);
  unsigned char *smem = smem_raw + ((1024 - (base_s & 1023)) & 1023);
  unsigned char *sA = smem;                          // S resident query slices
  unsigned char *sB = smem + kOSmax * kOChunk;       // the S slices of the current point tile
  double *red = reinterpret_cast<double *>(sA);      // [4][128], after the last MMA (aliases sA)
  uint64_t *full = reinterpret_cast<uint64_t *>(sB + kOSmax * kOChunk);  // [S] point slice landed
  uint64_t *empty = full + kOSmax;                                        // [S] point slice free
  uint64_t *tfull = empty + kOSmax;    // [2]
  uint64_t *tempty = tfull + 2;        // [2]
  uint64_t *afull = tempty + 2;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(afull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = f.S;
  const int64_t r0 = (int64_t)blockIdx.x * kOM;  // query rows of this CTA (local index)
  const int64_t nJ = (f.n + kON - 1) / kON;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kOSmax; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kOEpiWarps);
    }
    mbar_init(afull, 1);
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_holder, 256);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      // resident query slices (rows a0 + r0 .. of the sliced query matrix)
      mbar_arrive_expect_tx(afull, (uint32_t)S * kOChunk);
      for (int c = 0; c < S; ++c)
        tc::tma_load_2d(sA + c * kOChunk, &tmA, c * kOK, (int32_t)(f.a0 + r0), afull);
      // point tile J: all S slices resident; slot t is last used by level t (pair (0, t)),
      // so it is refilled for J+1 in the order t = S-1 .. 0 as the levels retire
      for (int64_t J = 0; J < nJ; ++J)
        for (int t = S - 1; t >= 0; --t) {
          if (J > 0) mbar_wait(&empty[t], (uint32_t)((J - 1) & 1));
          mbar_arrive_expect_tx(&full[t], kOChunk);
          tc::tma_load_2d(sB + t * kOChunk, &tmB, t * kOK, (int32_t)(J * kON), &full[t]);
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_i8(kOM, kON);
      mbar_wait(afull, 0);
      int64_t job = 0;
      for (int64_t J = 0; J < nJ; ++J)
        for (int h = S - 1; h >= 0; --h, ++job) {
          const int b = (int)(job & 1);
          if (job >= 2) mbar_wait(&tempty[b], (uint32_t)(((job >> 1) - 1) & 1));
          tc::fence_after();
          const uint32_t td = tmem + (uint32_t)(b * kON);
          for (int c = 0; c <= h; ++c) {
            const int t = h - c;
            mbar_wait(&full[t], (uint32_t)(J & 1));
            tc::fence_after();
            const uint32_t a0s = smem_u32(sA + c * kOChunk), b0s = smem_u32(sB + t * kOChunk);
#pragma unroll
            for (int kk = 0; kk < kOK / 32; ++kk)
              tc::mma_i8(td, tc::sdesc_k_sw128(a0s + kk * 32), tc::sdesc_k_sw128(b0s + kk * 32), idesc,
                         (c > 0 || kk > 0) ? 1u : 0u);
          }
          tc::mma_commit(&tfull[b]);
          tc::mma_commit(&empty[h]);  // slot h: no later level of tile J reads it
        }
    }
  } else {
    const int q = warp & 3, qt = (warp - 2) >> 2;  // lane quadrant, column quarter
    const int rl = q * 32 + lane;  // tile row
    const int64_t row = r0 + rl;
    const bool rok = row < f.m;
    const double pe = pow2i(rok ? f.ea[f.a0 + row] : 0);  // 2^(e_row); 2^(e_col) scale folded per column
    double acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.0;
    double rsum = 0.0;
    int64_t job = 0;
    for (int64_t J = 0; J < nJ; ++J) {
      for (int h = S - 1; h >= 0; --h, ++job) {
        const int b = (int)(job & 1);
        mbar_wait(&tfull[b], (uint32_t)((job >> 1) & 1));
        tc::fence_after();
        const double sc = pow2i(-12 - 7 * h);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t v[16];
          tc::tmem_ld16(tmem + (uint32_t)(b * kON + qt * 32 + hh * 16) + ((uint32_t)(q * 32) << 16), v);
          tc::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[hh * 16 + j] = fma((double)(int32_t)v[j], sc, acc[hh * 16 + j]);
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
      }
      // level 0 done for tile J: entries, weights, row sums (columns past n have w = 0
      // through the clamped index; their entries are finite and weightless)
      // lane l fetches column cb + l's weight and scale once; the row loop broadcasts them
      const int64_t cb = J * kON + qt * 32;
      const bool okl = cb + lane < f.n;
      const double pl = okl ? f.scale * pow2i(f.eb[cb + lane]) : 0.0;
      {
        const double wl = okl ? f.w[cb + lane] : 0.0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const double wj = __shfl_sync(0xffffffffu, wl, j);
          const double pj = __shfl_sync(0xffffffffu, pl, j);
          rsum = fma(exp_fast(acc[j] * pe * pj), wj, rsum);
          acc[j] = 0.0;
        }
      }
    }
    red[qt * kOM + rl] = rsum;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 256);
  if (threadIdx.x >= 64 && threadIdx.x < 64 + kOM) {
    const int rl = threadIdx.x - 64;
    const int64_t row = r0 + rl;
    if (row < f.m) {
      double v = (red[rl] + red[kOM + rl]) + (red[2 * kOM + rl] + red[3 * kOM + rl]);
      if (f.lambda != 0.0) v = fma(f.lambda, f.xdiag[row], v);
      f.out[row] = v;
    }
  }
}

}  // namespace

void otf_tc_init() {
  cudaFuncSetAttribute(otf_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOSmem);
}

cudaError_t oz_slices_make(OzSlices &o, const double *X, int64_t rows, int32_t d, int S, cudaStream_t s) {
  if (d > kOK || S > kOSmax || S < 1) return cudaErrorInvalidValue;
  const int64_t Kp = d <= 64 ? 64 : kOK;  // 64: the K = 64 slices of otf_tc2.cu
  if (!(o.s && o.rows == rows && o.S == S)) {
    oz_slices_free(o, s);
    cudaError_t e;
    if ((e = cudaMallocAsync(&o.s, (size_t)rows * S * Kp, s)) != cudaSuccess) return e;
    if ((e = cudaMallocAsync(&o.e, (size_t)rows * sizeof(int32_t), s)) != cudaSuccess) return e;
  }
  o.rows = rows;
  o.Kp = Kp;
  o.S = S;
  launch_ozaki_split(X, d, rows, d, 0, S, 0, o.s, o.e, Kp, s);
  return cudaGetLastError();
}

void oz_slices_free(OzSlices &o, cudaStream_t s) {
  if (o.s) cudaFreeAsync(o.s, s);
  if (o.e) cudaFreeAsync(o.e, s);
  o = OzSlices{};
}

cudaError_t launch_otf_tc(const OzSlices &A, int64_t a0, int64_t m, const OzSlices &B, int64_t n, double scale,
                          const double *w, double lambda, const double *xdiag, double *out, const int32_t *done,
                          cudaStream_t s) {
  if (m <= 0) return cudaSuccess;
  CUtensorMap ta, tb;
  const int64_t ld = (int64_t)A.S * A.Kp;
  if (!make_tmap_s8(&ta, A.s, A.rows, ld, ld, kOM) || !make_tmap_s8(&tb, B.s, B.rows, ld, ld, kON))
    return cudaErrorInvalidValue;
  OtfArgs f{};
  f.a0 = a0;
  f.m = m;
  f.n = n;
  f.S = A.S;
  f.ea = A.e;
  f.eb = B.e;
  f.scale = scale;
  f.lambda = lambda;
  f.w = w;
  f.xdiag = xdiag;
  f.out = out;
  f.done = done;
  otf_tc_kernel<false><<<(unsigned)((m + kOM - 1) / kOM), kOThreads, kOSmem, s>>>(ta, tb, f);
  return cudaGetLastError();
}

}  // namespace laker

namespace laker {

__global__ void max_rownorm2_kernel(const double *__restrict__ E, int64_t n, int d, unsigned long long *out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int k = 0; k < d; ++k) s = fma(E[i * d + k], E[i * d + k], s);
  atomicMax(out, (unsigned long long)__double_as_longlong(s));
}

// max_i ||e_i||^2 (bounds |<e_i, e_j>| by Cauchy-Schwarz): decides whether the
// branch-free exp of the tensor-core paths may be used (no overflow possible)
cudaError_t max_rownorm2(const double *E, int64_t n, int d, double *out, cudaStream_t s) {
  unsigned long long *dv = nullptr, hv = 0;
  cudaError_t e;
  if ((e = cudaMallocAsync(&dv, sizeof(unsigned long long), s)) != cudaSuccess) return e;
  cudaMemsetAsync(dv, 0, sizeof(unsigned long long), s);
  max_rownorm2_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(E, n, d, dv);
  cudaMemcpyAsync(&hv, dv, sizeof(hv), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(dv, s);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  *out = __builtin_bit_cast(double, hv);
  return cudaSuccess;
}

// FAST assembly: K rows [a0, a0 + m) (local row index) x all n columns, from the slices
// of E (ctx->ozE), entries exp(scale <e_i, e_j>) on the tcgen05 QK^T path

cudaError_t launch_kernel_matvec_ctx(laker_ctx ctx, int mode, const double *Eq, int64_t m, bool Eq_is_E,
                                     int64_t eq_row0, const double *w, double lambda, const double *xdiag,
                                     double *out, const int32_t *done, cudaStream_t s) {
  static int use_tc = -1;
  if (use_tc < 0) {
    const char *v = std::getenv("LAKER_OTF_TC");
    use_tc = (v && v[0] == '0') ? 0 : 1;
  }
  if (mode == LAKER_MODE_FAST && ctx->d <= kOK && use_tc && ctx->ozE_valid && ctx->ozE.Kp == 64) {
    // second-generation kernel (otf_tc2.cu), d <= 64
    if (Eq_is_E)
      return launch_otf_tc2_rect(ctx->ozE, eq_row0, m, ctx->ozE, ctx->n, ctx->scale, w, ctx->cf, lambda, xdiag, out,
                                 done, s);
    OzSlices q;
    cudaError_t e = oz_slices_make(q, Eq, m, ctx->d, ctx->ozE.S, s);
    if (e == cudaSuccess)
      e = launch_otf_tc2_rect(q, 0, m, ctx->ozE, ctx->n, ctx->scale, w, ctx->cf, lambda, xdiag, out, done, s);
    oz_slices_free(q, s);
    return e;
  }
  if (mode == LAKER_MODE_FAST && ctx->d <= kOK && use_tc && ctx->ozE_valid) {
    if (Eq_is_E)
      return launch_otf_tc(ctx->ozE, eq_row0, m, ctx->ozE, ctx->n, ctx->scale, w, lambda, xdiag, out, done, s);
    OzSlices q;
    cudaError_t e = oz_slices_make(q, Eq, m, ctx->d, ctx->ozE.S, s);
    if (e == cudaSuccess) e = launch_otf_tc(q, 0, m, ctx->ozE, ctx->n, ctx->scale, w, lambda, xdiag, out, done, s);
    oz_slices_free(q, s);
    return e;
  }
  if (mode != LAKER_MODE_FAST && !Eq_is_E) {  // EXACT predict: the query rows' maxima
    double *emq = nullptr;
    cudaError_t e = cudaMallocAsync(&emq, (size_t)std::max<int64_t>(m, 1) * sizeof(double), s);
    if (e != cudaSuccess) return e;
    launch_rowabsmax(Eq, m, ctx->d, emq, s);
    launch_kernel_matvec(mode, Eq, m, ctx->E, ctx->n, ctx->d, ctx->scale, w, lambda, xdiag, out, ctx->flags, done, s,
                         emq, ctx->emax);
    cudaFreeAsync(emq, s);
    return cudaGetLastError();
  }
  launch_kernel_matvec(mode, Eq, m, ctx->E, ctx->n, ctx->d, ctx->scale, w, lambda, xdiag, out, ctx->flags, done, s,
                       ctx->emax + (Eq_is_E ? eq_row0 : 0), ctx->emax);
  return cudaGetLastError();
}

}  // namespace laker
