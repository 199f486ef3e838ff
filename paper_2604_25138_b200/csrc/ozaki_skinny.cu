// Multi-RHS products of the block PCG on the
// 5th-gen tensor cores: C = alpha A X + beta Cin with A fixed for the whole
// solve (K, or the factors Q^T, M, Q of P) and X a block of up to 64
// right-hand sides, fp64 emulated with S int8 digit slices (Ozaki scheme,
// ozaki.cu).  A is sliced once per solve; X is sliced per product.
//
// One CTA owns 128 rows of A and all N <= 64 columns; ALL digit levels live in
// TMEM at once (level h = s + t in columns [64 h, 64 h + 64), S <= 7 -> 448 of
// 512 columns), so every 128-column K-block of A's S slices is read exactly
// once (8 bytes per entry per product, the same traffic as the fp64 GEMM) and
// multiplied against the S slices of X into the S(S+1)/2 slice pairs.  A slot s
// is refilled for the next K-block as soon as its pairs retire; X's slices are
// double-buffered per K-block.  The epilogue sums the levels in fp64 and
// applies 2^(e_row + f_col), alpha, beta Cin.  Split-K over CTAs when A has few
// row blocks (partials summed in a fixed order).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "laker_internal.h"
#include "tc_int8.cuh"

namespace laker {
bool make_tmap_s8(CUtensorMap *tm, const int8_t *base, int64_t rows, int64_t K, int64_t ld, int box_rows);
namespace {

constexpr int kSM = 128, kSN = 64, kSK = 128;
constexpr int kSSmax = 7;
constexpr uint32_t kSAChunk = kSM * kSK;  // 16 KiB
constexpr uint32_t kSBChunk = kSN * kSK;  // 8 KiB
constexpr size_t kSSmem = 1024 + kSSmax * kSAChunk + 2 * kSSmax * kSBChunk + 512;
constexpr int kSThreads = 10 * 32;

struct SkArgs {
  int64_t M, N, Kp;
  int S, nkb, splits;
  const int32_t *ea, *eb;
  double *C;
  int64_t ldc;
  const double *Cin;
  int64_t ldcin;
  double alpha, beta;
  double *part;  // splits > 1: [splits][M][kSN]
};

__device__ __forceinline__ double pow2d(int k) {
  return (k >= -1022 && k <= 1023) ? __longlong_as_double((long long)(k + 1023) << 52) : scalbn(1.0, k);
}

__global__ void __launch_bounds__(kSThreads, 1)
    oz_skinny_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const SkArgs f) {
  extern __shared__ unsigned char smem_raw[];
  const uint32_t base_s = smem_u32(smem_raw);
  unsigned char *smem = smem_raw + ((1024 - (base_s & 1023)) & 1023);
  unsigned char *sA = smem;                          // [S] A slices of the current K-block
  unsigned char *sB = smem + kSSmax * kSAChunk;      // [2][S] X slices
  uint64_t *afull = reinterpret_cast<uint64_t *>(sB + 2 * kSSmax * kSBChunk);
  uint64_t *aempty = afull + kSSmax;
  uint64_t *bfull = aempty + kSSmax;  // [2]
  uint64_t *bempty = bfull + 2;       // [2]
  uint64_t *tfull = bempty + 2;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = f.S;
  const int64_t m0 = (int64_t)blockIdx.x * kSM;
  const int z = blockIdx.y;
  const int kb0 = (int)((int64_t)f.nkb * z / f.splits), kb1 = (int)((int64_t)f.nkb * (z + 1) / f.splits);
  const int nb = kb1 - kb0;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kSSmax; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bfull[b], 1);
      mbar_init(&bempty[b], 1);
    }
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_holder, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < nb; ++i) {
        const int kb = kb0 + i, bb = i & 1;
        if (i >= 2) mbar_wait(&bempty[bb], (uint32_t)(((i >> 1) - 1) & 1));
        mbar_arrive_expect_tx(&bfull[bb], (uint32_t)S * kSBChunk);
        for (int t = 0; t < S; ++t)
          tc::tma_load_2d(sB + (bb * kSSmax + t) * kSBChunk, &tmB, (int32_t)(t * f.Kp + (int64_t)kb * kSK), 0,
                          &bfull[bb]);
        for (int s = 0; s < S; ++s) {
          if (i >= 1) mbar_wait(&aempty[s], (uint32_t)((i - 1) & 1));
          mbar_arrive_expect_tx(&afull[s], kSAChunk);
          tc::tma_load_2d(sA + s * kSAChunk, &tmA, (int32_t)(s * f.Kp + (int64_t)kb * kSK), (int32_t)m0, &afull[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_i8(kSM, kSN);
      for (int i = 0; i < nb; ++i) {
        const int bb = i & 1;
        mbar_wait(&bfull[bb], (uint32_t)((i >> 1) & 1));
        for (int s = 0; s < S; ++s) {
          mbar_wait(&afull[s], (uint32_t)(i & 1));
          tc::fence_after();
          const uint32_t a0 = smem_u32(sA + s * kSAChunk);
          for (int t = 0; t + s < S; ++t) {
            const uint32_t b0 = smem_u32(sB + (bb * kSSmax + t) * kSBChunk);
            const uint32_t td = tmem + (uint32_t)((s + t) * kSN);
#pragma unroll
            for (int kk = 0; kk < kSK / 32; ++kk)
              tc::mma_i8(td, tc::sdesc_k_sw128(a0 + kk * 32), tc::sdesc_k_sw128(b0 + kk * 32), idesc,
                         (i == 0 && s == 0 && kk == 0) ? 0u : 1u);
          }
          tc::mma_commit(&aempty[s]);
        }
        tc::mma_commit(&bempty[bb]);
      }
      tc::mma_commit(tfull);
    }
  } else {
    const int q = warp & 3, hf = (warp - 2) >> 2;  // lane quadrant, column half
    const int64_t row = m0 + q * 32 + lane;
    mbar_wait(tfull, 0);
    tc::fence_after();
    double acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.0;
    if (nb > 0) {
      for (int h = S - 1; h >= 0; --h) {
        uint32_t v[32];
        tc::tmem_ld32(tmem + (uint32_t)(h * kSN + hf * 32) + ((uint32_t)(q * 32) << 16), v);
        tc::tmem_ld_wait();
        const double sc = pow2d(-12 - 7 * h);
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = fma((double)(int32_t)v[j], sc, acc[j]);
      }
    }
    if (row < f.M) {
      const double pe = pow2d(f.ea[row]);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int64_t col = hf * 32 + j;
        if (col < f.N) {
          const double val = acc[j] * pe * pow2d(f.eb[col]);
          if (f.splits > 1) {
            f.part[((int64_t)z * f.M + row) * kSN + col] = val;
          } else {
            double out = __dmul_rn(f.alpha, val);
            if (f.beta != 0.0) out = __dadd_rn(out, __dmul_rn(f.beta, f.Cin[row * f.ldcin + col]));
            f.C[row * f.ldc + col] = out;
          }
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// C = alpha sum_z part[z] + beta Cin (fixed z order)
__global__ void oz_skinny_reduce_kernel(const SkArgs f) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= f.M * f.N) return;
  const int64_t row = e / f.N, col = e % f.N;
  double v = 0.0;
  for (int z = 0; z < f.splits; ++z) v = __dadd_rn(v, f.part[((int64_t)z * f.M + row) * kSN + col]);
  double out = __dmul_rn(f.alpha, v);
  if (f.beta != 0.0) out = __dadd_rn(out, __dmul_rn(f.beta, f.Cin[row * f.ldcin + col]));
  f.C[row * f.ldc + col] = out;
}

}  // namespace

void oz_skinny_init() {
  cudaFuncSetAttribute(oz_skinny_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSSmem);
}

int oz_skinny_max_slices() { return kSSmax; }

// slices of a rows x K matrix (K-contiguous, row stride ld; or K x rows if trans)
cudaError_t oz_slices_make_general(OzSlices &o, const double *X, int64_t ld, int64_t rows, int64_t K, int trans, int S,
                                   cudaStream_t s, unsigned long long *mx_buf) {
  const int64_t Kp = (K + kSK - 1) / kSK * kSK;
  if (!(o.s && o.rows == rows && o.Kp == Kp && o.S == S)) {
    oz_slices_free(o, s);
    cudaError_t e;
    if ((e = cudaMallocAsync(&o.s, (size_t)rows * S * Kp, s)) != cudaSuccess) return e;
    if ((e = cudaMallocAsync(&o.e, (size_t)rows * sizeof(int32_t), s)) != cudaSuccess) return e;
  }
  o.rows = rows;
  o.Kp = Kp;
  o.S = S;
  launch_ozaki_split(X, ld, rows, K, trans, S, 0, o.s, o.e, Kp, s, mx_buf);
  return cudaGetLastError();
}

// C (M x N) = alpha A op(B) + beta Cin: A = pre-sliced rows (M = A.rows), B = slices of the
// N <= 64 columns of op(B) (B.rows = N); part: workspace of >= splits * M * 64 doubles
cudaError_t launch_oz_skinny(const OzSlices &A, const OzSlices &B, int64_t N, double alpha, double beta,
                             const double *Cin, int64_t ldcin, double *C, int64_t ldc, double *part, int max_splits,
                             int num_sms, cudaStream_t s) {
  if (N > kSN || A.S != B.S || A.Kp != B.Kp || A.S > kSSmax) return cudaErrorInvalidValue;
  CUtensorMap ta, tb;
  const int64_t ld = (int64_t)A.S * A.Kp;
  if (!make_tmap_s8(&ta, A.s, A.rows, ld, ld, kSM) || !make_tmap_s8(&tb, B.s, B.rows, ld, ld, kSN))
    return cudaErrorInvalidValue;
  SkArgs f{};
  f.M = A.rows;
  f.N = N;
  f.Kp = A.Kp;
  f.S = A.S;
  f.nkb = (int)(A.Kp / kSK);
  const int tiles = (int)((A.rows + kSM - 1) / kSM);
  f.splits = std::max(1, std::min({max_splits, f.nkb, (num_sms + tiles - 1) / tiles}));
  f.ea = A.e;
  f.eb = B.e;
  f.C = C;
  f.ldc = ldc;
  f.Cin = Cin;
  f.ldcin = ldcin;
  f.alpha = alpha;
  f.beta = beta;
  f.part = part;
  oz_skinny_kernel<<<dim3((unsigned)tiles, (unsigned)f.splits), kSThreads, kSSmem, s>>>(ta, tb, f);
  if (f.splits > 1)
    oz_skinny_reduce_kernel<<<(unsigned)((f.M * N + 255) / 256), 256, 0, s>>>(f);
  return cudaGetLastError();
}

}  // namespace laker
