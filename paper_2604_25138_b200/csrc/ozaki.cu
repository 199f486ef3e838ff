// fp64 GEMM emulated on the int8 tensor cores (Ozaki scheme, split into
// integer slices; Ozaki, Ogita, Oishi & Rump, "Error-free transformations of
// matrix multiplication by using fast routines of matrix multiplication and
// its applications", Numer. Algorithms 59, 2012; int8 tensor-core variant of
// Ootomo et al. / Uchino et al.).  Puts the fp64 contractions of the method on
// tcgen05: tcgen05 has no fp64 kind on sm_100a.
//
// For C = A op(B) (A: M x K, op(B): K x N):
//  1. every row i of A (and every column j of op(B)) gets a power-of-two scale
//     2^e_i with max_k |A_ik| < 2^e_i;
//  2. x = A_ik 2^(6 - e_i) in (-64, 64) is split exactly into S signed digits
//     d_0 = rint(x), x_1 = 128 (x - d_0), d_1 = rint(x_1), ... (|d_s| <= 64), so
//     A_ik = 2^(e_i - 6) sum_s d_s 2^(-7 s) + O(2^(e_i - 7 S));
//  3. the products of digit slices with s + t = h are summed EXACTLY in one
//     int32 tensor-core GEMM over the concatenated K dimension (slices of A
//     stored in order, slices of B in reverse order, so the pairs (s, h - s)
//     are a contiguous K range of both);  |sum| <= (h+1) K 4096 < 2^31;
//  4. level h contributes 2^(e_i + f_j - 12 - 7 h) G_h, summed in fp64 from the
//     smallest level up; levels h >= S are dropped.
// S = 8 keeps 56 bits of every input (error ~ 2^-53 |A| |B|, the fp64 GEMM's
// own order); FAST-mode assembly uses S = 7 (entries <= 1e-13, tested).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "laker_internal.h"
#include "tc_int8.cuh"

namespace laker {
bool make_tmap_s8(CUtensorMap *tm, const int8_t *base, int64_t rows, int64_t K, int64_t ld, int box_rows);
bool make_tmap_s8_k64(CUtensorMap *tm, const int8_t *base, int64_t rows, int64_t K, int64_t ld, int box_rows);
namespace {

// ------------------------------------------------------------------ fused levels
// One CTA = one 128 x 128 output tile and ALL digit levels h = S-1 .. 0: the MMA
// thread accumulates level h (K_h = (h+1) Kp int8 columns) into TMEM buffer h % 2
// while the 8 epilogue warps add the previous level, v 2^(-12-7h), into fp64
// registers (64 per thread); the last level applies 2^(e_i + f_j) and the GEMM
// epilogue (alpha, beta Cin, diag, triangle mask).  No M x N workspace.
constexpr int kFM = 128, kFN = 128, kFK = 128;
constexpr int kFStages = 6;
constexpr uint32_t kFABytes = kFM * kFK, kFBBytes = kFN * kFK;
constexpr size_t kFSmem = 1024 + kFStages * (kFABytes + kFBBytes) + 512;
constexpr int kFThreads = 10 * 32;  // producer, MMA, 8 epilogue warps

struct FusedArgs {
  int64_t M, N, Kp;
  int S;
  const int32_t *ea, *eb;
  double *C;
  int64_t ldc;
  const double *Cin;
  int64_t ldcin;
  double alpha, beta, diag;
  int64_t diag_offset;
  int tri;
  int64_t tri_off;
};

__global__ void __launch_bounds__(kFThreads, 1)
    ozaki_fused_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const FusedArgs f) {
  // grouped rasterization: consecutive CTAs cover kGroupM tile-rows x ~148/kGroupM
  // tile-columns, so the concurrently streamed A and B slice chunks are shared in L2
  constexpr int kGroupM = 12;
  const int64_t tm = (f.M + kFM - 1) / kFM, tn = (f.N + kFN - 1) / kFN;
  const int64_t pid = blockIdx.x;
  const int64_t gsize = (int64_t)kGroupM * tn;
  const int64_t g0 = (pid / gsize) * kGroupM;
  const int64_t gm = (tm - g0) < kGroupM ? (tm - g0) : kGroupM;
  const int64_t m0 = (g0 + (pid % gsize) % gm) * kFM, n0 = ((pid % gsize) / gm) * kFN;
  if (f.tri == 1 && m0 + kFM - 1 + f.tri_off < n0) return;
  if (f.tri == 2 && m0 + f.tri_off >= n0 + kFN - 1) return;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t base_s = smem_u32(smem_raw);
  unsigned char *smem = smem_raw + ((1024 - (base_s & 1023)) & 1023);
  unsigned char *sA = smem;
  unsigned char *sB = smem + kFStages * kFABytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(sB + kFStages * kFBBytes);
  uint64_t *empty = full + kFStages;
  uint64_t *tfull = empty + kFStages;   // [2]
  uint64_t *tempty = tfull + 2;         // [2]
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = f.S;
  const int kpc = (int)(f.Kp / kFK);  // 128-byte chunks per slice

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kFStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_holder, 256);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      bool first = true;
      for (int h = S - 1; h >= 0; --h) {
        const int nk = (h + 1) * kpc;
        const int bcol0 = (S - 1 - h) * kpc;  // reversed B slices h .. 0
        for (int kb = 0; kb < nk; ++kb) {
          if (!first) mbar_wait(&empty[st], ph ^ 1u);
          mbar_arrive_expect_tx(&full[st], kFABytes + kFBBytes);
          tc::tma_load_2d(sA + st * kFABytes, &tmA, kb * kFK, (int32_t)m0, &full[st]);
          tc::tma_load_2d(sB + st * kFBBytes, &tmB, (bcol0 + kb) * kFK, (int32_t)n0, &full[st]);
          if (++st == kFStages) {
            st = 0;
            ph ^= 1u;
            first = false;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_i8(kFM, kFN);
      int st = 0;
      uint32_t ph = 0;
      int lev = 0;
      for (int h = S - 1; h >= 0; --h, ++lev) {
        const int b = lev & 1;
        if (lev >= 2) mbar_wait(&tempty[b], (uint32_t)(((lev >> 1) - 1) & 1));
        tc::fence_after();
        const uint32_t td = tmem + (uint32_t)(b * kFN);
        const int nk = (h + 1) * kpc;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[st], ph);
          tc::fence_after();
          const uint32_t a0 = smem_u32(sA + st * kFABytes), b0 = smem_u32(sB + st * kFBBytes);
#pragma unroll
          for (int kk = 0; kk < kFK / 32; ++kk)
            tc::mma_i8(td, tc::sdesc_k_sw128(a0 + kk * 32), tc::sdesc_k_sw128(b0 + kk * 32), idesc,
                       (kb > 0 || kk > 0) ? 1u : 0u);
          tc::mma_commit(&empty[st]);
          if (++st == kFStages) {
            st = 0;
            ph ^= 1u;
          }
        }
        tc::mma_commit(&tfull[b]);
      }
    }
  } else {
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int64_t row = m0 + q * 32 + lane;
    double acc[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) acc[j] = 0.0;
    int lev = 0;
    for (int h = S - 1; h >= 0; --h, ++lev) {
      const int b = lev & 1;
      mbar_wait(&tfull[b], (uint32_t)((lev >> 1) & 1));
      tc::fence_after();
      const double sc = scalbn(1.0, -12 - 7 * h);
#pragma unroll
      for (int c = 0; c < 64; c += 32) {
        uint32_t v[32];
        tc::tmem_ld32(tmem + (uint32_t)(b * kFN + half * 64 + c) + ((uint32_t)(q * 32) << 16), v);
        tc::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[c + j] = __dadd_rn(acc[c + j], __dmul_rn((double)(int32_t)v[j], sc));
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
    if (row < f.M) {
      const int ea = f.ea[row];
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const int64_t col = n0 + half * 64 + j;
        bool keep = col < f.N;
        if (f.tri != 0) {
          const int64_t gr = row + f.tri_off;
          keep = keep && (f.tri == 1 ? gr >= col : gr < col);
        }
        if (keep) {
          const double tot = scalbn(acc[j], ea + f.eb[col]);
          double out = __dmul_rn(f.alpha, tot);
          if (f.beta != 0.0) out = __dadd_rn(out, __dmul_rn(f.beta, f.Cin[row * f.ldcin + col]));
          if (f.diag != 0.0 && row - col == f.diag_offset) out = __dadd_rn(out, f.diag);
          f.C[row * f.ldc + col] = out;
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 256);
}

// ------------------------------------------------------------------ level groups
// One CTA = one 128 x 128 output tile; the S digit levels in groups of <= 4 (4 TMEM
// buffers x 128 columns = 512): for each 32-wide K chunk the S (or fewer) A slices and B
// slices are loaded ONCE and every slice pair (c, t) whose level c + t falls in the group
// is issued, level by level so consecutive MMAs accumulate into the same buffer.  The
// fused kernel above streams the pairs level by level over the whole K -- A_c and B_t are
// re-read for every level they meet, 4.5x the slice traffic at S = 8.  The slices are
// stored chunk-interleaved: row r holds, for each 32-wide K chunk kb, the S slices' 32
// bytes side by side (out[r][kb S 32 + s 32 + kk]), so one K chunk of 4 slices is ONE
// 128-byte TMA box row (SWIZZLE_128B, the fused kernel's tile shape); a 3-stage ring of
// chunk sets (64 KiB each).  (A first version with separate [s][Kp] slices, four 32-byte
// box rows per chunk and a 2-deep ring: 47.5 vs 40.8 ms on the directions product.)
// Levels are accumulated in the same order (S-1 .. 0) with the same fp64 operations and
// exact int32 level sums, so C is bitwise the fused kernel's.
constexpr int kLM = 128, kLN = 128, kLK = 32;
constexpr int kLSmax = 8;
constexpr int kLThreads = 10 * 32;  // producer, MMA, 8 epilogue warps
constexpr int kL2Stages = 3;
constexpr uint32_t kL2Box = 128 * 128;                 // 16 KiB: 128 rows x 4 slices x 32 B
constexpr uint32_t kL2Stage = 4 * kL2Box;              // A boxes 0, 1 + B boxes 0, 1
constexpr size_t kL2Smem = 1024 + kL2Stages * kL2Stage + 256;

__global__ void __launch_bounds__(kLThreads, 1)
    ozaki_lv2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const FusedArgs f) {
  constexpr int kGroupM = 12;
  const int64_t tm = (f.M + kLM - 1) / kLM, tn = (f.N + kLN - 1) / kLN;
  const int64_t pid = blockIdx.x;
  const int64_t gsize = (int64_t)kGroupM * tn;
  const int64_t g0 = (pid / gsize) * kGroupM;
  const int64_t gm = (tm - g0) < kGroupM ? (tm - g0) : kGroupM;
  const int64_t m0 = (g0 + (pid % gsize) % gm) * kLM, n0 = ((pid % gsize) / gm) * kLN;
  if (f.tri == 1 && m0 + kLM - 1 + f.tri_off < n0) return;
  if (f.tri == 2 && m0 + f.tri_off >= n0 + kLN - 1) return;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t base_s = smem_u32(smem_raw);
  unsigned char *smem = smem_raw + ((1024 - (base_s & 1023)) & 1023);  // [stage][A0 A1 B0 B1]
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kL2Stages * kL2Stage);  // [kL2Stages]
  uint64_t *empty = full + kL2Stages;                                          // [kL2Stages]
  uint64_t *tfull = empty + kL2Stages;                                         // [4]
  uint64_t *tempty = tfull + 4;                                                // [4]
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(tempty + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = f.S;
  const int nkb = (int)(f.Kp / kLK);
  const int ngrp = (S + 3) / 4;

  if (warp == 0 && lane == 0) {
    for (int b = 0; b < kL2Stages; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], 1);
    }
    for (int j = 0; j < 4; ++j) {
      mbar_init(&tfull[j], 1);
      mbar_init(&tempty[j], 8);
    }
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_holder, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      int use = 0;
      for (int g = 0; g < ngrp; ++g) {
        const int nbox = (S - 4 * g + 3) / 4;  // slices 0 .. S-1-4g of both operands
        for (int kb = 0; kb < nkb; ++kb, ++use) {
          if (use >= kL2Stages) mbar_wait(&empty[st], ph ^ 1u);
          mbar_arrive_expect_tx(&full[st], (uint32_t)(2 * nbox) * kL2Box);
          unsigned char *sb = smem + st * kL2Stage;
          for (int j = 0; j < nbox; ++j) {
            const int32_t x = (int32_t)((int64_t)kb * S * kLK + 128 * j);
            tc::tma_load_2d(sb + j * kL2Box, &tmA, x, (int32_t)m0, &full[st]);
            tc::tma_load_2d(sb + (2 + j) * kL2Box, &tmB, x, (int32_t)n0, &full[st]);
          }
          if (++st == kL2Stages) {
            st = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_i8(kLM, kLN);
      int st = 0;
      uint32_t ph = 0;
      for (int g = 0; g < ngrp; ++g) {
        const int hi = S - 1 - 4 * g, lo = hi - 3 > 0 ? hi - 3 : 0;
        if (g > 0)
          for (int j = 0; j <= hi - lo; ++j) mbar_wait(&tempty[j], (uint32_t)((g - 1) & 1));
        tc::fence_after();
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[st], ph);
          tc::fence_after();
          const uint32_t sa = smem_u32(smem + st * kL2Stage), sbb = sa + 2 * kL2Box;
          for (int h = hi; h >= lo; --h) {  // level-major: consecutive MMAs share the accumulator
            const uint32_t td = tmem + (uint32_t)((hi - h) * kLN);
            for (int c = 0; c <= h; ++c) {
              const int t = h - c;
              const uint64_t ad = tc::sdesc_k_sw128(sa + (uint32_t)((c >> 2) * kL2Box + (c & 3) * 32));
              const uint64_t bd = tc::sdesc_k_sw128(sbb + (uint32_t)((t >> 2) * kL2Box + (t & 3) * 32));
              tc::mma_i8(td, ad, bd, idesc, (kb > 0 || c > 0) ? 1u : 0u);
            }
          }
          tc::mma_commit(&empty[st]);
          if (++st == kL2Stages) {
            st = 0;
            ph ^= 1u;
          }
        }
        for (int j = 0; j <= hi - lo; ++j) tc::mma_commit(&tfull[j]);
      }
    }
  } else {
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int64_t row = m0 + q * 32 + lane;
    double acc[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) acc[j] = 0.0;
    for (int g = 0; g < ngrp; ++g) {
      const int hi = S - 1 - 4 * g, lo = hi - 3 > 0 ? hi - 3 : 0;
      for (int h = hi; h >= lo; --h) {
        const int jb = hi - h;
        mbar_wait(&tfull[jb], (uint32_t)(g & 1));
        tc::fence_after();
        const double sc = scalbn(1.0, -12 - 7 * h);
#pragma unroll
        for (int c = 0; c < 64; c += 32) {
          uint32_t v[32];
          tc::tmem_ld32(tmem + (uint32_t)(jb * kLN + half * 64 + c) + ((uint32_t)(q * 32) << 16), v);
          tc::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[c + j] = __dadd_rn(acc[c + j], __dmul_rn((double)(int32_t)v[j], sc));
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[jb]);
      }
    }
    if (row < f.M) {
      const int ea = f.ea[row];
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const int64_t col = n0 + half * 64 + j;
        bool keep = col < f.N;
        if (f.tri != 0) {
          const int64_t gr = row + f.tri_off;
          keep = keep && (f.tri == 1 ? gr >= col : gr < col);
        }
        if (keep) {
          const double tot = scalbn(acc[j], ea + f.eb[col]);
          double out = __dmul_rn(f.alpha, tot);
          if (f.beta != 0.0) out = __dadd_rn(out, __dmul_rn(f.beta, f.Cin[row * f.ldcin + col]));
          if (f.diag != 0.0 && row - col == f.diag_offset) out = __dadd_rn(out, f.diag);
          f.C[row * f.ldc + col] = out;
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// max-exponent of each row of X (element (r, k) = trans ? X[k ld + r] : X[r ld + k]);
// e[r] = e with max |x| < 2^e (frexp), 0 for an all-zero row
__global__ void __launch_bounds__(256) ozaki_rowexp_kernel(const double *__restrict__ X, int64_t ld, int64_t rows,
                                                           int64_t K, int trans, int32_t *__restrict__ e) {
  if (!trans) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * 8 + warp;
    if (r >= rows) return;
    double m = 0.0;
    for (int64_t k = lane; k < K; k += 32) m = fmax(m, fabs(X[r * ld + k]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
      int ex = 0;
      if (m > 0.0) frexp(m, &ex);
      e[r] = ex;
    }
  } else {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    double m = 0.0;
    for (int64_t k = 0; k < K; ++k) m = fmax(m, fabs(X[k * ld + r]));
    int ex = 0;
    if (m > 0.0) frexp(m, &ex);
    e[r] = ex;
  }
}

// column maxima of a K x rows matrix (the transposed layout): 32 columns x 8 k-lanes per
// CTA over a 1024-row chunk, |max| as IEEE bits (monotone for non-negative doubles) into
// mx[r] by atomicMax; ozaki_bits2exp_kernel turns them into frexp exponents
__global__ void __launch_bounds__(256) ozaki_colmax_kernel(const double *__restrict__ X, int64_t ld, int64_t rows,
                                                           int64_t K, unsigned long long *__restrict__ mx) {
  __shared__ double red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t r = (int64_t)blockIdx.x * 32 + tx;
  const int64_t k0 = (int64_t)blockIdx.y * 1024;
  double m = 0.0;
  if (r < rows)
    for (int64_t k = k0 + ty; k < k0 + 1024 && k < K; k += 8) m = fmax(m, fabs(X[k * ld + r]));
  red[ty][tx] = m;
  __syncthreads();
  if (ty == 0 && r < rows) {
    for (int i = 1; i < 8; ++i) m = fmax(m, red[i][tx]);
    atomicMax(&mx[r], (unsigned long long)__double_as_longlong(m));
  }
}

__global__ void ozaki_bits2exp_kernel(const unsigned long long *__restrict__ mx, int64_t rows, int32_t *__restrict__ e) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const double m = __longlong_as_double((long long)mx[r]);
  int ex = 0;
  if (m > 0.0) frexp(m, &ex);
  e[r] = ex;
}

// digits: out[r][slot(s) Kp + k] for s < S, slot(s) = rev ? S-1-s : s; 32 x 32 tiles
// staged through shared memory so both the fp64 reads and the int8 writes coalesce
__global__ void __launch_bounds__(256) ozaki_split_kernel(const double *__restrict__ X, int64_t ld, int64_t rows,
                                                          int64_t K, int trans, const int32_t *__restrict__ e,
                                                          int S, int rev, int8_t *__restrict__ out, int64_t Kp,
                                                          int il) {
  __shared__ double t[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int64_t r0 = (int64_t)blockIdx.y * 32, k0 = (int64_t)blockIdx.x * 32;
  for (int i = ty; i < 32; i += 8) {
    if (!trans) {
      const int64_t r = r0 + i, k = k0 + tx;
      t[i][tx] = (r < rows && k < K) ? X[r * ld + k] : 0.0;
    } else {
      const int64_t k = k0 + i, r = r0 + tx;
      t[tx][i] = (r < rows && k < K) ? X[k * ld + r] : 0.0;
    }
  }
  __syncthreads();
  const int64_t ldo = (int64_t)S * Kp;
  for (int i = ty; i < 32; i += 8) {
    const int64_t r = r0 + i, k = k0 + tx;
    if (r >= rows || k >= Kp) continue;
    double x = scalbn(t[i][tx], 6 - e[r]);  // |x| < 64, exact
    // il: chunk-interleaved (ozaki_lv2_kernel), out[r][(k / 32) S 32 + s 32 + k % 32]
    int8_t *o = out + r * ldo + (il ? (k >> 5) * S * 32 + (k & 31) : k);
    const int64_t sstride = il ? 32 : Kp;
    for (int s = 0; s < S; ++s) {
      const double d = rint(x);
      o[(int64_t)(rev ? S - 1 - s : s) * sstride] = (int8_t)(int)d;
      x = (x - d) * 128.0;  // exact: |x - d| <= 1/2 and x has <= 53 significant bits
    }
  }
}

// the same digits for the row-major (non-transposed) case without the shared-memory
// transpose: 16 rows x 128 k per CTA, each thread 8 consecutive k of one row, written as
// one 8-byte word per slice (the 32 x 32 kernel above stores single bytes)
__global__ void __launch_bounds__(256) ozaki_split_rows_kernel(const double *__restrict__ X, int64_t ld,
                                                               int64_t rows, int64_t K,
                                                               const int32_t *__restrict__ e, int S, int rev,
                                                               int8_t *__restrict__ out, int64_t Kp, int il) {
  const int64_t r = (int64_t)blockIdx.y * 16 + (threadIdx.x >> 4);
  const int64_t k0 = (int64_t)blockIdx.x * 128 + (threadIdx.x & 15) * 8;
  if (r >= rows || k0 >= Kp) return;
  const int sh = 6 - e[r];
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = k0 + j < K ? scalbn(X[r * ld + k0 + j], sh) : 0.0;  // |x| < 64, exact
  int8_t *o = out + r * (int64_t)S * Kp + (il ? (k0 >> 5) * S * 32 + (k0 & 31) : k0);
  const int64_t sstride = il ? 32 : Kp;
  for (int s = 0; s < S; ++s) {
    unsigned long long w = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double d = rint(x[j]);
      w |= (unsigned long long)(uint8_t)(int8_t)(int)d << (8 * j);
      x[j] = (x[j] - d) * 128.0;  // exact: |x - d| <= 1/2 and x has <= 53 significant bits
    }
    *reinterpret_cast<unsigned long long *>(o + (int64_t)(rev ? S - 1 - s : s) * sstride) = w;
  }
}

inline int ozaki_S() {
  return 8;  // B12: fewer slices (5) left P 1e-7 off the oracle's and indefinite at C5
}

}  // namespace

// scales + digit slices of a rows x K fp64 matrix (K-contiguous, or K x rows if trans):
// out[r][slot(s) Kp + k], slot(s) = rev ? S-1-s : s; e[r] the row's power-of-two exponent
void launch_ozaki_split(const double *X, int64_t ld, int64_t rows, int64_t K, int trans, int S, int rev,
                        int8_t *out, int32_t *e, int64_t Kp, cudaStream_t s, unsigned long long *mx_buf, int il) {
  if (trans) {
    unsigned long long *mx = mx_buf;
    if (!mx) cudaMallocAsync(&mx, (size_t)rows * sizeof(unsigned long long), s);
    cudaMemsetAsync(mx, 0, (size_t)rows * sizeof(unsigned long long), s);
    ozaki_colmax_kernel<<<dim3((unsigned)((rows + 31) / 32), (unsigned)((K + 1023) / 1024)), 256, 0, s>>>(X, ld, rows,
                                                                                                        K, mx);
    ozaki_bits2exp_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(mx, rows, e);
    if (!mx_buf) cudaFreeAsync(mx, s);
    ozaki_split_kernel<<<dim3((unsigned)((Kp + 31) / 32), (unsigned)((rows + 31) / 32)), 256, 0, s>>>(
        X, ld, rows, K, trans, e, S, rev, out, Kp, il);
  } else {
    ozaki_rowexp_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(X, ld, rows, K, 0, e);
    ozaki_split_rows_kernel<<<dim3((unsigned)((Kp + 127) / 128), (unsigned)((rows + 15) / 16)), 256, 0, s>>>(
        X, ld, rows, K, e, S, rev, out, Kp, il);
  }
}

bool ozaki_eligible(const GemmArgs &g) {
  // (lower_only -- the Cholesky trailing updates C -= P P^T -- runs as tri = 1: only the
  // entries on or below the diagonal are formed and written)
  if (g.dmma_only) return false;
  // pays above ~2^32 multiply-adds, with K long enough to amortize the slicing and
  // both output dimensions >= 512 (each input is re-sliced per call: a skinny product
  // such as the block solve's K X with 64 right-hand sides would re-slice the large
  // operand every iteration for little tensor work)
  return g.K >= 512 && g.M >= 512 && g.N >= 512 && (double)g.M * (double)g.N * (double)g.K >= 4.0e9;
}

cudaError_t launch_ozaki_gemm(const GemmArgs &g, bool b_kn, int S, cudaStream_t s, int kernel) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  if (S <= 0) S = ozaki_S();
  const int64_t M = g.M, N = g.N, K = g.K;
  const int64_t Kp = (K + 127) / 128 * 128;
  if ((double)K * S > 524288.0) return cudaErrorInvalidValue;  // int32 level sums could overflow
  int8_t *As = nullptr, *Bs = nullptr;
  int32_t *ea = nullptr, *eb = nullptr;
  const size_t la = (size_t)M * S * Kp, lb = (size_t)N * S * Kp;
  cudaError_t err;
  if ((err = cudaMallocAsync(&As, la, s)) != cudaSuccess) return err;
  if ((err = cudaMallocAsync(&Bs, lb, s)) != cudaSuccess) return err;
  if ((err = cudaMallocAsync(&ea, (M + N) * sizeof(int32_t), s)) != cudaSuccess) return err;
  eb = ea + M;
  // the level-group kernels cut the slice traffic 3x: the directions product (4096 x 16384 x
  // 16384) takes 47.9 ms fused, 47.5 with level groups, 40.8 with level groups on
  // chunk-interleaved slices (v2); at 4096^3 2.55 / 2.84 / 2.80 ms (tools/bench_ozaki_lv.py,
  // profiles/r02_ozaki_lv2.txt), so v2 serves the large products only (M N K >= 2^40);
  // `kernel` (diagnostic) forces one: 0 fused, 1 level groups, 2 level groups v2
  const bool big = (double)M * (double)N * (double)K >= 1099511627776.0;
  const bool lv2 = S <= kLSmax && (kernel >= 0 ? kernel != 0 : big);
  // scales and digit slices (A rows: K-contiguous; op(B) columns: B rows if !b_kn);
  // (B slices in reverse order for the level-streaming kernels: level h's pairs are a
  // contiguous K range; forward order for the level-group kernels, chunk-interleaved for v2)
  launch_ozaki_split(g.A, g.lda, M, K, 0, S, 0, As, ea, Kp, s, nullptr, lv2 ? 1 : 0);
  // (an exactly symmetric B: op(B)'s columns are B's rows, sliced by the row kernels)
  launch_ozaki_split(g.B, g.ldb, N, K, (b_kn && !g.b_sym) ? 1 : 0, S, lv2 ? 0 : 1, Bs, eb, Kp, s, nullptr,
                     lv2 ? 1 : 0);
  if (lv2) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(ozaki_lv2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kL2Smem);
      attr = true;
    }
    CUtensorMap ta, tb;
    const int64_t ldo = (int64_t)S * Kp;
    if (!make_tmap_s8(&ta, As, M, ldo, ldo, kLM) || !make_tmap_s8(&tb, Bs, N, ldo, ldo, kLN))
      return cudaErrorInvalidValue;
    FusedArgs f{};
    f.M = M; f.N = N; f.Kp = Kp; f.S = S; f.ea = ea; f.eb = eb; f.C = g.C; f.ldc = g.ldc; f.Cin = g.Cin;
    f.ldcin = g.ldcin; f.alpha = g.alpha; f.beta = g.beta; f.diag = g.diag; f.diag_offset = g.diag_offset;
    f.tri = g.lower_only ? 1 : g.tri; f.tri_off = g.lower_only ? 0 : g.tri_off;
    const unsigned grid = (unsigned)(((N + kLN - 1) / kLN) * ((M + kLM - 1) / kLM));
    ozaki_lv2_kernel<<<grid, kLThreads, kL2Smem, s>>>(ta, tb, f);
    cudaFreeAsync(As, s);
    cudaFreeAsync(Bs, s);
    cudaFreeAsync(ea, s);
    return cudaGetLastError();
  }
  {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(ozaki_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFSmem);
      attr = true;
    }
    CUtensorMap ta, tb;
    const int64_t ldo = (int64_t)S * Kp;
    if (!make_tmap_s8(&ta, As, M, ldo, ldo, kFM) || !make_tmap_s8(&tb, Bs, N, ldo, ldo, kFN))
      return cudaErrorInvalidValue;
    FusedArgs f{};
    f.M = M; f.N = N; f.Kp = Kp; f.S = S; f.ea = ea; f.eb = eb; f.C = g.C; f.ldc = g.ldc; f.Cin = g.Cin;
    f.ldcin = g.ldcin; f.alpha = g.alpha; f.beta = g.beta; f.diag = g.diag; f.diag_offset = g.diag_offset;
    f.tri = g.lower_only ? 1 : g.tri; f.tri_off = g.lower_only ? 0 : g.tri_off;
    const unsigned grid = (unsigned)(((N + kFN - 1) / kFN) * ((M + kFM - 1) / kFM));
    ozaki_fused_kernel<<<grid, kFThreads, kFSmem, s>>>(ta, tb, f);
    cudaFreeAsync(As, s);
    cudaFreeAsync(Bs, s);
    cudaFreeAsync(ea, s);
    return cudaGetLastError();
  }
}

}  // namespace laker

// Diagnostic: C = A B^T (A: M x K, B: N x K, fp64 row-major, DEVICE) via the Ozaki path.
extern "C" laker_status laker_debug_ozaki_gemm(const double *A, const double *B, double *C, int64_t M, int64_t N,
                                               int64_t K, int32_t slices, int32_t kernel) {
  if (!A || !B || !C || M < 1 || N < 1 || K < 1) return LAKER_ERR_INVALID_ARGUMENT;
  static bool inited = false;
  if (!inited) {
    laker::igemm_init();
    cudaMemPool_t pool;
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    inited = true;
  }
  laker::GemmArgs g{};
  g.M = M; g.N = N; g.K = K; g.A = A; g.lda = K; g.B = B; g.ldb = K; g.C = C; g.ldc = N; g.alpha = 1.0;
  if (laker::launch_ozaki_gemm(g, false, slices, 0, kernel) != cudaSuccess) return LAKER_ERR_CUDA;
  if (cudaDeviceSynchronize() != cudaSuccess) return LAKER_ERR_CUDA;
  return LAKER_OK;
}
