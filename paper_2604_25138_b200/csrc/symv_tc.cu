// Exact symmetric K apply on the int8 tensor cores (round 2): the same block-upper-
// triangle tiles, partials and finalize as symv.cu (K.p for the PCG, Alg. 1 l.16,
// P:306-321; rows a4/a9), with every product computed exactly in integers.
//
// K is stored as 8 signed 7-bit digit slices per entry with one global exponent,
//   K_ij = 2^(eK+1) sum_{s<8} d_ijs 2^(-7(s+1)),   d in [-64, 64],
// exact when every entry's mantissa falls on that 2^(eK-55) grid (the assembly checks
// it; K = exp(scale <e_i, e_j>) of the configs lies in [0.5, 4)), and x (the CG
// direction) as 16 slices with its own exponent, x_j = 2^(F+1) sum_{t<16} c_jt
// 2^(-7(t+1)) + (a remainder below 2^(F-111), ~2^-112 max|x|: under Dot2's own error).
// A row sum is then sum_{s,t} 2^(eK+F+2-7(s+t+2)) D_st with D_st = sum_j d_ijs c_jt an
// exact int32 (|D| <= 2^12 n < 2^31 for n <= 2^18): tcgen05 kind::i8 accumulates it in TMEM per
// slice pair, the level sums D_L = sum_{s+t=L} D_st are exact int64, and a TwoSum chain
// over the 23 levels gives the row's unrounded (s, c) pair -- the same contract as the
// fp64 kernel's compensated pairs (the finalize rounds once; correctly rounded in
// practice, so bitwise the oracle's O2 rows).  The fp64 work per matrix element drops
// from 14 operations (two offset-Fast2Sum products) to none: the apply streams K's
// slices (8 bytes per entry, as fp64) at the tile-stream rate.
//
// Per 128 x 64 tile (I, jt), one row-major SWIZZLE_64B shared-memory copy of the 8
// slices feeds both products (tools/mma_mn_major_test.cu):
//   rows    D_row[s] (M = 128, N = 16) += K_s (K-major: contraction over the 64 columns)
//           x x_J slices; accumulated over the whole block-row segment in TMEM;
//   columns D_col[s] (M = 64, N = 16)   = K_s^T (MN-major A, "transpose A": contraction
//           over the 128 rows) x x_I slices; read out per tile (off the diagonal block).
// TMEM (512 columns): D_row double-buffered [0, 256), D_col double-buffered [256, 512).
// Warps: 0 TMA producer, 1 MMA issuer, 2..5 epilogue (TMEM lane quadrants 2, 3, 0, 1).
#include <cuda.h>

#include <algorithm>
#include <cmath>

#include "laker_internal.h"
#include "tc_int8.cuh"
#include "tri.cuh"

namespace laker {
namespace {

constexpr int kTR = 128, kTC = 64;                 // tile rows / columns (symv.cu's plan)
constexpr int kSK = 8;                              // slices of K
constexpr int kSX = 16;                             // slices of x (MMA N)
constexpr int kStg = 3;                             // ring stages
constexpr uint32_t kSliceBytes = kTR * kTC;         // 8 KiB
constexpr uint32_t kKBytes = kSK * kSliceBytes;     // 64 KiB
constexpr uint32_t kXJBytes = kSX * kTC;            // 1 KiB
constexpr uint32_t kXIBytes = kSX * kTR;            // 2 KiB
constexpr int kTcThreads = 6 * 32;
constexpr int kLevels = kSK + kSX - 1;              // 23
// shared layout (1024-aligned base): [kStg][K 64 KiB] [kStg][xJ 1 KiB] [2][xI 2 KiB] barriers
constexpr size_t kOffXJ = (size_t)kStg * kKBytes;
constexpr size_t kOffXI = kOffXJ + (size_t)kStg * kXJBytes;
constexpr size_t kOffBar = kOffXI + 2 * kXIBytes;
constexpr size_t kTcSmem = 1024 + kOffBar + 256;

// descriptor of a K slice as the MN-major A operand of the column product (SWIZZLE_64B,
// 8-row atoms of 64 B, SBO 512 B between atoms along the contraction)
__device__ __forceinline__ uint64_t sdesc_mn_sw64(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *tm, int32_t c0, int32_t c1, int32_t c2,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// 2^e for a compile-time e (exact; folded once the level loop is unrolled)
__device__ __forceinline__ double pow2c(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }

// the exact level sums of one output (s slices x 16 t values read from TMEM columns
// base + 16 s), folded to an unrounded pair scaled by 2^escale
__device__ __forceinline__ dd_pair combine_levels(uint32_t taddr, int escale) {
  long long lv[kLevels];
#pragma unroll
  for (int L = 0; L < kLevels; ++L) lv[L] = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // two batches of 4 slices: 64 registers in flight
    uint32_t v[4][16];
#pragma unroll
    for (int s = 0; s < 4; ++s) tc::tmem_ld16(taddr + (uint32_t)(16 * (4 * h + s)), v[s]);
    tc::tmem_ld_wait();
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
      for (int t = 0; t < kSX; ++t) lv[4 * h + s + t] += (long long)(int32_t)v[s][t];
  }
  // sum_L lv_L 2^(-7L), each term exact in fp64 (|lv| < 2^34), TwoSum chain from L = 0
  dd_pair r = {(double)lv[0], 0.0};
#pragma unroll
  for (int L = 1; L < kLevels; ++L) {
    const double t = __dmul_rn((double)lv[L], pow2c(-7 * L));
    double s, e;
    two_sum(r.s, t, s, e);
    r.s = s;
    r.c = __dadd_rn(r.c, e);
  }
  r.s = ldexp(r.s, escale);
  r.c = ldexp(r.c, escale);
  return r;
}

struct TcArgs {
  SymvArgs t;
  const int *eK;  // global exponent of K's slices (device)
  const int *F;   // exponent of this x's slices (device, written by the slicing kernel)
};

__global__ void __launch_bounds__(kTcThreads, 1)
    symv_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmXJ,
                   const __grid_constant__ CUtensorMap tmXI, const TcArgs ta) {
  const SymvArgs &a = ta.t;
  if (a.state != nullptr && *(volatile int32_t *)&a.state->done) return;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t base_s = smem_u32(smem_raw);
  unsigned char *smem = smem_raw + ((1024 - (base_s & 1023)) & 1023);
  unsigned char *sK = smem;
  unsigned char *sXJ = smem + kOffXJ;
  unsigned char *sXI = smem + kOffXI;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kOffBar);  // [kStg]
  uint64_t *empty = full + kStg;                                  // [kStg]
  uint64_t *xif = empty + kStg;                                   // [2]
  uint64_t *xie = xif + 2;                                        // [2]
  uint64_t *rowf = xie + 2;                                       // [2]
  uint64_t *rowe = rowf + 2;                                      // [2]
  uint64_t *colf = rowe + 2;                                      // [2]
  uint64_t *cole = colf + 2;                                      // [2]
  uint32_t *holder = reinterpret_cast<uint32_t *>(cole + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t0 = a.T * blockIdx.x / gridDim.x, t1 = a.T * (blockIdx.x + 1) / gridDim.x;
  if (t0 >= t1) return;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStg; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&xif[b], 1);
      mbar_init(&xie[b], 1);
      mbar_init(&rowf[b], 1);
      mbar_init(&rowe[b], 4);
      mbar_init(&colf[b], 1);
      mbar_init(&cole[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(holder, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *holder;
  const int I0 = find_block_row(a.toff, a.nb, t0);

  if (warp == 0) {
    // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      int I = I0;
      int64_t rend = a.toff[I + 1];
      int slot = 0, xb = 0, nseg = 0;
      uint32_t ph = 0;
      bool first = true;
      for (int64_t t = t0; t < t1; ++t) {
        const bool newI = (t == t0) || (t >= rend);
        while (t >= rend) rend = a.toff[++I + 1];
        const int jt = 2 * I + (int)(t - a.toff[I]);
        if (newI) {
          if (nseg >= 2) mbar_wait(&xie[xb], (uint32_t)(((nseg - 2) >> 1) & 1));
          mbar_arrive_expect_tx(&xif[xb], kXIBytes);
          tc::tma_load_2d(sXI + xb * kXIBytes, &tmXI, I * kTR, 0, &xif[xb]);
          xb ^= 1;
          ++nseg;
        }
        if (!first) mbar_wait(&empty[slot], ph ^ 1u);
        mbar_arrive_expect_tx(&full[slot], kKBytes + kXJBytes);
        tma_load_3d(sK + slot * kKBytes, &tmK, jt * kTC, I * kTR, 0, &full[slot]);
        tc::tma_load_2d(sXJ + slot * kXJBytes, &tmXJ, jt * kTC, 0, &full[slot]);
        if (++slot == kStg) {
          slot = 0;
          ph ^= 1u;
          first = false;
        }
      }
    }
    return;
  }

  if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idr = tc::idesc_i8(kTR, kSX);
      constexpr uint32_t idc = tc::idesc_i8(kTC, kSX) | (1u << 15);  // A = K_s^T (MN-major)
      int I = I0;
      int64_t rend = a.toff[I + 1];
      int slot = 0, xb = 0, rb = 0, cb = 0, nseg = 0, ncol = 0;
      uint32_t ph = 0;
      bool acc = false;
      for (int64_t t = t0; t < t1; ++t) {
        const bool newI = (t == t0) || (t >= rend);
        while (t >= rend) rend = a.toff[++I + 1];
        const int jt = 2 * I + (int)(t - a.toff[I]);
        if (newI) {
          if (nseg >= 2) mbar_wait(&rowe[rb], (uint32_t)(((nseg - 2) >> 1) & 1));  // row buffer drained
          mbar_wait(&xif[xb], (uint32_t)((nseg >> 1) & 1));
          ++nseg;
          acc = false;
        }
        mbar_wait(&full[slot], ph);
        tc::fence_after();
        const uint32_t kb = smem_u32(sK + slot * kKBytes), xj = smem_u32(sXJ + slot * kXJBytes);
        const uint32_t trow = tmem + (uint32_t)(rb * 128);
#pragma unroll
        for (int s = 0; s < kSK; ++s)
#pragma unroll
          for (int kk = 0; kk < kTC / 32; ++kk)
            tc::mma_i8(trow + 16 * s, tc::sdesc_k_sw64(kb + s * kSliceBytes + kk * 32), tc::sdesc_k_sw64(xj + kk * 32),
                       idr, (acc || kk > 0) ? 1u : 0u);
        acc = true;
        if (jt / 2 != I + a.I0) {  // off the diagonal block: the column product of this tile
          if (ncol >= 2) mbar_wait(&cole[cb], (uint32_t)(((ncol - 2) >> 1) & 1));
          tc::fence_after();
          const uint32_t tcol = tmem + 256 + (uint32_t)(cb * 128);
          const uint32_t xi = smem_u32(sXI + xb * kXIBytes);
#pragma unroll
          for (int s = 0; s < kSK; ++s)
#pragma unroll
            for (int kk = 0; kk < kTR / 32; ++kk)
              tc::mma_i8(tcol + 16 * s, sdesc_mn_sw64(kb + s * kSliceBytes + kk * 2048), tc::sdesc_k_sw128(xi + kk * 32),
                         idc, kk > 0 ? 1u : 0u);
          tc::mma_commit(&colf[cb]);
          cb ^= 1;
          ++ncol;
        }
        tc::mma_commit(&empty[slot]);
        if (++slot == kStg) {
          slot = 0;
          ph ^= 1u;
        }
        if (t + 1 == t1 || t + 1 >= rend) {  // segment complete: rows to the epilogue, x_I slot free
          tc::mma_commit(&rowf[rb]);
          tc::mma_commit(&xie[xb]);
          rb ^= 1;
          xb ^= 1;
        }
      }
    }
    __syncwarp();
    // the allocating warp releases TMEM once the epilogue has drained every accumulator
    asm volatile("bar.sync 1, 160;" ::: "memory");
    tc::fence_after();
    tc::tmem_dealloc(tmem, 512);
    return;
  }

  // ------------------------------------------------------------ epilogue (warps 2..5)
  const int q = warp & 3;  // TMEM lane quadrant this warp may access
  const int escale = *ta.eK + *ta.F + 2 - 14;
  int I = I0;
  int64_t rend = a.toff[I + 1];
  int rb = 0, cb = 0, nseg = 0, ncol = 0;
  for (int64_t t = t0; t < t1; ++t) {
    const bool newI = (t == t0) || (t >= rend);
    while (t >= rend) rend = a.toff[++I + 1];
    if (newI) ++nseg;
    const int jt = 2 * I + (int)(t - a.toff[I]);
    if (jt / 2 != I + a.I0) {
      mbar_wait(&colf[cb], (uint32_t)((ncol >> 1) & 1));
      tc::fence_after();
      // M = 64 accumulator: columns 16 q .. 16 q + 15 in lanes 32 q .. 32 q + 15
      const uint32_t taddr = tmem + 256 + (uint32_t)(cb * 128) + ((uint32_t)(32 * q) << 16);
      const dd_pair v = combine_levels(taddr, escale);
      if (lane < 16) a.colpart[(int64_t)I * a.ldcp + (int64_t)jt * kTC + 16 * q + lane] = v;
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&cole[cb]);
      cb ^= 1;
      ++ncol;
    }
    if (t + 1 == t1 || t + 1 >= rend) {
      mbar_wait(&rowf[rb], (uint32_t)(((nseg - 1) >> 1) & 1));
      tc::fence_after();
      const uint32_t taddr = tmem + (uint32_t)(rb * 128) + ((uint32_t)(32 * q) << 16);
      const dd_pair v = combine_levels(taddr, escale);
      const int sg = (int)blockIdx.x - a.segfirst[I];
      a.rowpart[((int64_t)I * a.maxseg + sg) * kTR + 32 * q + lane] = v;
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&rowe[rb]);
      rb ^= 1;
    }
  }
  tc::fence_before();
  asm volatile("bar.sync 1, 160;" ::: "memory");
}

// x -> 16 digit slices with one exponent: F with max|x| < 2^F (from the per-CTA maxima
// parts), v = x 2^-(F+1), c_t = rint(128 v) digit by digit; xs is 16 rows x ldx bytes
__global__ void __launch_bounds__(256) slice_x_kernel(const double *__restrict__ x, int64_t n,
                                                      const double *__restrict__ parts, int nparts,
                                                      int8_t *__restrict__ xs, int64_t ldx, int *Fout,
                                                      const PcgState *st) {
  if (st && *(volatile const int32_t *)&st->done) return;
  double m = 0.0;
  for (int k = 0; k < nparts; ++k) m = fmax(m, parts[k]);
  int F = 0;
  if (m > 0.0) frexp(m, &F);  // m = f 2^F, f in [0.5, 1): |x| <= m < 2^F
  if (blockIdx.x == 0 && threadIdx.x == 0) *Fout = F;
  const double sc = ldexp(1.0, -(F + 1));
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double v = __dmul_rn(x[j], sc);  // exact (power of two), |v| < 0.5
#pragma unroll
    for (int t = 0; t < kSX; ++t) {
      v = __dmul_rn(v, 128.0);
      const double d = rint(v);
      v = __dsub_rn(v, d);
      xs[(int64_t)t * ldx + j] = (int8_t)(int)d;
    }
  }
}

// K (rows x n, stride ld) -> 8 slices (slice s: rows x ldk bytes at ks + s rows ldk, the
// padding columns n .. ldk zero) with the global exponent eK (max |K| < 2^eK); flag[0] = 1
// if some entry is not exact.  Thread: 8 consecutive columns of one row, 8-byte stores.
__global__ void __launch_bounds__(256) slice_k_kernel(const double *__restrict__ K, int64_t rows, int64_t n,
                                                      int64_t ld, int eK, int8_t *__restrict__ ks, int64_t ldk,
                                                      int *flag) {
  const double sc = ldexp(1.0, -(eK + 1));
  const int64_t j0 = 8 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  bool bad = false;
  if (j0 < ldk) {
    for (int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
      unsigned long long w[kSK];
#pragma unroll
      for (int s = 0; s < kSK; ++s) w[s] = 0ull;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (j0 + k >= n) break;
        double v = __dmul_rn(K[i * ld + j0 + k], sc);
#pragma unroll
        for (int s = 0; s < kSK; ++s) {
          v = __dmul_rn(v, 128.0);
          const double d = rint(v);
          v = __dsub_rn(v, d);
          w[s] |= (unsigned long long)(uint8_t)(int8_t)(int)d << (8 * k);
        }
        bad |= v != 0.0;
      }
#pragma unroll
      for (int s = 0; s < kSK; ++s)
        *reinterpret_cast<unsigned long long *>(ks + ((int64_t)s * rows + i) * ldk + j0) = w[s];
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
}

__global__ void absmax_reduce_kernel(const double *__restrict__ v, int64_t n, double *out) {
  __shared__ double sm[32];
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, fabs(v[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, sm[w]);
    *out = m;
  }
}

typedef CUresult (*PFN_enc)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_enc get_enc() {
  static PFN_enc fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_enc>(p);
  }
  return fn;
}

}  // namespace

struct SymvTc {
  int64_t n = 0, ldk = 0, ldx = 0;
  int8_t *ks = nullptr, *xs = nullptr;
  int *dexp = nullptr;  // [0] eK, [1] F of the last sliced x, [2] exactness flag
  double *dmax = nullptr;
  CUtensorMap tmK, tmXJ, tmXI;
};

void symv_tc_free(SymvTc *&p) {
  if (!p) return;
  cudaFree(p->ks);
  cudaFree(p->xs);
  cudaFree(p->dexp);
  cudaFree(p->dmax);
  delete p;
  p = nullptr;
}

void symv_tc_init() {
  cudaFuncSetAttribute(symv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem);
}

// Slice the (bitwise symmetric, single-rank) K into the int8 form; false if some entry is
// not exactly representable (the fp64 symmetric kernel stays in use then)
bool symv_tc_prepare(SymvTc *&p, const double *K, int64_t n, int64_t ld, const double *rowmax, cudaStream_t s) {
  if (n < 1 || n > (1 << 18)) return false;  // |D_st| <= 64 * 64 * n < 2^31 in the int32 accumulators
  PFN_enc enc = get_enc();
  if (!enc) return false;
  const int64_t ldk = (n + 127) / 128 * 128;
  if (!p || p->n != n) {
    symv_tc_free(p);
    p = new SymvTc();
    p->n = n;
    p->ldk = ldk;
    p->ldx = ldk;
    if (cudaMalloc(&p->ks, (size_t)kSK * n * ldk) != cudaSuccess ||
        cudaMalloc(&p->xs, (size_t)kSX * p->ldx) != cudaSuccess || cudaMalloc(&p->dexp, 4 * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&p->dmax, sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      symv_tc_free(p);
      return false;
    }
    cudaMemset(p->xs, 0, (size_t)kSX * p->ldx);
    cuuint64_t dk[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)kSK};
    cuuint64_t sk[2] = {(cuuint64_t)ldk, (cuuint64_t)ldk * (cuuint64_t)n};
    cuuint32_t bk[3] = {kTC, kTR, kSK}, es[3] = {1, 1, 1};
    cuuint64_t dx[2] = {(cuuint64_t)n, (cuuint64_t)kSX}, sx[1] = {(cuuint64_t)p->ldx};
    cuuint32_t bj[2] = {kTC, kSX}, bi[2] = {kTR, kSX};
    if (enc(&p->tmK, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, p->ks, dk, sk, bk, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS ||
        enc(&p->tmXJ, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, p->xs, dx, sx, bj, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS ||
        enc(&p->tmXI, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, p->xs, dx, sx, bi, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS) {
      symv_tc_free(p);
      return false;
    }
  }
  // global exponent from the row maxima (max |K| < 2^eK)
  absmax_reduce_kernel<<<1, 1024, 0, s>>>(rowmax, n, p->dmax);
  double hmax = 0.0;
  cudaMemcpyAsync(&hmax, p->dmax, sizeof(double), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  if (!(hmax > 0.0) || !std::isfinite(hmax)) return false;
  int eK = 0;
  std::frexp(hmax, &eK);
  int hexp[3] = {eK, 0, 0};
  cudaMemcpyAsync(p->dexp, hexp, 3 * sizeof(int), cudaMemcpyHostToDevice, s);
  const dim3 grid((unsigned)((ldk / 8 + 255) / 256), (unsigned)std::min<int64_t>(n, 65535));
  slice_k_kernel<<<grid, 256, 0, s>>>(K, n, n, ld, eK, p->ks, ldk, p->dexp + 2);
  int flag = 1;
  cudaMemcpyAsync(&flag, p->dexp + 2, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return false;
  return flag == 0;
}

// the tile pass of the exact tensor-core apply: x's slices, then the tiles; the caller
// (symv.cu) launches the shared finalize
void launch_symv_tc(SymvTc *p, const SymvArgs &a, const double *xparts, int nxparts, int grid, cudaStream_t s) {
  slice_x_kernel<<<(unsigned)std::min<int64_t>((p->n + 255) / 256, 296), 256, 0, s>>>(
      a.x, p->n, xparts, nxparts, p->xs, p->ldx, p->dexp + 1, a.state);
  TcArgs ta{};
  ta.t = a;
  ta.eK = p->dexp;
  ta.F = p->dexp + 1;
  symv_tc_kernel<<<grid, kTcThreads, kTcSmem, s>>>(p->tmK, p->tmXJ, p->tmXI, ta);
}

}  // namespace laker
