// Exact symmetric K apply on the int8 tensor cores (round 2): the block upper triangle of K
// streamed once, the partials and finalize of symv.cu (K.p for the PCG, Alg. 1 l.16,
// P:306-321; rows a4/a9), with every product computed exactly in integers.
//
// K is stored as 8 signed 7-bit digit slices per entry with one global exponent,
//   K_ij = 2^(eK+1) sum_{s<8} d_ijs 2^(-7(s+1)),   d in [-64, 64],
// exact when every entry's mantissa falls on that 2^(eK-55) grid (symv_tc_prepare checks
// it; K = exp(scale <e_i, e_j>) of the configs lies in [0.8, 2.9]), and x (the CG
// direction) as 16 slices with its own exponent, x_j = 2^(F+1) sum_{t<16} c_jt
// 2^(-7(t+1)) + (a remainder below 2^(F-112), ~2^-112 max|x|: under Dot2's own error).
// A row sum is then sum_{s,t} 2^(eK+F+2-7(s+t+2)) D_st with D_st = sum_j d_ijs c_jt an
// exact int32 (|D| <= 2^12 n < 2^31 for n <= 2^18): tcgen05 kind::i8 accumulates it in
// TMEM per slice pair, the level sums are folded exactly in int64 and a short TwoSum chain
// gives the row's unrounded (s, c) pair -- the same contract as the fp64 kernel's
// compensated pairs (the finalize rounds once; correctly rounded in practice, so bitwise
// the oracle's O2 rows).  The fp64 work per matrix element drops from 14 operations (two
// offset-Fast2Sum products) to none: the apply streams K's slices (8 bytes per entry,
// as fp64) at the tile-stream rate.
//
// Tiles are 128 x 128 (block-row I takes the column blocks J = I .. nb - 1; persistent
// CTAs take contiguous tile ranges).  The slices are stored tile-major, upper triangle only
// (n^2 / 2 entries x 8 bytes, as the fp64 triangle): slice s of tile t is 16 KiB contiguous,
// two 64-column halves of 128 rows x 64 B, already in the SWIZZLE_64B image, so the producer
// moves 4 slices (64 KiB) per ring slot with plain bulk copies (3 slots).  One slice feeds
// both products (tools/mma_mn128_test.cu):
//   rows    D_row[s] (M = 128, N = 16) += K_s (K-major, contraction over the 128 columns)
//           x x_J slices, accumulated over the block-row segment in TMEM (warp 1);
//   columns D_col[s] (M = 128, N = 16)  = K_s^T (MN-major A spanning both halves: LBO =
//           8 KiB, "transpose A"; contraction over the 128 rows) x x_I slices, read out per
//           tile off the diagonal block (warp 6).
// tools/mma_rate.cu, tools/mma_issue.cu: ~39 cycles per M = 128, N = 16 int8 MMA; the 64
// MMAs of a tile then take ~60% of its HBM time, and the kernel runs at the bulk-copy
// stream's rate (tools/tc_variants.sh: 170 us with the MMAs vs 159 us streaming alone at
// C3; TC work alone 104 us).  TMEM (512 columns): D_row double-buffered [0, 256), D_col
// [256, 512).  Warps: 0 producer, 1 row-product MMA issuer, 6 column-product MMA issuer,
// 2..5 epilogue (TMEM lane quadrants 2, 3, 0, 1).
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "laker_internal.h"
#include "tc_int8.cuh"
#include "tri.cuh"

// TC_EXP (tools/tc_variants.sh builds only; the library is built with 0): 1 = epilogue
// without the level combine, 2 = producer without K loads (TC + epilogue alone), 3 = MMA
// warp without MMAs (the bulk-copy stream alone), 4 = 1 + 2.
#ifndef TC_EXP
#define TC_EXP 0
#endif

namespace laker {
namespace {

constexpr int kT = 128;                             // tile rows = columns
constexpr int kSK = 8;                              // slices of K
constexpr int kSX = 16;                             // slices of x (MMA N)
constexpr int kSS = 4;                              // slices per ring slot (one mbarrier wait)
constexpr int kRing = 3;                            // ring slots (12 slices, 192 KiB in flight)
constexpr int kXJSlots = 3;                         // x_J tiles in flight
constexpr uint32_t kHalfBytes = kT * 64;            // 8 KiB: 128 rows x 64 columns
constexpr uint32_t kSliceBytes = 2 * kHalfBytes;    // 16 KiB
constexpr uint32_t kXBytes = kSX * kT;              // 2 KiB: 16 slices x 128
constexpr int kTcThreads = 7 * 32;
constexpr int kLevels = kSK + kSX - 1;              // 23 (8 groups of 3: tri.cuh kTcGroups)
static_assert((kLevels + 2) / 3 == kTcGroups, "level groups");
// shared layout (1024-aligned base): [kRing][kSS slices of 16 KiB] [kXJSlots][x_J] [2][x_I] barriers
constexpr size_t kOffXJ = (size_t)kRing * kSS * kSliceBytes;
constexpr size_t kOffXI = kOffXJ + (size_t)kXJSlots * kXBytes;
constexpr size_t kOffBar = kOffXI + 2 * kXBytes;
constexpr size_t kTcSmem = 1024 + kOffBar + 512;

// descriptor of a K slice as the MN-major A operand of the column product (SWIZZLE_64B,
// 8-row atoms of 64 B: SBO 512 B between atoms along the contraction, LBO 8 KiB between
// the two 64-column halves along M)
__device__ __forceinline__ uint64_t sdesc_mn_sw64(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)(kHalfBytes >> 4) << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}

// Single-thread tcgen05 operations issued from converged warp code: one lane is elected
// inside the asm block, so the surrounding loop stays warp-uniform and its operands live
// in uniform registers (no per-MMA ELECT / R2UR.BROADCAST loop: tools/mma_issue.cu
// measured 39 instead of 50 cycles per MMA in isolation, and far less under load)
__device__ __forceinline__ void mma_i8_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void commit_elect(uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(bar))
      : "memory");
}

// One output's exact level-group sums from its 8 x 16 slice-pair accumulators (TMEM
// columns base + 16 s, t = 0..15): level L = s + t carries 2^(-7L); three consecutive
// levels fold exactly into G_g = sum_{L in g} D_L 2^(7(3g+2-L)) (tri.cuh) -- |D_L| <= 8 *
// 2^12 n, so |G_g| < 2^48 per contribution and for the whole row.
__device__ __forceinline__ void level_groups(uint32_t taddr, long long (&G)[kTcGroups]) {
#pragma unroll
  for (int g = 0; g < kTcGroups; ++g) G[g] = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // two batches of 4 slices: 64 registers in flight
    uint32_t v[4][16];
#pragma unroll
    for (int s = 0; s < 4; ++s) tc::tmem_ld16(taddr + (uint32_t)(16 * (4 * h + s)), v[s]);
    tc::tmem_ld_wait();
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
      for (int t = 0; t < kSX; ++t) {
        const int L = 4 * h + s + t;
        G[L / 3] += (long long)(int32_t)v[s][t] << (7 * (2 - L % 3));
      }
  }
}

// add an output's groups to row i's accumulators (integer: exact whatever the order).
// Layout [W][8][cs]: the rows of rank c's shard (cs = n / W rows; one rank: cs = the padded
// n) are the contiguous block c, so the sharded apply reduce-scatters it as it stands.
__device__ __forceinline__ void red_groups(long long *yacc, int64_t cs, int64_t i, const long long (&G)[kTcGroups]) {
  const int64_t c = i / cs;
  long long *base = yacc + c * kTcGroups * cs + (i - c * cs);
#pragma unroll
  for (int g = 0; g < kTcGroups; ++g)
    atomicAdd(reinterpret_cast<unsigned long long *>(base + g * cs), (unsigned long long)G[g]);
}

struct TcArgs {
  const PcgState *state;
  int64_t n;
  const int64_t *toff;  // [nb + 1] first 128 x 128 tile of each (local) block-row
  const int32_t *jt;    // sharded plan: the column block of every tile (null: J = I0 + I ..)
  int32_t I0;           // global index of local block-row 0
  int64_t T;            // tiles
  int32_t nb;
  const int8_t *ks;     // the tile-major slice store
  long long *yacc;      // [W][8][cs] exact level-group sums per row (tri.cuh, red_groups)
  int64_t cs;
};

__device__ __forceinline__ int tile_col(const TcArgs &ta, int I, int64_t t) {
  return ta.jt != nullptr ? ta.jt[t] : ta.I0 + I + (int)(t - ta.toff[I]);
}

__global__ void __launch_bounds__(kTcThreads, 1)
    symv_tc_kernel(const __grid_constant__ CUtensorMap tmX, const TcArgs ta) {
  if (ta.state != nullptr && *(volatile int32_t *)&ta.state->done) return;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t base_s = smem_u32(smem_raw);
  unsigned char *smem = smem_raw + ((1024 - (base_s & 1023)) & 1023);
  unsigned char *sK = smem;
  unsigned char *sXJ = smem + kOffXJ;
  unsigned char *sXI = smem + kOffXI;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kOffBar);  // [kRing]
  uint64_t *empty = full + kRing;                                 // [kRing]
  uint64_t *xjf = empty + kRing;                                  // [kXJSlots]
  uint64_t *xje = xjf + kXJSlots;                                 // [kXJSlots]
  uint64_t *xif = xje + kXJSlots;                                 // [2]
  uint64_t *xie = xif + 2;                                        // [2]
  uint64_t *rowf = xie + 2;                                       // [2]
  uint64_t *rowe = rowf + 2;                                      // [2]
  uint64_t *colf = rowe + 2;                                      // [2]
  uint64_t *cole = colf + 2;                                      // [2]
  uint32_t *holder = reinterpret_cast<uint32_t *>(cole + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t0 = ta.T * blockIdx.x / gridDim.x, t1 = ta.T * (blockIdx.x + 1) / gridDim.x;
  if (t0 >= t1) return;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRing; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);
    }
    for (int s = 0; s < kXJSlots; ++s) {
      mbar_init(&xjf[s], 1);
      mbar_init(&xje[s], 1);
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
  const int I0 = find_block_row(ta.toff, ta.nb, t0);

  if (warp == 0) {
    // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      int I = I0;
      int64_t rend = ta.toff[I + 1];
      int xb = 0, nseg = 0, slot = 0, tb = 0;
      uint32_t ph = 0, tph = 0;
      bool ring_full = false, xj_full = false;  // past the first pass over the slots
      for (int64_t t = t0; t < t1; ++t) {
        const bool newI = (t == t0) || (t >= rend);
        while (t >= rend) rend = ta.toff[++I + 1];
        const int J = tile_col(ta, I, t);
        if (newI) {
          if (nseg >= 2) mbar_wait(&xie[xb], (uint32_t)(((nseg - 2) >> 1) & 1));
          mbar_arrive_expect_tx(&xif[xb], kXBytes);
          tc::tma_load_2d(sXI + xb * kXBytes, &tmX, (ta.I0 + I) * kT, 0, &xif[xb]);
          xb ^= 1;
          ++nseg;
        }
        if (xj_full) mbar_wait(&xje[tb], tph ^ 1u);
        mbar_arrive_expect_tx(&xjf[tb], kXBytes);
        tc::tma_load_2d(sXJ + tb * kXBytes, &tmX, J * kT, 0, &xjf[tb]);
        if (++tb == kXJSlots) {
          tb = 0;
          tph ^= 1u;
          xj_full = true;
        }
#pragma unroll 1
        for (int g = 0; g < kSK / kSS; ++g) {
          if (ring_full) mbar_wait(&empty[slot], ph ^ 1u);
          // slices g kSS .. of tile t: 16 KiB contiguous each in the tile-major store, one box each
#if TC_EXP == 2 || TC_EXP == 4
          mbar_arrive(&full[slot]);
#else
          mbar_arrive_expect_tx(&full[slot], kSS * kSliceBytes);
#pragma unroll
          for (int ss = 0; ss < kSS; ++ss)
            bulk_g2s(sK + (size_t)(slot * kSS + ss) * kSliceBytes, ta.ks + (t * kSK + g * kSS + ss) * kSliceBytes,
                     kSliceBytes, &full[slot], pol);
#endif
          if (++slot == kRing) {
            slot = 0;
            ph ^= 1u;
            ring_full = true;
          }
        }
      }
    }
    return;
  }

  if (warp == 1 || warp == 6) {
    // ---------------------------------------------------------- MMA issuers (whole warps,
    // one lane elected per MMA / commit): warp 1 the row products, warp 6 the column
    // products; each releases every ring slot (empty: 2 arrivals)
    const bool rows = warp == 1;
    constexpr uint32_t idr = tc::idesc_i8(kT, kSX);
    constexpr uint32_t idc = tc::idesc_i8(kT, kSX) | (1u << 15);  // A = K_s^T (MN-major)
    const uint64_t dK0 = rows ? tc::sdesc_k_sw64(smem_u32(sK)) : sdesc_mn_sw64(smem_u32(sK));
    const uint64_t dXJ0 = tc::sdesc_k_sw128(smem_u32(sXJ));
    const uint64_t dXI0 = tc::sdesc_k_sw128(smem_u32(sXI));
    int I = I0;
    int64_t rend = ta.toff[I + 1];
    int xb = 0, rb = 0, cb = 0, nseg = 0, ncol = 0;
    int slot = 0, tb = 0;
    uint32_t ph = 0, tph = 0;
    bool acc = false;
    for (int64_t t = t0; t < t1; ++t) {
      const bool newI = (t == t0) || (t >= rend);
      while (t >= rend) rend = ta.toff[++I + 1];
      const int J = tile_col(ta, I, t);
      const bool off = J != ta.I0 + I;  // off the diagonal block: the column product too
      if (newI) {
        if (rows) {
          if (nseg >= 2) mbar_wait(&rowe[rb], (uint32_t)(((nseg - 2) >> 1) & 1));  // row buffer drained
        } else {
          mbar_wait(&xif[xb], (uint32_t)((nseg >> 1) & 1));
        }
        ++nseg;
        acc = false;
      }
      if (rows) {
        mbar_wait(&xjf[tb], tph);
      } else if (off && ncol >= 2) {
        mbar_wait(&cole[cb], (uint32_t)(((ncol - 2) >> 1) & 1));
      }
      tc::fence_after();
      // descriptors: the start-address field is addr >> 4 in the low 14 bits, so an
      // offset inside shared memory is added to the base descriptor (no carry: < 256 KiB)
      const uint32_t td = rows ? tmem + (uint32_t)(rb * 128) : tmem + 256 + (uint32_t)(cb * 128);
      const uint64_t dX = rows ? dXJ0 + (uint64_t)((tb * kXBytes) >> 4) : dXI0 + (uint64_t)((xb * kXBytes) >> 4);
      const bool work = rows || off;
#pragma unroll 1
      for (int g = 0; g < kSK / kSS; ++g) {
        mbar_wait(&full[slot], ph);
        tc::fence_after();
#if TC_EXP != 3
        if (work) {
#pragma unroll
          for (int ss = 0; ss < kSS; ++ss) {
            const int s = g * kSS + ss;
            const uint64_t so = (uint64_t)(((slot * kSS + ss) * kSliceBytes) >> 4);
            if (rows) {
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)  // columns 32 kk ..: half kk / 2, +32 B inside it
                mma_i8_elect(td + 16 * s, dK0 + so + (uint64_t)(((kk >> 1) * kHalfBytes + (kk & 1) * 32) >> 4),
                             dX + (uint64_t)((kk * 32) >> 4), idr, (acc || kk > 0) ? 1u : 0u);
            } else {
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)  // rows 32 kk ..: 2 KiB into each half
                mma_i8_elect(td + 16 * s, dK0 + so + (uint64_t)((kk * 2048) >> 4), dX + (uint64_t)((kk * 32) >> 4),
                             idc, kk > 0 ? 1u : 0u);
            }
          }
        }
#endif
        commit_elect(&empty[slot]);
        if (++slot == kRing) {
          slot = 0;
          ph ^= 1u;
        }
      }
      acc = true;
      if (rows) {
        commit_elect(&xje[tb]);
        if (++tb == kXJSlots) {
          tb = 0;
          tph ^= 1u;
        }
      } else if (off) {
        commit_elect(&colf[cb]);
        cb ^= 1;
        ++ncol;
      }
      if (t + 1 == t1 || t + 1 >= rend) {  // segment complete: rows to the epilogue / x_I slot free
        if (rows) {
          commit_elect(&rowf[rb]);
          rb ^= 1;
        } else {
          commit_elect(&xie[xb]);
          xb ^= 1;
        }
      }
    }
    __syncwarp();
    // the allocating warp releases TMEM once both issuers and the epilogue are done
    asm volatile("bar.sync 1, 192;" ::: "memory");
    if (rows) {
      tc::fence_after();
      tc::tmem_dealloc(tmem, 512);
    }
    return;
  }

  // ------------------------------------------------------------ epilogue (warps 2..5)
  const int q = warp & 3;  // TMEM lane quadrant this warp may access
  int I = I0;
  int64_t rend = ta.toff[I + 1];
  int rb = 0, cb = 0, nseg = 0, ncol = 0;
  for (int64_t t = t0; t < t1; ++t) {
    const bool newI = (t == t0) || (t >= rend);
    while (t >= rend) rend = ta.toff[++I + 1];
    if (newI) ++nseg;
    const int J = tile_col(ta, I, t);
    if (J != ta.I0 + I) {  // the tile's column sums K_IJ^T x_I -> rows of block J
      mbar_wait(&colf[cb], (uint32_t)((ncol >> 1) & 1));
      tc::fence_after();
      long long G[kTcGroups];
#if TC_EXP == 1 || TC_EXP == 4
      for (int g = 0; g < kTcGroups; ++g) G[g] = 0;
#else
      level_groups(tmem + 256 + (uint32_t)(cb * 128) + ((uint32_t)(32 * q) << 16), G);
#endif
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&cole[cb]);
      red_groups(ta.yacc, ta.cs, (int64_t)J * kT + 32 * q + lane, G);
      cb ^= 1;
      ++ncol;
    }
    if (t + 1 == t1 || t + 1 >= rend) {  // the segment's row sums -> rows of block I
      mbar_wait(&rowf[rb], (uint32_t)(((nseg - 1) >> 1) & 1));
      tc::fence_after();
      long long G[kTcGroups];
      level_groups(tmem + (uint32_t)(rb * 128) + ((uint32_t)(32 * q) << 16), G);
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&rowe[rb]);
      red_groups(ta.yacc, ta.cs, (int64_t)(ta.I0 + I) * kT + 32 * q + lane, G);
      rb ^= 1;
    }
  }
  tc::fence_before();
  asm volatile("bar.sync 1, 192;" ::: "memory");
}

// x -> 16 digit slices with one exponent: F with max|x| < 2^F (from the per-CTA maxima
// parts), v = x 2^-(F+1), c_t = rint(128 v) digit by digit; xs is 16 rows x ldx bytes
__global__ void __launch_bounds__(256) slice_x_kernel(const double *__restrict__ x, int64_t n,
                                                      const double *__restrict__ parts, int nparts,
                                                      int8_t *__restrict__ xs, int64_t ldx, int *Fout,
                                                      const PcgState *st) {
  if (st && *(volatile const int32_t *)&st->done) return;
  __shared__ int sF;
  if (threadIdx.x < 32) {
    double m = 0.0;
    for (int k = threadIdx.x; k < nparts; k += 32) m = fmax(m, parts[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    int F = 0;
    if (m > 0.0) frexp(m, &F);  // m = f 2^F, f in [0.5, 1): |x| <= m < 2^F
    if (threadIdx.x == 0) {
      sF = F;
      if (blockIdx.x == 0) *Fout = F;
    }
  }
  __syncthreads();
  const double sc = ldexp(1.0, -(sF + 1));
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

// K (n x n, stride ld) -> the tile-major slice store: for upper-triangle tile t = (I, J)
// (plan order) and slice s, 16 KiB at ks + (8 t + s) 16 KiB holding [half h][row r][64 B]
// = the digits of K[128 I + r][128 J + 64 h + b] (zero past n): the shared-memory image of
// one ring slot before the SWIZZLE_64B the TMA applies.  eK: max |K| < 2^eK; flag[0] = 1
// if some entry is not exact.  Block: one tile; thread: 8 consecutive columns of a row per
// item, 8-byte stores.
__global__ void __launch_bounds__(256) slice_k_kernel(const double *__restrict__ K, int64_t rows, int64_t n,
                                                      int64_t ld, const int64_t *__restrict__ toff,
                                                      const int32_t *__restrict__ jt, int nb, int eK,
                                                      int8_t *__restrict__ ks, int *flag) {
  // K: this rank's rows (local block-row I = rows 128 I ..), all n columns
  const int64_t t = blockIdx.x;
  const int I = find_block_row(toff, nb, t);
  const int J = jt != nullptr ? jt[t] : I + (int)(t - toff[I]);
  const double sc = ldexp(1.0, -(eK + 1));
  bool bad = false;
#pragma unroll 1
  for (int it = threadIdx.x; it < 2 * kT * 8; it += blockDim.x) {
    const int h = it >> 10, r = (it >> 3) & (kT - 1), b8 = it & 7;
    const int64_t i = (int64_t)I * kT + r, j0 = (int64_t)J * kT + 64 * h + 8 * b8;
    unsigned long long w[kSK];
#pragma unroll
    for (int q = 0; q < kSK; ++q) w[q] = 0ull;
    if (i < rows) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (j0 + k >= n) break;
        double v = __dmul_rn(K[i * ld + j0 + k], sc);
#pragma unroll
        for (int q = 0; q < kSK; ++q) {
          v = __dmul_rn(v, 128.0);
          const double d = rint(v);
          v = __dsub_rn(v, d);
          w[q] |= (unsigned long long)(uint8_t)(int8_t)(int)d << (8 * k);
        }
        bad |= v != 0.0;
      }
    }
    // the SWIZZLE_64B image (16-byte chunk c of a 64-byte row r at chunk c ^ ((r >> 1) & 3)),
    // so a plain bulk copy lands the layout the MMA descriptors expect
    int8_t *dst = ks + ((t * kSK) * 2 * kT + h * kT + r) * 64 + 16 * ((b8 >> 1) ^ ((r >> 1) & 3)) + 8 * (b8 & 1);
#pragma unroll
    for (int q = 0; q < kSK; ++q)
      *reinterpret_cast<unsigned long long *>(dst + (int64_t)q * kSliceBytes) = w[q];
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
  int64_t n = 0, ldx = 0;
  int rank = 0, world = 1;
  int64_t rows = 0, cs = 0;   // this rank's K rows (n / W); yacc chunk per rank (one rank: ldx)
  int8_t *ks = nullptr, *xs = nullptr;
  int *dexp = nullptr;  // [0] eK, [1] F of the last sliced x, [2] exactness flag
  double *dmax = nullptr;
  long long *yacc = nullptr;  // [W][8][cs] exact level-group sums per row (zero between applies)
  CUtensorMap tmX;
  // the 128 x 128 tile plan for `grid` persistent CTAs (sharded: dist_tiles, jt per tile)
  int grid = 0, nb = 0, I0 = 0;
  int64_t T = 0;
  int64_t *toff = nullptr;
  int32_t *jt = nullptr;
};

void symv_tc_free(SymvTc *&p) {
  if (!p) return;
  cudaFree(p->ks);
  cudaFree(p->xs);
  cudaFree(p->dexp);
  cudaFree(p->dmax);
  cudaFree(p->yacc);
  cudaFree(p->toff);
  cudaFree(p->jt);
  delete p;
  p = nullptr;
}

void symv_tc_init() {
  cudaFuncSetAttribute(symv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem);
}

long long *symv_tc_groups(SymvTc *p, int64_t *cs) {
  if (cs) *cs = p->cs;
  return p->yacc;
}
const int *symv_tc_exponents(const SymvTc *p) { return p->dexp; }

namespace {
// One rank: block-row I takes tiles J = I .. nb - 1 (row-major order).  Sharded (rank r of
// W): the local block-rows' tile lists of dist_tiles (symv.cu; every pair of symmetric
// entries once over all ranks, n^2 / (2 W) entries per rank) at 128 x 128.  CTA b takes the
// range [T b / G, T (b + 1) / G), G = min(SMs, T).
cudaError_t tc_plan(SymvTc *p, int sms) {
  std::vector<int64_t> toff;
  std::vector<int32_t> jt;
  if (p->world == 1) {
    const int nb = (int)((p->n + kT - 1) / kT);
    toff.assign(nb + 1, 0);
    for (int I = 0; I < nb; ++I) toff[I + 1] = toff[I] + (nb - I);
    p->I0 = 0;
  } else {
    std::vector<int32_t> lo, hi;
    if (!dist_tiles(p->n, kT, kT, p->rank, p->world, toff, jt, lo, hi)) return cudaErrorInvalidValue;
    p->I0 = (int)(p->rank * (p->rows / kT));
  }
  const int nb = (int)toff.size() - 1;
  cudaError_t e;
  if ((e = cudaMalloc(&p->toff, toff.size() * sizeof(int64_t))) != cudaSuccess) return e;
  cudaMemcpy(p->toff, toff.data(), toff.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
  if (!jt.empty()) {
    if ((e = cudaMalloc(&p->jt, jt.size() * sizeof(int32_t))) != cudaSuccess) return e;
    cudaMemcpy(p->jt, jt.data(), jt.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  }
  p->nb = nb;
  p->T = toff[nb];
  p->grid = (int)std::max<int64_t>(1, std::min<int64_t>(sms, p->T));
  return cudaSuccess;
}
}  // namespace

// Slice this rank's rows of the (bitwise symmetric) K into the int8 form of its tiles; false
// if some entry is not exactly representable (the fp64 symmetric kernel stays in use then;
// sharded callers agree on the outcome across ranks).  rowmax: the maxima of all n rows.
bool symv_tc_prepare(SymvTc *&p, const double *K, int64_t n, int64_t ld, const double *rowmax, cudaStream_t s,
                     int rank, int world) {
  if (n < 1 || n > (1 << 18)) return false;  // |D_st| <= 64 * 64 * n < 2^31 in the int32 accumulators
  if (world > 1 && (n % world != 0 || (n / world) % (2 * kT) != 0)) return false;  // the dist_tiles shards
  PFN_enc enc = get_enc();
  if (!enc) return false;
  const int64_t ldx = (n + kT - 1) / kT * kT;
  if (!p || p->n != n || p->rank != rank || p->world != world) {
    symv_tc_free(p);
    p = new SymvTc();
    p->n = n;
    p->ldx = ldx;
    p->rank = rank;
    p->world = world;
    p->rows = n / world;
    p->cs = world == 1 ? ldx : n / world;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t ygroups = (size_t)kTcGroups * (world == 1 ? ldx : n);
    if (tc_plan(p, sms) != cudaSuccess || cudaMalloc(&p->ks, (size_t)p->T * kSK * kSliceBytes) != cudaSuccess ||
        cudaMalloc(&p->xs, (size_t)kSX * p->ldx) != cudaSuccess || cudaMalloc(&p->dexp, 4 * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&p->dmax, sizeof(double)) != cudaSuccess ||
        cudaMalloc(&p->yacc, ygroups * sizeof(long long)) != cudaSuccess) {
      cudaGetLastError();
      symv_tc_free(p);
      return false;
    }
    cudaMemset(p->xs, 0, (size_t)kSX * p->ldx);
    cudaMemset(p->yacc, 0, ygroups * sizeof(long long));
    // x slices: [16][ldx] bytes, boxes of 128 columns x 16 slices
    cuuint64_t dx[2] = {(cuuint64_t)p->ldx, (cuuint64_t)kSX}, sx[1] = {(cuuint64_t)p->ldx};
    cuuint32_t bx[2] = {kT, kSX}, es[2] = {1, 1};
    if (enc(&p->tmX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, p->xs, dx, sx, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
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
  slice_k_kernel<<<(unsigned)p->T, 256, 0, s>>>(K, p->rows, n, ld, p->toff, p->jt, p->nb, eK, p->ks, p->dexp + 2);
  int flag = 1;
  cudaMemcpyAsync(&flag, p->dexp + 2, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return false;
  return flag == 0;
}

// the tile pass of the exact tensor-core apply: x's slices, then the tiles adding every
// row's exact level groups to yacc; a's tensor-core fields point the finalize (launched by
// the caller: symv.cu on one rank, pcg_dist.cu after the reduce-scatter) at them
void launch_symv_tc(SymvTc *p, SymvArgs &a, cudaStream_t s) {
  slice_x_kernel<<<(unsigned)std::min<int64_t>((p->n + 255) / 256, 296), 256, 0, s>>>(
      a.x, p->n, a.xparts, a.nxparts, p->xs, p->ldx, p->dexp + 1, a.state);
  TcArgs ta{};
  ta.state = a.state;
  ta.n = p->n;
  ta.toff = p->toff;
  ta.jt = p->jt;
  ta.I0 = p->I0;
  ta.T = p->T;
  ta.nb = p->nb;
  ta.ks = p->ks;
  ta.yacc = p->yacc;
  ta.cs = p->cs;
  symv_tc_kernel<<<p->grid, kTcThreads, kTcSmem, s>>>(p->tmX, ta);
  a.yacc = p->yacc;
  a.ldy = p->cs;
  a.tc_exp = p->dexp;
}

}  // namespace laker
