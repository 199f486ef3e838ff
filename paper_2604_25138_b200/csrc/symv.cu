// Symmetric streaming Dot2 GEMV: the per-iteration
// K.p and P.r products of the PCG (Alg. 1 l.16-21; rows a4/a7/a9)
// reading only the block upper triangle of a bitwise-symmetric matrix, i.e.
// half the HBM bytes of gemv.cu.  K is symmetric by construction (P:141-147,
// K_ij = exp(scale <e_i, e_j>) with q = k, reading R2) and so is
// P = Sigma*^{-1/2} (formed bitwise symmetric, B4); the
// host verifies bitwise symmetry on the device before selecting this path
// (symv_check_kernel) and otherwise uses gemv.cu.
//
// Blocking: block-rows of 128 rows, tiles of 128 rows x 64 columns (64 KiB),
// block-row I streams the tiles with column index jt >= 2I.  The two tiles
// over the diagonal block contribute to rows only; every other tile (I, jt)
// contributes K_IJ x_J to its rows and K_IJ^T x_I to the rows of column
// block jt (K_ji = K_ij).  With tiles linearised row-major over the upper
// triangle, persistent CTA b owns the contiguous range [T b/G, T (b+1)/G).
//
// Roles (one CTA per SM): a producer warp loads each tile with one 2-D TMA
// (cp.async.bulk.tensor, OOB rows/columns zero-filled -> ragged n) plus the
// 64-entry slice of x with a 1-D bulk copy into a 3-stage mbarrier ring;
// 16 consumer warps (warp w: rows 8w .. 8w+7, columns 2 lane and 2 lane + 1) keep
// one Dot2 pair per row for the whole block-row segment and one Dot2 pair per
// column per tile; two reducer warps sum the 16 warps' column pairs of each
// tile in a fixed order and store one pair per column to `colpart[I][j]`.  At
// the end of a block-row segment each consumer warp reduces its 8 row pairs
// over its 32 lanes and stores them to `rowpart`.  (64-column tiles: 16
// elements per thread per tile amortise the per-tile barrier / offset / hand-off
// instructions, which at 32 columns were half of the issued instructions.)
//
// symv_finalize_kernel then forms, for every row i of block-row J,
//   y_i = RN( sum_{I<J} colpart[I][i] + sum_{segments} rowpart + lambda x_i )
// in a fixed order, plus the Dot2 pair x_i y_i per CTA, and the last CTA runs
// the PCG scalar epilogue (delta / beta / store), exactly as gemv.cu.  Every
// partial is an unrounded Dot2 pair combined by TwoSum, so y_i is the
// correctly rounded row sum in practice and bitwise equal to gemv.cu and to
// the oracle's sequential Dot2 (tests/test_gpu_symv.py).
#include <cuda.h>

#include <vector>

#include "laker_internal.h"
#include "tma.cuh"
#include "tri.cuh"

namespace laker {
namespace {

constexpr int kSR = 128;                 // rows per block-row
constexpr int kSC = 64;                  // columns per tile
constexpr int kCPT = kSC / 32;           // columns per consumer thread
constexpr int kTPD = kSR / kSC;          // tiles per diagonal block
constexpr int kRPT = 8;                  // rows per consumer thread
constexpr int kCons = 512;               // consumer threads
constexpr int kConsWarps = kCons / 32;   // 16
constexpr int kRedWarps = 2;             // warps 16, 17: column reducers (19 warps -> 96 registers)
constexpr int kRedWarp0 = kConsWarps;
constexpr int kProdWarp = kConsWarps + kRedWarps;  // warp 18: TMA producer
constexpr int kSymThreads = (kConsWarps + kRedWarps + 1) * 32;
constexpr int kSStages = 3;
constexpr uint32_t kTileBytes = kSR * kSC * 8;   // 65536
constexpr uint32_t kXBytes = kSC * 8;            // 512
constexpr size_t kStageBytes = kTileBytes + kXBytes;  // tile + x slice (keeps 512 B alignment)
constexpr int kRedBufs = 2;
constexpr size_t kRedBytes = kRedBufs * kConsWarps * kSC * sizeof(dd_pair);  // [2][16 warps][64 cols]
constexpr size_t kSymSmem = kSStages * kStageBytes + kRedBytes + 16 * sizeof(uint64_t);  // + static 1 KiB <= 227 KiB
constexpr int kFinThreads = 512;
constexpr int kXParts = 32;              // CTAs of absmax_parts_kernel

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *tm, int32_t c0, int32_t c1,
                                            uint64_t *bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *tm) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tm)) : "memory");
}

// ROWOFF: the row accumulators carry offsets (at most kMaxOffTiles products each, n <=
// 16384); otherwise they are plain Dot2 pairs (the offset-sum error grows with the
// products per accumulator) and only the 8-product column chains use offsets
constexpr int kMaxOffTiles = 512;  // products per row accumulator: nct kCPT
template <bool ROWOFF>
__global__ void __launch_bounds__(kSymThreads, 1)
    symv_dot2_kernel(const __grid_constant__ CUtensorMap tm, const SymvArgs a) {
  if (a.state != nullptr && *(volatile int32_t *)&a.state->done) return;
  extern __shared__ __align__(128) unsigned char smem[];  // 128 B suffices for unswizzled TMA
  dd_pair *red = reinterpret_cast<dd_pair *>(smem + kSStages * kStageBytes);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kSStages * kStageBytes + kRedBytes);
  uint64_t *empty = full + kSStages;
  uint64_t *rfull = empty + kSStages;  // [kRedBufs]
  uint64_t *rempty = rfull + kRedBufs;  // [kRedBufs]
  __shared__ int s_I0;
  __shared__ double s_xr[kConsWarps][kRPT];  // x at the consumer warp's 8 rows (warp-private)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t t0 = a.T * blockIdx.x / gridDim.x;
  const int64_t t1 = a.T * (blockIdx.x + 1) / gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < kSStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsWarps);
    }
    for (int b = 0; b < kRedBufs; ++b) {
      mbar_init(&rfull[b], kConsWarps);
      mbar_init(&rempty[b], kRedWarps);
    }
    fence_mbar_init();
    s_I0 = find_block_row(a.toff, a.nb, t0);
  }
  if (warp == kProdWarp && lane == 0) prefetch_tmap(&tm);
  __syncthreads();
  if (t0 >= t1) return;
  const int I0 = s_I0;

  if (warp == kProdWarp) {
    // ------------------------------------------------ TMA producer (one lane)
    if (lane == 0) {
      const uint64_t pol_a = a.evict_first ? l2_policy_evict_first() : l2_policy_evict_last();
      const uint64_t pol_x = l2_policy_evict_last();
      int I = I0;
      int64_t rbeg = a.toff[I], rend = a.toff[I + 1];
      int slot = 0;
      uint32_t ph = 0;
      bool first = true;
      for (int64_t t = t0; t < t1; ++t) {
        while (t >= rend) {
          rbeg = rend;
          rend = a.toff[++I + 1];
        }
        const int jt = a.jt_of ? a.jt_of[t] : kTPD * I + (int)(t - rbeg);
        if (!first) mbar_wait(&empty[slot], ph ^ 1u);
        unsigned char *st = smem + slot * kStageBytes;
        mbar_arrive_expect_tx(&full[slot], kTileBytes + kXBytes);
        tma_load_2d(st, &tm, jt * kSC, I * kSR, &full[slot], pol_a);
        bulk_g2s(st + kTileBytes, a.x + (int64_t)jt * kSC, kXBytes, &full[slot], pol_x);
        if (++slot == kSStages) {
          slot = 0;
          ph ^= 1u;
          first = false;
        }
      }
    }
    return;
  }

  if (warp >= kRedWarp0) {
    // ------------------------------------------------ column reducers: warp r owns columns
    // 32h + 16r .. 32h + 16r + 15 (h = 0, 1); lane l sums the pairs of warps 8q .. 8q+7
    // (q = l / 16) of its column in warp order, then the two q-partials are combined by
    // one shuffle.
    const int r = warp - kRedWarp0, q = lane >> 4;
    int I = I0;
    int64_t rbeg = a.toff[I], rend = a.toff[I + 1];
    int b = 0;
    uint32_t rph = 0;
    for (int64_t t = t0; t < t1; ++t) {
      while (t >= rend) {
        rbeg = rend;
        rend = a.toff[++I + 1];
      }
      const int jt = a.jt_of ? a.jt_of[t] : kTPD * I + (int)(t - rbeg);
      if (jt / kTPD == I + a.I0) continue;  // diagonal-block tile: rows only
      mbar_wait(&rfull[b], rph);
#pragma unroll
      for (int h = 0; h < kCPT; ++h) {
        const dd_pair *rb = red + b * kConsWarps * kSC + 8 * q * kSC + 32 * h + 16 * r + (lane & 15);
        dd_pair w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) w[k] = rb[k * kSC];
        if (h == kCPT - 1) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&rempty[b]);
        }
        pair_add(w[0], w[1]);
        pair_add(w[2], w[3]);
        pair_add(w[4], w[5]);
        pair_add(w[6], w[7]);
        pair_add(w[0], w[2]);
        pair_add(w[4], w[6]);
        pair_add(w[0], w[4]);
        dd_pair v0 = w[0];
        dd_pair o;
        o.s = __shfl_down_sync(0xffffffffu, v0.s, 16);
        o.c = __shfl_down_sync(0xffffffffu, v0.c, 16);
        if (q == 0) {
          pair_add(v0, o);
          a.colpart[(int64_t)I * a.ldcp + (int64_t)jt * kSC + 32 * h + 16 * r + lane] = v0;
        }
      }
      if (++b == kRedBufs) {
        b = 0;
        rph ^= 1u;
      }
    }
    return;
  }

  // -------------------------------------------------- consumer warps
  // Every accumulator carries a power-of-two offset C >= 2 sum |a_ij x_j| of what it will
  // add (row: <= nct kCPT products of |a| <= rowmax_i, |x| <= xmax; column: 8 products), so
  // each step is TwoProd + Fast2Sum (dot2_step_off, 7 fp64 ops instead of 10); the offset
  // is removed exactly before the pair leaves the thread.
  const int c = lane;  // column within the tile; rows 8 warp .. 8 warp + 7
  dd_pair acc[kRPT];
  double *xr = s_xr[warp];
  double xm = 0.0;
  for (int k = 0; k < a.nxparts; ++k) xm = fmax(xm, a.xparts[k]);
  const double mrow = 2.0 * (double)a.nct * kCPT;
  int curI = -1;
  int64_t rbeg = 0, rend = 0;
  int slot = 0, b = 0;
  uint32_t ph = 0, rph = 0;
  bool rfirst = true;

  auto flush_rows = [&](int I) {
    // reduce the 8 row pairs over the warp's 32 columns; lane k stores row k
    const int s = blockIdx.x - a.segfirst[I];
    dd_pair *dst = a.rowpart + ((int64_t)I * a.maxseg + s) * kSR + warp * kRPT;
    const double *rmr = a.rowmax + (int64_t)(I + a.I0) * kSR + warp * kRPT;
#pragma unroll
    for (int k = 0; k < kRPT; ++k) {
      dd_pair v = acc[k];
      if (ROWOFF) v.s = __dsub_rn(v.s, pow2_above(rmr[k] * xm * mrow));  // exact: v.s in [C/2, 3C/2]
      v = warp_reduce_pair(v);
      v.s = __shfl_sync(0xffffffffu, v.s, 0);
      v.c = __shfl_sync(0xffffffffu, v.c, 0);
      if (lane == k) dst[k] = v;
    }
  };

  for (int64_t t = t0; t < t1; ++t) {
    if (t >= rend) {
      if (curI >= 0) flush_rows(curI);
      curI = (curI < 0) ? I0 : curI + 1;
      while (t >= a.toff[curI + 1]) ++curI;
      rbeg = a.toff[curI];
      rend = a.toff[curI + 1];
      __syncwarp();
      if (lane < kRPT) xr[lane] = a.x[(int64_t)(curI + a.I0) * kSR + warp * kRPT + lane];
      __syncwarp();
      const double *rmr = a.rowmax + (int64_t)(curI + a.I0) * kSR + warp * kRPT;
#pragma unroll
      for (int k = 0; k < kRPT; ++k) acc[k] = dd_pair{ROWOFF ? pow2_above(rmr[k] * xm * mrow) : 0.0, 0.0};
    }
    const int I = curI;
    const int jt = a.jt_of ? a.jt_of[t] : kTPD * I + (int)(t - rbeg);
    const bool diag = jt / kTPD == I + a.I0;
    // column offsets from the column maxima (L2-resident; loaded before the data wait)
    static_assert(kCPT == 2, "two column halves per thread");
    // this thread's columns are 2c and 2c + 1 (16-byte loads of the tile, x and maxima)
    const double2 cm = diag ? double2{0.0, 0.0} : __ldg(reinterpret_cast<const double2 *>(a.rowmax + (int64_t)jt * kSC) + c);
    if (!diag && !rfirst) mbar_wait(&rempty[b], rph ^ 1u);  // this tile's column-pair buffer is free
    mbar_wait(&full[slot], ph);
    const double *tile = reinterpret_cast<const double *>(smem + slot * kStageBytes);
    if (diag) {
#pragma unroll
      for (int h = 0; h < kCPT; ++h) {
        const double xc = tile[kSR * kSC + 2 * c + h];
        const double *tp = tile + warp * kRPT * kSC + 2 * c + h;
#pragma unroll
        for (int k = 0; k < kRPT; ++k) {
          if (ROWOFF)
            dot2_step_off(acc[k], tp[k * kSC], xc);
          else
            dot2_step(acc[k], tp[k * kSC], xc);
        }
      }
    } else {
      // k-major over the thread's two columns: per row k the products with x_{2c} and
      // x_{2c+1} (in that order, as the diagonal tiles do), and two independent column chains
      const double2 xcv = reinterpret_cast<const double2 *>(tile + kSR * kSC)[c];
      const double xc0 = xcv.x, xc1 = xcv.y;
      const double *tp = tile + warp * kRPT * kSC + 2 * c;
      const double ccol0 = pow2_above(cm.x * xm * 16.0), ccol1 = pow2_above(cm.y * xm * 16.0);
      dd_pair c0 = {ccol0, 0.0}, c1 = {ccol1, 0.0};
#pragma unroll
      for (int k = 0; k < kRPT; ++k) {
        const double2 vv = *reinterpret_cast<const double2 *>(tp + k * kSC);
        const double v0 = vv.x, v1 = vv.y;
        if (ROWOFF) {
          dot2_step_off(acc[k], v0, xc0);
          dot2_step_off(acc[k], v1, xc1);
        } else {
          dot2_step(acc[k], v0, xc0);
          dot2_step(acc[k], v1, xc1);
        }
        dot2_step_off(c0, v0, xr[k]);
        dot2_step_off(c1, v1, xr[k]);
      }
      c0.s = __dsub_rn(c0.s, ccol0);
      c1.s = __dsub_rn(c1.s, ccol1);
      red[b * kConsWarps * kSC + warp * kSC + 2 * c] = c0;
      red[b * kConsWarps * kSC + warp * kSC + 2 * c + 1] = c1;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (++slot == kSStages) {
      slot = 0;
      ph ^= 1u;
    }
    if (!diag) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&rfull[b]);
      if (++b == kRedBufs) {
        b = 0;
        rph ^= 1u;
        rfirst = false;
      }
    }
  }
  if (curI >= 0) flush_rows(curI);
}

// y_i = RN(sum of the partial pairs of row i in a fixed order + lambda x_i); Dot2 x.y
// per CTA; the last CTA reduces the CTA pairs in CTA order and runs the epilogue.
// 32-row groups grid-strided over a persistent grid (coalesced partial loads).
__device__ __forceinline__ dd_pair ldcg_pair(const dd_pair *p) {
  const double2 v = __ldcg(reinterpret_cast<const double2 *>(p));  // pairs are 16-byte aligned
  return dd_pair{v.x, v.y};
}

template <int BR, bool TCP>
__global__ void __launch_bounds__(kFinThreads) symv_finalize_kernel(const SymvArgs a) {
  if (a.state != nullptr && *(volatile int32_t *)&a.state->done) return;
  __shared__ dd_pair sred[kFinThreads / 32];
  __shared__ dd_pair spart[kFinThreads / 32][32];
  __shared__ int s_last;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kW = kFinThreads / 32;  // 16 warps
  static_assert(BR % 32 == 0, "a 32-row group lies in one block-row");
  dd_pair dotp = {0.0, 0.0};
  if constexpr (TCP) {
    // the exact tensor-core apply (symv_tc.cu): row i's 8 exact level groups -> its pair
    // (zeroing them for the next apply); one 32-row group per warp, lane = row
    const int escale = a.tc_exp[0] + a.tc_exp[1] + 2 - 14;
    for (int64_t g = (int64_t)blockIdx.x * kW + warp; g * 32 < a.n; g += (int64_t)gridDim.x * kW) {
      const int64_t i = g * 32 + lane;
      if (i >= a.n) continue;
      long long G[kTcGroups];
#pragma unroll
      for (int q = 0; q < kTcGroups; ++q) {
        G[q] = __ldcg(&a.yacc[q * a.ldy + i]);
        a.yacc[q * a.ldy + i] = 0;
      }
      dd_pair t = tc_groups_to_pair(G, escale);
      const double xi = a.x[i];
      if (a.lambda != 0.0) dot2_step(t, a.lambda, xi);
      const double yv = pair_value(t);
      a.y[i] = yv;
      dot2_step(dotp, xi, yv);
    }
  } else {
  // one 32-row group per iteration: lane = row, warp w sums the column partials I = w
  // (mod 16) of the block-rows above (each load: 32 consecutive 16-byte pairs) and the
  // row segments q = w (mod 16); warp 0 then combines the 16 warp sums in warp order
  for (int64_t g = blockIdx.x; g * 32 < a.n; g += gridDim.x) {
    const int64_t i = g * 32 + lane;
    const bool valid = i < a.n;
    const int J = (int)((g * 32) / BR), r = (int)(i % BR);
    const double xi = (warp == 0 && valid) ? a.x[i] : 0.0;  // issued before the partial loads
    dd_pair v = {0.0, 0.0};
    if (valid) {
      int I = warp;
      for (; I + 3 * kW < J; I += 4 * kW) {
        dd_pair o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) o[q] = ldcg_pair(&a.colpart[(int64_t)(I + q * kW) * a.ldcp + i]);
#pragma unroll
        for (int q = 0; q < 4; ++q) pair_add(v, o[q]);
      }
      for (; I < J; I += kW) pair_add(v, ldcg_pair(&a.colpart[(int64_t)I * a.ldcp + i]));
      const int ns = a.nseg[J];
      for (int q = warp; q < ns; q += kW) pair_add(v, ldcg_pair(a.rowpart + ((int64_t)J * a.maxseg + q) * BR + r));
    }
    spart[warp][lane] = v;
    __syncthreads();
    if (warp == 0) {
      dd_pair t = spart[0][lane];
#pragma unroll
      for (int w = 1; w < kW; ++w) pair_add(t, spart[w][lane]);
      if (valid) {
        if (a.lambda != 0.0) dot2_step(t, a.lambda, xi);
        const double yv = pair_value(t);
        a.y[i] = yv;
        dot2_step(dotp, xi, yv);
      }
    }
    __syncthreads();
  }
  }
  dotp = warp_reduce_pair(dotp);
  if (lane == 0) sred[warp] = dotp;
  __syncthreads();
  if (a.upd.on) {
    // ---- the PCG update step fused in (all CTAs co-resident, grid <= symv_fused_grid)
    if (tid == 0) {
      dd_pair t = sred[0];
      for (int w = 1; w < kFinThreads / 32; ++w) pair_add(t, sred[w]);
      a.partials[blockIdx.x] = t;
    }
    grid_barrier(a.upd.bar, a.upd.bar + 1, 1, kFinThreads);
    __shared__ double s_delta;
    __shared__ int s_ok;
    PcgState *st = a.state;
    if (warp == 0) {  // p.q over the CTA pairs in CTA order: the same value in every CTA
      dd_pair v = {0.0, 0.0};
      for (int b = lane; b < (int)gridDim.x; b += 32) pair_add(v, ldcg_pair(&a.partials[b]));
      v = warp_reduce_pair(v);
      if (lane == 0) {
        const double pq = pair_value(v);
        s_ok = pq > 0.0;
        s_delta = s_ok ? __ddiv_rn(st->rho, pq) : 0.0;
      }
    }
    __syncthreads();
    const bool ok = s_ok != 0;
    const double delta = s_delta;
    __syncthreads();
    if (blockIdx.x == 0 && tid == 0) {
      if (!ok) {
        st->term = LAKER_TERM_BREAKDOWN;
        st->done = 1;
      } else {
        pcg_set_delta(st, delta);
      }
    }
    if (!ok) return;
    const FusedUpdate &u = a.upd;
    dd_pair v0 = {0.0, 0.0}, v1 = {0.0, 0.0};
    for (int64_t g = blockIdx.x + (int64_t)warp * gridDim.x; g * 32 < a.n; g += (int64_t)kW * gridDim.x) {
      const int64_t i = g * 32 + lane;
      if (i >= a.n) continue;
      u.alpha[i] = __fma_rn(delta, u.p[i], u.alpha[i]);
      const double ri = __fma_rn(-delta, __ldcg(&a.y[i]), u.r[i]);
      u.r[i] = ri;
      dot2_step(v0, ri, ri);
      if (u.pk == LAKER_PRECOND_JACOBI) {
        const double th = __dmul_rn(u.dvec[i], ri);
        u.theta[i] = th;
        dot2_step(v1, ri, th);
      }
    }
    v0 = warp_reduce_pair(v0);
    v1 = warp_reduce_pair(v1);
    __shared__ dd_pair sr2[kFinThreads / 32][2];
    if (lane == 0) {
      sr2[warp][0] = v0;
      sr2[warp][1] = v1;
    }
    __syncthreads();
    if (tid == 0) {
      dd_pair t0 = sr2[0][0], t1 = sr2[0][1];
      for (int w = 1; w < kW; ++w) {
        pair_add(t0, sr2[w][0]);
        pair_add(t1, sr2[w][1]);
      }
      u.partials2[2 * blockIdx.x] = t0;
      u.partials2[2 * blockIdx.x + 1] = t1;
      __threadfence();
      s_last = (atomicAdd(u.counter2, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last || warp != 0) return;
    __threadfence();
    dd_pair t0 = {0.0, 0.0}, t1 = {0.0, 0.0};
    for (int b = lane; b < (int)gridDim.x; b += 32) {
      pair_add(t0, ldcg_pair(&u.partials2[2 * b]));
      pair_add(t1, ldcg_pair(&u.partials2[2 * b + 1]));
    }
    t0 = warp_reduce_pair(t0);
    t1 = warp_reduce_pair(t1);
    if (lane != 0) return;
    *u.counter2 = 0u;
    // the termination / beta epilogue of pcg_update_kernel
    const double rr = pair_value(t0);
    const double rel = __ddiv_rn(__dsqrt_rn(rr), st->ynorm);
    const int it = st->iters + 1;
    st->iters = it;
    st->rel = rel;
    if (u.hist) u.hist[it - 1] = rel;
    if (rel <= st->tol) {
      st->term = LAKER_TERM_RESIDUAL_TOL;
      st->done = 1;
      return;
    }
    if (u.pk != LAKER_PRECOND_EXTERNAL_DENSE && u.pk != LAKER_PRECOND_LEARNED) {
      const double rho_new = (u.pk == LAKER_PRECOND_NONE) ? rr : pair_value(t1);
      if (!(rho_new > 0.0)) {
        st->term = LAKER_TERM_INDEFINITE;
        st->done = 1;
        return;
      }
      pcg_set_beta(st, __ddiv_rn(rho_new, st->rho));
      st->rho = rho_new;
      if (it >= st->max_iters) {
        st->term = LAKER_TERM_MAX_ITERS;
        st->done = 1;
      }
    }
    return;
  }
  if (tid == 0) {
    dd_pair t = sred[0];
    for (int w = 1; w < kFinThreads / 32; ++w) pair_add(t, sred[w]);
    a.partials[blockIdx.x] = t;
    __threadfence();
    s_last = (atomicAdd(a.counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  // last CTA: one CTA pair per thread, then a fixed-shape block reduction
  __threadfence();
  dd_pair v = tid < (int)gridDim.x ? ldcg_pair(&a.partials[tid]) : dd_pair{0.0, 0.0};
  for (int b = tid + kFinThreads; b < (int)gridDim.x; b += kFinThreads) pair_add(v, ldcg_pair(&a.partials[b]));
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    dd_pair o;
    o.s = __shfl_down_sync(0xffffffffu, v.s, off);
    o.c = __shfl_down_sync(0xffffffffu, v.c, off);
    if ((lane & (2 * off - 1)) == 0) pair_add(v, o);
  }
  __syncthreads();
  if (lane == 0) sred[warp] = v;
  __syncthreads();
  if (tid != 0) return;
  v = sred[0];
  for (int w = 1; w < kFinThreads / 32; ++w) pair_add(v, sred[w]);
  *a.counter = 0u;
  PcgState *st = a.state;
  const double dv = pair_value(v);
  switch (a.epi) {
    case kEpiDelta:
      if (!(dv > 0.0)) {
        st->term = LAKER_TERM_BREAKDOWN;
        st->done = 1;
      } else {
        pcg_set_delta(st, __ddiv_rn(st->rho, dv));
      }
      break;
    case kEpiBeta:
      if (!(dv > 0.0)) {
        st->term = LAKER_TERM_INDEFINITE;
        st->done = 1;
      } else {
        pcg_set_beta(st, __ddiv_rn(dv, st->rho));
        st->rho = dv;
      }
      break;
    case kEpiStoreDot:
      if (a.dot_out) *a.dot_out = dv;
      break;
    case kEpiStorePair:
      if (a.pair_out) *a.pair_out = v;
      break;
    default:
      break;
  }
}

// Row-sharded finalize (tri_plan_dist): for every row i < n the unrounded pair of this
// rank's partials -- the column partials of the local block-rows [cr_lo, cr_hi) of i's
// column tile and, for the rank's own rows, the row segments -- summed in the order of
// symv_finalize_kernel (warp w: block-rows cr_lo + w (mod 16), then segments w (mod 16);
// warps combined in order), so at W = 1 the pair is the one that kernel rounds.
template <int BR, int TC>
__global__ void __launch_bounds__(kFinThreads) tri_finalize_dist_kernel(const SymvArgs a) {
  if (a.state != nullptr && *(volatile int32_t *)&a.state->done) return;
  __shared__ dd_pair spart[kFinThreads / 32][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kW = kFinThreads / 32;
  static_assert(BR % 32 == 0 && TC % 32 == 0, "a 32-row group lies in one block-row and one column tile");
  for (int64_t g = blockIdx.x; g * 32 < a.n; g += gridDim.x) {
    const int64_t i = g * 32 + lane;
    const bool valid = i < a.n;
    const int jt = (int)((g * 32) / TC);
    dd_pair v = {0.0, 0.0};
    if (valid) {
      const int hi = a.cr_hi[jt];
      int I = a.cr_lo[jt] + warp;
      for (; I + 3 * kW < hi; I += 4 * kW) {
        dd_pair o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) o[q] = ldcg_pair(&a.colpart[(int64_t)(I + q * kW) * a.ldcp + i]);
#pragma unroll
        for (int q = 0; q < 4; ++q) pair_add(v, o[q]);
      }
      for (; I < hi; I += kW) pair_add(v, ldcg_pair(&a.colpart[(int64_t)I * a.ldcp + i]));
      if (i >= a.own0 && i < a.own1) {
        const int J = (int)((i - a.own0) / BR), r = (int)((i - a.own0) % BR);
        const int ns = a.nseg[J];
        for (int q = warp; q < ns; q += kW) pair_add(v, ldcg_pair(a.rowpart + ((int64_t)J * a.maxseg + q) * BR + r));
      }
    }
    spart[warp][lane] = v;
    __syncthreads();
    if (warp == 0 && valid) {
      dd_pair t = spart[0][lane];
#pragma unroll
      for (int w = 1; w < kW; ++w) pair_add(t, spart[w][lane]);
      a.ypair[i] = t;
    }
    __syncthreads();
  }
}

// rm[i] = max_j |A_ij| over the `rows` rows of A (n columns; one warp per row)
__global__ void rowmax_kernel(const double *__restrict__ A, int64_t rows, int64_t n, int64_t ld,
                              double *__restrict__ rm) {
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= rows) return;
  double m = 0.0;
  for (int64_t j = lane; j < n; j += 32) m = fmax(m, fabs(A[i * ld + j]));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  if (lane == 0) rm[i] = m;
}

// parts[b] = max |x_i| over CTA b's grid-stride share
__global__ void __launch_bounds__(256) absmax_parts_kernel(const double *__restrict__ x, int64_t n, double *parts,
                                                           const PcgState *state) {
  if (state != nullptr && *(volatile const int32_t *)&state->done) return;
  __shared__ double sm[8];
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
    m = fmax(m, fabs(x[i]));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) m = fmax(m, sm[w]);
    parts[blockIdx.x] = m;
  }
}

// flag[0] = 1 if A (n x n, row stride ld) is not bitwise symmetric
__global__ void symv_check_kernel(const double *__restrict__ A, int64_t n, int64_t ld, int *flag) {
  __shared__ double tI[32][33];
  __shared__ double tJ[32][33];
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (bj < bi) return;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = (int64_t)bi * 32 + r, j = (int64_t)bj * 32 + tx;
    tI[r][tx] = (i < n && j < n) ? A[i * ld + j] : 0.0;
    const int64_t i2 = (int64_t)bj * 32 + r, j2 = (int64_t)bi * 32 + tx;
    tJ[r][tx] = (i2 < n && j2 < n) ? A[i2 * ld + j2] : 0.0;
  }
  __syncthreads();
  bool bad = false;
  for (int r = ty; r < 32; r += 8)
    bad |= __double_as_longlong(tI[r][tx]) != __double_as_longlong(tJ[tx][r]);
  if (__syncthreads_or(bad) && tx == 0 && ty == 0) atomicExch(flag, 1);
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                     const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

}  // namespace

struct SymvPlan {
  int64_t n = 0, ld = 0, T = 0, ldcp = 0;
  int nb = 0, nct = 0, maxseg = 0, grid = 0, fin_grid = 0, br = 0, tc = 0;
  int rank = 0, world = 1;  // tri_plan_dist: nb local block-rows starting at global I0
  bool dist = false;        // built by tri_plan_dist (also at world = 1: the sharded pipeline)
  int32_t I0 = 0;
  int32_t *jt_of = nullptr, *cr_lo = nullptr, *cr_hi = nullptr;
  int64_t *toff = nullptr;
  int32_t *segfirst = nullptr, *nseg = nullptr;
  dd_pair *colpart = nullptr, *rowpart = nullptr;
  double *rowmax[2] = {nullptr, nullptr};  // symv: per-row max |A_ij| of K / P, zero-padded
  double *xparts = nullptr;  // [kXParts] when the caller supplies none
  CUtensorMap tm[2];
  const void *tm_base[2] = {nullptr, nullptr};
};

size_t symv_smem_bytes() { return kSymSmem; }

// CTAs of symv_finalize_kernel<kSR, *> guaranteed co-resident (the fused update's grid barrier)
int fused_fin_grid() {
  static int g = 0;
  if (g == 0) {
    int per = 0, sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int per2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, symv_finalize_kernel<kSR, false>, kFinThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, symv_finalize_kernel<kSR, true>, kFinThreads, 0);
    g = std::max(1, std::min(per, per2)) * sms;
  }
  return g;
}

void symv_init() {
  cudaFuncSetAttribute(symv_dot2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSymSmem);
  cudaFuncSetAttribute(symv_dot2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSymSmem);
}

void symv_free(SymvPlan *&p) {
  if (!p) return;
  cudaFree(p->toff);
  cudaFree(p->jt_of);
  cudaFree(p->cr_lo);
  cudaFree(p->cr_hi);
  cudaFree(p->segfirst);
  cudaFree(p->nseg);
  cudaFree(p->colpart);
  cudaFree(p->rowpart);
  cudaFree(p->rowmax[0]);
  cudaFree(p->rowmax[1]);
  cudaFree(p->xparts);
  delete p;
  p = nullptr;
}

bool dist_tiles(int64_t n, int br, int tc, int rank, int world, std::vector<int64_t> &toff,
                std::vector<int32_t> &jt, std::vector<int32_t> &cr_lo, std::vector<int32_t> &cr_hi) {
  if (world < 1 || rank < 0 || rank >= world || br % tc != 0 || n % world != 0) return false;
  const int64_t nloc = n / world;
  if (nloc % br != 0 || (world % 2 == 0 && world > 1 && nloc % (2 * br) != 0)) return false;
  const int L = (int)(nloc / br), tpd = br / tc, tpb = (int)(nloc / tc);  // column tiles per block
  const int nct = (int)(n / tc), W = world, w = rank;
  const int I0 = w * L;
  const int D = (W % 2 == 1) ? (W - 1) / 2 : W / 2 - 1;
  const int hc = (W % 2 == 0 && W > 1) ? (w + W / 2) % W : -1;  // the half-shared block
  toff.assign(L + 1, 0);
  jt.clear();
  cr_lo.assign(nct, 0);
  cr_hi.assign(nct, 0);
  for (int I = 0; I < L; ++I) {
    for (int j = tpd * (I0 + I); j < (w + 1) * tpb; ++j) jt.push_back(j);  // own block, from the diagonal
    for (int d = 1; d <= D; ++d) {
      const int c = (w + d) % W;
      for (int j = c * tpb; j < (c + 1) * tpb; ++j) jt.push_back(j);
    }
    if (hc >= 0) {
      if (w < hc) {
        if (I < L / 2)
          for (int j = hc * tpb; j < (hc + 1) * tpb; ++j) jt.push_back(j);
      } else {
        for (int j = hc * tpb + tpb / 2; j < (hc + 1) * tpb; ++j) jt.push_back(j);
      }
    }
    toff[I + 1] = (int64_t)jt.size();
  }
  // column partials: own block -> the local block-rows above the tile's diagonal block;
  // blocks at distance 1..D -> all; the half block -> the half this rank streams
  for (int j = w * tpb; j < (w + 1) * tpb; ++j) cr_hi[j] = j / tpd - I0;
  for (int d = 1; d <= D; ++d) {
    const int c = (w + d) % W;
    for (int j = c * tpb; j < (c + 1) * tpb; ++j) cr_hi[j] = L;
  }
  if (hc >= 0) {
    if (w < hc)
      for (int j = hc * tpb; j < (hc + 1) * tpb; ++j) cr_hi[j] = L / 2;
    else
      for (int j = hc * tpb + tpb / 2; j < (hc + 1) * tpb; ++j) cr_hi[j] = L;
  }
  return true;
}

static cudaError_t tri_plan_common(SymvPlan *p, const std::vector<int64_t> &toff, int br) {
  p->T = toff[p->nb];
  p->grid = (int)std::max<int64_t>(1, std::min<int64_t>(p->grid, p->T));
  std::vector<int32_t> segfirst(p->nb), nseg(p->nb);
  auto cta_of = [&](int64_t t) {  // CTA b with floor(T b / G) <= t < floor(T (b+1) / G)
    int64_t b = (t * p->grid) / p->T;
    while (b + 1 < p->grid && p->T * (b + 1) / p->grid <= t) ++b;
    while (b > 0 && p->T * b / p->grid > t) --b;
    return (int)b;
  };
  p->maxseg = 1;
  for (int I = 0; I < p->nb; ++I) {
    segfirst[I] = cta_of(toff[I]);
    nseg[I] = cta_of(toff[I + 1] - 1) - segfirst[I] + 1;
    p->maxseg = std::max(p->maxseg, (int)nseg[I]);
  }
  p->ldcp = (int64_t)p->nct * p->tc;
  const int64_t groups = (p->n + 31) / 32;  // 32-row groups of the finalize
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  p->fin_grid = (int)std::min<int64_t>(4 * sms, groups);
  cudaError_t e;
  if ((e = cudaMalloc(&p->toff, toff.size() * sizeof(int64_t))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&p->segfirst, segfirst.size() * sizeof(int32_t))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&p->nseg, nseg.size() * sizeof(int32_t))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&p->colpart, (size_t)p->nb * p->ldcp * sizeof(dd_pair))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&p->rowpart, (size_t)p->nb * p->maxseg * br * sizeof(dd_pair))) != cudaSuccess) return e;
  cudaMemcpy(p->toff, toff.data(), toff.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
  cudaMemcpy(p->segfirst, segfirst.data(), segfirst.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  cudaMemcpy(p->nseg, nseg.data(), nseg.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  return cudaSuccess;
}

cudaError_t tri_plan(SymvPlan *&p, int64_t n, int br, int tc, int grid) {
  if (p && p->n == n && p->br == br && p->tc == tc && !p->dist && p->grid == (int)std::max<int64_t>(1, grid))
    return cudaSuccess;
  symv_free(p);
  p = new SymvPlan();
  p->n = n;
  p->br = br;
  p->tc = tc;
  p->nb = (int)((n + br - 1) / br);
  p->nct = (int)((n + tc - 1) / tc);
  p->grid = grid;
  const int tpd = br / tc;
  std::vector<int64_t> toff(p->nb + 1, 0);
  for (int I = 0; I < p->nb; ++I) toff[I + 1] = toff[I] + (p->nct - tpd * I);
  return tri_plan_common(p, toff, br);
}

cudaError_t tri_plan_dist(SymvPlan *&p, int64_t n, int br, int tc, int grid, int rank, int world) {
  if (p && p->dist && p->n == n && p->br == br && p->tc == tc && p->rank == rank && p->world == world &&
      p->grid == (int)std::max<int64_t>(1, grid))
    return cudaSuccess;
  std::vector<int64_t> toff;
  std::vector<int32_t> jt, lo, hi;
  if (!dist_tiles(n, br, tc, rank, world, toff, jt, lo, hi)) return cudaErrorInvalidValue;
  symv_free(p);
  p = new SymvPlan();
  p->n = n;
  p->br = br;
  p->tc = tc;
  p->rank = rank;
  p->world = world;
  p->dist = true;
  p->nb = (int)(toff.size() - 1);
  p->I0 = rank * p->nb;
  p->nct = (int)(n / tc);
  p->grid = grid;
  cudaError_t e;
  if ((e = cudaMalloc(&p->jt_of, std::max<size_t>(jt.size(), 1) * sizeof(int32_t))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&p->cr_lo, lo.size() * sizeof(int32_t))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&p->cr_hi, hi.size() * sizeof(int32_t))) != cudaSuccess) return e;
  cudaMemcpy(p->jt_of, jt.data(), jt.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  cudaMemcpy(p->cr_lo, lo.data(), lo.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  cudaMemcpy(p->cr_hi, hi.data(), hi.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  return tri_plan_common(p, toff, br);
}

bool tri_is_dist(const SymvPlan *p) { return p && p->dist; }

cudaError_t symv_plan(SymvPlan *&p, int64_t n, int64_t ld, int num_sms, int rank, int world, bool dist) {
  if (p && p->n == n && p->ld == ld && p->br == kSR && p->tc == kSC && p->dist == dist && p->rank == rank &&
      p->world == world)
    return cudaSuccess;
  cudaError_t e = dist ? tri_plan_dist(p, n, kSR, kSC, num_sms, rank, world) : tri_plan(p, n, kSR, kSC, num_sms);
  if (e != cudaSuccess) return e;
  p->ld = ld;
  const size_t len = (size_t)p->nct * kSC;
  for (int w = 0; w < 2; ++w) {
    if ((e = cudaMalloc(&p->rowmax[w], len * sizeof(double))) != cudaSuccess) return e;
    if ((e = cudaMemset(p->rowmax[w], 0, len * sizeof(double))) != cudaSuccess) return e;
  }
  return cudaMalloc(&p->xparts, kXParts * sizeof(double));
}

void tri_fill(const SymvPlan *p, SymvArgs &a) {
  a.n = p->n;
  a.nb = p->nb;
  a.nct = p->nct;
  a.maxseg = p->maxseg;
  a.T = p->T;
  a.toff = p->toff;
  a.segfirst = p->segfirst;
  a.nseg = p->nseg;
  a.colpart = p->colpart;
  a.ldcp = p->ldcp;
  a.rowpart = p->rowpart;
  a.I0 = p->I0;
  a.jt_of = p->jt_of;
  a.cr_lo = p->cr_lo;
  a.cr_hi = p->cr_hi;
  a.own0 = (int64_t)p->I0 * p->br;
  a.own1 = a.own0 + (int64_t)p->nb * p->br;
}

int tri_grid(const SymvPlan *p) { return p->grid; }
int64_t tri_n(const SymvPlan *p) { return p->n; }
int tri_br(const SymvPlan *p) { return p->br; }

void launch_tri_finalize(const SymvPlan *p, const SymvArgs &a, cudaStream_t s) {
  if (p->dist) {
    if (p->br == 128 && p->tc == 64)
      tri_finalize_dist_kernel<128, 64><<<p->fin_grid, kFinThreads, 0, s>>>(a);
    else if (p->br == 128 && p->tc == 128)
      tri_finalize_dist_kernel<128, 128><<<p->fin_grid, kFinThreads, 0, s>>>(a);
    else
      tri_finalize_dist_kernel<64, 64><<<p->fin_grid, kFinThreads, 0, s>>>(a);
    return;
  }
  if (p->br == 128)
    symv_finalize_kernel<128, false><<<p->fin_grid, kFinThreads, 0, s>>>(a);
  else
    symv_finalize_kernel<64, false><<<p->fin_grid, kFinThreads, 0, s>>>(a);
}

int symv_finalize_grid(const SymvPlan *p) { return p->fin_grid; }

// which = 0 (K) or 1 (P): the row maxima of the (new) contents of A (sharded: of the
// rank's rows, into their global slots; the caller all-gathers the rest)
void symv_rowmax(SymvPlan *p, int which, const double *A, cudaStream_t s) {
  const int64_t rows = p->dist ? (int64_t)p->nb * p->br : p->n;
  const int64_t r0 = p->dist ? (int64_t)p->I0 * p->br : 0;
  rowmax_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(A, rows, p->n, p->ld, p->rowmax[which] + r0);
}

double *symv_rowmax_ptr(SymvPlan *p, int which) { return p->rowmax[which]; }

// which = 0 (K) or 1 (P); (re)encodes the tensor map when the base pointer changed
bool symv_bind(SymvPlan *p, int which, const double *A) {
  if (p->tm_base[which] == A) return true;
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  // the rows this rank stores: all n, or its n / W (sharded; tile rows are local)
  const int64_t rows = p->dist ? (int64_t)p->nb * p->br : p->n;
  cuuint64_t dims[2] = {(cuuint64_t)p->n, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)p->ld * sizeof(double)};
  cuuint32_t box[2] = {kSC, kSR};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&p->tm[which], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(A), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  p->tm_base[which] = A;
  return true;
}

void launch_symv(const SymvPlan *p, int which, const GemvArgs &g, cudaStream_t s) {
  SymvArgs a{};
  tri_fill(p, a);
  a.x = g.x;
  a.y = g.y;
  a.lambda = g.lambda;
  a.state = g.state;
  a.epi = g.epi;
  a.dot_out = g.dot_out;
  a.pair_out = g.pair_out;
  a.partials = g.partials;
  a.counter = g.counter;
  a.evict_first = g.evict_first ? 1 : 0;
  a.rowmax = p->rowmax[which];
  if (g.xparts) {
    a.xparts = g.xparts;
    a.nxparts = g.nxparts;
  } else {
    absmax_parts_kernel<<<dim3(kXParts), dim3(256), 0, s>>>(g.x, (int64_t)p->n, p->xparts, (const PcgState *)g.state);
    a.xparts = p->xparts;
    a.nxparts = kXParts;
  }
  a.ypair = g.ypair;
  a.upd = g.upd;
  const bool tc = g.tc != nullptr && which == 0;
  if (tc) {
    launch_symv_tc(g.tc, a, s);
    if (p->dist) return;  // the sharded apply reduce-scatters the groups and combines (pcg_dist.cu)
  } else if ((int64_t)p->nct * kCPT <= kMaxOffTiles)
    symv_dot2_kernel<true><<<dim3(p->grid), dim3(kSymThreads), kSymSmem, s>>>(p->tm[which], a);
  else
    symv_dot2_kernel<false><<<dim3(p->grid), dim3(kSymThreads), kSymSmem, s>>>(p->tm[which], a);
  if (p->dist)
    tri_finalize_dist_kernel<kSR, kSC><<<dim3(p->fin_grid), dim3(kFinThreads), 0, s>>>(a);
  else if (tc)  // one 32-row group per warp: a small grid (a cheap grid barrier), co-resident
    symv_finalize_kernel<kSR, true><<<dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(
                                           fused_fin_grid(), (p->n + 32 * (kFinThreads / 32) - 1) /
                                                                 (32 * (kFinThreads / 32))))),
                                       dim3(kFinThreads), 0, s>>>(a);
  else if (g.upd.on)
    symv_finalize_kernel<kSR, false><<<dim3(std::min(p->fin_grid, fused_fin_grid())), dim3(kFinThreads), 0, s>>>(a);
  else
    symv_finalize_kernel<kSR, false><<<dim3(p->fin_grid), dim3(kFinThreads), 0, s>>>(a);
}

void launch_symv_check(const double *A, int64_t n, int64_t ld, int *flag, cudaStream_t s) {
  const int nt = (int)((n + 31) / 32);
  symv_check_kernel<<<dim3(nt, nt), dim3(32, 8), 0, s>>>(A, n, ld, flag);
}

}  // namespace laker
