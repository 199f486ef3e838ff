// Symmetric on-the-fly operator apply ("compute each
// off-diagonal tile once in K7 (half the flops and exps)"):
//
//   q = lambda p + K p,   K_ij = exp(scale <e_i, e_j>) never stored
//
// K is symmetric (q = k, reading R2), so every off-diagonal tile K_IJ (J > I) is
// computed once and used twice: its rows give K_IJ p_J to the rows of block I and
// its columns K_IJ^T p_I = K_JI p_I to the rows of block J.  The tiles of the
// block upper triangle are split over a persistent grid exactly as the stored
// symmetric apply (tri.cuh); the per-row and per-column Dot2 pairs go to
// rowpart / colpart and the shared finalize kernel forms q_i (and the PCG
// epilogue, so the on-the-fly operator gets the fused p.q like the stored one).
//
// FAST: the tcgen05 tiles of otf_tc2.cu (kSym).
// EXACT (this file, otf_sym_exact_kernel): each entry exactly as assembly forms it
// (sequential Dot2 over k, RN(scale x), correctly rounded exp -- the (i, j) and
// (j, i) entries are the same bits), accumulated as Dot2 pairs; so q equals the
// materialized apply and the oracle's row sums bitwise in practice (T19).
// 64 x 64 tiles, 256 threads, 4 x 4 entries per thread.
#include <algorithm>
#include <cstdlib>

#include "exp_cr.cuh"
#include "laker_internal.h"
#include "tri.cuh"

namespace laker {
namespace {

constexpr int kXT = 64;       // tile rows = tile columns = block rows
constexpr int kXThreads = 256;

struct OtfSymArgs {
  SymvArgs t;
  const double *E;
  int d, ldE;  // smem row stride (d + 1)
  double scale;
  unsigned long long *flags;
  const double *emax;  // max_k |e_ik| per row (offsets of the compensated dots, assemble.cu)
};

__global__ void __launch_bounds__(kXThreads) otf_sym_exact_kernel(const OtfSymArgs f) {
  const SymvArgs &a = f.t;
  if (a.state != nullptr && *(volatile int32_t *)&a.state->done) return;
  extern __shared__ double sm[];
  double *EI = sm;                        // [64][d + 1] rows of block I
  double *EJ = EI + kXT * f.ldE;          // [64][d + 1] rows of block J
  double *wI = EJ + kXT * f.ldE;          // [64]
  double *wJ = wI + kXT;                  // [64]
  dd_pair *cred = reinterpret_cast<dd_pair *>(wJ + kXT);  // [8 warps][64 columns]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4, warp = tid >> 5, lane = tid & 31;
  const int d = f.d, ldE = f.ldE;
  const int64_t n = a.n;
  const int64_t t0 = a.T * blockIdx.x / gridDim.x, t1 = a.T * (blockIdx.x + 1) / gridDim.x;
  if (t0 >= t1) return;
  int I = find_block_row(a.toff, a.nb, t0);
  int64_t rend = a.toff[I + 1];
  unsigned int inc = 0, ovf = 0;

  auto load_rows = [&](double *dst, double *wdst, int blk) {
    const int64_t r0 = (int64_t)blk * kXT;
    for (int idx = tid; idx < kXT * d; idx += kXThreads) {
      const int r = idx / d, c = idx - r * d;
      dst[r * ldE + c] = (r0 + r < n) ? f.E[(r0 + r) * d + c] : 0.0;
    }
    if (tid < kXT) wdst[tid] = (r0 + tid < n) ? a.x[r0 + tid] : 0.0;
  };
  auto flush_rows = [&](int Iblk, dd_pair (&row)[4]) {
    const int s = blockIdx.x - a.segfirst[Iblk];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      dd_pair v = row[i];
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) {  // the 16 column threads of the row, fixed butterfly
        dd_pair o;
        o.s = __shfl_xor_sync(0xffffffffu, v.s, off);
        o.c = __shfl_xor_sync(0xffffffffu, v.c, off);
        pair_add(v, o);
      }
      if (tx == 0) a.rowpart[((int64_t)Iblk * a.maxseg + s) * kXT + ty + 16 * i] = v;
      row[i] = dd_pair{0.0, 0.0};
    }
  };

  dd_pair row[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) row[i] = dd_pair{0.0, 0.0};
  load_rows(EI, wI, I);
  for (int64_t t = t0; t < t1; ++t) {
    if (t >= rend) {
      flush_rows(I, row);
      ++I;
      rend = a.toff[I + 1];
      __syncthreads();
      load_rows(EI, wI, I);
    }
    const int J = I + (int)(t - a.toff[I]);
    const bool diag = J == I;
    __syncthreads();  // previous tile's EJ / cred consumers done
    load_rows(EJ, wJ, J);
    __syncthreads();
    double ei[4], ej[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      ei[i] = (int64_t)I * kXT + ty + 16 * i < n ? f.emax[(int64_t)I * kXT + ty + 16 * i] * (2.0 * d) : 0.0;
      ej[i] = (int64_t)J * kXT + tx + 16 * i < n ? f.emax[(int64_t)J * kXT + tx + 16 * i] : 0.0;
    }
    dd_pair acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = dd_pair{pow2_above(ei[i] * ej[j]), 0.0};
    for (int k = 0; k < d; ++k) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = EI[(ty + 16 * i) * ldE + k];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = EJ[(tx + 16 * j) * ldE + k];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dot2_step_off(acc[i][j], av[i], bv[j]);
    }
    dd_pair col[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) col[j] = dd_pair{0.0, 0.0};
    const int64_t jb = (int64_t)J * kXT, ib = (int64_t)I * kXT;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool cok = jb + tx + 16 * j < n;
      const double wj = wJ[tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const bool rok = ib + ty + 16 * i < n;
        if (!(rok && cok)) continue;
        dd_pair ac = acc[i][j];
        ac.s = __dsub_rn(ac.s, pow2_above(ei[i] * ej[j]));  // exact (Sterbenz)
        const double kv = exp_cr(__dmul_rn(f.scale, pair_value(ac)), inc, ovf);
        dot2_step(row[i], kv, wj);
        if (!diag) dot2_step(col[j], kv, wI[ty + 16 * i]);
      }
    }
    if (!diag) {
      // column pairs: lanes l and l ^ 16 (ty, ty ^ 1) by shuffle, then the 8 warps in order
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        dd_pair o;
        o.s = __shfl_xor_sync(0xffffffffu, col[j].s, 16);
        o.c = __shfl_xor_sync(0xffffffffu, col[j].c, 16);
        pair_add(col[j], o);
        if (lane < 16) cred[warp * kXT + tx + 16 * j] = col[j];
      }
      __syncthreads();
      if (tid < kXT) {
        dd_pair v = cred[tid];
#pragma unroll
        for (int w = 1; w < kXThreads / 32; ++w) pair_add(v, cred[w * kXT + tid]);
        a.colpart[(int64_t)I * a.ldcp + jb + tid] = v;
      }
    }
  }
  flush_rows(I, row);
  if (inc) atomicAdd(&f.flags[0], (unsigned long long)inc);
  if (ovf) atomicAdd(&f.flags[1], (unsigned long long)ovf);
}

size_t exact_smem(int d) { return (size_t)(2 * kXT * (d + 1) + 2 * kXT) * sizeof(double) + 8 * kXT * sizeof(dd_pair); }

}  // namespace

void otf_sym_init() {
  cudaFuncSetAttribute(otf_sym_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)exact_smem(128));
}

// the tile partition of the symmetric on-the-fly apply (at assembly: plans allocate,
// which a captured solve may not)
cudaError_t otf_sym_prepare(laker_ctx ctx) {
  if (ctx->world != 1 || ctx->storage != LAKER_STORE_ON_THE_FLY) return cudaSuccess;
  if (ctx->mode == LAKER_MODE_FAST) {
    // tcgen05 tiles of 128 x 128, one persistent CTA per SM (otf_tc2.cu)
    if (!(ctx->ozE_valid && ctx->ozE.Kp == 64)) return cudaSuccess;
    return tri_plan(ctx->otf_sym, ctx->n, 128, 128, ctx->num_sms);
  }
  if (ctx->d > 128) return cudaSuccess;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, otf_sym_exact_kernel, kXThreads, exact_smem(ctx->d));
  return tri_plan(ctx->otf_sym, ctx->n, kXT, kXT, std::max(1, per_sm) * ctx->num_sms);
}

// q = (lambda I + K) p over all n rows with K recomputed on the fly, each tile of the
// block upper triangle once; epi / state / dot_out as the stored applies.  Returns
// false (nothing launched) when the symmetric path does not apply.
bool launch_operator_otf_sym(laker_ctx ctx, const double *p, double *q, PcgState *st, int epi, double *dot_out,
                             cudaStream_t s) {
  static int enabled = -1;
  if (enabled < 0) {
    const char *v = std::getenv("LAKER_OTF_SYM");
    enabled = (v && v[0] == '0') ? 0 : 1;
  }
  if (!enabled || ctx->world != 1 || ctx->storage != LAKER_STORE_ON_THE_FLY || !ctx->otf_sym ||
      tri_n(ctx->otf_sym) != ctx->n)
    return false;
  const bool fast = ctx->mode == LAKER_MODE_FAST;
  if (fast ? !(ctx->ozE_valid && ctx->ozE.Kp == 64 && tri_br(ctx->otf_sym) == 128)
           : (ctx->d > 128 || tri_br(ctx->otf_sym) != kXT))
    return false;
  SymvArgs t{};
  tri_fill(ctx->otf_sym, t);
  t.x = p;
  t.y = q;
  t.lambda = ctx->lambda;
  t.state = st;
  t.epi = epi;
  t.dot_out = dot_out;
  t.partials = ctx->partials;
  t.counter = ctx->counters + kCtrGemv;
  if (fast) {
    if (launch_otf_tc2_sym(ctx->ozE, ctx->n, ctx->scale, p, ctx->cf, t, tri_grid(ctx->otf_sym), s) != cudaSuccess)
      return false;
  } else {
    OtfSymArgs f{};
    f.t = t;
    f.E = ctx->E;
    f.d = ctx->d;
    f.ldE = ctx->d + 1;
    f.scale = ctx->scale;
    f.flags = ctx->flags;
    f.emax = ctx->emax;
    otf_sym_exact_kernel<<<tri_grid(ctx->otf_sym), kXThreads, exact_smem(ctx->d), s>>>(f);
  }
  launch_tri_finalize(ctx->otf_sym, t, s);
  return true;
}

}  // namespace laker
