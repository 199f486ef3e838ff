// Streaming fp64 Dot2 GEMV: the per-iteration K.p and P.r products of the PCG
// (Alg. 1 l.16-21) -- HBM-bound.
//
// Layout: A is the local row block of K (or P), row-major with a padded stride
// `ld` (multiple of 256 doubles, zero padding).  Work unit = a group of ROWS
// rows x one 1024-column chunk plus the matching 1024-entry chunk(s) of the
// input vector.  One persistent CTA per SM owns a contiguous range of row
// groups.  A producer warp streams the units into a 3-stage shared-memory
// ring with 1-D bulk copies (cp.async.bulk, TMA engine; A with an L2
// evict-first policy, vectors evict-last) signalled on mbarriers; 16 consumer
// warps read the ring, each thread 2 columns x ROWS rows, so the vector never
// costs a dependent global load.  Each thread keeps one Dot2 pair per row;
// rows are reduced warp -> CTA in a fixed order, so
// y_i = RN(lambda x_i + sum_j A_ij x_j) is correctly rounded in practice and
// bitwise equal to the oracle's sequential Dot2.  The CTA also accumulates
// dot(x_local, y) as a Dot2 pair; the last CTA to finish reduces the per-CTA
// pairs in CTA order and runs the PCG scalar epilogue in the same kernel.
//
// Fused PCG modes (single rank, dense P: the whole iteration is 2 kernels):
//   FUSE_K: x = p_new = fma(beta, p_old, theta) formed on the fly from two
//           staged chunks (Alg. 1 l.21), own rows of p_new written out;
//           epilogue delta = rho / p.q (l.16).
//   FUSE_P: x = r_new = fma(-delta, q, r_old) on the fly (l.18); own rows:
//           r_new written, alpha = fma(delta, p, alpha) (l.17), ||r||^2 pair;
//           epilogue: ||r||/||y|| test (l.19), then beta = r.theta / rho (l.20).
// The fma/Dot2 operations are exactly those of the unfused kernels, so the
// fused iteration is bitwise the same recurrence.
#include "laker_internal.h"
#include "tma.cuh"
#include "pdl.cuh"

namespace laker {
namespace {

constexpr int kConsumers = 512;
constexpr int kWarps = kConsumers / 32;
constexpr int kStages = 3;
constexpr int kThreads = kConsumers + 32;
enum { FUSE_NONE = 0, FUSE_K = 1, FUSE_P = 2 };

template <int FUSE>
struct Cfg {
  static constexpr int NX = FUSE == FUSE_NONE ? 1 : 2;     // staged vector chunks
  static constexpr int ROWS = FUSE == FUSE_NONE ? 8 : 7;   // rows per group (stage = 9 x 8 KiB)
  static constexpr int CPT = 2;                            // columns per consumer thread
  static constexpr int CHUNK = kConsumers * CPT;           // 1024 / 512 columns per unit
  static constexpr size_t STAGE = (size_t)(ROWS + NX) * CHUNK;
  static constexpr size_t SMEM = kStages * STAGE * sizeof(double) + 2 * kWarps * ROWS * sizeof(dd_pair) +
                                 2 * kStages * sizeof(uint64_t) + 16;
};

__device__ __forceinline__ void run_epilogue(const GemvArgs &a, double v) {
  PcgState *st = a.state;
  switch (a.epi) {
    case kEpiDelta:
      if (!(v > 0.0)) {
        st->term = LAKER_TERM_BREAKDOWN;
        st->done = 1;
      } else {
        pcg_set_delta(st, __ddiv_rn(st->rho, v));
      }
      break;
    case kEpiBeta:
      if (!(v > 0.0)) {
        st->term = LAKER_TERM_INDEFINITE;
        st->done = 1;
      } else {
        pcg_set_beta(st, __ddiv_rn(v, st->rho));
        st->rho = v;
      }
      break;
    case kEpiStoreDot:
      if (a.dot_out) *a.dot_out = v;
      break;
    default:
      break;
  }
}

// FUSE_P epilogue: rr (termination) first, then beta from r.theta (+ budget)
__device__ __forceinline__ void fused_p_epilogue(const GemvArgs &a, double rtheta, double rr) {
  PcgState *st = a.state;
  const double rel = __ddiv_rn(__dsqrt_rn(rr), st->ynorm);
  const int it = st->iters + 1;
  st->iters = it;
  st->rel = rel;
  if (a.hist) a.hist[it - 1] = rel;
  if (rel <= st->tol) {
    st->term = LAKER_TERM_RESIDUAL_TOL;
    st->done = 1;
    return;
  }
  if (!(rtheta > 0.0)) {
    st->term = LAKER_TERM_INDEFINITE;
    st->done = 1;
    return;
  }
  pcg_set_beta(st, __ddiv_rn(rtheta, st->rho));
  st->rho = rtheta;
  if (it >= st->max_iters) {
    st->term = LAKER_TERM_MAX_ITERS;
    st->done = 1;
  }
}

template <int FUSE>
__global__ void __launch_bounds__(kThreads, 1) gemv_dot2_kernel(const GemvArgs a) {
  pdl_prologue();
  using C = Cfg<FUSE>;
  constexpr int ROWS = C::ROWS;
  constexpr int kCPT = C::CPT;
  constexpr int kChunk = C::CHUNK;
  if (a.state != nullptr && *(volatile int32_t *)&a.state->done) return;
  extern __shared__ __align__(128) unsigned char smem[];
  double *ring = reinterpret_cast<double *>(smem);
  dd_pair *red = reinterpret_cast<dd_pair *>(smem + kStages * C::STAGE * sizeof(double));
  uint64_t *full = reinterpret_cast<uint64_t *>(red + 2 * kWarps * ROWS);
  uint64_t *empty = full + kStages;
  __shared__ int s_last;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // rows split evenly over the CTAs (time ~ rows streamed), groups of ROWS from each start
  const int64_t rbeg = a.rows * blockIdx.x / gridDim.x;
  const int64_t rend = a.rows * (blockIdx.x + 1) / gridDim.x;
  const int64_t ncp = (a.ncols + 255) / 256 * 256;  // padded columns actually streamed
  const int64_t nchunks = (ncp + kChunk - 1) / kChunk;
  // fused: x = fma(xs, xa, xb) with xs = beta (K) or -delta (P)
  double xs = 0.0, delta = 0.0;
  if (FUSE == FUSE_K) xs = a.state->beta;
  if (FUSE == FUSE_P) {
    delta = a.state->delta;
    xs = -delta;
  }
  const double *xsrc0 = FUSE == FUSE_NONE ? a.x : a.xa;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kWarps) {
    // ---------------- producer warp: one elected lane issues the bulk copies
    if (lane == 0) {
      const uint64_t pol_a = a.evict_first ? l2_policy_evict_first() : l2_policy_evict_last();
      const uint64_t pol_x = l2_policy_evict_last();
      int slot = 0;
      uint32_t ph = 0;
      bool first = true;
      for (int64_t rb = rbeg; rb < rend; rb += ROWS) {
        const int nr = (int)imin64(ROWS, rend - rb);
        for (int64_t c = 0; c < nchunks; ++c) {
          if (!first) mbar_wait(&empty[slot], ph ^ 1u);
          const int64_t col0 = c * kChunk;
          const int width = (int)imin64(kChunk, ncp - col0);
          const uint32_t bytes = (uint32_t)width * 8u;
          mbar_arrive_expect_tx(&full[slot], bytes * (uint32_t)(nr + C::NX));
          double *dst = ring + slot * C::STAGE;
          bulk_g2s(dst + ROWS * kChunk, xsrc0 + col0, bytes, &full[slot], pol_x);
          if (C::NX == 2) bulk_g2s(dst + (ROWS + 1) * kChunk, a.xb + col0, bytes, &full[slot], pol_x);
          for (int r = 0; r < nr; ++r)
            bulk_g2s(dst + r * kChunk, a.A + (rb + r) * a.ld + col0, bytes, &full[slot], pol_a);
          if (++slot == kStages) {
            slot = 0;
            ph ^= 1u;
            first = false;
          }
        }
      }
    }
    return;
  }

  // ---------------- consumer warps
  __shared__ double xrow_buf[2][ROWS];  // x at the group's own row indices, captured from the ring
  __shared__ dd_pair spart[kWarps][2];
  dd_pair part = {0.0, 0.0}, part2 = {0.0, 0.0};
  const int cb = tid * kCPT;
  int slot = 0, gpar = 0;
  uint32_t ph = 0;
  for (int64_t rb = rbeg; rb < rend; rb += ROWS, gpar ^= 1) {
    const int nr = (int)imin64(ROWS, rend - rb);
    double *xrow = xrow_buf[FUSE == FUSE_NONE ? gpar : 0];
    const int64_t own0 = a.row0 + rb;  // global index of the group's first row
    dd_pair acc[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) acc[r] = dd_pair{0.0, 0.0};
    double pcur_i = 0.0, alpha_i = 0.0;  // FUSE_P own-row operands, prefetched off the critical path
    if (FUSE == FUSE_P && warp == 0 && lane < nr) {
      pcur_i = a.pcur[own0 + lane];
      alpha_i = a.alpha[own0 + lane];
    }
    for (int64_t c = 0; c < nchunks; ++c) {
      mbar_wait(&full[slot], ph);
      const int64_t col0 = c * kChunk;
      const int width = (int)imin64(kChunk, ncp - col0);
      if (cb < width) {
        const double *sp = ring + slot * C::STAGE + cb;
        if (kCPT == 2) {
          double2 x0 = *reinterpret_cast<const double2 *>(sp + ROWS * kChunk);
          if (C::NX == 2) {
            const double2 xb = *reinterpret_cast<const double2 *>(sp + (ROWS + 1) * kChunk);
            x0.x = __fma_rn(xs, x0.x, xb.x);
            x0.y = __fma_rn(xs, x0.y, xb.y);
          }
          const int64_t o = own0 - (col0 + cb);  // own row indices falling in this thread's columns
          if (o > -ROWS && o < kCPT) {
            if (o <= 0 && -o < nr) xrow[-o] = x0.x;
            if (o <= 1 && 1 - o < nr) xrow[1 - o] = x0.y;
          }
#pragma unroll
          for (int r = 0; r < ROWS; ++r) {
            if (r < nr) {
              const double2 v0 = *reinterpret_cast<const double2 *>(sp + r * kChunk);
              dot2_step(acc[r], v0.x, x0.x);
              dot2_step(acc[r], v0.y, x0.y);
            }
          }
        } else {
          double x0 = sp[ROWS * kChunk];
          if (C::NX == 2) x0 = __fma_rn(xs, x0, sp[(ROWS + 1) * kChunk]);
          const int64_t o = own0 - (col0 + cb);
          if (o <= 0 && -o < nr) xrow[-o] = x0;
#pragma unroll
          for (int r = 0; r < ROWS; ++r)
            if (r < nr) dot2_step(acc[r], sp[r * kChunk], x0);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++slot == kStages) {
        slot = 0;
        ph ^= 1u;
      }
    }
    if constexpr (FUSE == FUSE_NONE) {
      // rows: reduce-scatter inside the warp (row R ends in lane 4R: 9 pair adds per
      // lane instead of 40), then warp R combines the 16 warps' pairs of row R by a
      // fixed-shape shuffle tree; red / xrow double-buffered by group parity, so one
      // CTA barrier per group
      static_assert(ROWS == 8, "reduce-scatter layout assumes 8 rows");
      dd_pair v4[4], v2[2], v1;
      const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const dd_pair snd = b4 ? acc[j] : acc[4 + j];
        dd_pair rcv;
        rcv.s = __shfl_xor_sync(0xffffffffu, snd.s, 16);
        rcv.c = __shfl_xor_sync(0xffffffffu, snd.c, 16);
        v4[j] = b4 ? acc[4 + j] : acc[j];
        pair_add(v4[j], rcv);
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const dd_pair snd = b3 ? v4[j] : v4[2 + j];
        dd_pair rcv;
        rcv.s = __shfl_xor_sync(0xffffffffu, snd.s, 8);
        rcv.c = __shfl_xor_sync(0xffffffffu, snd.c, 8);
        v2[j] = b3 ? v4[2 + j] : v4[j];
        pair_add(v2[j], rcv);
      }
      {
        const dd_pair snd = b2 ? v2[0] : v2[1];
        dd_pair rcv;
        rcv.s = __shfl_xor_sync(0xffffffffu, snd.s, 4);
        rcv.c = __shfl_xor_sync(0xffffffffu, snd.c, 4);
        v1 = b2 ? v2[1] : v2[0];
        pair_add(v1, rcv);
      }
#pragma unroll
      for (int off = 2; off > 0; off >>= 1) {
        dd_pair rcv;
        rcv.s = __shfl_xor_sync(0xffffffffu, v1.s, off);
        rcv.c = __shfl_xor_sync(0xffffffffu, v1.c, off);
        pair_add(v1, rcv);
      }
      dd_pair *rb_red = red + gpar * kWarps * ROWS;
      if ((lane & 3) == 0) rb_red[warp * ROWS + (lane >> 2)] = v1;
      named_bar_sync(1, kConsumers);
      if (warp < nr) {
        const int R = warp;
        dd_pair t = lane < kWarps ? rb_red[lane * ROWS + R] : dd_pair{0.0, 0.0};
#pragma unroll
        for (int off = 1; off < kWarps; off <<= 1) {
          dd_pair o;
          o.s = __shfl_down_sync(0xffffffffu, t.s, off);
          o.c = __shfl_down_sync(0xffffffffu, t.c, off);
          if ((lane & (2 * off - 1)) == 0) pair_add(t, o);
        }
        if (lane == 0) {
          const int64_t gi = a.row0 + rb + R;
          const double xi = a.xd != nullptr ? a.xd[gi] : xrow[R];
          if (a.lambda != 0.0) dot2_step(t, a.lambda, xi);  // the lambda x_i term of the row
          const double yv = pair_value(t);
          a.y[rb + R] = yv;
          dot2_step(part, xi, yv);
        }
      }
      continue;
    }
    // fused variants: warp butterfly, then the warp pairs in warp order
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const dd_pair v = warp_reduce_pair(acc[r]);
      if (lane == 0) red[warp * ROWS + r] = v;
    }
    named_bar_sync(1, kConsumers);
    if (warp == 0 && lane < nr) {
      const double xi = xrow[lane];
      dd_pair t = red[lane];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) pair_add(t, red[w * ROWS + lane]);
      if (a.lambda != 0.0) dot2_step(t, a.lambda, xi);  // the lambda x_i term of the row
      const double yv = pair_value(t);
      const int64_t li = rb + lane, gi = own0 + lane;
      a.y[li] = yv;
      if (FUSE != FUSE_NONE) {
        a.xown[gi] = xi;  // own rows of p_new (K) / r_new (P)
        if (FUSE == FUSE_P) {
          a.alpha[gi] = __fma_rn(delta, pcur_i, alpha_i);
          dot2_step(part2, xi, xi);
        }
      }
      dot2_step(part, xi, yv);
    }
    named_bar_sync(1, kConsumers);
  }

  // ---------------- CTA partials, then the last CTA reduces in CTA order
  if (FUSE == FUSE_NONE) {  // row partials live in lane 0 of warps 0..7: gather them in warp order
    if (lane == 0) spart[warp][0] = part;
    named_bar_sync(1, kConsumers);
    if (warp == 0) {
      part = lane < kWarps ? spart[lane][0] : dd_pair{0.0, 0.0};
#pragma unroll
      for (int off = 1; off < kWarps; off <<= 1) {
        dd_pair o;
        o.s = __shfl_down_sync(0xffffffffu, part.s, off);
        o.c = __shfl_down_sync(0xffffffffu, part.c, off);
        if ((lane & (2 * off - 1)) == 0) pair_add(part, o);
      }
    }
  }
  if (warp == 0) {
    const dd_pair v = FUSE == FUSE_NONE ? part : warp_reduce_pair(part);
    const dd_pair v2 = warp_reduce_pair(part2);
    if (lane == 0) {
      a.partials[2 * blockIdx.x] = v;
      a.partials[2 * blockIdx.x + 1] = v2;
      __threadfence();
      const unsigned int ticket = atomicAdd(a.counter, 1u);
      s_last = (ticket == gridDim.x - 1);
    }
  }
  named_bar_sync(1, kConsumers);
  if (s_last && warp == 0) {
    __threadfence();
    dd_pair v = {0.0, 0.0}, v2 = {0.0, 0.0};
    for (int i = lane; i < (int)gridDim.x; i += 32) {
      dd_pair o = {__ldcg(&a.partials[2 * i].s), __ldcg(&a.partials[2 * i].c)};
      pair_add(v, o);
      if (FUSE == FUSE_P) {
        dd_pair o2 = {__ldcg(&a.partials[2 * i + 1].s), __ldcg(&a.partials[2 * i + 1].c)};
        pair_add(v2, o2);
      }
    }
    v = warp_reduce_pair(v);
    if (FUSE == FUSE_P) v2 = warp_reduce_pair(v2);
    if (lane == 0) {
      *a.counter = 0u;
      if (FUSE == FUSE_P)
        fused_p_epilogue(a, pair_value(v), pair_value(v2));
      else if (a.epi == kEpiStorePair)
        *a.pair_out = v;
      else
        run_epilogue(a, pair_value(v));
    }
  }
}

}  // namespace

size_t gemv_smem_bytes() { return Cfg<FUSE_NONE>::SMEM; }

int gemv_max_grid(int num_sms) { return num_sms; }

void gemv_init() {
  cudaFuncSetAttribute(gemv_dot2_kernel<FUSE_NONE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)Cfg<FUSE_NONE>::SMEM);
  cudaFuncSetAttribute(gemv_dot2_kernel<FUSE_K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)Cfg<FUSE_K>::SMEM);
  cudaFuncSetAttribute(gemv_dot2_kernel<FUSE_P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)Cfg<FUSE_P>::SMEM);
}

void launch_gemv(const GemvArgs &a, int grid, cudaStream_t s) {
  const int rows_per = a.fuse == FUSE_NONE ? Cfg<FUSE_NONE>::ROWS : Cfg<FUSE_K>::ROWS;
  const int64_t groups = (a.rows + rows_per - 1) / rows_per;
  const int g = (int)imin64(grid, imax64(groups, 1));
  switch (a.fuse) {
    case FUSE_K:
      gemv_dot2_kernel<FUSE_K><<<g, kThreads, Cfg<FUSE_K>::SMEM, s>>>(a);
      break;
    case FUSE_P:
      gemv_dot2_kernel<FUSE_P><<<g, kThreads, Cfg<FUSE_P>::SMEM, s>>>(a);
      break;
    default:
      launch_pdl(gemv_dot2_kernel<FUSE_NONE>, dim3(g), dim3(kThreads), Cfg<FUSE_NONE>::SMEM, s, a);
  }
}

}  // namespace laker
