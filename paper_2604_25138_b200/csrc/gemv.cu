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
#include "laker_internal.h"
#include "tma.cuh"

namespace laker {
namespace {

constexpr int kConsumers = 512;
constexpr int kWarps = kConsumers / 32;
constexpr int kStages = 3;
constexpr int kThreads = kConsumers + 32;
struct Cfg {
  static constexpr int NX = 1;                  // staged vector chunks
  static constexpr int ROWS = 8;                // rows per group (stage = 9 x 8 KiB)
  static constexpr int CPT = 2;                 // columns per consumer thread
  static constexpr int CHUNK = kConsumers * CPT;  // 1024 columns per unit
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

__global__ void __launch_bounds__(kThreads, 1) gemv_dot2_kernel(const GemvArgs a) {
  using C = Cfg;
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
  const double rho_old = a.pu_p != nullptr ? a.state->rho : 0.0;  // read before any CTA updates it
  // rows split evenly over the CTAs (time ~ rows streamed), groups of ROWS from each start
  const int64_t rbeg = a.rows * blockIdx.x / gridDim.x;
  const int64_t rend = a.rows * (blockIdx.x + 1) / gridDim.x;
  const int64_t ncp = (a.ncols + 255) / 256 * 256;  // padded columns actually streamed
  const int64_t nchunks = (ncp + kChunk - 1) / kChunk;
  const double *xsrc0 = a.x;

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
  dd_pair part = {0.0, 0.0};
  const int cb = tid * kCPT;
  int slot = 0, gpar = 0;
  uint32_t ph = 0;
  for (int64_t rb = rbeg; rb < rend; rb += ROWS, gpar ^= 1) {
    const int nr = (int)imin64(ROWS, rend - rb);
    double *xrow = xrow_buf[gpar];
    const int64_t own0 = a.row0 + rb;  // global index of the group's first row
    dd_pair acc[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) acc[r] = dd_pair{0.0, 0.0};
    for (int64_t c = 0; c < nchunks; ++c) {
      mbar_wait(&full[slot], ph);
      const int64_t col0 = c * kChunk;
      const int width = (int)imin64(kChunk, ncp - col0);
      if (cb < width) {
        const double *sp = ring + slot * C::STAGE + cb;
        {
          const double2 x0 = *reinterpret_cast<const double2 *>(sp + ROWS * kChunk);
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
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++slot == kStages) {
        slot = 0;
        ph ^= 1u;
      }
    }
    {
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
          if (a.ypair != nullptr) {
            a.ypair[rb + R] = t;  // unrounded row pair (sharded partial sums, pcg_dist.cu)
          } else {
            const double yv = pair_value(t);
            a.y[rb + R] = yv;
            dot2_step(part, xi, yv);
          }
        }
      }
    }
  }

  // ---------------- CTA partials, then the last CTA reduces in CTA order
  {  // row partials live in lane 0 of warps 0..7: gather them in warp order
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
  if (a.pu_p != nullptr) {
    // ---- fused direction update: r.theta over the CTA pairs in CTA order (the same value in
    // every CTA), beta, then p = fma(beta, p, theta) on this CTA's rows (pcg_pupdate_kernel)
    if (warp == 0 && lane == 0) a.partials[blockIdx.x] = part;
    grid_barrier(a.pu_bar, a.pu_bar + 1, 1, kConsumers);
    __shared__ double s_beta;
    __shared__ int s_ok;
    if (warp == 0) {
      dd_pair v = {0.0, 0.0};
      for (int i = lane; i < (int)gridDim.x; i += 32) {
        dd_pair o = {__ldcg(&a.partials[i].s), __ldcg(&a.partials[i].c)};
        pair_add(v, o);
      }
      v = warp_reduce_pair(v);
      if (lane == 0) {
        const double rt = pair_value(v);
        s_ok = rt > 0.0;
        s_beta = s_ok ? __ddiv_rn(rt, rho_old) : 0.0;
        if (blockIdx.x == 0) {
          PcgState *st = a.state;
          if (!s_ok) {
            st->term = LAKER_TERM_INDEFINITE;
            st->done = 1;
          } else {
            pcg_set_beta(st, s_beta);
            st->rho = rt;
          }
        }
      }
    }
    named_bar_sync(1, kConsumers);
    if (!s_ok) return;
    const double beta = s_beta;
    double m = 0.0;
    for (int64_t i = rbeg + tid; i < rend; i += kConsumers) {
      const double pi = __fma_rn(beta, a.pu_p[a.row0 + i], __ldcg(&a.y[i]));
      a.pu_p[a.row0 + i] = pi;
      m = fmax(m, fabs(pi));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    __shared__ double s_m[kWarps];
    if (lane == 0) s_m[warp] = m;
    named_bar_sync(1, kConsumers);
    if (tid == 0) {
      for (int w = 1; w < kWarps; ++w) m = fmax(m, s_m[w]);
      a.pu_pmax[blockIdx.x] = m;
      if (blockIdx.x == gridDim.x - 1 && a.pu_budget && a.state->iters >= a.state->max_iters) {
        a.state->term = LAKER_TERM_MAX_ITERS;
        a.state->done = 1;
      }
    }
    return;
  }
  if (warp == 0) {
    if (lane == 0) {
      a.partials[blockIdx.x] = part;
      __threadfence();
      const unsigned int ticket = atomicAdd(a.counter, 1u);
      s_last = (ticket == gridDim.x - 1);
    }
  }
  named_bar_sync(1, kConsumers);
  if (s_last && warp == 0) {
    __threadfence();
    dd_pair v = {0.0, 0.0};
    for (int i = lane; i < (int)gridDim.x; i += 32) {
      dd_pair o = {__ldcg(&a.partials[i].s), __ldcg(&a.partials[i].c)};
      pair_add(v, o);
    }
    v = warp_reduce_pair(v);
    if (lane == 0) {
      *a.counter = 0u;
      if (a.epi == kEpiStorePair)
        *a.pair_out = v;
      else
        run_epilogue(a, pair_value(v));
    }
  }
}

}  // namespace

size_t gemv_smem_bytes() { return Cfg::SMEM; }

int gemv_max_grid(int num_sms) { return num_sms; }

void gemv_init() {
  cudaFuncSetAttribute(gemv_dot2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
}

void launch_gemv(const GemvArgs &a, int grid, cudaStream_t s) {
  const int64_t groups = (a.rows + Cfg::ROWS - 1) / Cfg::ROWS;
  const int g = (int)imin64(grid, imax64(groups, 1));
  gemv_dot2_kernel<<<g, kThreads, Cfg::SMEM, s>>>(a);
}

}  // namespace laker
