// Streaming fp64 Dot2 GEMV: the per-iteration K.p and P.r products of the PCG
// (Alg. 1 l.16-21) -- HBM-bound.
//
// Layout: A is the local row block of K (or P), row-major with a padded stride
// `ld` (multiple of 256 doubles, zero padding).  Work unit = a group of 8 rows
// x one 1024-column chunk (64 KiB) plus the matching 1024-entry chunk of x
// (8 KiB).  One persistent CTA per SM owns a contiguous range of row groups.
// A producer warp streams the units into a 3-stage shared-memory ring with
// 1-D bulk copies (cp.async.bulk, TMA engine; A with an L2 evict-first policy,
// x evict-last) signalled on mbarriers; 16 consumer warps read the ring, each
// thread 2 columns x 8 rows, so the x chunk never costs a dependent global
// load.  Each thread keeps one Dot2 pair per row; rows are reduced warp ->
// CTA in a fixed order, so y_i = RN(lambda x_i + sum_j A_ij x_j) is correctly
// rounded in practice and bitwise equal to the oracle's sequential Dot2.
// The CTA also accumulates dot(x_local, y) as a Dot2 pair; the last CTA to
// finish reduces the per-CTA pairs in CTA order and runs the PCG scalar
// epilogue (delta = rho / p.q, or beta = rho'/rho) in the same kernel.
#include "laker_internal.h"
#include "tma.cuh"

namespace laker {
namespace {

constexpr int kRows = 8;
constexpr int kCPT = 2;
constexpr int kConsumers = 512;
constexpr int kWarps = kConsumers / 32;
constexpr int kChunk = kConsumers * kCPT;  // 1024 doubles
constexpr int kStages = 3;
constexpr int kThreads = kConsumers + 32;
constexpr size_t kStageDoubles = (size_t)(kRows + 1) * kChunk;  // 8 rows of A + the x chunk
constexpr size_t kSmem = kStages * kStageDoubles * sizeof(double) + kWarps * kRows * sizeof(dd_pair) +
                         2 * kStages * sizeof(uint64_t) + 16;

__device__ __forceinline__ void run_epilogue(const GemvArgs &a, double v) {
  PcgState *st = a.state;
  switch (a.epi) {
    case kEpiDelta:
      if (!(v > 0.0)) {
        st->term = LAKER_TERM_BREAKDOWN;
        st->done = 1;
      } else {
        st->delta = __ddiv_rn(st->rho, v);
      }
      break;
    case kEpiBeta:
      if (!(v > 0.0)) {
        st->term = LAKER_TERM_INDEFINITE;
        st->done = 1;
      } else {
        st->beta = __ddiv_rn(v, st->rho);
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
  if (a.state != nullptr && *(volatile int32_t *)&a.state->done) return;
  extern __shared__ __align__(128) unsigned char smem[];
  double *ring = reinterpret_cast<double *>(smem);
  dd_pair *red = reinterpret_cast<dd_pair *>(smem + kStages * kStageDoubles * sizeof(double));
  uint64_t *full = reinterpret_cast<uint64_t *>(red + kWarps * kRows);
  uint64_t *empty = full + kStages;
  __shared__ int s_last;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t groups = (a.rows + kRows - 1) / kRows;
  const int64_t g0 = groups * blockIdx.x / gridDim.x;
  const int64_t g1 = groups * (blockIdx.x + 1) / gridDim.x;
  const int64_t ncp = (a.ncols + 255) / 256 * 256;  // padded columns actually streamed
  const int64_t nchunks = (ncp + kChunk - 1) / kChunk;

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
      int64_t it = 0;
      for (int64_t g = g0; g < g1; ++g) {
        const int64_t rb = g * kRows;
        const int nr = (int)imin64(kRows, a.rows - rb);
        for (int64_t c = 0; c < nchunks; ++c, ++it) {
          const int slot = (int)(it % kStages);
          if (it >= kStages) mbar_wait(&empty[slot], (uint32_t)(((it / kStages) - 1) & 1));
          const int64_t col0 = c * kChunk;
          const int width = (int)imin64(kChunk, ncp - col0);
          const uint32_t bytes = (uint32_t)width * 8u;
          mbar_arrive_expect_tx(&full[slot], bytes * (uint32_t)(nr + 1));
          double *dst = ring + slot * kStageDoubles;
          bulk_g2s(dst + kRows * kChunk, a.x + col0, bytes, &full[slot], pol_x);
          for (int r = 0; r < nr; ++r)
            bulk_g2s(dst + r * kChunk, a.A + (rb + r) * a.ld + col0, bytes, &full[slot], pol_a);
        }
      }
    }
    return;
  }

  // ---------------- consumer warps
  dd_pair part = {0.0, 0.0};
  const int cb = tid * kCPT;
  int64_t it = 0;
  for (int64_t g = g0; g < g1; ++g) {
    const int64_t rb = g * kRows;
    const int nr = (int)imin64(kRows, a.rows - rb);
    dd_pair acc[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) acc[r] = dd_pair{0.0, 0.0};
    if (tid == 0 && a.lambda != 0.0) {
#pragma unroll
      for (int r = 0; r < kRows; ++r)
        if (r < nr) dot2_step(acc[r], a.lambda, a.x[a.row0 + rb + r]);
    }
    for (int64_t c = 0; c < nchunks; ++c, ++it) {
      const int slot = (int)(it % kStages);
      mbar_wait(&full[slot], (uint32_t)((it / kStages) & 1));
      const int64_t col0 = c * kChunk;
      const int width = (int)imin64(kChunk, ncp - col0);
      if (cb < width) {
        const double *sp = ring + slot * kStageDoubles + cb;
        const double2 x0 = *reinterpret_cast<const double2 *>(sp + kRows * kChunk);
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
          if (r < nr) {
            const double2 v0 = *reinterpret_cast<const double2 *>(sp + r * kChunk);
            dot2_step(acc[r], v0.x, x0.x);
            dot2_step(acc[r], v0.y, x0.y);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
    // rows: warp butterfly, then the warp pairs in warp order
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const dd_pair v = warp_reduce_pair(acc[r]);
      if (lane == 0) red[warp * kRows + r] = v;
    }
    named_bar_sync(1, kConsumers);
    if (warp == 0 && lane < nr) {
      dd_pair t = red[lane];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) pair_add(t, red[w * kRows + lane]);
      const double yv = pair_value(t);
      a.y[rb + lane] = yv;
      dot2_step(part, a.x[a.row0 + rb + lane], yv);
    }
    named_bar_sync(1, kConsumers);
  }

  // ---------------- CTA partial of dot(x_local, y), then the last CTA reduces
  if (warp == 0) {
    const dd_pair v = warp_reduce_pair(part);
    if (lane == 0) {
      a.partials[blockIdx.x] = v;
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
      dd_pair o;
      o.s = __ldcg(&a.partials[i].s);
      o.c = __ldcg(&a.partials[i].c);
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

size_t gemv_smem_bytes() { return kSmem; }

int gemv_max_grid(int num_sms) { return num_sms; }

void gemv_init() {
  cudaFuncSetAttribute(gemv_dot2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
}

void launch_gemv(const GemvArgs &a, int grid, cudaStream_t s) {
  const int64_t groups = (a.rows + kRows - 1) / kRows;
  int g = (int)imin64(grid, imax64(groups, 1));
  gemv_dot2_kernel<<<g, kThreads, kSmem, s>>>(a);
}

}  // namespace laker
