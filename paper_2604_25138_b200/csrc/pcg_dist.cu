// Row-sharded PCG over NCCL (BASELINE.json north_star: "K is sharded by row
// blocks. Each iteration all-gathers the search direction and all-reduces the
// scalars").  Rank r owns rows [r n/W, (r+1) n/W) of K
// and P and the same slices of alpha, r, q, theta; p is kept full on every
// rank and updated redundantly.  Per iteration (dense P):
//   q_loc = (lambda I + K_loc) p            gemv, unrounded Dot2 pair of p_loc.q_loc
//   allgather(pair)                          -> every rank sums the W pairs in rank
//                                               order: identical delta everywhere
//   alpha_loc, r_loc update; pair ||r_loc||^2 (and r.theta for Jacobi)
//   allgather([r_loc | pairs])               -> full r; ||r||/||y|| test on every rank
//   theta_loc = P_loc r                      gemv, pair r_loc.theta_loc
//   allgather([theta_loc | pair])            -> full theta; beta
//   p = theta + beta p                       (full, redundant)
// With P = I or Jacobi the second and third exchanges merge into one.
// Shipping the unrounded (s, c) pairs and rounding once after the rank-order
// combine keeps every scalar the correctly rounded global value in practice, so
// iteration counts and alpha do not depend on W.
#include <chrono>
#include <thread>

#include "pcg_kernels.cuh"
#include "tri.cuh"

namespace laker {
namespace {

__device__ __forceinline__ double sum_rank_pairs(const double *buf, int64_t stride, int64_t off, int W) {
  dd_pair t = {0.0, 0.0};
  for (int w = 0; w < W; ++w) {
    dd_pair o = {buf[w * stride + off], buf[w * stride + off + 1]};
    pair_add(t, o);
  }
  return pair_value(t);
}

// delta from the gathered p.q pairs; alpha_loc, r_loc update; pack [vec | rr | rt].
// send == null: r_loc is not packed (the factored P needs only the local r); the four
// pair doubles [rr | rt] go to pairs_out (default send + nloc).
__global__ void __launch_bounds__(kVecThreads) dist_update_kernel(
    int64_t nloc, int64_t r0, int pk, const double *__restrict__ dvec, const double *__restrict__ p_full,
    const double *__restrict__ q_loc, double *__restrict__ alpha_loc, double *__restrict__ r_loc,
    double *__restrict__ send, const double *__restrict__ pq_recv, int W, PcgState *st, dd_pair *partials,
    unsigned int *counter, double *pairs_out) {
  if (*(volatile int32_t *)&st->done) return;
  const double pq = sum_rank_pairs(pq_recv, 2, 0, W);
  if (!(pq > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->term = LAKER_TERM_BREAKDOWN;
      st->done = 1;
    }
    return;
  }
  const double delta = __ddiv_rn(st->rho, pq);
  dd_pair v[2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += (int64_t)gridDim.x * blockDim.x) {
    alpha_loc[i] = __fma_rn(delta, p_full[r0 + i], alpha_loc[i]);
    const double ri = __fma_rn(-delta, q_loc[i], r_loc[i]);
    r_loc[i] = ri;
    dot2_step(v[0], ri, ri);
    double th = ri;
    if (pk == LAKER_PRECOND_JACOBI) {
      th = __dmul_rn(dvec[r0 + i], ri);
      dot2_step(v[1], ri, th);
    }
    if (send) send[i] = (pk == LAKER_PRECOND_JACOBI) ? th : ri;
  }
  if (!pairs_out) pairs_out = send + nloc;
  double tot[2];
  // reduce to one pair per quantity; the last block stores the unrounded pairs
  __shared__ dd_pair sred[kVecThreads / 32][2];
  __shared__ int s_last;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int k = 0; k < 2; ++k) {
    dd_pair r = warp_reduce_pair(v[k]);
    if (lane == 0) sred[warp][k] = r;
  }
  __syncthreads();
  if (tid == 0) {
    for (int k = 0; k < 2; ++k) {
      dd_pair t = sred[0][k];
      for (int w = 1; w < kVecThreads / 32; ++w) pair_add(t, sred[w][k]);
      partials[blockIdx.x * 2 + k] = t;
    }
    __threadfence();
    s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  (void)tot;
  if (s_last && warp == 0) {
    __threadfence();
    for (int k = 0; k < 2; ++k) {
      dd_pair t = {0.0, 0.0};
      for (int b = lane; b < (int)gridDim.x; b += 32) {
        dd_pair o = {__ldcg(&partials[b * 2 + k].s), __ldcg(&partials[b * 2 + k].c)};
        pair_add(t, o);
      }
      t = warp_reduce_pair(t);
      if (lane == 0) {
        pairs_out[2 * k] = t.s;
        pairs_out[2 * k + 1] = t.c;
      }
    }
    if (lane == 0) {
      *counter = 0u;
      pcg_set_delta(st, delta);
    }
  }
}

// Unpack [vec | rr | rt] x W into the full vector; block 0 runs the scalar step:
// rel = ||r||/||y||, termination; for P = I / Jacobi also beta.
__global__ void __launch_bounds__(kVecThreads) dist_unpack_r_kernel(int64_t nloc, int W, int pk,
                                                                   const double *__restrict__ recv,
                                                                   double *__restrict__ full, PcgState *st,
                                                                   double *history) {
  if (*(volatile int32_t *)&st->done) return;
  const int64_t stride = nloc + 4;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nloc * W; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = e / nloc, i = e % nloc;
    full[w * nloc + i] = recv[w * stride + i];
  }
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const double rr = sum_rank_pairs(recv, stride, nloc, W);
  const double rel = __ddiv_rn(__dsqrt_rn(rr), st->ynorm);
  const int it = st->iters + 1;
  st->iters = it;
  st->rel = rel;
  if (history) history[it - 1] = rel;
  if (rel <= st->tol) {
    st->term = LAKER_TERM_RESIDUAL_TOL;
    st->done = 1;
    return;
  }
  if (pk == LAKER_PRECOND_NONE || pk == LAKER_PRECOND_JACOBI) {
    const double rho_new = (pk == LAKER_PRECOND_NONE) ? rr : sum_rank_pairs(recv, stride, nloc + 2, W);
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
}

// Dense P: unpack [theta_loc | r.theta pair] x W; beta (or rho at init); budget.
__global__ void __launch_bounds__(kVecThreads) dist_unpack_theta_kernel(int64_t nloc, int W,
                                                                       const double *__restrict__ recv,
                                                                       double *__restrict__ theta_full,
                                                                       double *__restrict__ p_full, int init,
                                                                       PcgState *st) {
  if (*(volatile int32_t *)&st->done) return;
  const int64_t stride = nloc + 2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nloc * W; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = e / nloc, i = e % nloc;
    const double th = recv[w * stride + i];
    theta_full[w * nloc + i] = th;
    if (init) p_full[w * nloc + i] = th;
  }
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const double rho_new = sum_rank_pairs(recv, stride, nloc, W);
  if (!(rho_new > 0.0)) {
    st->term = LAKER_TERM_INDEFINITE;
    st->done = 1;
    return;
  }
  if (init) {
    st->rho = rho_new;
    return;
  }
  pcg_set_beta(st, __ddiv_rn(rho_new, st->rho));
  st->rho = rho_new;
  if (st->iters >= st->max_iters) {
    st->term = LAKER_TERM_MAX_ITERS;
    st->done = 1;
  }
}

// Sharded factored P: the W gathered [z partial pairs (nrp) | rr pair | spare pair] blocks
// -> z_k = RN(sum of the W pairs in rank order) on every rank (the single-GPU Dot2 z_k in
// practice); block 0 then runs the ||r||/||y|| test exactly as dist_unpack_r_kernel
// (skipped at init, before the first iteration).
__global__ void __launch_bounds__(kVecThreads) dist_unpack_z_kernel(int64_t nrp, int W, const double *__restrict__ recv,
                                                                   double *__restrict__ z, PcgState *st,
                                                                   double *history, int init) {
  if (*(volatile int32_t *)&st->done) return;
  const int64_t stride = 2 * nrp + 4;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nrp; k += (int64_t)gridDim.x * blockDim.x)
    z[k] = sum_rank_pairs(recv, stride, 2 * k, W);
  if (init || blockIdx.x != 0 || threadIdx.x != 0) return;
  const double rr = sum_rank_pairs(recv, stride, 2 * nrp, W);
  const double rel = __ddiv_rn(__dsqrt_rn(rr), st->ynorm);
  const int it = st->iters + 1;
  st->iters = it;
  st->rel = rel;
  if (history) history[it - 1] = rel;
  if (rel <= st->tol) {
    st->term = LAKER_TERM_RESIDUAL_TOL;
    st->done = 1;
  }
}

// unrounded pair of x.y over n elements, stored by the last block (on-the-fly operator)
__global__ void __launch_bounds__(kVecThreads) local_pair_kernel(int64_t n, const double *__restrict__ x,
                                                                 const double *__restrict__ y, double *out,
                                                                 const PcgState *st, dd_pair *partials,
                                                                 unsigned int *counter, int residual) {
  if (st && *(volatile const int32_t *)&st->done) return;
  __shared__ dd_pair sred[kVecThreads / 32];
  __shared__ int s_last;
  dd_pair v = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (residual) {
      const double t = __dsub_rn(x[i], y[i]);
      dot2_step(v, t, t);
    } else {
      dot2_step(v, x[i], y[i]);
    }
  }
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  v = warp_reduce_pair(v);
  if (lane == 0) sred[warp] = v;
  __syncthreads();
  if (tid == 0) {
    dd_pair t = sred[0];
    for (int w = 1; w < kVecThreads / 32; ++w) pair_add(t, sred[w]);
    partials[blockIdx.x] = t;
    __threadfence();
    s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last && warp == 0) {
    __threadfence();
    dd_pair t = {0.0, 0.0};
    for (int b = lane; b < (int)gridDim.x; b += 32) {
      dd_pair o = {__ldcg(&partials[b].s), __ldcg(&partials[b].c)};
      pair_add(t, o);
    }
    t = warp_reduce_pair(t);
    if (lane == 0) {
      out[0] = t.s;
      out[1] = t.c;
      *counter = 0u;
    }
  }
}

// The sharded symmetric K apply, own rows: q_i = RN(own pair + the pairs received from
// ranks w - 1, ..., w - D (in that order) + lambda p_i) -- the row's partials summed
// unrounded and rounded once, as symv_finalize_kernel does on one rank; the unrounded
// Dot2 pair p_loc.q_loc -> pair_out (last block).
// own rows of the sharded symmetric apply: q_i = RN(row pair + lambda p_i) and the Dot2
// pair p_loc.q_loc.  fp64 tiles: the row pair is this rank's pair plus the D received pairs
// in rank order; tensor-core tiles (yg != null): the pair of the row's 8 exact level groups,
// already summed over all ranks by the integer reduce-scatter ([8][nloc], tri.cuh).
__global__ void __launch_bounds__(kVecThreads) symv_combine_kernel(
    int64_t nloc, int64_t r0, const dd_pair *__restrict__ own, const dd_pair *__restrict__ recv, int D,
    double lambda, const double *__restrict__ p_full, double *__restrict__ q_loc, const PcgState *st,
    dd_pair *partials, unsigned int *counter, double *pair_out, const long long *__restrict__ yg,
    const int *tc_exp) {
  if (st && *(volatile const int32_t *)&st->done) return;
  __shared__ dd_pair sred[kVecThreads / 32];
  __shared__ int s_last;
  dd_pair v = {0.0, 0.0};
  const int escale = yg != nullptr ? tc_exp[0] + tc_exp[1] + 2 - 14 : 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += (int64_t)gridDim.x * blockDim.x) {
    dd_pair t;
    if (yg != nullptr) {
      long long G[kTcGroups];
#pragma unroll
      for (int g = 0; g < kTcGroups; ++g) G[g] = __ldcg(&yg[g * nloc + i]);
      t = tc_groups_to_pair(G, escale);
    } else {
      const double2 o = __ldcg(reinterpret_cast<const double2 *>(own + i));
      t = dd_pair{o.x, o.y};
      for (int d = 0; d < D; ++d) {
        const double2 r = __ldcg(reinterpret_cast<const double2 *>(recv + (int64_t)d * nloc + i));
        pair_add(t, dd_pair{r.x, r.y});
      }
    }
    const double pi = p_full[r0 + i];
    if (lambda != 0.0) dot2_step(t, lambda, pi);
    const double q = pair_value(t);
    q_loc[i] = q;
    dot2_step(v, pi, q);
  }
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  v = warp_reduce_pair(v);
  if (lane == 0) sred[warp] = v;
  __syncthreads();
  if (tid == 0) {
    dd_pair t = sred[0];
    for (int w = 1; w < kVecThreads / 32; ++w) pair_add(t, sred[w]);
    partials[blockIdx.x] = t;
    __threadfence();
    s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last && warp == 0) {
    __threadfence();
    dd_pair t = {0.0, 0.0};
    for (int b = lane; b < (int)gridDim.x; b += 32) {
      dd_pair o = {__ldcg(&partials[b].s), __ldcg(&partials[b].c)};
      pair_add(t, o);
    }
    t = warp_reduce_pair(t);
    if (lane == 0) {
      if (pair_out) {
        pair_out[0] = t.s;
        pair_out[1] = t.c;
      }
      *counter = 0u;
    }
  }
}

__global__ void dist_true_residual_kernel(const double *recv, int W, const PcgState *st, double *out) {
  const double rr = sum_rank_pairs(recv, 2, 0, W);
  *out = st->ynorm > 0.0 ? __ddiv_rn(__dsqrt_rn(rr), st->ynorm) : 0.0;
}

}  // namespace

laker_status nccl_err(laker_ctx ctx, ncclResult_t r, const char *what) {
  return set_err(ctx, LAKER_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

// Wait for `ev` while watching the communicator: a failed peer or link surfaces as an
// asynchronous NCCL error, on which the communicator is aborted (so no rank blocks in a
// collective forever) and the context loses it (later collective calls fail NOT_READY /
// NCCL).  SPEC's failure kinds map to LAKER_ERR_NCCL here.
laker_status dist_wait(laker_ctx ctx, cudaEvent_t ev) {
  if (!ctx->comm) {
    LAKER_CUDA(ctx, cudaEventSynchronize(ev));
    return LAKER_OK;
  }
  for (int spin = 0;; ++spin) {
    const cudaError_t e = cudaEventQuery(ev);
    if (e == cudaSuccess) return LAKER_OK;
    if (e != cudaErrorNotReady) return cuda_err(ctx, e, "dist_wait");
    ncclResult_t ae = ncclSuccess;
    if (ncclCommGetAsyncError(ctx->comm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress) {
      ncclCommAbort(ctx->comm);
      ctx->comm = nullptr;
      return set_err(ctx, LAKER_ERR_NCCL, std::string("NCCL asynchronous error, communicator aborted: ") +
                                              ncclGetErrorString(ae));
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(spin > 4096 ? 200 : 5));
  }
}

laker_status dist_sync(laker_ctx ctx, cudaStream_t s) {
  cudaEvent_t ev;
  LAKER_CUDA(ctx, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  cudaEventRecord(ev, s);
  const laker_status st = dist_wait(ctx, ev);
  cudaEventDestroy(ev);
  return st;
}

// Workspace of the sharded symmetric apply: the n row pairs of this rank's tiles and the
// pairs received for its rows from ranks w - 1 .. w - D
struct SymvDistBufs {
  dd_pair *ypair = nullptr, *recv = nullptr;
  long long *yown = nullptr;  // tensor-core tiles: this rank's [8][nloc] groups after the reduce-scatter
};

// Sharded symmetric K (tri_plan_dist, symv.cu): this rank's tiles -> row pairs of all n
// rows; the pairs of the rows of ranks w + d (d = 1 .. D = W/2) go to them, the pairs of
// this rank's rows come from ranks w - d; symv_combine_kernel rounds each own row once.
// Per apply a rank streams n^2 / (2 W) entries (the single-GPU triangle / W) and sends and
// receives D n / W pairs.
static laker_status symv_dist_apply(laker_ctx ctx, const double *p_full, double *q_loc, PcgState *st,
                                    double *pair_out, const SymvDistBufs &b, laker_status &err) {
  const int64_t nloc = ctx->r1 - ctx->r0;
  const int W = ctx->world, w = ctx->rank, D = dist_nsend(W);
  const int g = (int)std::min<int64_t>(2 * ctx->num_sms, (nloc + kVecThreads - 1) / kVecThreads);
  if (ctx->k_tc && b.yown) {
    // tensor-core tiles (symv_tc.cu, B13): every row's exact level groups from this rank's
    // tiles, summed over the ranks by an int64 reduce-scatter (exact, order-free: the
    // reduce-scatter of the transposed contributions), then rounded once per own row
    GemvArgs a{};
    a.x = p_full; a.state = st; a.evict_first = true; a.tc = ctx->symv_tc;
    launch_symv(ctx->symv, 0, a, ctx->stream);
    ctx->stats.kernel_launches += 2;
    int64_t cs = 0;
    long long *yacc = symv_tc_groups(ctx->symv_tc, &cs);
    if (ctx->comm) {
      if (ncclReduceScatter(yacc, b.yown, (size_t)kTcGroups * nloc, ncclInt64, ncclSum, ctx->comm, ctx->stream) !=
          ncclSuccess)
        err = LAKER_ERR_NCCL;
    } else {  // detached shard (tests): its own contributions only
      cudaMemcpyAsync(b.yown, yacc + (int64_t)w * kTcGroups * nloc, (size_t)kTcGroups * nloc * sizeof(long long),
                      cudaMemcpyDeviceToDevice, ctx->stream);
    }
    cudaMemsetAsync(yacc, 0, (size_t)kTcGroups * ctx->n * sizeof(long long), ctx->stream);
    symv_combine_kernel<<<g, kVecThreads, 0, ctx->stream>>>(nloc, ctx->r0, nullptr, nullptr, 0, ctx->lambda, p_full,
                                                            q_loc, st, ctx->partials, ctx->counters + kCtrMisc,
                                                            pair_out, b.yown, symv_tc_exponents(ctx->symv_tc));
    ctx->stats.kernel_launches++;
    return err;
  }
  GemvArgs a{};
  a.x = p_full; a.state = st; a.evict_first = true; a.ypair = b.ypair;
  launch_symv(ctx->symv, 0, a, ctx->stream);
  ctx->stats.kernel_launches += 3;
  if (D > 0 && ctx->comm) {
    if (ncclGroupStart() != ncclSuccess) err = LAKER_ERR_NCCL;
    for (int d = 1; d <= D; ++d) {
      const int c = (w + d) % W, src = (w - d + W) % W;
      if (ncclSend(b.ypair + (int64_t)c * nloc, 2 * nloc, ncclDouble, c, ctx->comm, ctx->stream) != ncclSuccess ||
          ncclRecv(b.recv + (int64_t)(d - 1) * nloc, 2 * nloc, ncclDouble, src, ctx->comm, ctx->stream) != ncclSuccess)
        err = LAKER_ERR_NCCL;
    }
    if (ncclGroupEnd() != ncclSuccess) err = LAKER_ERR_NCCL;
  }
  symv_combine_kernel<<<g, kVecThreads, 0, ctx->stream>>>(nloc, ctx->r0, b.ypair + ctx->r0, b.recv,
                                                          ctx->comm ? D : 0, ctx->lambda, p_full, q_loc, st,
                                                          ctx->partials, ctx->counters + kCtrMisc, pair_out,
                                                          nullptr, nullptr);
  return err;
}

static laker_status symv_dist_alloc(laker_ctx ctx, SymvDistBufs &b) {
  const int64_t nloc = ctx->r1 - ctx->r0;
  const int D = dist_nsend(ctx->world);
  LAKER_CUDA(ctx, cudaMallocAsync(&b.ypair, ((size_t)ctx->n + (size_t)std::max(D, 1) * nloc) * sizeof(dd_pair),
                                  ctx->stream));
  b.recv = b.ypair + ctx->n;
  if (ctx->k_tc)
    LAKER_CUDA(ctx, cudaMallocAsync(&b.yown, (size_t)kTcGroups * nloc * sizeof(long long), ctx->stream));
  return LAKER_OK;
}

// q_loc = (lambda I + K_loc) p_full; the unrounded local pair p_loc.q_loc -> pair_out
static void dist_operator(laker_ctx ctx, const double *p_full, double *q_loc, PcgState *st, double *pair_out,
                          const SymvDistBufs *sb = nullptr, laker_status *err = nullptr) {
  const int64_t nloc = ctx->r1 - ctx->r0;
  if (ctx->storage == LAKER_STORE_MATERIALIZED && ctx->k_sym && sb) {
    laker_status e = LAKER_OK;
    symv_dist_apply(ctx, p_full, q_loc, st, pair_out, *sb, e);
    if (e != LAKER_OK && err) *err = e;
    return;
  }
  if (ctx->storage == LAKER_STORE_MATERIALIZED) {
    GemvArgs a{};
    a.A = ctx->K; a.ld = ctx->ld; a.rows = nloc; a.ncols = ctx->n; a.x = p_full; a.row0 = ctx->r0;
    a.y = q_loc; a.lambda = ctx->lambda; a.state = st; a.partials = ctx->partials;
    a.counter = ctx->counters + kCtrGemv; a.epi = pair_out ? kEpiStorePair : kEpiNone;
    a.pair_out = reinterpret_cast<dd_pair *>(pair_out); a.evict_first = true;
    launch_gemv(a, ctx->gemv_grid, ctx->stream);
  } else {
    launch_kernel_matvec_ctx(ctx, ctx->mode, ctx->E + ctx->r0 * ctx->d, nloc, true, ctx->r0, p_full, ctx->lambda,
                             p_full + ctx->r0, q_loc, st ? &st->done : nullptr, ctx->stream);
    if (pair_out) {
      const int g = (int)std::min<int64_t>(2 * ctx->num_sms, (nloc + kVecThreads - 1) / kVecThreads);
      local_pair_kernel<<<g, kVecThreads, 0, ctx->stream>>>(nloc, p_full + ctx->r0, q_loc, pair_out, st,
                                                             ctx->partials, ctx->counters + kCtrMisc, 0);
      ctx->stats.kernel_launches++;
    }
  }
  ctx->stats.kernel_launches++;
}

laker_status apply_operator_dist(laker_ctx ctx, const double *x, double *y) {
  const int64_t nloc = ctx->r1 - ctx->r0;
  cudaStream_t s = ctx->stream;
  double *xp = nullptr, *ql = nullptr;
  LAKER_CUDA(ctx, cudaMallocAsync(&xp, ctx->ld * sizeof(double), s));
  LAKER_CUDA(ctx, cudaMallocAsync(&ql, nloc * sizeof(double), s));
  LAKER_CUDA(ctx, cudaMemsetAsync(xp, 0, ctx->ld * sizeof(double), s));
  LAKER_CUDA(ctx, cudaMemcpyAsync(xp, x, ctx->n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  SymvDistBufs sb;
  if (ctx->k_sym) LAKER_TRY(symv_dist_alloc(ctx, sb));
  laker_status err = LAKER_OK;
  dist_operator(ctx, xp, ql, nullptr, nullptr, &sb, &err);
  if (err != LAKER_OK) return set_err(ctx, err, "apply: NCCL exchange failed");
  LAKER_NCCL(ctx, ncclAllGather(ql, y, nloc, ncclDouble, ctx->comm, s));
  LAKER_CUDA(ctx, cudaGetLastError());
  cudaFreeAsync(xp, s);
  cudaFreeAsync(ql, s);
  if (sb.ypair) cudaFreeAsync(sb.ypair, s);
  if (sb.yown) cudaFreeAsync(sb.yown, s);
  return LAKER_OK;
}

laker_status pcg_solve_dist(laker_ctx ctx, const double *y, double *alpha_out, const laker_solve_opts &o,
                            laker_solve_report *rep, double *history) {
  const int64_t n = ctx->n, ld = ctx->ld, r0 = ctx->r0, nloc = ctx->r1 - ctx->r0;
  const int W = ctx->world;
  const int pk = ctx->precond_kind;
  const bool dense = (pk == LAKER_PRECOND_LEARNED || pk == LAKER_PRECOND_EXTERNAL_DENSE);
  // factored P (SURVEY §8(f) NEXT-1 on the sharded path), rank-local factors (fit.cu):
  // z = Q^T r = sum over ranks of Q_loc^T r_loc, so each rank streams its columns of Q^T
  // against its own r rows into N_r unrounded Dot2 pairs, the W blocks are all-gathered
  // (with the ||r||^2 pair) and every rank sums them in rank order and rounds once: the
  // single-GPU z in practice, and no r exchange.  Then theta_loc = a^{-1/2} r_loc +
  // QM_loc z (QM form), or w = M z by row blocks of M + all-gather and theta_loc =
  // a^{-1/2} r_loc + Q_loc w (three passes).  P bytes per rank: 16 (n/W) N_r (+ 8 N_r^2 / W).
  const bool fac = dense && ctx->p_factored && ctx->f_local;
  if (dense && !fac) LAKER_TRY(ensure_dense_p(ctx));  // a factored P is expanded once to its rows
  if (dense && !fac && !ctx->P) return set_err(ctx, LAKER_ERR_NOT_READY, "dense preconditioner not set");
  if (pk == LAKER_PRECOND_JACOBI && !ctx->Pdiag) return set_err(ctx, LAKER_ERR_NOT_READY, "Jacobi diagonal not set");
  const int32_t max_iters = o.max_iters > 0 ? o.max_iters : (int32_t)std::min<int64_t>(10 * n, 1 << 30);
  cudaStream_t s = ctx->stream;

  // full vectors (ld): y, r (full copy for dense P), theta, p, alpha_full; local: alpha, r, q;
  // exchange buffers: pq pair, [vec|4] send/recv, [theta|2] send/recv, scalars.
  // (r_loc is zero padded to a whole number of GEMV chunks: it streams against Q^T's columns)
  double *base = nullptr;
  const int64_t ldl = padded_ld(nloc), nzp = fac ? 2 * ctx->f_nrp + 4 : 0;
  const size_t nfull = 5 * (size_t)ld, nl = 2 * (size_t)nloc + ldl;
  const size_t nx = 2 + 2 * (size_t)W + (nloc + 4) + (size_t)W * (nloc + 4) + (nloc + 2) + (size_t)W * (nloc + 2) + 4 +
                    (size_t)(W + 1) * nzp;
  LAKER_CUDA(ctx, cudaMallocAsync(&base, (nfull + nl + nx) * sizeof(double), s));
  LAKER_CUDA(ctx, cudaMemsetAsync(base, 0, (nfull + nl + nx) * sizeof(double), s));
  double *yf = base, *rf = yf + ld, *thf = rf + ld, *pf = thf + ld, *af = pf + ld;
  double *al = af + ld, *rl = al + nloc, *ql = rl + ldl;
  double *pq_send = ql + nloc, *pq_recv = pq_send + 2, *vsend = pq_recv + 2 * W, *vrecv = vsend + (nloc + 4);
  double *tsend = vrecv + (size_t)W * (nloc + 4), *trecv = tsend + (nloc + 2), *scal = trecv + (size_t)W * (nloc + 2);
  double *zsend = scal + 4, *zrecv = zsend + nzp;
  SymvDistBufs sb;
  if (ctx->k_sym && ctx->storage == LAKER_STORE_MATERIALIZED) LAKER_TRY(symv_dist_alloc(ctx, sb));
  PcgState *st = nullptr;
  double *hist = nullptr;
  LAKER_CUDA(ctx, cudaMallocAsync(&st, sizeof(PcgState), s));
  LAKER_CUDA(ctx, cudaMallocAsync(&hist, (size_t)3 * max_iters * sizeof(double), s));
  double *dh = hist + max_iters, *bh = dh + max_iters;  // CG coefficients (Lanczos estimates)
  LAKER_CUDA(ctx, cudaMemcpyAsync(yf, y, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  LAKER_CUDA(ctx, cudaMemcpyAsync(rl, y + r0, nloc * sizeof(double), cudaMemcpyDeviceToDevice, s));
  PcgState h0{};
  h0.tol = o.tol;
  h0.max_iters = max_iters;
  h0.dh = dh;
  h0.bh = bh;
  LAKER_CUDA(ctx, cudaMemcpyAsync(st, &h0, sizeof(PcgState), cudaMemcpyHostToDevice, s));

  const int vg = (int)std::min<int64_t>(2 * ctx->num_sms, (n + kVecThreads - 1) / kVecThreads);
  const int lg = (int)std::min<int64_t>(2 * ctx->num_sms, (nloc + kVecThreads - 1) / kVecThreads);
  cudaEvent_t ev0, ev1;
  cudaEventCreate(&ev0);
  cudaEventCreate(&ev1);
  cudaEventRecord(ev0, s);
  // init: ||y|| on the full (replicated) y; alpha = 0; r_full = y
  laker_status err = LAKER_OK;
  // theta_loc (-> tsend, r_loc.theta_loc pair -> tsend + nloc) = P r for the full r in rf
  auto apply_p = [&]() {
    GemvArgs a{};
    a.state = st; a.partials = ctx->partials; a.counter = ctx->counters + kCtrGemv; a.evict_first = true;
    if (!fac) {
      a.A = ctx->P; a.ld = ld; a.rows = nloc; a.ncols = n; a.x = rf; a.row0 = r0; a.y = tsend; a.lambda = 0.0;
      a.epi = kEpiStorePair; a.pair_out = reinterpret_cast<dd_pair *>(tsend + nloc);
      launch_gemv(a, ctx->gemv_grid, s);
      return;
    }
    const int64_t nrp = ctx->f_nrp, ldq = ctx->f_ldq;
    // z (fz) was formed from the gathered partials (z_partials + dist_unpack_z_kernel)
    if (ctx->p_qm) {  // R21: theta_loc = a^-1/2 r_loc + QM_loc z
      GemvArgs t = a;
      t.A = ctx->QMf; t.ld = ldq; t.rows = nloc; t.ncols = nrp; t.x = ctx->fz; t.row0 = 0; t.y = tsend;
      t.lambda = ctx->f_ainv; t.xd = rl; t.epi = kEpiStorePair; t.pair_out = reinterpret_cast<dd_pair *>(tsend + nloc);
      launch_gemv(t, ctx->gemv_grid, s);
      ctx->stats.kernel_launches += 1;
      return;
    }
    // w = M z by row blocks of M (all of it on every rank when W does not divide nrp)
    const bool split = nrp % W == 0;
    const int64_t nk = split ? nrp / W : nrp, k0 = split ? nk * ctx->rank : 0;
    GemvArgs w = a;  // w[k0 .. k0+nk) = M[k0.., :] z
    w.A = ctx->Mf + k0 * ldq; w.ld = ldq; w.rows = nk; w.ncols = nrp; w.x = ctx->fz; w.row0 = k0; w.y = ctx->fw + k0;
    w.epi = kEpiNone; w.evict_first = false;
    launch_gemv(w, ctx->gemv_grid, s);
    if (split && W > 1 && ncclAllGather(ctx->fw + k0, ctx->fw, nk, ncclDouble, ctx->comm, s) != ncclSuccess)
      err = LAKER_ERR_NCCL;
    GemvArgs t = a;  // theta_loc = a^{-1/2} r_loc + Q_loc w, pair r_loc.theta_loc
    t.A = ctx->Qr; t.ld = ldq; t.rows = nloc; t.ncols = nrp; t.x = ctx->fw; t.row0 = 0; t.y = tsend;
    t.lambda = ctx->f_ainv; t.xd = rl; t.epi = kEpiStorePair; t.pair_out = reinterpret_cast<dd_pair *>(tsend + nloc);
    launch_gemv(t, ctx->gemv_grid, s);
    ctx->stats.kernel_launches += 2;
  };
  // the unrounded pairs of Q_loc^T r_loc (nrp) -> zsend, all-gathered, summed in rank order
  auto z_partials = [&](int init) {
    const int64_t nrp = ctx->f_nrp;
    GemvArgs z{};
    z.A = ctx->Qt; z.ld = ctx->f_ldl; z.rows = nrp; z.ncols = nloc; z.x = rl; z.row0 = 0;
    z.ypair = reinterpret_cast<dd_pair *>(zsend); z.state = st; z.partials = ctx->partials;
    z.counter = ctx->counters + kCtrGemv; z.epi = kEpiNone; z.evict_first = true;
    launch_gemv(z, ctx->gemv_grid, s);
    if (ncclAllGather(zsend, zrecv, 2 * nrp + 4, ncclDouble, ctx->comm, s) != ncclSuccess) err = LAKER_ERR_NCCL;
    const int zg = (int)std::min<int64_t>(ctx->num_sms, (nrp + kVecThreads - 1) / kVecThreads);
    dist_unpack_z_kernel<<<zg, kVecThreads, 0, s>>>(nrp, W, zrecv, ctx->fz, st, hist, init);
    ctx->stats.kernel_launches += 2;
  };
  pcg_init_kernel<<<vg, kVecThreads, 0, s>>>(n, yf, af, rf, st, ctx->partials, ctx->counters + kCtrInit);
  ctx->stats.kernel_launches++;
  if (dense) {
    if (fac) z_partials(1);
    apply_p();
    LAKER_NCCL(ctx, ncclAllGather(tsend, trecv, nloc + 2, ncclDouble, ctx->comm, s));
    dist_unpack_theta_kernel<<<vg, kVecThreads, 0, s>>>(nloc, W, trecv, thf, pf, 1, st);
    ctx->stats.kernel_launches += 2;
  } else {
    // theta = r (none) or d o r (Jacobi) on the full vector, p = theta, rho = r.theta
    pcg_first_dir_kernel<<<vg, kVecThreads, 0, s>>>(n, pk, ctx->Pdiag, rf, thf, pf, st, ctx->partials,
                                                    ctx->counters + kCtrInit);
    ctx->stats.kernel_launches++;
  }
  LAKER_CUDA(ctx, cudaGetLastError());

  const double *theta_src = dense ? thf : (pk == LAKER_PRECOND_NONE ? rf : thf);
  const int chunk = n >= 8192 ? 8 : (n >= 2048 ? 32 : 64);
  const bool instr = o.instrument != 0;
  std::vector<cudaEvent_t> evs;
  if (instr) {
    evs.resize(4 * chunk);
    for (auto &e : evs) cudaEventCreate(&e);
  }
  auto record_iteration = [&](int j) {
    if (instr) cudaEventRecordWithFlags(evs[4 * j + 0], s, cudaEventRecordExternal);
    dist_operator(ctx, pf, ql, st, pq_send, &sb, &err);
    if (instr) cudaEventRecordWithFlags(evs[4 * j + 1], s, cudaEventRecordExternal);
    if (ncclAllGather(pq_send, pq_recv, 2, ncclDouble, ctx->comm, s) != ncclSuccess) err = LAKER_ERR_NCCL;
    if (fac) {
      // sharded factored P: no r exchange -- the local r feeds the z partials, which
      // travel with the ||r||^2 pair
      dist_update_kernel<<<lg, kVecThreads, 0, s>>>(nloc, r0, pk, ctx->Pdiag, pf, ql, al, rl, nullptr, pq_recv, W,
                                                    st, ctx->partials, ctx->counters + kCtrUpdate, zsend + 2 * ctx->f_nrp);
      ctx->stats.kernel_launches++;
    } else {
      dist_update_kernel<<<lg, kVecThreads, 0, s>>>(nloc, r0, pk, ctx->Pdiag, pf, ql, al, rl, vsend, pq_recv, W, st,
                                                    ctx->partials, ctx->counters + kCtrUpdate, nullptr);
      if (ncclAllGather(vsend, vrecv, nloc + 4, ncclDouble, ctx->comm, s) != ncclSuccess) err = LAKER_ERR_NCCL;
      // dense: the exchange carried r; otherwise theta (Jacobi) or r (= theta, none)
      dist_unpack_r_kernel<<<vg, kVecThreads, 0, s>>>(nloc, W, pk, vrecv,
                                                      dense ? rf : (pk == LAKER_PRECOND_NONE ? rf : thf), st, hist);
      ctx->stats.kernel_launches += 2;
    }
    if (dense) {
      if (instr) cudaEventRecordWithFlags(evs[4 * j + 2], s, cudaEventRecordExternal);
      if (fac) z_partials(0);
      apply_p();
      if (instr) cudaEventRecordWithFlags(evs[4 * j + 3], s, cudaEventRecordExternal);
      if (ncclAllGather(tsend, trecv, nloc + 2, ncclDouble, ctx->comm, s) != ncclSuccess) err = LAKER_ERR_NCCL;
      dist_unpack_theta_kernel<<<vg, kVecThreads, 0, s>>>(nloc, W, trecv, thf, pf, 0, st);
      ctx->stats.kernel_launches += 2;
    }
    pcg_pupdate_kernel<<<vg, kVecThreads, 0, s>>>(n, theta_src, pf, st);
    ctx->stats.kernel_launches++;
  };

  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  const int64_t launches_before = ctx->stats.kernel_launches;
  LAKER_CUDA(ctx, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int j = 0; j < chunk; ++j) record_iteration(j);
  LAKER_CUDA(ctx, cudaStreamEndCapture(s, &graph));
  if (err != LAKER_OK) return set_err(ctx, err, "ncclAllGather failed during capture");
  const int64_t per_chunk = ctx->stats.kernel_launches - launches_before;
  ctx->stats.kernel_launches = launches_before;
  LAKER_CUDA(ctx, cudaGraphInstantiate(&gexec, graph, 0));

  PcgState *hs = nullptr;
  LAKER_CUDA(ctx, cudaMallocHost(&hs, 2 * sizeof(PcgState)));
  LAKER_CUDA(ctx, cudaMemcpyAsync(hs, st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
  LAKER_TRY(dist_sync(ctx, s));
  int32_t iters_prev = 0;
  if (!instr && !hs->done) {
    // one chunk always queued ahead of the host's check (as pcg.cu): every rank decides
    // termination from identical scalars, so all ranks launch the same number of chunks
    // and the collectives inside them match; chunks after termination are no-ops
    cudaEvent_t ce[2];
    cudaEventCreateWithFlags(&ce[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ce[1], cudaEventDisableTiming);
    PcgState *slot[2] = {hs, hs + 1};
    int cur = 0;
    LAKER_CUDA(ctx, cudaGraphLaunch(gexec, s));
    ctx->stats.kernel_launches += per_chunk;
    LAKER_CUDA(ctx, cudaMemcpyAsync(slot[0], st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    cudaEventRecord(ce[0], s);
    laker_status werr = LAKER_OK;
    for (;;) {
      LAKER_CUDA(ctx, cudaGraphLaunch(gexec, s));
      ctx->stats.kernel_launches += per_chunk;
      LAKER_CUDA(ctx, cudaMemcpyAsync(slot[cur ^ 1], st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
      cudaEventRecord(ce[cur ^ 1], s);
      if ((werr = dist_wait(ctx, ce[cur])) != LAKER_OK) break;
      if (slot[cur]->done) break;
      cur ^= 1;
    }
    if (werr == LAKER_OK) werr = dist_sync(ctx, s);
    cudaEventDestroy(ce[0]);
    cudaEventDestroy(ce[1]);
    if (werr != LAKER_OK) return werr;
    *hs = *slot[cur ^ 1];
  }
  while (!hs->done) {
    LAKER_CUDA(ctx, cudaGraphLaunch(gexec, s));
    ctx->stats.kernel_launches += per_chunk;
    LAKER_CUDA(ctx, cudaMemcpyAsync(hs, st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    LAKER_TRY(dist_sync(ctx, s));
    if (instr) {
      const int ran = hs->iters - iters_prev;
      for (int j = 0; j < std::min(ran, chunk); ++j) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, evs[4 * j + 0], evs[4 * j + 1]) != cudaSuccess) { cudaGetLastError(); ms = 0.f; }
        ctx->stats.op_ms += ms;
        ctx->stats.op_launches++;
        if (dense && (j < ran - 1 || !hs->done || hs->term != LAKER_TERM_RESIDUAL_TOL)) {
          if (cudaEventElapsedTime(&ms, evs[4 * j + 2], evs[4 * j + 3]) != cudaSuccess) { cudaGetLastError(); ms = 0.f; }
          ctx->stats.prec_ms += ms;
          ctx->stats.prec_launches++;
        }
      }
    }
    iters_prev = hs->iters;
  }
  cudaEventRecord(ev1, s);

  // alpha_full on every rank, true residual over the shards
  LAKER_NCCL(ctx, ncclAllGather(al, af, nloc, ncclDouble, ctx->comm, s));
  dist_operator(ctx, af, ql, nullptr, nullptr, &sb, &err);
  local_pair_kernel<<<lg, kVecThreads, 0, s>>>(nloc, yf + r0, ql, pq_send, nullptr, ctx->partials,
                                               ctx->counters + kCtrMisc, 1);
  LAKER_NCCL(ctx, ncclAllGather(pq_send, pq_recv, 2, ncclDouble, ctx->comm, s));
  dist_true_residual_kernel<<<1, 1, 0, s>>>(pq_recv, W, st, scal);
  ctx->stats.kernel_launches += 2;
  LAKER_CUDA(ctx, cudaMemcpyAsync(alpha_out, af, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  double true_rel = 0.0;
  LAKER_CUDA(ctx, cudaMemcpyAsync(&true_rel, scal, sizeof(double), cudaMemcpyDeviceToHost, s));
  LAKER_CUDA(ctx, cudaMemcpyAsync(hs, st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  if (history && hs->iters > 0)
    LAKER_CUDA(ctx, cudaMemcpyAsync(history, hist, (size_t)hs->iters * sizeof(double), cudaMemcpyDeviceToHost, s));
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev0, ev1);
  ctx->stats.solve_ms = ms;
  if (rep) {
    if (hs->iters > 0) {
      LAKER_CUDA(ctx, cudaStreamSynchronize(s));
      std::vector<double> hd(hs->iters), hb(hs->iters);
      cudaMemcpy(hd.data(), dh, hs->iters * sizeof(double), cudaMemcpyDeviceToHost);
      cudaMemcpy(hb.data(), bh, hs->iters * sizeof(double), cudaMemcpyDeviceToHost);
      lanczos_extremes(hd, hb, hs->iters, rep->lanczos_lmin, rep->lanczos_lmax);
    }
    rep->iters = hs->iters;
    rep->termination = hs->term;
    rep->rel_residual = hs->iters > 0 ? hs->rel : (hs->term == LAKER_TERM_ZERO_RHS ? 0.0 : 1.0);
    rep->true_rel_residual = true_rel;
    rep->seconds = ms * 1e-3;
  }
  const int term = hs->term;
  cudaFreeHost(hs);
  for (auto &e : evs) cudaEventDestroy(e);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  cudaGraphExecDestroy(gexec);
  cudaGraphDestroy(graph);
  cudaFreeAsync(base, s);
  if (sb.ypair) cudaFreeAsync(sb.ypair, s);
  if (sb.yown) cudaFreeAsync(sb.yown, s);
  cudaFreeAsync(st, s);
  cudaFreeAsync(hist, s);
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  if (term == LAKER_TERM_BREAKDOWN) return set_err(ctx, LAKER_ERR_BREAKDOWN_ZERO_CURVATURE, "p.(lambda I + K)p <= 0");
  if (term == LAKER_TERM_INDEFINITE) return set_err(ctx, LAKER_ERR_INDEFINITE_PRECONDITIONER, "r.theta <= 0");
  return LAKER_OK;
}

}  // namespace laker

// ------------------------------------------------------------------ test hooks
// (include/laker.h: the pieces of the sharded symmetric apply on a detached shard)
namespace {
laker_status copy_in(laker_ctx ctx, double *dst, const double *src, size_t count) {
  LAKER_CUDA(ctx, cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyDefault, ctx->stream));
  return LAKER_OK;
}
}  // namespace

extern "C" laker_status laker_debug_dist_tiles(int64_t n, int32_t br, int32_t tc, int32_t rank, int32_t world,
                                               int64_t *counts, int64_t *toff, int32_t *jt, int32_t *cr_lo,
                                               int32_t *cr_hi) {
  std::vector<int64_t> t;
  std::vector<int32_t> j, lo, hi;
  if (!counts || !laker::dist_tiles(n, br, tc, rank, world, t, j, lo, hi)) return LAKER_ERR_INVALID_ARGUMENT;
  counts[0] = (int64_t)t.size() - 1;
  counts[1] = (int64_t)j.size();
  counts[2] = (int64_t)lo.size();
  if (toff) std::copy(t.begin(), t.end(), toff);
  if (jt) std::copy(j.begin(), j.end(), jt);
  if (cr_lo) std::copy(lo.begin(), lo.end(), cr_lo);
  if (cr_hi) std::copy(hi.begin(), hi.end(), cr_hi);
  return LAKER_OK;
}

extern "C" laker_status laker_debug_dist_symv_partials(laker_ctx ctx, const double *x, const double *rowmax,
                                                       double *pairs) {
  using namespace laker;
  if (!ctx || !x || !pairs) return LAKER_ERR_INVALID_ARGUMENT;
  if (!ctx->k_sym || !tri_is_dist(ctx->symv)) return set_err(ctx, LAKER_ERR_NOT_READY, "no sharded symmetric K");
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  double *xp = nullptr, *yp = nullptr;
  LAKER_CUDA(ctx, cudaMallocAsync(&xp, ctx->ld * sizeof(double), s));
  LAKER_CUDA(ctx, cudaMallocAsync(&yp, 2 * ctx->n * sizeof(double), s));
  LAKER_CUDA(ctx, cudaMemsetAsync(xp, 0, ctx->ld * sizeof(double), s));
  LAKER_TRY(copy_in(ctx, xp, x, ctx->n));
  if (rowmax) LAKER_TRY(copy_in(ctx, symv_rowmax_ptr(ctx->symv, 0), rowmax, ctx->n));
  GemvArgs a{};
  a.x = xp; a.evict_first = true; a.ypair = reinterpret_cast<dd_pair *>(yp);
  launch_symv(ctx->symv, 0, a, s);
  LAKER_CUDA(ctx, cudaMemcpyAsync(pairs, yp, 2 * ctx->n * sizeof(double), cudaMemcpyDefault, s));
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  cudaFree(xp);
  cudaFree(yp);
  return LAKER_OK;
}

extern "C" laker_status laker_debug_dist_symv_combine(laker_ctx ctx, const double *x, const double *own,
                                                      const double *recv, double *q_loc, double *pq_pair) {
  using namespace laker;
  if (!ctx || !x || !own || !q_loc) return LAKER_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  const int64_t nloc = ctx->r1 - ctx->r0;
  const int D = dist_nsend(ctx->world);
  double *xp = nullptr, *buf = nullptr, *q = nullptr;
  LAKER_CUDA(ctx, cudaMallocAsync(&xp, ctx->ld * sizeof(double), s));
  LAKER_CUDA(ctx, cudaMallocAsync(&buf, (2 * nloc * (1 + std::max(D, 1)) + nloc + 2) * sizeof(double), s));
  q = buf + 2 * nloc * (1 + std::max(D, 1));
  LAKER_CUDA(ctx, cudaMemsetAsync(xp, 0, ctx->ld * sizeof(double), s));
  LAKER_TRY(copy_in(ctx, xp, x, ctx->n));
  LAKER_TRY(copy_in(ctx, buf, own, 2 * nloc));
  if (D > 0 && recv) LAKER_TRY(copy_in(ctx, buf + 2 * nloc, recv, 2 * nloc * D));
  const int g = (int)std::min<int64_t>(2 * ctx->num_sms, (nloc + kVecThreads - 1) / kVecThreads);
  symv_combine_kernel<<<g, kVecThreads, 0, s>>>(nloc, ctx->r0, reinterpret_cast<const dd_pair *>(buf),
                                                reinterpret_cast<const dd_pair *>(buf + 2 * nloc), recv ? D : 0,
                                                ctx->lambda, xp, q, nullptr, ctx->partials, ctx->counters + kCtrMisc,
                                                q + nloc, nullptr, nullptr);
  LAKER_CUDA(ctx, cudaMemcpyAsync(q_loc, q, nloc * sizeof(double), cudaMemcpyDefault, s));
  if (pq_pair) LAKER_CUDA(ctx, cudaMemcpyAsync(pq_pair, q + nloc, 2 * sizeof(double), cudaMemcpyDefault, s));
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  cudaFree(xp);
  cudaFree(buf);
  return LAKER_OK;
}

extern "C" laker_status laker_debug_tc_groups(laker_ctx ctx, const double *x, const double *rowmax, int64_t *groups) {
  using namespace laker;
  if (!ctx || !x || !groups) return LAKER_ERR_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  if (!ctx->k_sym || ctx->storage != LAKER_STORE_MATERIALIZED)
    return set_err(ctx, LAKER_ERR_NOT_READY, "no symmetric stored K");
  if (rowmax) {  // the full row maxima -> the global slice exponent of K (re-slices this rank's tiles)
    LAKER_TRY(copy_in(ctx, symv_rowmax_ptr(ctx->symv, 0), rowmax, ctx->n));
    ctx->k_tc = symv_tc_prepare(ctx->symv_tc, ctx->K, ctx->n, ctx->ld, symv_rowmax_ptr(ctx->symv, 0), s, ctx->rank,
                                ctx->world);
  }
  if (!ctx->k_tc) return set_err(ctx, LAKER_ERR_NOT_READY, "K does not use the tensor-core apply");
  const int64_t n = ctx->n;
  std::vector<double> hx(n);
  LAKER_CUDA(ctx, cudaMemcpy(hx.data(), x, n * sizeof(double), cudaMemcpyDefault));
  double xm = 0.0;
  for (double v : hx) xm = std::max(xm, std::fabs(v));
  double *xp = nullptr;
  LAKER_CUDA(ctx, cudaMallocAsync(&xp, (ctx->ld + 1) * sizeof(double), s));
  LAKER_CUDA(ctx, cudaMemsetAsync(xp, 0, ctx->ld * sizeof(double), s));
  LAKER_CUDA(ctx, cudaMemcpyAsync(xp, hx.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
  LAKER_CUDA(ctx, cudaMemcpyAsync(xp + ctx->ld, &xm, sizeof(double), cudaMemcpyHostToDevice, s));
  SymvArgs a{};
  a.x = xp;
  a.xparts = xp + ctx->ld;  // max |x| as the single per-CTA part
  a.nxparts = 1;
  launch_symv_tc(ctx->symv_tc, a, s);
  int64_t cs = 0;
  long long *yacc = symv_tc_groups(ctx->symv_tc, &cs);
  const int64_t chunks = (ctx->world == 1) ? 1 : ctx->world;
  std::vector<long long> h((size_t)chunks * kTcGroups * cs);
  LAKER_CUDA(ctx, cudaMemcpyAsync(h.data(), yacc, h.size() * sizeof(long long), cudaMemcpyDeviceToHost, s));
  LAKER_CUDA(ctx, cudaMemsetAsync(yacc, 0, h.size() * sizeof(long long), s));
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  cudaFree(xp);
  std::vector<int64_t> out((size_t)kTcGroups * n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t c = i / cs;
    for (int g = 0; g < kTcGroups; ++g) out[(size_t)g * n + i] = h[(size_t)(c * kTcGroups + g) * cs + (i - c * cs)];
  }
  LAKER_CUDA(ctx, cudaMemcpy(groups, out.data(), out.size() * sizeof(int64_t), cudaMemcpyDefault));
  return LAKER_OK;
}
