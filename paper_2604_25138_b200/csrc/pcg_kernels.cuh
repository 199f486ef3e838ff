// Shared PCG vector kernels (single-rank solver in pcg.cu, row-sharded solver
// in pcg_dist.cu).  Each translation unit gets its own copy (anonymous namespace).
#pragma once
#include <cmath>
#include <vector>

#include "laker_internal.h"

namespace laker {
namespace {


constexpr int kVecThreads = 256;

// Block pair-reduction + last-block ticket.  Each block contributes NP pairs;
// the last block returns the NP totals (reduced over blocks in block order).
template <int NP>
__device__ bool reduce_pairs_last_block(dd_pair (&v)[NP], dd_pair *partials, unsigned int *counter,
                                        double (&tot)[NP]) {
  __shared__ dd_pair sred[kVecThreads / 32][NP];
  __shared__ int s_last;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    dd_pair r = warp_reduce_pair(v[k]);
    if (lane == 0) sred[warp][k] = r;
  }
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      dd_pair t = sred[0][k];
      for (int w = 1; w < kVecThreads / 32; ++w) pair_add(t, sred[w][k]);
      partials[blockIdx.x * NP + k] = t;
    }
    __threadfence();
    s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  if (warp == 0) {
    __threadfence();
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      dd_pair t = {0.0, 0.0};
      for (int b = lane; b < (int)gridDim.x; b += 32) {
        dd_pair o;
        o.s = __ldcg(&partials[b * NP + k].s);
        o.c = __ldcg(&partials[b * NP + k].c);
        pair_add(t, o);
      }
      t = warp_reduce_pair(t);
      tot[k] = pair_value(t);
    }
    if (lane == 0) *counter = 0u;
  }
  return lane == 0 && warp == 0;
}

// alpha = 0, r = y; ||y||^2.  Last block: ynorm, ZERO_RHS.
__global__ void __launch_bounds__(kVecThreads) pcg_init_kernel(int64_t n, const double *__restrict__ y,
                                                               double *__restrict__ alpha,
                                                               double *__restrict__ r, PcgState *st,
                                                               dd_pair *partials, unsigned int *counter) {
  dd_pair v[1] = {{0.0, 0.0}};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double yi = y[i];
    alpha[i] = 0.0;
    r[i] = yi;
    dot2_step(v[0], yi, yi);
  }
  double tot[1];
  if (reduce_pairs_last_block<1>(v, partials, counter, tot)) {
    st->ynorm = __dsqrt_rn(tot[0]);
    st->iters = 0;
    st->rel = 1.0;
    if (st->ynorm == 0.0) {
      st->done = 1;
      st->term = LAKER_TERM_ZERO_RHS;
    }
  }
}

// theta^0 = P r^0 (none: r, jacobi: d o r; dense: already in theta), p^0 = theta^0,
// rho = r.theta.  For dense, rho_in_state = 1 (the P gemv stored it).
// per-block max of m over the block's threads -> pmax[blockIdx.x] (pmax may be null)
__device__ __forceinline__ void block_absmax(double m, double *pmax) {
  if (pmax == nullptr) return;
  __shared__ double sm[kVecThreads / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kVecThreads / 32; ++w) m = fmax(m, sm[w]);
    pmax[blockIdx.x] = m;
  }
}

__global__ void __launch_bounds__(kVecThreads) pcg_first_dir_kernel(
    int64_t n, int pk, const double *__restrict__ dvec, const double *__restrict__ r,
    double *__restrict__ theta, double *__restrict__ p, PcgState *st, dd_pair *partials,
    unsigned int *counter, double *pmax = nullptr) {
  if (*(volatile int32_t *)&st->done) return;
  dd_pair v[1] = {{0.0, 0.0}};
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double ri = r[i];
    double th;
    if (pk == LAKER_PRECOND_NONE) {
      th = ri;
    } else if (pk == LAKER_PRECOND_JACOBI) {
      th = __dmul_rn(dvec[i], ri);
      theta[i] = th;
    } else {
      th = theta[i];
    }
    p[i] = th;
    m = fmax(m, fabs(th));
    dot2_step(v[0], ri, th);
  }
  block_absmax(m, pmax);
  double tot[1];
  if (reduce_pairs_last_block<1>(v, partials, counter, tot)) {
    st->rho = tot[0];
    if (!(tot[0] > 0.0)) {
      st->done = 1;
      st->term = LAKER_TERM_INDEFINITE;
    }
  }
}

// alpha = fma(delta, p, alpha); r = fma(-delta, q, r); ||r||^2 (and r.theta for Jacobi).
__global__ void __launch_bounds__(kVecThreads) pcg_update_kernel(
    int64_t n, int pk, const double *__restrict__ dvec, const double *__restrict__ p,
    const double *__restrict__ q, double *__restrict__ alpha, double *__restrict__ r,
    double *__restrict__ theta, PcgState *st, double *history, dd_pair *partials, unsigned int *counter) {
  if (*(volatile int32_t *)&st->done) return;
  const double delta = st->delta;
  dd_pair v[2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    alpha[i] = __fma_rn(delta, p[i], alpha[i]);
    const double ri = __fma_rn(-delta, q[i], r[i]);
    r[i] = ri;
    dot2_step(v[0], ri, ri);
    if (pk == LAKER_PRECOND_JACOBI) {
      const double th = __dmul_rn(dvec[i], ri);
      theta[i] = th;
      dot2_step(v[1], ri, th);
    }
  }
  double tot[2];
  if (reduce_pairs_last_block<2>(v, partials, counter, tot)) {
    const double rel = __ddiv_rn(__dsqrt_rn(tot[0]), st->ynorm);
    const int it = st->iters + 1;
    st->iters = it;
    st->rel = rel;
    if (history) history[it - 1] = rel;
    if (rel <= st->tol) {
      st->term = LAKER_TERM_RESIDUAL_TOL;
      st->done = 1;
      return;
    }
    if (pk != LAKER_PRECOND_EXTERNAL_DENSE && pk != LAKER_PRECOND_LEARNED) {
      const double rho_new = (pk == LAKER_PRECOND_NONE) ? tot[0] : tot[1];
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
}

// dense P only: after theta = P r and beta, close the iteration budget.
__global__ void pcg_budget_kernel(PcgState *st) {
  if (st->done) return;
  if (st->iters >= st->max_iters) {
    st->term = LAKER_TERM_MAX_ITERS;
    st->done = 1;
  }
}

// p = fma(beta, p, theta); with budget = 1 (dense P, single rank) the last block
// also closes the iteration budget (MAX_ITERS after the last allowed update).
__global__ void __launch_bounds__(kVecThreads) pcg_pupdate_kernel(int64_t n, const double *__restrict__ theta,
                                                                  double *__restrict__ p, PcgState *st,
                                                                  int budget = 0, double *pmax = nullptr) {
  if (*(volatile const int32_t *)&st->done) return;
  const double beta = st->beta;
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double pi = __fma_rn(beta, p[i], theta[i]);
    p[i] = pi;
    m = fmax(m, fabs(pi));
  }
  block_absmax(m, pmax);
  if (budget && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0 && st->iters >= st->max_iters) {
    st->term = LAKER_TERM_MAX_ITERS;
    st->done = 1;
  }
}

// true residual ||y - q|| / ||y|| with q = (lambda I + K) alpha
__global__ void __launch_bounds__(kVecThreads) true_residual_kernel(int64_t n, const double *__restrict__ y,
                                                                    const double *__restrict__ q,
                                                                    const PcgState *st, double *out,
                                                                    dd_pair *partials,
                                                                    unsigned int *counter) {
  dd_pair v[1] = {{0.0, 0.0}};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double t = __dsub_rn(y[i], q[i]);
    dot2_step(v[0], t, t);
  }
  double tot[1];
  if (reduce_pairs_last_block<1>(v, partials, counter, tot))
    *out = st->ynorm > 0.0 ? __ddiv_rn(__dsqrt_rn(tot[0]), st->ynorm) : 0.0;
}

// delta epilogue for the on-the-fly operator: p.q over the vector
__global__ void __launch_bounds__(kVecThreads) dot_delta_kernel(int64_t n, const double *__restrict__ p,
                                                                const double *__restrict__ q, PcgState *st,
                                                                dd_pair *partials, unsigned int *counter) {
  if (*(volatile int32_t *)&st->done) return;
  dd_pair v[1] = {{0.0, 0.0}};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dot2_step(v[0], p[i], q[i]);
  double tot[1];
  if (reduce_pairs_last_block<1>(v, partials, counter, tot)) {
    if (!(tot[0] > 0.0)) {
      st->term = LAKER_TERM_BREAKDOWN;
      st->done = 1;
    } else {
      pcg_set_delta(st, __ddiv_rn(st->rho, tot[0]));
    }
  }
}

__global__ void strided_copy_kernel(int64_t n, const double *__restrict__ src, double *__restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

struct Workspace {
  double *alpha = nullptr, *r = nullptr, *theta = nullptr, *p = nullptr, *q = nullptr, *y = nullptr;
  double *hist = nullptr, *scal = nullptr;
  PcgState *st = nullptr;
  size_t cap_n = 0;
  int32_t cap_hist = 0;
};

}  // namespace
}  // namespace laker
