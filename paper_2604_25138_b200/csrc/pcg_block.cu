// Multi-RHS PCG (BASELINE config C4: 64 independent radio
// maps, reading R13): m independent Alg. 1 recurrences that share
// every pass over K and P, so each operator / preconditioner apply is a GEMM
// Q = (lambda I + K) X, Theta = P R with X, R, Q, Theta n x m row-major
// (m contiguous RHS per row).
//
//  * EXACT: `gemm_dot2_kernel` -- one Dot2 pair per output entry, so column c
//    of every apply equals the single-RHS Dot2 GEMV bitwise and the block
//    solve reproduces the single-RHS solves column by column (T18).  fp64 ALU
//    bound (10 flops per K-element and RHS).
//  * FAST: the DMMA GEMM (dgemm.cu), K-element reuse m-fold: fp64 tensor bound.
//
// Per-column scalars (delta, beta, termination) come from fixed-order Dot2
// column reductions; a converged column is frozen (its delta/beta are not
// applied) while the others continue; the loop ends when every column is done.
//
// laker_block_cg_solve runs O'Leary's block PCG instead (B14) through the same
// operator / preconditioner products: m x m Gram matrices and SPD solves per step, the
// columns in independent groups of `block`.
#include <cstdlib>

#include "pcg_kernels.cuh"

namespace laker {
namespace {

constexpr int kBR = 32;   // rows of A per CTA
constexpr int kBK = 32;   // k chunk
constexpr int kBM = 64;   // RHS per CTA (columns)

// rm[i] = max_j |A[i][j]| (one warp per row)
__global__ void rowmax_abs_kernel(const double *__restrict__ A, int64_t rows, int64_t cols, int64_t lda,
                                  double *__restrict__ rm) {
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= rows) return;
  double v = 0.0;
  for (int64_t j = lane; j < cols; j += 32) v = fmax(v, fabs(A[i * lda + j]));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
  if (lane == 0) rm[i] = v;
}

// cm[c] = max_j |X[j][c]| (c < m; X row-major, ldx): block of 64 columns x 4 row lanes,
// atomicMax on the bits (non-negative doubles order as integers); cm zeroed beforehand
__global__ void __launch_bounds__(256) colmax_abs_kernel(const double *__restrict__ X, int64_t rows, int64_t m,
                                                         int64_t ldx, unsigned long long *cm,
                                                         const int32_t *__restrict__ all_done) {
  if (all_done && *(volatile const int32_t *)all_done) return;
  const int c = (int)blockIdx.y * 64 + (threadIdx.x & 63), rl = threadIdx.x >> 6;
  double v = 0.0;
  if (c < m)
    for (int64_t j = (int64_t)blockIdx.x * 4 + rl; j < rows; j += (int64_t)gridDim.x * 4) v = fmax(v, fabs(X[j * ldx + c]));
  __shared__ double sv[4][64];
  const int cl = threadIdx.x & 63;
  sv[rl][cl] = v;
  __syncthreads();
  if (rl == 0 && c < m) {
    v = fmax(fmax(sv[0][cl], sv[1][cl]), fmax(sv[2][cl], sv[3][cl]));
    atomicMax(&cm[c], (unsigned long long)__double_as_longlong(v));
  }
}

// Q[i][c] = RN(lambda Xd[row0+i][c] + sum_j A[i][j] X[j][c]), one compensated sum per entry
// (Xd = X for the operator; Xd = R for the last pass of the factored P, Q (M (Q^T R)) +
// a^-1/2 R).  With rmax / cmax (row maxima of A, column maxima of X) each accumulator
// carries the power-of-two offset C >= 2 kdim rmax_i cmax_c and every step is TwoProd +
// Fast2Sum (dot2_step_off, 7 fp64 ops instead of Dot2's 10; exact error capture, see
// symv.cu); the offset is removed exactly before lambda Xd is added.
template <bool OFF>
__global__ void __launch_bounds__(256) gemm_dot2_kernel(const double *__restrict__ A, int64_t lda, int64_t rows,
                                                        int64_t kdim, const double *__restrict__ X, int64_t ldx,
                                                        int64_t m, double *__restrict__ Q, int64_t ldq,
                                                        double lambda, int64_t row0,
                                                        const int32_t *__restrict__ all_done,
                                                        const double *__restrict__ Xd,
                                                        const double *__restrict__ rmax,
                                                        const double *__restrict__ cmax,
                                                        dd_pair *__restrict__ Qpair = nullptr) {
  if (all_done && *(volatile const int32_t *)all_done) return;
  __shared__ double As[kBR][kBK + 1];
  __shared__ __align__(16) double Xs[kBK][kBM];
  const int tid = threadIdx.x;
  const int tr = (tid >> 4) * 2;       // 2 rows
  const int tc = (tid & 15) * 4;       // 4 columns
  const int64_t R0 = (int64_t)blockIdx.x * kBR;
  const int64_t C0 = (int64_t)blockIdx.y * kBM;
  // offset accumulators cover kOffChunk products each and are folded into the Dot2 pair
  // `tot` at chunk ends: the offset-sum error grows with the products per accumulator
  // (~k^2 u^2 max|a x|), which at k = 512 stays far below ulp(q) as in symv.cu
  constexpr int kOffChunk = 512;
  constexpr bool off = OFF;
  double ra[2] = {0.0, 0.0}, cb[4] = {0.0, 0.0, 0.0, 0.0};
  if (off) {
#pragma unroll
    for (int a = 0; a < 2; ++a) ra[a] = R0 + tr + a < rows ? rmax[R0 + tr + a] * (2.0 * (double)kOffChunk) : 0.0;
#pragma unroll
    for (int b = 0; b < 4; ++b) cb[b] = C0 + tc + b < m ? cmax[C0 + tc + b] : 0.0;
  }
  dd_pair acc[2][4], tot[2][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      acc[a][b] = dd_pair{off ? pow2_above(ra[a] * cb[b]) : 0.0, 0.0};
      tot[a][b] = dd_pair{0.0, 0.0};
    }
  for (int64_t k0 = 0; k0 < kdim; k0 += kBK) {
    __syncthreads();
    for (int e = tid; e < kBR * kBK; e += 256) {
      const int r = e / kBK, c = e % kBK;
      As[r][c] = (R0 + r < rows && k0 + c < kdim) ? A[(R0 + r) * lda + k0 + c] : 0.0;
    }
    for (int e = tid; e < kBK * kBM; e += 256) {
      const int r = e / kBM, c = e % kBM;
      Xs[r][c] = (k0 + r < kdim && C0 + c < m) ? X[(k0 + r) * ldx + C0 + c] : 0.0;
    }
    __syncthreads();
    if constexpr (OFF) {
      if (k0 > 0 && k0 % kOffChunk == 0) {  // fold the finished chunk (offset removed exactly)
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const double cab = pow2_above(ra[a] * cb[b]);
            pair_add(tot[a][b], dd_pair{__dsub_rn(acc[a][b].s, cab), acc[a][b].c});
            acc[a][b] = dd_pair{cab, 0.0};
          }
      }
#pragma unroll 4
      for (int j = 0; j < kBK; ++j) {
        const double a0 = As[tr][j], a1 = As[tr + 1][j];
        const double2 x01 = *reinterpret_cast<const double2 *>(&Xs[j][tc]);
        const double2 x23 = *reinterpret_cast<const double2 *>(&Xs[j][tc + 2]);
        dot2_step_off(acc[0][0], a0, x01.x);
        dot2_step_off(acc[0][1], a0, x01.y);
        dot2_step_off(acc[0][2], a0, x23.x);
        dot2_step_off(acc[0][3], a0, x23.y);
        dot2_step_off(acc[1][0], a1, x01.x);
        dot2_step_off(acc[1][1], a1, x01.y);
        dot2_step_off(acc[1][2], a1, x23.x);
        dot2_step_off(acc[1][3], a1, x23.y);
      }
    } else {
#pragma unroll 4
      for (int j = 0; j < kBK; ++j) {
        const double a0 = As[tr][j], a1 = As[tr + 1][j];
        const double2 x01 = *reinterpret_cast<const double2 *>(&Xs[j][tc]);
        const double2 x23 = *reinterpret_cast<const double2 *>(&Xs[j][tc + 2]);
        dot2_step(acc[0][0], a0, x01.x);
        dot2_step(acc[0][1], a0, x01.y);
        dot2_step(acc[0][2], a0, x23.x);
        dot2_step(acc[0][3], a0, x23.y);
        dot2_step(acc[1][0], a1, x01.x);
        dot2_step(acc[1][1], a1, x01.y);
        dot2_step(acc[1][2], a1, x23.x);
        dot2_step(acc[1][3], a1, x23.y);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (R0 + tr + a < rows && C0 + tc + b < m) {
        dd_pair v = acc[a][b];
        if constexpr (OFF) {
          v.s = __dsub_rn(v.s, pow2_above(ra[a] * cb[b]));  // exact (Sterbenz)
          pair_add(tot[a][b], v);
          v = tot[a][b];
        }
        if (lambda != 0.0) dot2_step(v, lambda, Xd[(row0 + R0 + tr + a) * ldx + C0 + tc + b]);
        if (Qpair)  // unrounded entry (row-sharded partial products, pcg_solve_block_dist)
          Qpair[(R0 + tr + a) * ldq + C0 + tc + b] = v;
        else
          Q[(R0 + tr + a) * ldq + C0 + tc + b] = pair_value(v);
      }
}

enum ColMode { kColInit = 0, kColDelta = 1, kColUpdate = 2, kColBeta = 3, kColTrue = 4 };

struct BlockArgs {
  int64_t n, m, ldv;   // rows, RHS count, row stride of the n x m blocks
  int mode, pk;
  const double *Y;
  double *alpha, *r, *theta, *p, *q;
  const double *dvec;
  PcgState *st;        // [m]
  double *hist;        // [max_iters] column 0
  int32_t *all_done;
  double *true_rel;    // [m]
  dd_pair *partials;   // [grid][m][2]
  unsigned int *counter;
  int64_t ldy;         // column stride of Y (n; the row-sharded solve passes Y + r0)
  double *pair_out;    // row-sharded: the last block stores the unrounded column pairs
                       // [m][2] here instead of running the column epilogue
};

__device__ void column_epilogue(const BlockArgs &a, int col, dd_pair t0, dd_pair t1);

// Column Dot2 reductions over the n x m blocks with the per-element work and
// the per-column scalar logic of each PCG phase.  Block b owns a contiguous
// row range; thread = (column c = tid % m, row lane = tid / m).
__global__ void __launch_bounds__(256) block_col_kernel(const BlockArgs a) {
  if (a.mode != kColTrue && a.all_done && *(volatile int32_t *)a.all_done) return;
  const int64_t m = a.m;
  const int lanes = 256 / (int)m;
  const int c = threadIdx.x % m, ln = threadIdx.x / m;
  const bool act = ln < lanes;
  const int64_t rows_per = (a.n + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * rows_per, i1 = imin64(a.n, i0 + rows_per);
  PcgState &st = a.st[c];
  const bool col_done = st.done != 0;
  double delta = 0.0;
  if (a.mode == kColUpdate && !col_done) delta = st.delta;
  dd_pair v0 = {0.0, 0.0}, v1 = {0.0, 0.0};
  if (act && (!col_done || a.mode == kColInit || a.mode == kColTrue)) {
    for (int64_t i = i0 + ln; i < i1; i += lanes) {
      const int64_t e = i * a.ldv + c;
      switch (a.mode) {
        case kColInit: {  // alpha = 0, r = y, ||y||^2; theta^0 = P r (none/jacobi), p = theta, rho
          const double yi = a.Y[i + c * a.ldy];
          a.alpha[e] = 0.0;
          a.r[e] = yi;
          dot2_step(v0, yi, yi);
          if (a.pk != LAKER_PRECOND_EXTERNAL_DENSE && a.pk != LAKER_PRECOND_LEARNED) {
            const double th = (a.pk == LAKER_PRECOND_JACOBI) ? __dmul_rn(a.dvec[i], yi) : yi;
            a.theta[e] = th;
            a.p[e] = th;
            dot2_step(v1, yi, th);
          }
          break;
        }
        case kColDelta:  // p.q
          dot2_step(v0, a.p[e], a.q[e]);
          break;
        case kColUpdate: {
          a.alpha[e] = __fma_rn(delta, a.p[e], a.alpha[e]);
          const double ri = __fma_rn(-delta, a.q[e], a.r[e]);
          a.r[e] = ri;
          dot2_step(v0, ri, ri);
          if (a.pk == LAKER_PRECOND_JACOBI) {
            const double th = __dmul_rn(a.dvec[i], ri);
            a.theta[e] = th;
            dot2_step(v1, ri, th);
          } else if (a.pk == LAKER_PRECOND_NONE) {
            a.theta[e] = ri;
          }
          break;
        }
        case kColBeta:  // r.theta (dense P); kColInit for dense also lands here via rho0
          dot2_step(v0, a.r[e], a.theta[e]);
          break;
        case kColTrue: {
          const double t = __dsub_rn(a.Y[i + c * a.ldy], a.q[e]);
          dot2_step(v0, t, t);
          break;
        }
      }
    }
  }
  // reduce over the row lanes of this block (fixed order), then over blocks
  __shared__ dd_pair red[256][2];
  red[threadIdx.x][0] = v0;
  red[threadIdx.x][1] = v1;
  __syncthreads();
  __shared__ int s_last;
  if (threadIdx.x < m) {
    dd_pair t0 = red[threadIdx.x][0], t1 = red[threadIdx.x][1];
    for (int l = 1; l < lanes; ++l) {
      pair_add(t0, red[l * m + threadIdx.x][0]);
      pair_add(t1, red[l * m + threadIdx.x][1]);
    }
    a.partials[((int64_t)blockIdx.x * m + threadIdx.x) * 2] = t0;
    a.partials[((int64_t)blockIdx.x * m + threadIdx.x) * 2 + 1] = t1;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(a.counter, 1u) == gridDim.x - 1);
  __syncthreads();
  const bool last = s_last != 0;
  if (last) {
    // the per-block pairs of each column: thread groups g = 0..G-1 (G = 256 / m) take the
    // blocks b = g, g + G, ... with their loads issued in batches of 8, then group 0 adds
    // the G group sums in group order -- a fixed order for every run
    __threadfence();
    const int G = 256 / (int)m;
    const int col = threadIdx.x % (int)m, grp = threadIdx.x / (int)m;
    dd_pair t0 = {0.0, 0.0}, t1 = {0.0, 0.0};
    if (grp < G) {
      for (unsigned b0 = grp; b0 < gridDim.x; b0 += 8u * G) {
        dd_pair o0[8], o1[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const unsigned b = b0 + (unsigned)(u * G);
          if (b < gridDim.x) {
            const dd_pair *pp = a.partials + ((int64_t)b * m + col) * 2;
            o0[u] = dd_pair{__ldcg(&pp[0].s), __ldcg(&pp[0].c)};
            o1[u] = dd_pair{__ldcg(&pp[1].s), __ldcg(&pp[1].c)};
          } else {
            o0[u] = o1[u] = dd_pair{0.0, 0.0};
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          pair_add(t0, o0[u]);
          pair_add(t1, o1[u]);
        }
      }
    }
    __syncthreads();  // red[] reused for the group sums
    red[threadIdx.x][0] = t0;
    red[threadIdx.x][1] = t1;
    __syncthreads();
    if (threadIdx.x < m) {
      dd_pair s0 = red[threadIdx.x][0], s1 = red[threadIdx.x][1];
      for (int g = 1; g < G; ++g) {
        pair_add(s0, red[g * m + threadIdx.x][0]);
        pair_add(s1, red[g * m + threadIdx.x][1]);
      }
      if (a.pair_out) {
        double *o = a.pair_out + 4 * threadIdx.x;
        o[0] = s0.s; o[1] = s0.c; o[2] = s1.s; o[3] = s1.c;
      } else {
        column_epilogue(a, threadIdx.x, s0, s1);
      }
    }
  }
  __syncthreads();
  if (last && threadIdx.x == 0 && a.pair_out) {
    *a.counter = 0u;
    return;
  }
  if (last && threadIdx.x == 0) {
    int all = 1;
    for (int k = 0; k < (int)m; ++k) all &= a.st[k].done != 0;
    *a.all_done = all;
    *a.counter = 0u;
  }
}

__device__ void column_epilogue(const BlockArgs &a, int col, dd_pair t0, dd_pair t1) {
  const double s0 = pair_value(t0), s1 = pair_value(t1);
  PcgState &S = a.st[col];
  switch (a.mode) {
    case kColInit:
      S.ynorm = __dsqrt_rn(s0);
      S.iters = 0;
      S.rel = 1.0;
      if (S.ynorm == 0.0) {
        S.done = 1;
        S.term = LAKER_TERM_ZERO_RHS;
      } else if (a.pk != LAKER_PRECOND_EXTERNAL_DENSE && a.pk != LAKER_PRECOND_LEARNED) {
        S.rho = s1;
        if (!(s1 > 0.0)) {
          S.done = 1;
          S.term = LAKER_TERM_INDEFINITE;
        }
      }
      break;
    case kColDelta:
      if (!S.done) {
        if (!(s0 > 0.0)) {
          S.done = 1;
          S.term = LAKER_TERM_BREAKDOWN;
          S.delta = 0.0;
        } else {
          S.delta = __ddiv_rn(S.rho, s0);
        }
      }
      break;
    case kColUpdate:
      if (!S.done) {
        const double rel = __ddiv_rn(__dsqrt_rn(s0), S.ynorm);
        const int it = S.iters + 1;
        S.iters = it;
        S.rel = rel;
        if (col == 0 && a.hist) a.hist[it - 1] = rel;
        if (rel <= S.tol) {
          S.term = LAKER_TERM_RESIDUAL_TOL;
          S.done = 1;
        } else if (a.pk == LAKER_PRECOND_NONE || a.pk == LAKER_PRECOND_JACOBI) {
          const double rho_new = (a.pk == LAKER_PRECOND_NONE) ? s0 : s1;
          if (!(rho_new > 0.0)) {
            S.term = LAKER_TERM_INDEFINITE;
            S.done = 1;
          } else {
            S.beta = __ddiv_rn(rho_new, S.rho);
            S.rho = rho_new;
            if (it >= S.max_iters) {
              S.term = LAKER_TERM_MAX_ITERS;
              S.done = 1;
            }
          }
        }
      }
      break;
    case kColBeta:
      if (!S.done) {
        if (!(s0 > 0.0)) {
          S.term = LAKER_TERM_INDEFINITE;
          S.done = 1;
        } else if (S.iters == 0 && S.rho == 0.0) {  // initial rho for dense P
          S.rho = s0;
        } else {
          S.beta = __ddiv_rn(s0, S.rho);
          S.rho = s0;
          if (S.iters >= S.max_iters) {
            S.term = LAKER_TERM_MAX_ITERS;
            S.done = 1;
          }
        }
      }
      break;
    case kColTrue:
      a.true_rel[col] = S.ynorm > 0.0 ? __ddiv_rn(__dsqrt_rn(s0), S.ynorm) : 0.0;
      break;
  }
}

// Row-sharded block solve: the W gathered [m][2] column pairs -> summed in rank order,
// then the column epilogue of `a.mode` (identical on every rank), then all_done.
__global__ void block_combine_kernel(const BlockArgs a, const double *__restrict__ recv, int W) {
  if (a.mode != kColTrue && a.mode != kColInit && *(volatile int32_t *)a.all_done) return;
  const int c = threadIdx.x;
  if (c < a.m) {
    dd_pair t0 = {0.0, 0.0}, t1 = {0.0, 0.0};
    for (int w = 0; w < W; ++w) {
      const double *o = recv + (int64_t)w * 4 * a.m + 4 * c;
      pair_add(t0, dd_pair{o[0], o[1]});
      pair_add(t1, dd_pair{o[2], o[3]});
    }
    column_epilogue(a, c, t0, t1);
  }
  __syncthreads();
  if (c == 0) {
    int all = 1;
    for (int k = 0; k < (int)a.m; ++k) all &= a.st[k].done != 0;
    *a.all_done = all;
  }
}

// Z (nrp x ldz) = the rank-order sum of the W gathered partial products (EXACT: unrounded
// pairs, rounded once; FAST: fp64 values summed in rank order)
__global__ void block_zcombine_kernel(int64_t rows, int64_t m, int64_t ldz, const double *__restrict__ recv, int W,
                                      int pairs, double *__restrict__ Z, const int32_t *all_done) {
  if (*(volatile const int32_t *)all_done) return;
  const int64_t per = rows * ldz * (pairs ? 2 : 1);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * ldz; e += (int64_t)gridDim.x * blockDim.x) {
    if (e % ldz >= m) continue;
    if (pairs) {
      dd_pair t = {0.0, 0.0};
      for (int w = 0; w < W; ++w) pair_add(t, dd_pair{recv[w * per + 2 * e], recv[w * per + 2 * e + 1]});
      Z[e] = pair_value(t);
    } else {
      double t = recv[e];
      for (int w = 1; w < W; ++w) t = __dadd_rn(t, recv[w * per + e]);
      Z[e] = t;
    }
  }
}

// p = theta + beta p for active columns; p = theta at init (dense)
__global__ void block_pupdate_kernel(int64_t n, int64_t m, int64_t ldv, const double *__restrict__ theta,
                                     double *__restrict__ p, const PcgState *st, int init,
                                     const int32_t *all_done) {
  if (*(volatile const int32_t *)all_done) return;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * m; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / m, c = e % m;
    if (st[c].done) continue;
    const int64_t k = i * ldv + c;
    p[k] = init ? theta[k] : __fma_rn(st[c].beta, p[k], theta[k]);
  }
}

// ---------------------------------------------------------------- block CG (O'Leary)
// The block-CG variant of C4 (O'Leary, Linear Algebra Appl. 29, 1980):
// the m columns share one block Krylov space, every step needs the m x m Gram matrices
// D^T Q, Z^T R (and R^T R for the stopping test) and two m x m SPD solves.  Grams: each CTA
// sums its rows' outer products in a fixed order, partials reduced in CTA order; the
// solves: one CTA (Cholesky + substitutions); the block updates V +- D C: one pass per row
// block with the m x m coefficients in shared memory.  m <= 64.
constexpr int kBcgGrid = 128;

// part[g] = sum over the rows of CTA g of A[i][:]^T B[i][:] (64 x 64, columns >= m zero)
__global__ void __launch_bounds__(256) bcg_gram_kernel(const double *__restrict__ A, const double *__restrict__ B,
                                                       int64_t n, int m, int64_t ld, double *__restrict__ part) {
  __shared__ double As[32][65], Bs[32][65];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  double acc[4][4] = {};
  for (int64_t i0 = (int64_t)blockIdx.x * 32; i0 < n; i0 += (int64_t)gridDim.x * 32) {
    for (int e = tid; e < 32 * 64; e += 256) {
      const int r = e >> 6, c = e & 63;
      const bool ok = i0 + r < n && c < m;
      As[r][c] = ok ? A[(i0 + r) * ld + c] : 0.0;
      Bs[r][c] = ok ? B[(i0 + r) * ld + c] : 0.0;
    }
    __syncthreads();
    for (int r = 0; r < 32; ++r) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = As[r][4 * ty + u];
        b[u] = Bs[r][4 * tx + u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = __fma_rn(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
  double *o = part + (int64_t)blockIdx.x * 4096;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) o[(4 * ty + u) * 64 + 4 * tx + v] = acc[u][v];
}

// out = the reduced Gram, masked to its bs x bs diagonal blocks (column groups of bs solved
// as independent block recurrences: a block-diagonal Gram keeps every factor and
// coefficient block-diagonal)
__global__ void bcg_gram_reduce_kernel(const double *__restrict__ part, int G, int bs, double *__restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 4096) return;
  double v = 0.0;
  if ((e >> 6) / bs == (e & 63) / bs)
    for (int g = 0; g < G; ++g) v = __dadd_rn(v, part[(int64_t)g * 4096 + e]);
  out[e] = v;
}

// X = G^{-1} B for the m x m SPD G (64 x 64 storage): Cholesky in shared memory, then one
// thread per right-hand-side column for the two triangular solves; *fail = 1 when a pivot
// is not positive (G not numerically positive definite: breakdown)
// Columns of a converged (frozen) group: their rows / columns of G are replaced by the
// identity's and their rows of B by zeros, so their coefficients are zero (no update).
__global__ void __launch_bounds__(256) bcg_spd_solve_kernel(const double *__restrict__ G, const double *__restrict__ B,
                                                            double *__restrict__ X, int m, int *fail,
                                                            const int *__restrict__ frozen) {
  __shared__ double L[64][65];
  const int tid = threadIdx.x;
  for (int e = tid; e < 4096; e += 256) {
    const int i = e >> 6, k = e & 63;
    L[i][k] = (frozen[i] || frozen[k]) ? (i == k ? 1.0 : 0.0) : G[e];
  }
  __syncthreads();
  for (int j = 0; j < m; ++j) {
    const double d = L[j][j];
    if (!(d > 0.0)) {
      if (tid == 0) *fail = 1;
      return;  // uniform: every thread read the same pivot
    }
    const double piv = __dsqrt_rn(d);
    __syncthreads();
    if (tid == 0) L[j][j] = piv;
    if (tid > j && tid < m) L[tid][j] = __ddiv_rn(L[tid][j], piv);
    __syncthreads();
    for (int e = tid; e < 4096; e += 256) {
      const int i = e >> 6, k = e & 63;
      if (i > j && i < m && k > j && k <= i) L[i][k] = __fma_rn(-L[i][j], L[k][j], L[i][k]);
    }
    __syncthreads();
  }
  if (tid < 64) {
    const int c = tid;
    double y[64];
    for (int i = 0; i < m; ++i) {
      double v = (c < m && !frozen[i] && !frozen[c]) ? B[i * 64 + c] : 0.0;
      for (int k = 0; k < i; ++k) v = __fma_rn(-L[i][k], y[k], v);
      y[i] = __ddiv_rn(v, L[i][i]);
    }
    for (int i = m - 1; i >= 0; --i) {
      double v = y[i];
      for (int k = i + 1; k < m; ++k) v = __fma_rn(-L[k][i], y[k], v);
      y[i] = __ddiv_rn(v, L[i][i]);
    }
    for (int i = 0; i < 64; ++i) X[i * 64 + c] = (i < m && c < m) ? y[i] : 0.0;
  }
}

// out[i][c] = add[i][c] + sgn sum_{k < m} D[i][k] C[k][c]  (c < m; out may alias add, not D)
__global__ void __launch_bounds__(256) bcg_update_kernel(double *out, const double *add, const double *__restrict__ D,
                                                         const double *__restrict__ C, int64_t n, int m, int64_t ld,
                                                         double sgn) {
  __shared__ double Cs[64][64];
  __shared__ double Ds[16][65];
  const int tid = threadIdx.x;
  for (int e = tid; e < 4096; e += 256) Cs[e >> 6][e & 63] = C[e];
  const int r = tid >> 4, c0 = (tid & 15) * 4;
  for (int64_t i0 = (int64_t)blockIdx.x * 16; i0 < n; i0 += (int64_t)gridDim.x * 16) {
    __syncthreads();
    for (int e = tid; e < 16 * 64; e += 256) {
      const int rr = e >> 6, k = e & 63;
      Ds[rr][k] = (i0 + rr < n && k < m) ? D[(i0 + rr) * ld + k] : 0.0;
    }
    __syncthreads();
    const int64_t i = i0 + r;
    if (i >= n) continue;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < m; ++k) {
      const double dk = Ds[r][k];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __fma_rn(dk, Cs[k][c0 + u], v[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (c0 + u < m) out[i * ld + c0 + u] = __fma_rn(sgn, v[u], add[i * ld + c0 + u]);
  }
}

__global__ void bcg_jacobi_kernel(double *__restrict__ th, const double *__restrict__ r,
                                  const double *__restrict__ dvec, int64_t n, int m, int64_t ld) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * m; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / m;
    const int c = (int)(e % m);
    th[i * ld + c] = __dmul_rn(dvec[i], r[i * ld + c]);
  }
}

}  // namespace


laker_status pcg_solve_block(laker_ctx ctx, int32_t m, const double *Y, double *alpha_out,
                             const laker_solve_opts &o, laker_solve_report *reps, double *history, int block_cg) {
  if (ctx->comm) return pcg_solve_block_dist(ctx, m, Y, alpha_out, o, reps, history);
  if (ctx->world != 1) return set_err(ctx, LAKER_ERR_NOT_READY, "multi-RHS: detached shard (no NCCL communicator)");
  if (ctx->storage != LAKER_STORE_MATERIALIZED) return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "multi-RHS needs MATERIALIZED");
  if (m > 256) return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "multi-RHS: nrhs <= 256");
  const int64_t n = ctx->n, ld = ctx->ld;
  const int pk = ctx->precond_kind;
  const bool dense = (pk == LAKER_PRECOND_LEARNED || pk == LAKER_PRECOND_EXTERNAL_DENSE);
  const bool fac = dense && ctx->p_factored;
  if (dense && !ctx->P && !fac) return set_err(ctx, LAKER_ERR_NOT_READY, "dense preconditioner not set");
  if (pk == LAKER_PRECOND_JACOBI && !ctx->Pdiag) return set_err(ctx, LAKER_ERR_NOT_READY, "Jacobi diagonal not set");
  const int32_t max_iters = o.max_iters > 0 ? o.max_iters : (int32_t)std::min<int64_t>(10 * n, 1 << 30);
  const int64_t mp = (m + 1) / 2 * 2;  // even row stride for the DMMA epilogue
  cudaStream_t s = ctx->stream;
  double *base = nullptr;
  const size_t blk = (size_t)ld * mp;
  LAKER_CUDA(ctx, cudaMallocAsync(&base, 5 * blk * sizeof(double), s));
  LAKER_CUDA(ctx, cudaMemsetAsync(base, 0, 5 * blk * sizeof(double), s));
  double *al = base, *rr = al + blk, *th = rr + blk, *pp = th + blk, *qq = pp + blk;
  double *zb = nullptr, *wb = nullptr;  // factored P: Q^T R and M Q^T R (nrp x mp)
  if (fac) {
    LAKER_CUDA(ctx, cudaMallocAsync(&zb, 2 * (size_t)ctx->f_nrp * mp * sizeof(double), s));
    LAKER_CUDA(ctx, cudaMemsetAsync(zb, 0, 2 * (size_t)ctx->f_nrp * mp * sizeof(double), s));
    wb = zb + (size_t)ctx->f_nrp * mp;
  }
  PcgState *st = nullptr;
  double *hist = nullptr, *trel = nullptr;
  int32_t *all_done = nullptr;
  dd_pair *parts = nullptr;
  const int cg = (int)std::min<int64_t>(2 * ctx->num_sms, (n + 63) / 64);
  LAKER_CUDA(ctx, cudaMallocAsync(&st, m * sizeof(PcgState), s));
  LAKER_CUDA(ctx, cudaMallocAsync(&hist, (size_t)max_iters * sizeof(double), s));
  LAKER_CUDA(ctx, cudaMallocAsync(&trel, m * sizeof(double), s));
  LAKER_CUDA(ctx, cudaMallocAsync(&all_done, sizeof(int32_t), s));
  LAKER_CUDA(ctx, cudaMallocAsync(&parts, (size_t)cg * m * 2 * sizeof(dd_pair), s));
  LAKER_CUDA(ctx, cudaMemsetAsync(all_done, 0, sizeof(int32_t), s));
  std::vector<PcgState> h0(m);
  for (auto &x : h0) {
    x = PcgState{};
    x.tol = o.tol;
    x.max_iters = max_iters;
  }
  LAKER_CUDA(ctx, cudaMemcpyAsync(st, h0.data(), m * sizeof(PcgState), cudaMemcpyHostToDevice, s));

  BlockArgs ba{};
  ba.n = n; ba.m = m; ba.ldv = mp; ba.pk = pk; ba.Y = Y; ba.alpha = al; ba.r = rr; ba.theta = th; ba.p = pp;
  ba.q = qq; ba.dvec = ctx->Pdiag; ba.st = st; ba.hist = hist; ba.all_done = all_done; ba.true_rel = trel;
  ba.partials = parts; ba.counter = ctx->counters + kCtrMisc; ba.ldy = n;
  auto col = [&](int mode) {
    BlockArgs b = ba;
    b.mode = mode;
    block_col_kernel<<<cg, 256, 0, s>>>(b);
    ctx->stats.kernel_launches++;
  };
  const bool exact = ctx->mode == LAKER_MODE_EXACT;
  // EXACT: row maxima of every matrix the solve multiplies (once) and a column-maxima
  // buffer for the right-hand-side blocks (per product): the offsets of gemm_dot2_kernel
  const char *offenv = std::getenv("LAKER_BLOCK_OFFSET");
  const bool use_off = exact && !(offenv && offenv[0] == '0');
  // the factored P in the form the single-RHS solve applies (QM form R21, or three passes),
  // so that every column is that solve bitwise (T18)
  const bool qm = fac && ctx->p_qm;
  double *rmK = nullptr, *rmP = nullptr, *rmQt = nullptr, *rmM = nullptr, *rmQr = nullptr;
  unsigned long long *cmx = nullptr;
  if (use_off) {
    const int64_t nrp = fac ? ctx->f_nrp : 0;
    LAKER_CUDA(ctx, cudaMallocAsync(&rmK, (size_t)(3 * n + 2 * nrp) * sizeof(double) + 256 * sizeof(double), s));
    rmP = rmK + n;
    rmQt = rmP + n;
    rmM = rmQt + nrp;
    rmQr = rmM + nrp;  // rows of Q (three passes) or of QM (QM form)
    cmx = reinterpret_cast<unsigned long long *>(rmQr + n);
    auto rowmax = [&](const double *A, int64_t rows, int64_t cols, int64_t lda, double *out) {
      rowmax_abs_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(A, rows, cols, lda, out);
      ctx->stats.kernel_launches++;
    };
    rowmax(ctx->K, n, n, ld, rmK);
    if (dense && !fac) rowmax(ctx->P, n, n, ld, rmP);
    if (fac) {
      rowmax(ctx->Qt, nrp, n, ld, rmQt);
      if (qm) {
        rowmax(ctx->QMf, n, nrp, ctx->f_ldq, rmQr);
      } else {
        rowmax(ctx->Mf, nrp, nrp, ctx->f_ldq, rmM);
        rowmax(ctx->Qr, n, nrp, ctx->f_ldq, rmQr);
      }
    }
  }
  auto rowmax_of = [&](const double *Amat) -> const double * {
    if (!use_off) return nullptr;
    if (Amat == ctx->K) return rmK;
    if (Amat == ctx->P) return rmP;
    if (fac && Amat == ctx->Qt) return rmQt;
    if (fac && Amat == ctx->Mf) return rmM;
    if (fac && !qm && Amat == ctx->Qr) return rmQr;
    if (qm && Amat == ctx->QMf) return rmQr;
    return nullptr;
  };
  // Out (rows x m) = A (rows x kdim, lda) X + lam Xd
  auto gemm = [&](const double *Amat, int64_t lda, int64_t rows, int64_t kdim, double lam, const double *X,
                  const double *Xd, double *Out, bool gated) {
    if (exact) {
      dim3 grid((unsigned)((rows + kBR - 1) / kBR), (unsigned)((m + kBM - 1) / kBM));
      const double *rmx = rowmax_of(Amat);
      if (rmx) {
        cudaMemsetAsync(cmx, 0, 256 * sizeof(unsigned long long), s);
        colmax_abs_kernel<<<dim3((unsigned)std::min<int64_t>(2 * ctx->num_sms, (kdim + 3) / 4),
                                 (unsigned)((m + 63) / 64)), 256, 0, s>>>(X, kdim, m, mp, cmx,
                                                                          gated ? all_done : nullptr);
        ctx->stats.kernel_launches++;
      }
      if (rmx)
        gemm_dot2_kernel<true><<<grid, 256, 0, s>>>(Amat, lda, rows, kdim, X, mp, m, Out, mp, lam, 0,
                                                    gated ? all_done : nullptr, Xd, rmx,
                                                    reinterpret_cast<const double *>(cmx));
      else
        gemm_dot2_kernel<false><<<grid, 256, 0, s>>>(Amat, lda, rows, kdim, X, mp, m, Out, mp, lam, 0,
                                                     gated ? all_done : nullptr, Xd, nullptr, nullptr);
    } else {
      GemmArgs g{};
      g.M = rows; g.N = mp; g.K = kdim; g.A = Amat; g.lda = lda; g.B = X; g.ldb = mp; g.C = Out; g.ldc = mp;
      g.alpha = 1.0; g.beta = lam; g.Cin = Xd; g.ldcin = mp;
      launch_dgemm(g, true, s);
    }
    ctx->stats.kernel_launches++;
  };
  auto apply = [&](const double *Amat, double lam, const double *X, double *Out, bool gated = true) {
    gemm(Amat, ld, n, ld, lam, X, X, Out, gated);
  };
  // FAST: the operator product K X on the tcgen05 int8 tensor cores (ozaki_skinny.cu),
  // K sliced once per solve and the right-hand-side block per product.  K's entries
  // lie in a narrow range (exp of small arguments), so per-row digit scaling keeps
  // ~2^-46 of every entry; the preconditioner factors (Q, M: entries spanning many
  // binades, M indefinite-sign) stay on the DMMA GEMM -- sliced, their small entries
  // lost enough precision to make r.theta <= 0 near convergence (tested).
  const char *tcenv = std::getenv("LAKER_BLOCK_TC");
  // (block CG keeps FAST's K products on the DMMA GEMM: its few, coupled steps are far more
  // sensitive to the S = 7 digit products -- C4, groups of 16: 90 steps / 0.23 s on DMMA,
  // 132 steps / 0.27 s with true residuals 6e-8 on the int8 products; B14)
  const bool tcb = !exact && m <= 64 && !(tcenv && tcenv[0] == '0') && !block_cg;
  const int Stc = oz_skinny_max_slices();
  OzSlices sK, sQt, sM, sQr, sXn, sXr;  // sXn / sXr: RHS-block slices for K-dim n / N_r
  double *part = nullptr;
  unsigned long long *mxb = nullptr;
  if (tcb) {
    LAKER_CUDA(ctx, oz_slices_make_general(sK, ctx->K, ld, n, n, 0, Stc, s));
    LAKER_CUDA(ctx, cudaMallocAsync(&part, (size_t)16 * std::max<int64_t>(n, 128) * 64 * sizeof(double), s));
    LAKER_CUDA(ctx, cudaMallocAsync(&mxb, 64 * sizeof(unsigned long long), s));
    // allocate the per-product slice buffers now: nothing may be allocated inside the graph capture
    LAKER_CUDA(ctx, oz_slices_make_general(sXn, rr, mp, m, n, 1, Stc, s, mxb));
  }
  // Out (rows x m) = A X + lam Xd with A pre-sliced; X (kdim x m) sliced per product
  auto gemm_tc = [&](const OzSlices &A, int64_t kdim, double lam, const double *X, const double *Xd, double *Out) {
    OzSlices &sX = (kdim == n) ? sXn : sXr;
    oz_slices_make_general(sX, X, mp, m, kdim, 1, Stc, s, mxb);
    launch_oz_skinny(A, sX, m, 1.0, lam, Xd, mp, Out, mp, part, 16, ctx->num_sms, s);
    ctx->stats.kernel_launches += 4;
  };
  // theta = P R: dense rows, or the factored passes Z = Q^T R, W = M Z, Theta = Q W + a^-1/2 R
  // (QM form: Z = Q^T R, Theta = QM Z + a^-1/2 R)
  auto apply_p = [&](const double *R, double *Th) {
    if (!fac) {
      apply(ctx->P, 0.0, R, Th);
      return;
    }
    const int64_t nrp = ctx->f_nrp, ldq = ctx->f_ldq;
    gemm(ctx->Qt, ld, nrp, ld, 0.0, R, R, zb, true);
    if (qm) {
      gemm(ctx->QMf, ldq, n, nrp, ctx->f_ainv, zb, R, Th, true);
      return;
    }
    gemm(ctx->Mf, ldq, nrp, nrp, 0.0, zb, zb, wb, true);
    gemm(ctx->Qr, ldq, n, nrp, ctx->f_ainv, wb, R, Th, true);
  };
  const int vg = 2 * ctx->num_sms;
  if (block_cg) {
    // ------------------------------------------------ block CG (oracle.block_pcg)
    // X0 = 0, R0 = Y, Z0 = P R0, D0 = Z0; Q = A D; alpha = (D^T Q)^{-1} (Z^T R);
    // X += D alpha; R -= Q alpha; stop when every ||R_c|| / ||Y_c|| <= tol; Z = P R;
    // beta = (Z_old^T R_old)^{-1} (Z^T R); D = Z + D beta.  Products as the batched solve's.
    double *sm = nullptr, *d2 = nullptr;
    int *fail = nullptr;  // [0] breakdown flag, [1 .. 64] frozen (converged) columns
    LAKER_CUDA(ctx, cudaMallocAsync(&sm, ((size_t)kBcgGrid * 4096 + 6 * 4096) * sizeof(double), s));
    LAKER_CUDA(ctx, cudaMallocAsync(&d2, blk * sizeof(double), s));
    LAKER_CUDA(ctx, cudaMallocAsync(&fail, 65 * sizeof(int), s));
    LAKER_CUDA(ctx, cudaMemsetAsync(d2, 0, blk * sizeof(double), s));
    LAKER_CUDA(ctx, cudaMemsetAsync(fail, 0, 65 * sizeof(int), s));
    int *frozen = fail + 1;
    std::vector<int> hfrozen(64, 0);
    double *gpart = sm, *Gzr = sm + (size_t)kBcgGrid * 4096, *Gnew = Gzr + 4096, *Gpq = Gnew + 4096,
           *Grr = Gpq + 4096, *Am = Grr + 4096, *Bm = Am + 4096;
    const int bs = (block_cg > 0 && block_cg < m) ? block_cg : m;  // column groups of bs
    auto gram = [&](const double *A, const double *B, double *out) {
      bcg_gram_kernel<<<kBcgGrid, 256, 0, s>>>(A, B, n, m, mp, gpart);
      bcg_gram_reduce_kernel<<<16, 256, 0, s>>>(gpart, kBcgGrid, bs, out);
      ctx->stats.kernel_launches += 2;
    };
    auto spd_solve = [&](const double *G, const double *B, double *X) {
      bcg_spd_solve_kernel<<<1, 256, 0, s>>>(G, B, X, m, fail, frozen);
      ctx->stats.kernel_launches++;
    };
    auto upd = [&](double *out, const double *add, const double *D, const double *C, double sgn) {
      bcg_update_kernel<<<(unsigned)std::min<int64_t>(2 * ctx->num_sms, (n + 15) / 16), 256, 0, s>>>(
          out, add, D, C, n, m, mp, sgn);
      ctx->stats.kernel_launches++;
    };
    auto precond = [&](const double *R) -> const double * {  // Z = P R
      if (dense) {
        apply_p(R, th);
        return th;
      }
      if (pk == LAKER_PRECOND_JACOBI) {
        bcg_jacobi_kernel<<<vg, 256, 0, s>>>(th, R, ctx->Pdiag, n, m, mp);
        ctx->stats.kernel_launches++;
        return th;
      }
      return R;
    };
    cudaEvent_t b0, b1;
    cudaEventCreate(&b0);
    cudaEventCreate(&b1);
    cudaEventRecord(b0, s);
    col(kColInit);  // X = 0, R = Y
    std::vector<double> hg(4096), ynorm(m);
    gram(rr, rr, Grr);
    LAKER_CUDA(ctx, cudaMemcpyAsync(hg.data(), Grr, 4096 * sizeof(double), cudaMemcpyDeviceToHost, s));
    LAKER_CUDA(ctx, cudaStreamSynchronize(s));
    for (int c = 0; c < m; ++c) ynorm[c] = std::sqrt(hg[c * 64 + c]);
    const double *Z = precond(rr);
    LAKER_CUDA(ctx, cudaMemcpyAsync(pp, Z, blk * sizeof(double), cudaMemcpyDeviceToDevice, s));
    gram(Z, rr, Gzr);
    int32_t it = 0, term = LAKER_TERM_MAX_ITERS;
    std::vector<double> rel(m, 1.0);
    double *D = pp, *Dn = d2;
    int hfail = 0;
    bool zero = false;
    for (int c = 0; c < m; ++c) zero = zero || !(ynorm[c] > 0.0);
    if (zero) term = LAKER_TERM_ZERO_RHS;
    while (!zero && it < max_iters) {
      if (tcb)
        gemm_tc(sK, n, ctx->lambda, D, D, qq);
      else
        apply(ctx->K, ctx->lambda, D, qq, false);
      gram(D, qq, Gpq);
      spd_solve(Gpq, Gzr, Am);
      upd(al, al, D, Am, 1.0);
      upd(rr, rr, qq, Am, -1.0);
      ++it;
      gram(rr, rr, Grr);
      LAKER_CUDA(ctx, cudaMemcpyAsync(hg.data(), Grr, 4096 * sizeof(double), cudaMemcpyDeviceToHost, s));
      LAKER_CUDA(ctx, cudaMemcpyAsync(&hfail, fail, sizeof(int), cudaMemcpyDeviceToHost, s));
      LAKER_CUDA(ctx, cudaStreamSynchronize(s));
      if (hfail) {
        term = LAKER_TERM_BREAKDOWN;
        break;
      }
      bool all = true, newly = false;
      for (int c = 0; c < m; ++c) {
        rel[c] = std::sqrt(std::max(hg[c * 64 + c], 0.0)) / ynorm[c];
        all = all && rel[c] <= o.tol;
      }
      for (int g0 = 0; g0 < m; g0 += bs) {  // a group whose columns all converged stops
        bool gdone = true;
        for (int c = g0; c < g0 + bs; ++c) gdone = gdone && rel[c] <= o.tol;
        if (gdone && !hfrozen[g0]) {
          for (int c = g0; c < g0 + bs; ++c) hfrozen[c] = 1;
          newly = true;
        }
      }
      if (newly && !all)
        LAKER_CUDA(ctx, cudaMemcpyAsync(frozen, hfrozen.data(), 64 * sizeof(int), cudaMemcpyHostToDevice, s));
      if (history) history[it - 1] = rel[0];
      if (all) {
        term = LAKER_TERM_RESIDUAL_TOL;
        break;
      }
      Z = precond(rr);
      gram(Z, rr, Gnew);
      spd_solve(Gzr, Gnew, Bm);
      upd(Dn, Z, D, Bm, 1.0);
      std::swap(D, Dn);
      std::swap(Gzr, Gnew);
    }
    LAKER_CUDA(ctx, cudaMemcpyAsync(&hfail, fail, sizeof(int), cudaMemcpyDeviceToHost, s));
    LAKER_CUDA(ctx, cudaStreamSynchronize(s));
    if (hfail && term != LAKER_TERM_BREAKDOWN) term = LAKER_TERM_INDEFINITE;  // Z^T R not positive definite
    cudaEventRecord(b1, s);
    apply(ctx->K, ctx->lambda, al, qq, false);
    col(kColTrue);
    LAKER_CUDA(ctx, cudaMemcpy2DAsync(alpha_out, sizeof(double), al, mp * sizeof(double), sizeof(double), n,
                                      cudaMemcpyDeviceToDevice, s));
    for (int32_t c = 1; c < m; ++c)
      LAKER_CUDA(ctx, cudaMemcpy2DAsync(alpha_out + (size_t)c * n, sizeof(double), al + c, mp * sizeof(double),
                                        sizeof(double), n, cudaMemcpyDeviceToDevice, s));
    std::vector<double> htr(m);
    LAKER_CUDA(ctx, cudaMemcpyAsync(htr.data(), trel, m * sizeof(double), cudaMemcpyDeviceToHost, s));
    LAKER_CUDA(ctx, cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, b0, b1);
    ctx->stats.solve_ms = ms;
    for (int32_t c = 0; c < m && reps; ++c) {
      reps[c].iters = it;
      reps[c].termination = term;
      reps[c].rel_residual = zero ? 0.0 : rel[c];
      reps[c].true_rel_residual = htr[c];
      reps[c].seconds = ms * 1e-3;
      reps[c].lanczos_lmin = reps[c].lanczos_lmax = 0.0;
    }
    cudaEventDestroy(b0);
    cudaEventDestroy(b1);
    cudaFreeAsync(sm, s);
    cudaFreeAsync(d2, s);
    cudaFreeAsync(fail, s);
    cudaFreeAsync(base, s);
    if (zb) cudaFreeAsync(zb, s);
    if (rmK) cudaFreeAsync(rmK, s);
    if (part) cudaFreeAsync(part, s);
    oz_slices_free(sK, s);
    oz_slices_free(sQt, s);
    oz_slices_free(sM, s);
    oz_slices_free(sQr, s);
    oz_slices_free(sXn, s);
    oz_slices_free(sXr, s);
    if (mxb) cudaFreeAsync(mxb, s);
    cudaFreeAsync(st, s);
    cudaFreeAsync(hist, s);
    cudaFreeAsync(trel, s);
    cudaFreeAsync(all_done, s);
    cudaFreeAsync(parts, s);
    LAKER_CUDA(ctx, cudaStreamSynchronize(s));
    if (term == LAKER_TERM_BREAKDOWN)
      return set_err(ctx, LAKER_ERR_BREAKDOWN_ZERO_CURVATURE, "block CG: D^T (lambda I + K) D not positive definite");
    if (term == LAKER_TERM_INDEFINITE)
      return set_err(ctx, LAKER_ERR_INDEFINITE_PRECONDITIONER, "block CG: Z^T R not positive definite");
    return LAKER_OK;
  }
  cudaEvent_t ev0, ev1;
  cudaEventCreate(&ev0);
  cudaEventCreate(&ev1);
  cudaEventRecord(ev0, s);
  col(kColInit);
  if (dense) {
    apply_p(rr, th);
    col(kColBeta);  // initial rho = r.theta
    block_pupdate_kernel<<<vg, 256, 0, s>>>(n, m, mp, th, pp, st, 1, all_done);
    ctx->stats.kernel_launches++;
  }
  const double *theta_src = th;
  const int chunk = 4;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  const int64_t before = ctx->stats.kernel_launches;
  LAKER_CUDA(ctx, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int j = 0; j < chunk; ++j) {
    if (tcb)
      gemm_tc(sK, n, ctx->lambda, pp, pp, qq);
    else
      apply(ctx->K, ctx->lambda, pp, qq);
    col(kColDelta);
    col(kColUpdate);
    if (dense) {
      apply_p(rr, th);
      col(kColBeta);
    }
    block_pupdate_kernel<<<vg, 256, 0, s>>>(n, m, mp, theta_src, pp, st, 0, all_done);
    ctx->stats.kernel_launches++;
  }
  LAKER_CUDA(ctx, cudaStreamEndCapture(s, &graph));
  const int64_t per_chunk = ctx->stats.kernel_launches - before;
  ctx->stats.kernel_launches = before;
  LAKER_CUDA(ctx, cudaGraphInstantiate(&gexec, graph, 0));
  int32_t *hd = nullptr;
  LAKER_CUDA(ctx, cudaMallocHost(&hd, sizeof(int32_t)));
  LAKER_CUDA(ctx, cudaMemcpyAsync(hd, all_done, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  while (!*hd) {
    LAKER_CUDA(ctx, cudaGraphLaunch(gexec, s));
    ctx->stats.kernel_launches += per_chunk;
    LAKER_CUDA(ctx, cudaMemcpyAsync(hd, all_done, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  }
  cudaEventRecord(ev1, s);
  // true residuals, alpha out (column-major n x m)
  apply(ctx->K, ctx->lambda, al, qq, false);
  col(kColTrue);
  LAKER_CUDA(ctx, cudaMemcpy2DAsync(alpha_out, sizeof(double), al, mp * sizeof(double), sizeof(double), n,
                                    cudaMemcpyDeviceToDevice, s));
  for (int32_t c = 1; c < m; ++c)
    LAKER_CUDA(ctx, cudaMemcpy2DAsync(alpha_out + (size_t)c * n, sizeof(double), al + c, mp * sizeof(double),
                                      sizeof(double), n, cudaMemcpyDeviceToDevice, s));
  std::vector<PcgState> hs(m);
  std::vector<double> htr(m);
  LAKER_CUDA(ctx, cudaMemcpyAsync(hs.data(), st, m * sizeof(PcgState), cudaMemcpyDeviceToHost, s));
  LAKER_CUDA(ctx, cudaMemcpyAsync(htr.data(), trel, m * sizeof(double), cudaMemcpyDeviceToHost, s));
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  if (history && hs[0].iters > 0)
    LAKER_CUDA(ctx, cudaMemcpyAsync(history, hist, (size_t)hs[0].iters * sizeof(double), cudaMemcpyDeviceToHost, s));
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev0, ev1);
  ctx->stats.solve_ms = ms;
  int worst = LAKER_TERM_RESIDUAL_TOL;
  for (int32_t c = 0; c < m; ++c) {
    if (reps) {
      reps[c].iters = hs[c].iters;
      reps[c].termination = hs[c].term;
      reps[c].rel_residual = hs[c].iters > 0 ? hs[c].rel : (hs[c].term == LAKER_TERM_ZERO_RHS ? 0.0 : 1.0);
      reps[c].true_rel_residual = htr[c];
      reps[c].seconds = ms * 1e-3;
    }
    if (hs[c].term == LAKER_TERM_BREAKDOWN || hs[c].term == LAKER_TERM_INDEFINITE) worst = hs[c].term;
  }
  cudaFreeHost(hd);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  cudaGraphExecDestroy(gexec);
  cudaGraphDestroy(graph);
  cudaFreeAsync(base, s);
  if (zb) cudaFreeAsync(zb, s);
  if (rmK) cudaFreeAsync(rmK, s);
  if (part) cudaFreeAsync(part, s);
  oz_slices_free(sK, s);
  oz_slices_free(sQt, s);
  oz_slices_free(sM, s);
  oz_slices_free(sQr, s);
  oz_slices_free(sXn, s);
  oz_slices_free(sXr, s);
  if (mxb) cudaFreeAsync(mxb, s);
  cudaFreeAsync(st, s);
  cudaFreeAsync(hist, s);
  cudaFreeAsync(trel, s);
  cudaFreeAsync(all_done, s);
  cudaFreeAsync(parts, s);
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  if (worst == LAKER_TERM_BREAKDOWN) return set_err(ctx, LAKER_ERR_BREAKDOWN_ZERO_CURVATURE, "p.(lambda I + K)p <= 0");
  if (worst == LAKER_TERM_INDEFINITE) return set_err(ctx, LAKER_ERR_INDEFINITE_PRECONDITIONER, "r.theta <= 0");
  return LAKER_OK;
}

}  // namespace laker

namespace laker {

// Row-sharded multi-RHS PCG (C4 on W GPUs): rank w holds rows [r0, r1) of
// K (full rows), of alpha, R, Q, Theta, and its part of the factored P (fit.cu: Q^T's
// columns, QM's / Q's rows); P (the search directions) is kept whole on every rank.
// Every column reduction is a per-rank unrounded Dot2 pair, all-gathered and summed in
// rank order (block_combine_kernel), so every rank takes identical per-column decisions;
// the factored P's N_r x m product Z = Q^T R is formed from the W partial products the
// same way (block_zcombine_kernel).  Per iteration and rank: K_loc X (8 n^2 / W bytes),
// Z_loc = Q^T_loc R_loc and Theta_loc = QM_loc Z + a^-1/2 R_loc (16 n N_r / W bytes).
// Exchanges: the column pairs of p.q, ||r||^2 (+ r.theta), r.theta (4 m doubles each),
// the partial Z (2 N_r m doubles, EXACT) and the Theta rows (n m / W doubles).
laker_status pcg_solve_block_dist(laker_ctx ctx, int32_t m, const double *Y, double *alpha_out,
                                  const laker_solve_opts &o, laker_solve_report *reps, double *history) {
  if (ctx->storage != LAKER_STORE_MATERIALIZED) return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "multi-RHS needs MATERIALIZED");
  if (m > 256) return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "multi-RHS: nrhs <= 256");
  const int W = ctx->world;
  const int64_t n = ctx->n, ld = ctx->ld, r0 = ctx->r0, nloc = ctx->r1 - ctx->r0;
  const int pk = ctx->precond_kind;
  const bool dense = (pk == LAKER_PRECOND_LEARNED || pk == LAKER_PRECOND_EXTERNAL_DENSE);
  const bool fac = dense && ctx->p_factored && ctx->f_local;
  if (dense && !fac && !ctx->P) return set_err(ctx, LAKER_ERR_NOT_READY, "dense preconditioner not set");
  if (pk == LAKER_PRECOND_JACOBI && !ctx->Pdiag) return set_err(ctx, LAKER_ERR_NOT_READY, "Jacobi diagonal not set");
  const bool qm = fac && ctx->p_qm;
  const int32_t max_iters = o.max_iters > 0 ? o.max_iters : (int32_t)std::min<int64_t>(10 * n, 1 << 30);
  const int64_t mp = (m + 1) / 2 * 2;
  const bool exact = ctx->mode == LAKER_MODE_EXACT;
  const int64_t nrp = fac ? ctx->f_nrp : 0, ldq = fac ? ctx->f_ldq : 0;
  cudaStream_t s = ctx->stream;
  // local n/W x mp blocks: alpha, R, Theta_loc, Q; whole ld x mp: P, Theta; exchanges
  const size_t lb = (size_t)nloc * mp, fb = (size_t)ld * mp;
  const size_t zb = fac ? (size_t)nrp * mp : 0, zp = exact ? 2 * zb : zb;
  const size_t cs = 4 * (size_t)m;
  const size_t total = 4 * lb + 2 * fb + 2 * zb + (1 + W) * zp + (1 + W) * cs + 8;
  double *base = nullptr;
  LAKER_CUDA(ctx, cudaMallocAsync(&base, total * sizeof(double), s));
  LAKER_CUDA(ctx, cudaMemsetAsync(base, 0, total * sizeof(double), s));
  double *al = base, *rr = al + lb, *thl = rr + lb, *qq = thl + lb, *pp = qq + lb, *thf = pp + fb;
  double *Zb = thf + fb, *Wb = Zb + zb, *zsend = Wb + zb, *zrecv = zsend + zp, *csend = zrecv + W * zp,
         *crecv = csend + cs;
  PcgState *st = nullptr;
  double *hist = nullptr, *trel = nullptr;
  int32_t *all_done = nullptr;
  dd_pair *parts = nullptr;
  const int cg = (int)std::min<int64_t>(2 * ctx->num_sms, (nloc + 63) / 64);
  LAKER_CUDA(ctx, cudaMallocAsync(&st, m * sizeof(PcgState), s));
  LAKER_CUDA(ctx, cudaMallocAsync(&hist, (size_t)max_iters * sizeof(double), s));
  LAKER_CUDA(ctx, cudaMallocAsync(&trel, m * sizeof(double), s));
  LAKER_CUDA(ctx, cudaMallocAsync(&all_done, sizeof(int32_t), s));
  LAKER_CUDA(ctx, cudaMallocAsync(&parts, (size_t)cg * m * 2 * sizeof(dd_pair), s));
  LAKER_CUDA(ctx, cudaMemsetAsync(all_done, 0, sizeof(int32_t), s));
  std::vector<PcgState> h0(m);
  for (auto &x : h0) {
    x = PcgState{};
    x.tol = o.tol;
    x.max_iters = max_iters;
  }
  LAKER_CUDA(ctx, cudaMemcpyAsync(st, h0.data(), m * sizeof(PcgState), cudaMemcpyHostToDevice, s));
  laker_status err = LAKER_OK;

  BlockArgs ba{};
  ba.n = nloc; ba.m = m; ba.ldv = mp; ba.pk = pk; ba.Y = Y + r0; ba.ldy = n; ba.alpha = al; ba.r = rr;
  ba.theta = thl; ba.p = pp + (size_t)r0 * mp; ba.q = qq; ba.dvec = ctx->Pdiag ? ctx->Pdiag + r0 : nullptr;
  ba.st = st; ba.hist = hist; ba.all_done = all_done; ba.true_rel = trel; ba.partials = parts;
  ba.counter = ctx->counters + kCtrMisc; ba.pair_out = csend;
  // a column reduction on the local rows, its W pair blocks gathered and combined in rank order
  auto col = [&](int mode) {
    BlockArgs b = ba;
    b.mode = mode;
    block_col_kernel<<<cg, 256, 0, s>>>(b);
    if (ncclAllGather(csend, crecv, cs, ncclDouble, ctx->comm, s) != ncclSuccess) err = LAKER_ERR_NCCL;
    block_combine_kernel<<<1, 256, 0, s>>>(b, crecv, W);
    ctx->stats.kernel_launches += 2;
  };
  // EXACT offsets: row maxima of the local matrices, column maxima of each right-hand block
  double *rmK = nullptr, *rmQt = nullptr, *rmQ = nullptr, *rmM = nullptr;
  unsigned long long *cmx = nullptr;
  if (exact) {
    LAKER_CUDA(ctx, cudaMallocAsync(&rmK, (size_t)(2 * nloc + 2 * nrp + 256) * sizeof(double), s));
    rmQt = rmK + nloc;
    rmQ = rmQt + nrp;
    rmM = rmQ + nloc;
    cmx = reinterpret_cast<unsigned long long *>(rmM + nrp);
    auto rowmax = [&](const double *A, int64_t rows, int64_t cols, int64_t lda, double *out) {
      rowmax_abs_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(A, rows, cols, lda, out);
      ctx->stats.kernel_launches++;
    };
    rowmax(ctx->K, nloc, n, ld, rmK);
    if (fac) {
      rowmax(ctx->Qt, nrp, nloc, ctx->f_ldl, rmQt);
      rowmax(qm ? ctx->QMf : ctx->Qr, nloc, nrp, ldq, rmQ);
      if (!qm) rowmax(ctx->Mf, nrp, nrp, ldq, rmM);
    }
  }
  // Out (rows x m) = A (rows x kdim) X + lam Xd[row0 ..] -- EXACT compensated (pair output
  // when Op != null) or the DMMA GEMM (FAST)
  auto gemm = [&](const double *A, int64_t lda, int64_t rows, int64_t kdim, double lam, const double *X,
                  const double *Xd, int64_t row0, double *Out, const double *rmx, dd_pair *Op) {
    if (exact) {
      cudaMemsetAsync(cmx, 0, 256 * sizeof(unsigned long long), s);
      colmax_abs_kernel<<<dim3((unsigned)std::min<int64_t>(2 * ctx->num_sms, (kdim + 3) / 4), (unsigned)((m + 63) / 64)),
                          256, 0, s>>>(X, kdim, m, mp, cmx, all_done);
      dim3 grid((unsigned)((rows + kBR - 1) / kBR), (unsigned)((m + kBM - 1) / kBM));
      gemm_dot2_kernel<true><<<grid, 256, 0, s>>>(A, lda, rows, kdim, X, mp, m, Out, mp, lam, row0, all_done, Xd, rmx,
                                                  reinterpret_cast<const double *>(cmx), Op);
      ctx->stats.kernel_launches += 2;
    } else {
      GemmArgs g{};
      g.M = rows; g.N = mp; g.K = kdim; g.A = A; g.lda = lda; g.B = X; g.ldb = mp; g.C = Out; g.ldc = mp;
      g.alpha = 1.0; g.beta = lam; g.Cin = Xd ? Xd + row0 * mp : nullptr; g.ldcin = mp;
      launch_dgemm(g, true, s);
      ctx->stats.kernel_launches++;
    }
  };
  // Theta_loc = P R_loc (factored, from the local R); Theta gathered whole afterwards
  auto apply_p = [&]() {
    gemm(ctx->Qt, ctx->f_ldl, nrp, nloc, 0.0, rr, nullptr, 0, zsend, rmQt,
         exact ? reinterpret_cast<dd_pair *>(zsend) : nullptr);
    if (ncclAllGather(zsend, zrecv, zp, ncclDouble, ctx->comm, s) != ncclSuccess) err = LAKER_ERR_NCCL;
    block_zcombine_kernel<<<2 * ctx->num_sms, 256, 0, s>>>(nrp, m, mp, zrecv, W, exact ? 1 : 0, Zb, all_done);
    ctx->stats.kernel_launches++;
    if (qm) {
      gemm(ctx->QMf, ldq, nloc, nrp, ctx->f_ainv, Zb, rr, 0, thl, rmQ, nullptr);
    } else {
      gemm(ctx->Mf, ldq, nrp, nrp, 0.0, Zb, nullptr, 0, Wb, rmM, nullptr);
      gemm(ctx->Qr, ldq, nloc, nrp, ctx->f_ainv, Wb, rr, 0, thl, rmQ, nullptr);
    }
  };
  auto gather_theta = [&]() {  // Theta_loc (nloc x mp) -> rows [r0, r1) of Theta on every rank
    if (ncclAllGather(thl, thf, lb, ncclDouble, ctx->comm, s) != ncclSuccess) err = LAKER_ERR_NCCL;
  };
  const int vg = 2 * ctx->num_sms;
  cudaEvent_t ev0, ev1;
  cudaEventCreate(&ev0);
  cudaEventCreate(&ev1);
  cudaEventRecord(ev0, s);
  col(kColInit);
  if (dense) {
    if (!fac) return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "sharded multi-RHS: dense P rows not supported");
    apply_p();
    col(kColBeta);  // initial rho = r.theta
  }
  gather_theta();
  block_pupdate_kernel<<<vg, 256, 0, s>>>(n, m, mp, thf, pp, st, 1, all_done);
  ctx->stats.kernel_launches++;
  LAKER_CUDA(ctx, cudaGetLastError());
  const int chunk = 4;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  const int64_t before = ctx->stats.kernel_launches;
  LAKER_CUDA(ctx, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int j = 0; j < chunk; ++j) {
    gemm(ctx->K, ld, nloc, n, ctx->lambda, pp, pp, r0, qq, rmK, nullptr);
    col(kColDelta);
    col(kColUpdate);
    if (dense) {
      apply_p();
      col(kColBeta);
    }
    gather_theta();
    block_pupdate_kernel<<<vg, 256, 0, s>>>(n, m, mp, thf, pp, st, 0, all_done);
    ctx->stats.kernel_launches++;
  }
  LAKER_CUDA(ctx, cudaStreamEndCapture(s, &graph));
  if (err != LAKER_OK) return set_err(ctx, err, "sharded multi-RHS: NCCL call failed during capture");
  const int64_t per_chunk = ctx->stats.kernel_launches - before;
  ctx->stats.kernel_launches = before;
  LAKER_CUDA(ctx, cudaGraphInstantiate(&gexec, graph, 0));
  int32_t *hd = nullptr;
  LAKER_CUDA(ctx, cudaMallocHost(&hd, sizeof(int32_t)));
  LAKER_CUDA(ctx, cudaMemcpyAsync(hd, all_done, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  LAKER_TRY(dist_sync(ctx, s));
  while (!*hd) {
    LAKER_CUDA(ctx, cudaGraphLaunch(gexec, s));
    ctx->stats.kernel_launches += per_chunk;
    LAKER_CUDA(ctx, cudaMemcpyAsync(hd, all_done, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    LAKER_TRY(dist_sync(ctx, s));
  }
  cudaEventRecord(ev1, s);
  // true residuals on the local rows (combined), alpha gathered (column-major n x m out)
  LAKER_NCCL(ctx, ncclAllGather(al, thf, lb, ncclDouble, ctx->comm, s));   // alpha rows of every rank -> thf
  LAKER_CUDA(ctx, cudaMemsetAsync(all_done, 0, sizeof(int32_t), s));
  gemm(ctx->K, ld, nloc, n, ctx->lambda, thf, thf, r0, qq, rmK, nullptr);
  {
    BlockArgs b = ba;
    b.mode = kColTrue;
    block_col_kernel<<<cg, 256, 0, s>>>(b);
    LAKER_NCCL(ctx, ncclAllGather(csend, crecv, cs, ncclDouble, ctx->comm, s));
    block_combine_kernel<<<1, 256, 0, s>>>(b, crecv, W);
    ctx->stats.kernel_launches += 2;
  }
  for (int32_t c = 0; c < m; ++c)
    LAKER_CUDA(ctx, cudaMemcpy2DAsync(alpha_out + (size_t)c * n, sizeof(double), thf + c, mp * sizeof(double),
                                      sizeof(double), n, cudaMemcpyDeviceToDevice, s));
  std::vector<PcgState> hs(m);
  std::vector<double> htr(m);
  LAKER_CUDA(ctx, cudaMemcpyAsync(hs.data(), st, m * sizeof(PcgState), cudaMemcpyDeviceToHost, s));
  LAKER_CUDA(ctx, cudaMemcpyAsync(htr.data(), trel, m * sizeof(double), cudaMemcpyDeviceToHost, s));
  LAKER_TRY(dist_sync(ctx, s));
  if (history && hs[0].iters > 0)
    LAKER_CUDA(ctx, cudaMemcpyAsync(history, hist, (size_t)hs[0].iters * sizeof(double), cudaMemcpyDeviceToHost, s));
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev0, ev1);
  ctx->stats.solve_ms = ms;
  int worst = LAKER_TERM_RESIDUAL_TOL;
  for (int32_t c = 0; c < m; ++c) {
    if (reps) {
      reps[c].iters = hs[c].iters;
      reps[c].termination = hs[c].term;
      reps[c].rel_residual = hs[c].iters > 0 ? hs[c].rel : (hs[c].term == LAKER_TERM_ZERO_RHS ? 0.0 : 1.0);
      reps[c].true_rel_residual = htr[c];
      reps[c].seconds = ms * 1e-3;
    }
    if (hs[c].term == LAKER_TERM_BREAKDOWN || hs[c].term == LAKER_TERM_INDEFINITE) worst = hs[c].term;
  }
  cudaFreeHost(hd);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  cudaGraphExecDestroy(gexec);
  cudaGraphDestroy(graph);
  cudaFreeAsync(base, s);
  if (rmK) cudaFreeAsync(rmK, s);
  cudaFreeAsync(st, s);
  cudaFreeAsync(hist, s);
  cudaFreeAsync(trel, s);
  cudaFreeAsync(all_done, s);
  cudaFreeAsync(parts, s);
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  if (worst == LAKER_TERM_BREAKDOWN) return set_err(ctx, LAKER_ERR_BREAKDOWN_ZERO_CURVATURE, "p.(lambda I + K)p <= 0");
  if (worst == LAKER_TERM_INDEFINITE) return set_err(ctx, LAKER_ERR_INDEFINITE_PRECONDITIONER, "r.theta <= 0");
  return LAKER_OK;
}

}  // namespace laker
