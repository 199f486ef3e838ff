// Small dense factorizations for the CCCP fit, blocked so that the bulk of the
// work is the DMMA GEMM (dgemm.cu): right-looking Cholesky (64 x 64 diagonal
// blocks factored in shared memory, panel solve, lower-only trailing GEMM
// update) and the lower-triangular solve with many right-hand sides
// (64-row diagonal solves with the solution held in registers, GEMM updates
// of the rows below).
#include <algorithm>

#include "laker_internal.h"

namespace laker {
namespace {

constexpr int NB = 64;

// Factor the 64 x 64 diagonal block at (j0, j0); zero its strict upper part.
// Right-looking, 256 threads as a 16 x 16 grid, the block held in registers: thread
// (ty, tx) owns A_ik for rows i = ty + 16a, columns k = tx + 16b (a, b < 4).  Step j:
// every thread takes 1/sqrt(A_jj) from the pivot slot, the owners of column j
// (tx == j mod 16) scale it into the shared column buffer, then every thread applies
// A_ik -= L_ij L_kj to its entries with j < k <= i and the owner of A_{j+1,j+1}
// publishes the next pivot -- the textbook operations (the same per-entry sequence
// as a shared-memory right-looking loop), two barriers and 8 broadcast loads per step
// instead of a shared read-modify-write of the whole trailing triangle.
__global__ void __launch_bounds__(256) potrf_diag_kernel(double *A, int64_t lda, int64_t j0, int *flag) {
  __shared__ double col[NB];
  __shared__ double pivot;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  double v[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) v[a][b] = A[(j0 + ty + 16 * a) * lda + j0 + tx + 16 * b];
  if (tid == 0) pivot = v[0][0];
  __syncthreads();
#pragma unroll
  for (int jb = 0; jb < 4; ++jb) {
    for (int jt = 0; jt < 16; ++jt) {
      const int j = 16 * jb + jt;
      double d = pivot;
      if (!(d > 0.0)) {
        if (tid == 0) atomicExch(flag, 1);
        d = 1.0;
      }
      // 1/sqrt(d) directly (hardware approximation + Newton steps, ~1 ulp) and the pivot as
      // d / sqrt(d): the step's dependent chain was the IEEE sqrt followed by the IEEE
      // reciprocal; the fit only needs P to ~1e-8 of the oracle's (tests/test_gpu_fit.py)
      const double rpiv = rsqrt(d);
      if (tx == jt) {
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int i = ty + 16 * a;
          if (i > j) {
            const double l = __dmul_rn(v[a][jb], rpiv);
            v[a][jb] = l;
            col[i] = l;
          } else if (i == j) {
            v[a][jb] = __dmul_rn(d, rpiv);
          }
        }
      }
      __syncthreads();
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int i = ty + 16 * a;
        if (i > j) {
          const double lij = col[i];
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int k = tx + 16 * b;
            if (k > j && k <= i) v[a][b] = __fma_rn(-lij, col[k], v[a][b]);
          }
        }
      }
      // the next pivot A_{j+1,j+1}: row and column j + 1 are owned by ty == tx == (j+1) mod 16
      const int jn = j + 1, an = jn >> 4;
      if (jn < NB && tx == (jn & 15) && ty == (jn & 15)) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
          if (a == an) pivot = v[a][a];
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = ty + 16 * a, k = tx + 16 * b;
      A[(j0 + i) * lda + j0 + k] = k <= i ? v[a][b] : 0.0;
    }
}

// Rows [r0, r0 + nrows) of column block j0: X = A L^{-T}, L = A[j0.., j0..] (factored).
// Four threads per row (thread k holds entries c = k, k+4, ... in registers),
// right-looking: x_c = a_c / L_cc from its owner by a shuffle, then
// a_i -= x_c L_ic for i > c -- per entry the same fma sequence as the dot form.
constexpr int kPanelThreads = 128;
constexpr int kPanelRows = kPanelThreads / 4;
__global__ void __launch_bounds__(kPanelThreads) potrf_panel_kernel(double *A, int64_t lda, int64_t j0, int64_t r0,
                                                                    int64_t nrows) {
  __shared__ double Ls[NB][NB + 1];
  __shared__ double rd[NB];  // 1 / L_cc: the 64-step chain multiplies instead of dividing
#pragma unroll 8
  for (int e = threadIdx.x; e < NB * NB; e += kPanelThreads) {
    const int r = e / NB, c = e % NB;
    Ls[r][c] = A[(j0 + r) * lda + j0 + c];
  }
  __syncthreads();
  if (threadIdx.x < NB) rd[threadIdx.x] = __drcp_rn(Ls[threadIdx.x][threadIdx.x]);
  __syncthreads();
  const int lane = threadIdx.x & 31, k = lane & 3;
  const int64_t row = r0 + (int64_t)blockIdx.x * kPanelRows + (threadIdx.x >> 2);
  const bool ok = row < r0 + nrows;
  double *a = A + (ok ? row : r0) * lda + j0;
  double x[NB / 4];
#pragma unroll
  for (int t = 0; t < NB / 4; ++t) x[t] = ok ? a[4 * t + k] : 0.0;
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    double xc = 0.0;
    if (k == (c & 3)) {
      xc = __dmul_rn(x[c >> 2], rd[c]);
      x[c >> 2] = xc;
    }
    xc = __shfl_sync(0xffffffffu, xc, (lane & ~3) | (c & 3));
#pragma unroll
    for (int t = 0; t < NB / 4; ++t) {
      const int i = 4 * t + k;
      if (4 * t + 3 > c && i > c) x[t] = __fma_rn(-xc, Ls[i][c], x[t]);
    }
  }
  if (ok) {
#pragma unroll
    for (int t = 0; t < NB / 4; ++t) a[4 * t + k] = x[t];
  }
}

__global__ void zero_upper_kernel(double *A, int64_t lda, int64_t n) {
  const int64_t r = blockIdx.y;
  for (int64_t c = r + 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    A[r * lda + c] = 0.0;
}

// X[b] = L[b,b]^{-1} B[b] for one 64-row block.  Four threads per column (lanes
// 4c .. 4c+3 of a warp), thread k holding rows k, k+4, ... of the column in
// registers: step r takes x_r = b_r / L_rr from its owner by a shuffle and every
// thread updates its rows i > r, b_i -= L_ir x_r -- per entry the same fma
// sequence as the dot-product form.  8 columns per warp, 4 warps per CTA: 4x the
// warps of a thread-per-column solve for the latency-bound 64-step chain.
constexpr int kTrsmThreads = 128;
constexpr int kTrsmCols = kTrsmThreads / 4;
__global__ void __launch_bounds__(kTrsmThreads) trsm_diag_kernel(const double *L, int64_t ldl, int64_t b0, double *B,
                                                                 int64_t ldb, int64_t ncols) {
  __shared__ double Ls[NB][NB + 1];
  __shared__ double rd[NB];  // 1 / L_rr
#pragma unroll 8
  for (int e = threadIdx.x; e < NB * NB; e += kTrsmThreads) {
    const int r = e / NB, c = e % NB;
    Ls[r][c] = L[(b0 + r) * ldl + b0 + c];
  }
  __syncthreads();
  if (threadIdx.x < NB) rd[threadIdx.x] = __drcp_rn(Ls[threadIdx.x][threadIdx.x]);
  __syncthreads();
  const int lane = threadIdx.x & 31, k = lane & 3;
  const int64_t j = (int64_t)blockIdx.x * kTrsmCols + (threadIdx.x >> 2);
  const bool ok = j < ncols;
  double x[NB / 4];
#pragma unroll
  for (int t = 0; t < NB / 4; ++t) x[t] = ok ? B[(b0 + 4 * t + k) * ldb + j] : 0.0;
#pragma unroll
  for (int r = 0; r < NB; ++r) {
    // owner k == r % 4 holds row r in x[r / 4]
    double xr = 0.0;
    if (k == (r & 3)) {
      xr = __dmul_rn(x[r >> 2], rd[r]);
      x[r >> 2] = xr;
    }
    xr = __shfl_sync(0xffffffffu, xr, (lane & ~3) | (r & 3));
#pragma unroll
    for (int t = 0; t < NB / 4; ++t) {
      const int i = 4 * t + k;
      if (4 * t + 3 > r && i > r) x[t] = __fma_rn(-Ls[i][r], xr, x[t]);
    }
  }
  if (ok) {
#pragma unroll
    for (int t = 0; t < NB / 4; ++t) B[(b0 + 4 * t + k) * ldb + j] = x[t];
  }
}

__global__ void transpose_kernel(const double *__restrict__ A, int64_t rows, int64_t cols, int64_t lda,
                                 double *__restrict__ B, int64_t ldb) {
  __shared__ double t[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    t[k][threadIdx.x] = (r < rows && c < cols) ? A[r * lda + c] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = c0 + k, c = r0 + threadIdx.x;  // B[c][r] = A[r][c]
    if (r < cols && c < rows) B[r * ldb + c] = t[threadIdx.x][k];
  }
}

}  // namespace

// Two-level blocking: 64-wide diagonal steps inside 256-wide block columns, so the
// bulk of the flops is in K = 256 GEMM updates (a K = 64 DMMA GEMM runs at a
// fraction of the rate: its 3-stage ring never fills) -- same operations per entry.
constexpr int NB2 = 512;

void cholesky_lower(double *A, int64_t lda, int64_t n, int *flag, cudaStream_t s, int64_t *launches) {
  cholesky_lower_aug(A, lda, n, n, flag, s, launches);
}

// Rows [0, m) x columns [0, n) of A, m >= n: the lower Cholesky factor L of the leading
// n x n block and, in rows [n, m), B L^{-T} for the block B stored there -- the blocked
// factorization of [[A11, *], [B, *]] run over its first n columns (every panel solve and
// update also covers rows [n, m); the trailing matrix of rows >= n is never formed).
void cholesky_lower_aug(double *A, int64_t lda, int64_t n, int64_t m, int *flag, cudaStream_t s,
                        int64_t *launches) {
  for (int64_t J0 = 0; J0 < n; J0 += NB2) {
    const int64_t Jend = std::min<int64_t>(n, J0 + NB2);
    for (int64_t j0 = J0; j0 < Jend; j0 += NB) {
      potrf_diag_kernel<<<1, 256, 0, s>>>(A, lda, j0, flag);
      ++*launches;
      const int64_t rest = m - j0 - NB;
      if (rest <= 0) break;
      potrf_panel_kernel<<<(unsigned)((rest + kPanelRows - 1) / kPanelRows), kPanelThreads, 0, s>>>(A, lda, j0,
                                                                                                    j0 + NB, rest);
      ++*launches;
      const int64_t inblk = Jend - j0 - NB;  // remaining columns of this block column
      if (inblk <= 0) continue;
      GemmArgs g{};  // A[j0+64.., j0+64 .. Jend) -= P P[0:inblk]^T  (lower tiles)
      g.M = rest;
      g.N = inblk;
      g.K = NB;
      g.A = A + (j0 + NB) * lda + j0;
      g.lda = lda;
      g.B = g.A;
      g.ldb = lda;
      g.C = A + (j0 + NB) * lda + j0 + NB;
      g.ldc = lda;
      g.Cin = g.C;
      g.ldcin = lda;
      g.alpha = -1.0;
      g.beta = 1.0;
      g.lower_only = true;
      launch_dgemm(g, false, s);
      ++*launches;
    }
    const int64_t rest = m - Jend;
    if (n - Jend <= 0) break;
    GemmArgs g{};  // trailing matrix: A[Jend.., Jend..n) -= P P[0:n-Jend]^T with P = A[Jend.., J0 .. Jend)
    g.M = rest;
    g.N = n - Jend;
    g.K = Jend - J0;
    g.A = A + Jend * lda + J0;
    g.lda = lda;
    g.B = g.A;
    g.ldb = lda;
    g.C = A + Jend * lda + Jend;
    g.ldc = lda;
    g.Cin = g.C;
    g.ldcin = lda;
    g.alpha = -1.0;
    g.beta = 1.0;
    g.lower_only = true;
    launch_dgemm(g, false, s);
    ++*launches;
  }
  zero_upper_kernel<<<dim3(8, (unsigned)n), 256, 0, s>>>(A, lda, n);
  ++*launches;
}

void trsm_lower_left(const double *L, int64_t ldl, int64_t n, double *B, int64_t ldb, int64_t ncols,
                     cudaStream_t s, int64_t *launches) {
  for (int64_t B0 = 0; B0 < n; B0 += NB2) {
    const int64_t Bend = std::min<int64_t>(n, B0 + NB2);
    for (int64_t b0 = B0; b0 < Bend; b0 += NB) {
      trsm_diag_kernel<<<(unsigned)((ncols + kTrsmCols - 1) / kTrsmCols), kTrsmThreads, 0, s>>>(L, ldl, b0, B, ldb,
                                                                                                ncols);
      ++*launches;
      const int64_t inblk = Bend - b0 - NB;
      if (inblk <= 0) continue;
      GemmArgs g{};  // rows b0+64 .. Bend of the block: -= L[., b0:b0+64] X_b
      g.M = inblk;
      g.N = ncols;
      g.K = NB;
      g.A = L + (b0 + NB) * ldl + b0;
      g.lda = ldl;
      g.B = B + b0 * ldb;
      g.ldb = ldb;
      g.C = B + (b0 + NB) * ldb;
      g.ldc = ldb;
      g.Cin = g.C;
      g.ldcin = ldb;
      g.alpha = -1.0;
      g.beta = 1.0;
      launch_dgemm(g, true, s);
      ++*launches;
    }
    const int64_t rest = n - Bend;
    if (rest <= 0) break;
    GemmArgs g{};  // rows below the block: -= L[Bend.., B0:Bend] X_[B0:Bend]  (K = 256)
    g.M = rest;
    g.N = ncols;
    g.K = Bend - B0;
    g.A = L + Bend * ldl + B0;
    g.lda = ldl;
    g.B = B + B0 * ldb;
    g.ldb = ldb;
    g.C = B + Bend * ldb;
    g.ldc = ldb;
    g.Cin = g.C;
    g.ldcin = ldb;
    g.alpha = -1.0;
    g.beta = 1.0;
    launch_dgemm(g, true, s);
    ++*launches;
  }
}

void launch_transpose(const double *A, int64_t rows, int64_t cols, int64_t lda, double *B, int64_t ldb,
                      cudaStream_t s) {
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(A, rows, cols, lda, B, ldb);
}

}  // namespace laker
