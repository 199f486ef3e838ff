// Small dense factorizations for the CCCP fit, blocked so that the bulk of the
// work is the DMMA GEMM (dgemm.cu): right-looking Cholesky (64 x 64 diagonal
// blocks factored in shared memory, panel solve, lower-only trailing GEMM
// update) and the lower-triangular solve with many right-hand sides
// (64-row diagonal solves with the solution held in registers, GEMM updates
// of the rows below).
#include "laker_internal.h"

namespace laker {
namespace {

constexpr int NB = 64;

// Factor the 64 x 64 diagonal block at (j0, j0); zero its strict upper part.
__global__ void __launch_bounds__(256) potrf_diag_kernel(double *A, int64_t lda, int64_t j0, int *flag) {
  __shared__ double S[NB][NB + 1];
  const int tid = threadIdx.x;
  for (int e = tid; e < NB * NB; e += 256) {
    const int r = e / NB, c = e % NB;
    S[r][c] = A[(j0 + r) * lda + j0 + c];
  }
  __syncthreads();
  for (int j = 0; j < NB; ++j) {
    if (tid == 0) {
      const double d = S[j][j];
      if (!(d > 0.0)) {
        atomicExch(flag, 1);
        S[j][j] = 1.0;
      } else {
        S[j][j] = __dsqrt_rn(d);
      }
    }
    __syncthreads();
    const double piv = S[j][j];
    for (int i = j + 1 + tid; i < NB; i += 256) S[i][j] = __ddiv_rn(S[i][j], piv);
    __syncthreads();
    const int m = NB - j - 1;
    for (int e = tid; e < m * m; e += 256) {
      const int i = j + 1 + e / m, k = j + 1 + e % m;
      if (k <= i) S[i][k] = __fma_rn(-S[i][j], S[k][j], S[i][k]);
    }
    __syncthreads();
  }
  for (int e = tid; e < NB * NB; e += 256) {
    const int r = e / NB, c = e % NB;
    A[(j0 + r) * lda + j0 + c] = c <= r ? S[r][c] : 0.0;
  }
}

// Rows [r0, r0 + nrows) of column block j0: X = A L^{-T}, L = A[j0.., j0..] (factored).
// One CTA = 64 rows, one thread per row (the row held in registers).
__global__ void __launch_bounds__(64) potrf_panel_kernel(double *A, int64_t lda, int64_t j0, int64_t r0,
                                                         int64_t nrows) {
  __shared__ double Ls[NB][NB + 1];
  const int tid = threadIdx.x;
  for (int e = tid; e < NB * NB; e += 64) {
    const int r = e / NB, c = e % NB;
    Ls[r][c] = A[(j0 + r) * lda + j0 + c];
  }
  __syncthreads();
  const int64_t row = r0 + (int64_t)blockIdx.x * NB + tid;
  if (row >= r0 + nrows) return;
  double *a = A + row * lda + j0;
  double x[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    double s = a[c];
#pragma unroll
    for (int k = 0; k < c; ++k) s = __fma_rn(-x[k], Ls[c][k], s);
    x[c] = __ddiv_rn(s, Ls[c][c]);
  }
#pragma unroll
  for (int c = 0; c < NB; ++c) a[c] = x[c];
}

__global__ void zero_upper_kernel(double *A, int64_t lda, int64_t n) {
  const int64_t r = blockIdx.y;
  for (int64_t c = r + 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    A[r * lda + c] = 0.0;
}

// X[b] = L[b,b]^{-1} B[b] for one 64-row block; one thread per column, solution in registers.
__global__ void __launch_bounds__(128) trsm_diag_kernel(const double *L, int64_t ldl, int64_t b0, double *B,
                                                        int64_t ldb, int64_t ncols) {
  __shared__ double Ls[NB][NB + 1];
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    Ls[r][c] = L[(b0 + r) * ldl + b0 + c];
  }
  __syncthreads();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ncols) return;
  double x[NB];
#pragma unroll
  for (int r = 0; r < NB; ++r) {
    double s = B[(b0 + r) * ldb + j];
#pragma unroll
    for (int k = 0; k < r; ++k) s = __fma_rn(-Ls[r][k], x[k], s);
    x[r] = __ddiv_rn(s, Ls[r][r]);
  }
#pragma unroll
  for (int r = 0; r < NB; ++r) B[(b0 + r) * ldb + j] = x[r];
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

void cholesky_lower(double *A, int64_t lda, int64_t n, int *flag, cudaStream_t s, int64_t *launches) {
  for (int64_t j0 = 0; j0 < n; j0 += NB) {
    potrf_diag_kernel<<<1, 256, 0, s>>>(A, lda, j0, flag);
    ++*launches;
    const int64_t rest = n - j0 - NB;
    if (rest <= 0) break;
    potrf_panel_kernel<<<(unsigned)((rest + NB - 1) / NB), 64, 0, s>>>(A, lda, j0, j0 + NB, rest);
    ++*launches;
    GemmArgs g{};
    g.M = rest;
    g.N = rest;
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
  zero_upper_kernel<<<dim3(8, (unsigned)n), 256, 0, s>>>(A, lda, n);
  ++*launches;
}

void trsm_lower_left(const double *L, int64_t ldl, int64_t n, double *B, int64_t ldb, int64_t ncols,
                     cudaStream_t s, int64_t *launches) {
  for (int64_t b0 = 0; b0 < n; b0 += NB) {
    trsm_diag_kernel<<<(unsigned)((ncols + 127) / 128), 128, 0, s>>>(L, ldl, b0, B, ldb, ncols);
    ++*launches;
    const int64_t rest = n - b0 - NB;
    if (rest <= 0) break;
    GemmArgs g{};
    g.M = rest;
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
}

void launch_transpose(const double *A, int64_t rows, int64_t cols, int64_t lda, double *B, int64_t ldb,
                      cudaStream_t s) {
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(A, rows, cols, lda, B, ldb);
}

}  // namespace laker
