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
// Right-looking in shared memory, 256 threads as a 16 x 16 grid: step j divides
// column j by the pivot sqrt(A_jj) (taken by every thread itself), then thread
// (ty, tx) applies A_ik -= L_ij L_kj to rows i = j+1+ty+16a, columns
// k = j+1+tx+16b with k <= i -- the textbook operations, two barriers per step.
__global__ void __launch_bounds__(256) potrf_diag_kernel(double *A, int64_t lda, int64_t j0, int *flag) {
  __shared__ double S[NB][NB + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
#pragma unroll 4
  for (int e = tid; e < NB * NB; e += 256) {
    const int r = e / NB, c = e % NB;
    S[r][c] = A[(j0 + r) * lda + j0 + c];
  }
  __syncthreads();
  for (int j = 0; j < NB; ++j) {
    double d = S[j][j];
    if (!(d > 0.0)) {
      if (tid == 0) atomicExch(flag, 1);
      d = 1.0;
    }
    const double piv = __dsqrt_rn(d);
    // column j below the diagonal (rows j+1+tid), the pivot itself by thread 63
    if (tid < NB - 1 - j) S[j + 1 + tid][j] = __ddiv_rn(S[j + 1 + tid][j], piv);
    __syncthreads();
    if (tid == NB - 1) S[j][j] = piv;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = j + 1 + ty + 16 * a;
      if (i < NB) {
        const double lij = S[i][j];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int k = j + 1 + tx + 16 * b;
          if (k <= i) S[i][k] = __fma_rn(-lij, S[k][j], S[i][k]);
        }
      }
    }
    __syncthreads();
  }
#pragma unroll 4
  for (int e = tid; e < NB * NB; e += 256) {
    const int r = e / NB, c = e % NB;
    A[(j0 + r) * lda + j0 + c] = c <= r ? S[r][c] : 0.0;
  }
}

// Rows [r0, r0 + nrows) of column block j0: X = A L^{-T}, L = A[j0.., j0..] (factored).
// One thread per row (the row held in registers), right-looking substitution:
// x_c = a_c / L_cc, then a_k -= x_c L_kc for k > c -- per entry the same fma
// sequence as the dot-product form, with 64 independent chains of ILP.
constexpr int kPanelThreads = 32;
__global__ void __launch_bounds__(kPanelThreads) potrf_panel_kernel(double *A, int64_t lda, int64_t j0, int64_t r0,
                                                                    int64_t nrows) {
  __shared__ double Ls[NB][NB + 1];
  const int tid = threadIdx.x;
#pragma unroll 16
  for (int e = tid; e < NB * NB; e += kPanelThreads) {
    const int r = e / NB, c = e % NB;
    Ls[r][c] = A[(j0 + r) * lda + j0 + c];
  }
  __syncthreads();
  const int64_t row = r0 + (int64_t)blockIdx.x * kPanelThreads + tid;
  if (row >= r0 + nrows) return;
  double *a = A + row * lda + j0;
  double x[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) x[c] = a[c];
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    x[c] = __ddiv_rn(x[c], Ls[c][c]);
#pragma unroll
    for (int k = c + 1; k < NB; ++k) x[k] = __fma_rn(-x[c], Ls[k][c], x[k]);
  }
#pragma unroll
  for (int c = 0; c < NB; ++c) a[c] = x[c];
}

__global__ void zero_upper_kernel(double *A, int64_t lda, int64_t n) {
  const int64_t r = blockIdx.y;
  for (int64_t c = r + 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    A[r * lda + c] = 0.0;
}

// X[b] = L[b,b]^{-1} B[b] for one 64-row block; one thread per column, solution
// in registers, right-looking (x_r = b_r / L_rr, then b_k -= L_kr x_r for k > r):
// per entry the same fma sequence as the dot-product form, 64 chains of ILP.
constexpr int kTrsmThreads = 32;
__global__ void __launch_bounds__(kTrsmThreads) trsm_diag_kernel(const double *L, int64_t ldl, int64_t b0, double *B,
                                                                 int64_t ldb, int64_t ncols) {
  __shared__ double Ls[NB][NB + 1];
#pragma unroll 16
  for (int e = threadIdx.x; e < NB * NB; e += kTrsmThreads) {
    const int r = e / NB, c = e % NB;
    Ls[r][c] = L[(b0 + r) * ldl + b0 + c];
  }
  __syncthreads();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ncols) return;
  double x[NB];
#pragma unroll
  for (int r = 0; r < NB; ++r) x[r] = B[(b0 + r) * ldb + j];
#pragma unroll
  for (int r = 0; r < NB; ++r) {
    x[r] = __ddiv_rn(x[r], Ls[r][r]);
#pragma unroll
    for (int k = r + 1; k < NB; ++k) x[k] = __fma_rn(-Ls[k][r], x[r], x[k]);
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
    potrf_panel_kernel<<<(unsigned)((rest + kPanelThreads - 1) / kPanelThreads), kPanelThreads, 0, s>>>(A, lda, j0,
                                                                                                      j0 + NB, rest);
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
    trsm_diag_kernel<<<(unsigned)((ncols + kTrsmThreads - 1) / kTrsmThreads), kTrsmThreads, 0, s>>>(L, ldl, b0, B, ldb,
                                                                                                    ncols);
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
