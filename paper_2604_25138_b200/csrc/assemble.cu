// Kernel assembly K_ij = exp(scale <e_i, e_j>) (Eq. sc-exp-kernel, P:141-147;
// Alg. 1 l.3) and the Jacobi diagonal
// d_i = 1 / (lambda + K_ii) (row a2).
//
// EXACT mode: each entry is RN(exp_cr(RN(scale * <e_i, e_j>))) with the dot product
// correctly rounded in practice -- a compensated sum over k whose accumulator carries
// the power-of-two offset C_ij >= 2 d max_k|e_ik| max_k|e_jk| (emax), so each step is
// TwoProd + Fast2Sum (dot2_step_off: exact error capture, 7 fp64 ops instead of Dot2's
// 10), the offset removed exactly before rounding -- bitwise the oracle's sequential
// Dot2 (and exp_cr is correctly rounded, exp_cr.cuh).  64 x 64 tiles, 256 threads, 4 x 4 entries
// per thread, E tiles staged through shared memory in 32-wide k chunks.
// Single-rank: only tiles J >= I are computed and mirrored through a shared-
// memory transpose, so K is bitwise symmetric and half the exps are saved.
//
// FAST mode: see assemble_fast.cu (fp64 DMMA tensor-core tiles).
#include "exp_cr.cuh"
#include "laker_internal.h"

namespace laker {
namespace {

constexpr int kT = 64;
constexpr int kKC = 32;

__device__ __forceinline__ void flag_add(unsigned long long *flags, unsigned int inc, unsigned int ovf) {
  if (inc) atomicAdd(&flags[0], (unsigned long long)inc);
  if (ovf) atomicAdd(&flags[1], (unsigned long long)ovf);
}

// sym = 1: grid (nt, nt) over the whole matrix, only J >= I tiles work, mirrored.
// sym = 0: grid (nt_cols, nt_local_rows): rows [r0, r1) x all columns.
__global__ void __launch_bounds__(256) assemble_exact_kernel(const double *__restrict__ E, int64_t n,
                                                             int d, double scale, int64_t r0,
                                                             int64_t r1, double *__restrict__ K,
                                                             int64_t ld, int sym,
                                                             unsigned long long *flags,
                                                             const double *__restrict__ emax) {
  __shared__ double buf[2 * kT * (kKC + 1)];
  double(*Ei)[kKC + 1] = reinterpret_cast<double(*)[kKC + 1]>(buf);
  double(*Ej)[kKC + 1] = reinterpret_cast<double(*)[kKC + 1]>(buf + kT * (kKC + 1));

  const int64_t I0 = sym ? (int64_t)blockIdx.y * kT : r0 + (int64_t)blockIdx.y * kT;
  const int64_t J0 = (int64_t)blockIdx.x * kT;
  if (sym && blockIdx.x < blockIdx.y) return;
  const int64_t rowEnd = sym ? n : r1;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;

  double ei[4], ej[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gi = I0 + ty + 16 * i, gj = J0 + tx + 16 * i;
    ei[i] = gi < rowEnd ? emax[gi] * (2.0 * d) : 0.0;
    ej[i] = gj < n ? emax[gj] : 0.0;
  }
  dd_pair acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = dd_pair{pow2_above(ei[i] * ej[j]), 0.0};

  for (int k0 = 0; k0 < d; k0 += kKC) {
    const int kc = min(kKC, d - k0);
    for (int idx = tid; idx < kT * kKC; idx += 256) {
      const int r = idx / kKC, c = idx % kKC;
      const int64_t gi = I0 + r, gj = J0 + r;
      Ei[r][c] = (gi < rowEnd && c < kc) ? E[gi * d + k0 + c] : 0.0;
      Ej[r][c] = (gj < n && c < kc) ? E[gj * d + k0 + c] : 0.0;
    }
    __syncthreads();
    for (int kk = 0; kk < kc; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = Ei[ty + 16 * i][kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Ej[tx + 16 * j][kk];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dot2_step_off(acc[i][j], av[i], bv[j]);
    }
    __syncthreads();
  }

  unsigned int inc = 0, ovf = 0;
  double v[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      dd_pair a = acc[i][j];
      a.s = __dsub_rn(a.s, pow2_above(ei[i] * ej[j]));  // exact (Sterbenz)
      v[i][j] = exp_cr(__dmul_rn(scale, pair_value(a)), inc, ovf);
    }
  flag_add(flags, inc, ovf);

  const int64_t rowBase = sym ? 0 : r0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gi = I0 + ty + 16 * i;
    if (gi >= rowEnd) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gj = J0 + tx + 16 * j;
      if (gj < n) K[(gi - rowBase) * ld + gj] = v[i][j];
    }
  }
  if (sym && blockIdx.x != blockIdx.y) {
    // mirrored tile K[J0.., I0..] via a shared-memory transpose (coalesced stores)
    double(*tr)[kT + 1] = reinterpret_cast<double(*)[kT + 1]>(buf);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) tr[ty + 16 * i][tx + 16 * j] = v[i][j];
    __syncthreads();
    const int cc = tid & 63;
    for (int rr = tid >> 6; rr < kT; rr += 4) {
      const int64_t gi = J0 + rr, gj = I0 + cc;
      if (gi < n && gj < n) K[gi * ld + gj] = tr[cc][rr];
    }
  }
}

__global__ void jacobi_diag_kernel(const double *__restrict__ E, int64_t n, int d, double scale,
                                   double lambda, double *__restrict__ dv, unsigned long long *flags) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  dd_pair acc = {0.0, 0.0};
  for (int k = 0; k < d; ++k) dot2_step(acc, E[i * d + k], E[i * d + k]);
  unsigned int inc = 0, ovf = 0;
  const double kii = exp_cr(__dmul_rn(scale, pair_value(acc)), inc, ovf);
  flag_add(flags, inc, ovf);
  dv[i] = __ddiv_rn(1.0, __dadd_rn(lambda, kii));
}

}  // namespace

void launch_assemble_exact_sym(const double *E, int64_t n, int32_t d, double scale, double *K,
                               int64_t ld, unsigned long long *flags, const double *emax, cudaStream_t s) {
  const unsigned nt = (unsigned)((n + kT - 1) / kT);
  assemble_exact_kernel<<<dim3(nt, nt), 256, 0, s>>>(E, n, d, scale, 0, n, K, ld, 1, flags, emax);
}

void launch_assemble_exact_rows(const double *E, int64_t n, int32_t d, double scale, int64_t r0,
                                int64_t r1, double *K, int64_t ld, unsigned long long *flags,
                                const double *emax, cudaStream_t s) {
  const unsigned ntc = (unsigned)((n + kT - 1) / kT);
  const unsigned ntr = (unsigned)((r1 - r0 + kT - 1) / kT);
  assemble_exact_kernel<<<dim3(ntc, ntr), 256, 0, s>>>(E, n, d, scale, r0, r1, K, ld, 0, flags, emax);
}

// out[i] = max_k |X_ik| (the offsets of the EXACT entry kernels)
__global__ void rowabsmax_kernel(const double *__restrict__ X, int64_t rows, int d, double *__restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  double m = 0.0;
  for (int k = 0; k < d; ++k) m = fmax(m, fabs(X[i * d + k]));
  out[i] = m;
}

void launch_rowabsmax(const double *X, int64_t rows, int32_t d, double *out, cudaStream_t s) {
  if (rows > 0) rowabsmax_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(X, rows, d, out);
}

void launch_jacobi_diag(const double *E, int64_t n, int32_t d, double scale, double lambda,
                        double *dvec, unsigned long long *flags, cudaStream_t s) {
  jacobi_diag_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(E, n, d, scale, lambda, dvec, flags);
}

}  // namespace laker
