// LEARNED preconditioner: Alg. 1 l.5-14 and P = Sigma*^{-1/2}
// (Eq. preconditioner-Sigmma) on the GPU, in the exact structured
// form of DESIGN.md O4' (the same restatement the oracle pins against the
// literal n x n iteration):
//
//  1. directions  U = (lambda I + K) Z, ubar_k = u_k / ||u_k||
//     -- DMMA / Ozaki GEMM, Dot2 column norms;  Z from the caller or a Philox
//     stream; with ON_THE_FLY storage K's rows are assembled chunk by chunk
//     into a transient buffer feeding the GEMM (K is never stored);
//  2. thin QR  Ubar = Q R by shifted CholeskyQR3 (Fukaya et al., SIAM J. Sci.
//     Comput. 2020): three Gram / Cholesky / triangular-solve passes, all
//     GEMM-shaped; R = R3 R2 R1 with a positive diagonal (the oracle's sign
//     convention for its Householder R);
//  3. CCCP in N_r space: Sigma_t = a_t I + Ubar diag(b_t) Ubar^T,
//     T_t = a_t I + R diag(b_t) R^T, qf_k = ||L_T^{-1} R e_k||^2,
//     w = 1/(qf + eps), a' = (1-rho) gamma/(1+gamma/n) + rho,
//     b' = (1-rho)(n/N_r) w/(1+gamma/n), (a, b) <- n (a', b') / tr(Sigma~);
//     stop on ||Sigma_{t+1}-Sigma_t||_F / ||Sigma_t||_F <= fp_tol (reading R8),
//     evaluated exactly through C = Ubar^T Ubar;
//  4. T^{-1/2} by the coupled Newton-Schulz iteration (GEMMs only);
//  5. P = a^{-1/2} I + Q (T^{-1/2} - a^{-1/2} I) Q^T, kept factored (one rank)
//     or dense and row-sharded like K.
// N_r is padded to a multiple of 128 with an identity block in R (zero
// directions), which leaves every quantity of the first N_r rows unchanged.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "laker_internal.h"

namespace laker {
namespace {

// ------------------------------------------------------------ Philox normals
__device__ __forceinline__ void philox_round(uint32_t (&c)[4], uint32_t (&k)[2]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
  const uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
  const uint32_t n0 = hi1 ^ c[1] ^ k[0], n2 = hi0 ^ c[3] ^ k[1];
  c[0] = n0;
  c[1] = lo1;
  c[2] = n2;
  c[3] = lo0;
  k[0] += 0x9E3779B9u;
  k[1] += 0xBB67AE85u;
}

// Zt[k][i] ~ N(0,1) for k < nr, i < n (Philox4x32-10 + Box-Muller); padding zero.
__global__ void philox_normal_kernel(double *Zt, int64_t ldz, int64_t n, int64_t nr, uint64_t seed) {
  const int64_t total = nr * n;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; 2 * p < total; p += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c[4] = {(uint32_t)p, (uint32_t)(p >> 32), 0x4c414b45u, 0x52u};
    uint32_t k[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
#pragma unroll
    for (int r = 0; r < 10; ++r) philox_round(c, k);
    const double u1 = ((double)(((uint64_t)c[0] << 21) ^ (c[1] >> 11)) + 0.5) * 0x1p-53;
    const double u2 = ((double)(((uint64_t)c[2] << 21) ^ (c[3] >> 11)) + 0.5) * 0x1p-53;
    const double rad = sqrt(-2.0 * log(u1));
    double s, co;
    sincospi(2.0 * u2, &s, &co);
    const int64_t f0 = 2 * p, f1 = 2 * p + 1;
    Zt[(f0 / n) * ldz + f0 % n] = rad * co;
    if (f1 < total) Zt[(f1 / n) * ldz + f1 % n] = rad * s;
  }
}

// ------------------------------------------------------------ small kernels
// row norms of Ut (nr rows, n cols): Dot2 sum of squares, then scale the row.
__global__ void __launch_bounds__(256) normalize_rows_kernel(double *Ut, int64_t ld, int64_t n) {
  __shared__ dd_pair red[8];
  __shared__ double s_norm;
  double *row = Ut + (int64_t)blockIdx.x * ld;
  dd_pair acc = {0.0, 0.0};
  for (int64_t i = threadIdx.x; i < n; i += 256) dot2_step(acc, row[i], row[i]);
  acc = warp_reduce_pair(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    dd_pair t = red[0];
    for (int w = 1; w < 8; ++w) pair_add(t, red[w]);
    s_norm = __dsqrt_rn(pair_value(t));
  }
  __syncthreads();
  const double nr = s_norm;
  for (int64_t i = threadIdx.x; i < n; i += 256) row[i] = __ddiv_rn(row[i], nr);
}

// A[i][i] += v for i in [i0, i1)
__global__ void add_diag_kernel(double *A, int64_t lda, int64_t i0, int64_t i1, double v) {
  const int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < i1) A[i * lda + i] += v;
}

__global__ void copy_diag_kernel(const double *A, int64_t lda, int64_t n, double *d) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = A[i * lda + i];
}

// S = R diag(sqrt(b)) (b padded with zeros)
__global__ void scale_cols_sqrt_kernel(const double *R, double *S, int64_t ld, int64_t nrp, const double *b) {
  const int64_t r = blockIdx.y;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nrp; c += (int64_t)gridDim.x * blockDim.x)
    S[r * ld + c] = R[r * ld + c] * __dsqrt_rn(b[c]);
}

// qf[k] = sum_j X[k][j]^2 over columns [0, cols) for rows k < nr (Dot2 per lane, lanes
// combined by the fixed xor tree): one warp per row
__global__ void row_sumsq_kernel(const double *X, int64_t ld, int64_t cols, int64_t nr, double *qf) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= nr) return;
  dd_pair acc = {0.0, 0.0};
  for (int64_t j = lane; j < cols; j += 32) {
    const double v = X[k * ld + j];
    dot2_step(acc, v, v);
  }
  acc = warp_reduce_pair(acc);
  if (lane == 0) qf[k] = pair_value(acc);
}

struct CccpScalars {
  double a, a_new, tr, change, d2, s2, rho, gamma, eps, nn, nr;
  double sum_db_cd, sum_b_cd;
};

// One CTA: w, b', tr, (a, b) update and the linear pieces of the Frobenius
// change.  b_old kept in bo for the quadratic forms.
__global__ void __launch_bounds__(1024) cccp_update_kernel(const double *qf, const double *cd, double *b,
                                                           double *bo, double *db, int64_t nr, CccpScalars *sc) {
  __shared__ dd_pair red[32][3];
  __shared__ double s_tr, s_anew;
  const double rho = sc->rho, gamma = sc->gamma, eps = sc->eps, n = sc->nn, NR = sc->nr;
  const double den = 1.0 + gamma / n;
  const double a1 = (1.0 - rho) * gamma / den + rho;
  dd_pair acc = {0.0, 0.0};
  for (int64_t k = threadIdx.x; k < nr; k += blockDim.x) {
    const double w = 1.0 / (qf[k] + eps);
    const double b1 = (1.0 - rho) * (n / NR) * w / den;
    db[k] = b1;  // temporarily b'
    dot2_step(acc, b1, cd[k]);
  }
  acc = warp_reduce_pair(acc);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp][0] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    dd_pair t = {0.0, 0.0};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) pair_add(t, red[w][0]);
    double s = 0.0, e = 0.0;
    two_prod(n, a1, s, e);
    dd_pair tt = {s, e};
    pair_add(tt, t);
    s_tr = pair_value(tt);
    s_anew = n * a1 / s_tr;
  }
  __syncthreads();
  const double tr = s_tr, anew = s_anew, aold = sc->a;
  dd_pair p1 = {0.0, 0.0}, p2 = {0.0, 0.0};
  for (int64_t k = threadIdx.x; k < nr; k += blockDim.x) {
    const double bnew = n * db[k] / tr;
    const double bold = b[k];
    bo[k] = bold;
    b[k] = bnew;
    const double d = bnew - bold;
    db[k] = d;
    dot2_step(p1, d, cd[k]);
    dot2_step(p2, bold, cd[k]);
  }
  p1 = warp_reduce_pair(p1);
  p2 = warp_reduce_pair(p2);
  if (lane == 0) {
    red[warp][1] = p1;
    red[warp][2] = p2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    dd_pair t1 = {0.0, 0.0}, t2 = {0.0, 0.0};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      pair_add(t1, red[w][1]);
      pair_add(t2, red[w][2]);
    }
    sc->sum_db_cd = pair_value(t1);
    sc->sum_b_cd = pair_value(t2);
    sc->tr = tr;
    sc->a_new = anew;
  }
}

// quadratic forms q1 = db^T (C o C) db, q2 = bo^T (C o C) bo; one warp per row
// (coalesced), per-CTA pairs then the last CTA finishes the change.
__global__ void __launch_bounds__(256) cccp_quadform_kernel(const double *C, int64_t ld, int64_t nr,
                                                            const double *db, const double *bo,
                                                            dd_pair *partials, unsigned int *counter,
                                                            CccpScalars *sc) {
  __shared__ dd_pair red[8][2];
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  dd_pair q1 = {0.0, 0.0}, q2 = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * 8 + warp; i < nr; i += (int64_t)gridDim.x * 8) {
    dd_pair r1 = {0.0, 0.0}, r2 = {0.0, 0.0};
    for (int64_t k = lane; k < nr; k += 32) {
      const double c = C[i * ld + k];
      const double c2 = c * c;
      dot2_step(r1, c2, db[k]);
      dot2_step(r2, c2, bo[k]);
    }
    r1 = warp_reduce_pair(r1);
    r2 = warp_reduce_pair(r2);
    // row contribution: db_i * (C o C db)_i
    dot2_step(q1, db[i], pair_value(r1));
    dot2_step(q2, bo[i], pair_value(r2));
  }
  if (lane == 0) {
    red[warp][0] = q1;
    red[warp][1] = q2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    dd_pair t1 = red[0][0], t2 = red[0][1];
    for (int w = 1; w < 8; ++w) {
      pair_add(t1, red[w][0]);
      pair_add(t2, red[w][1]);
    }
    partials[2 * blockIdx.x] = t1;
    partials[2 * blockIdx.x + 1] = t2;
    __threadfence();
    s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    dd_pair t1 = {0.0, 0.0}, t2 = {0.0, 0.0};
    for (unsigned b = 0; b < gridDim.x; ++b) {
      dd_pair o1 = {__ldcg(&partials[2 * b].s), __ldcg(&partials[2 * b].c)};
      dd_pair o2 = {__ldcg(&partials[2 * b + 1].s), __ldcg(&partials[2 * b + 1].c)};
      pair_add(t1, o1);
      pair_add(t2, o2);
    }
    *counter = 0u;
    const double n = sc->nn, a = sc->a, an = sc->a_new, da = an - a;
    const double d2 = n * da * da + 2.0 * da * sc->sum_db_cd + pair_value(t1);
    const double s2 = n * a * a + 2.0 * a * sc->sum_b_cd + pair_value(t2);
    sc->d2 = d2;
    sc->s2 = s2;
    sc->change = __dsqrt_rn(fmax(d2, 0.0)) / __dsqrt_rn(s2);
    sc->a = an;
  }
}

// ||W - I||_F^2 partial sums (NS convergence), symmetric averaging of Y, Z.
__global__ void __launch_bounds__(256) frob_minus_identity_kernel(const double *W, int64_t ld, int64_t n,
                                                                  double *out) {
  __shared__ double red[8];
  double s = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    const double v = W[i * ld + j] - (i == j ? 1.0 : 0.0);
    s += v * v;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    atomicAdd(out, t);
  }
}

__global__ void symmetrize_kernel(double *A, int64_t ld, int64_t n) {
  const int64_t i = blockIdx.y;
  for (int64_t j = i + 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const double v = 0.5 * (A[i * ld + j] + A[j * ld + i]);
    A[i * ld + j] = v;
    A[j * ld + i] = v;
  }
}

__global__ void scale_kernel(double *A, int64_t ld, int64_t rows, int64_t cols, double s) {
  const int64_t r = blockIdx.y;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += (int64_t)gridDim.x * blockDim.x)
    A[r * ld + c] *= s;
}

__global__ void set_identity_kernel(double *A, int64_t ld, int64_t n) {
  const int64_t r = blockIdx.y;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    A[r * ld + c] = (r == c) ? 1.0 : 0.0;
}

// power iteration step: y = A x / ||x||, returns ||A x|| estimate via atomic
__global__ void __launch_bounds__(256) matvec_kernel(const double *A, int64_t ld, int64_t n, const double *x,
                                                     double *y) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t i = (int64_t)blockIdx.x * 8 + warp; i < n; i += (int64_t)gridDim.x * 8) {
    double s = 0.0;
    for (int64_t k = lane; k < n; k += 32) s = __fma_rn(A[i * ld + k], x[k], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[i] = s;
  }
}

__global__ void __launch_bounds__(1024) normalize_vec_kernel(double *x, int64_t n, double *norm_out) {
  __shared__ double red[32];
  __shared__ double s_n;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = __fma_rn(x[i], x[i], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    s_n = sqrt(t);
    *norm_out = s_n;
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x[i] /= s_n;
}

__global__ void fill_kernel(double *x, int64_t n, double v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = v;
}

inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

struct DevMem {
  std::vector<void *> ptrs;
  cudaStream_t s;
  ~DevMem() {
    for (void *p : ptrs) cudaFreeAsync(p, s);
  }
  template <class T>
  cudaError_t alloc(T **p, size_t count) {
    cudaError_t e = cudaMallocAsync((void **)p, std::max<size_t>(count, 1) * sizeof(T), s);
    if (e == cudaSuccess) ptrs.push_back(*p);
    return e;
  }
};

double host_rho(int64_t nr, int64_t n, double gamma, double lmin, double rho_floor) {
  double rho;
  if (nr >= n) {
    rho = rho_floor;
  } else {
    rho = rho_floor + 0.5 * (1.0 - (double)nr / (double)n) * std::min(1.0, 10.0 * gamma);
    rho = std::min(std::max(rho, rho_floor), 0.9);
  }
  if (lmin < 1e-6) rho = std::max(rho, 0.2);
  return rho;
}

}  // namespace

void free_factors(laker_ctx ctx) {
  cudaFree(ctx->Qt);
  cudaFree(ctx->Qr);
  cudaFree(ctx->Mf);
  cudaFree(ctx->QMf);
  ctx->QMf = nullptr;
  ctx->p_qm = false;
  cudaFree(ctx->fz);
  ctx->Qt = ctx->Qr = ctx->Mf = ctx->fz = ctx->fw = nullptr;
  ctx->p_factored = false;
  ctx->f_local = false;
  ctx->f_nr = ctx->f_nrp = ctx->f_ldq = 0;
  ctx->f_alloc_nrp = ctx->f_alloc_n = 0;
}

// P = a^{-1/2} I + Q M Q^T, rows [r0, r1) into ctx->P.  P_ij = W_i . Q_j for i >= j
// and Q_i . W_j for i < j (+ a^{-1/2} on the diagonal) with W = Q M: the upper
// entry (i, j) is the same DMMA dot product as the lower entry (j, i) (the product
// is commutative in its operands), so P is bitwise symmetric, every row is
// independent of the row sharding (each rank holds W and Q in full), and the work
// is one n_loc x n x N_r GEMM split in two (B4).
laker_status form_dense_p(laker_ctx ctx, const double *Ut, const double *Mm, int64_t ldm, int64_t nrp,
                          double ainv) {
  const int64_t n = ctx->n, ld = ctx->ld;
  cudaStream_t s = ctx->stream;
  int64_t &L = ctx->stats.kernel_launches;
  DevMem mem{{}, s};
  double *Wt, *Qr, *Wr;  // Wt = M Q^T (nrp x ld); Qr, Wr row-major ld x nrp (k contiguous)
  LAKER_CUDA(ctx, mem.alloc(&Wt, (size_t)nrp * ld));
  LAKER_CUDA(ctx, mem.alloc(&Qr, (size_t)ld * nrp));
  LAKER_CUDA(ctx, mem.alloc(&Wr, (size_t)ld * nrp));
  GemmArgs g{};
  g.M = nrp; g.N = ld; g.K = nrp; g.A = Mm; g.lda = ldm; g.B = Ut; g.ldb = ld; g.C = Wt; g.ldc = ld;
  g.alpha = 1.0;
  launch_dgemm(g, true, s);
  launch_transpose(Ut, nrp, ld, ld, Qr, nrp, s);
  launch_transpose(Wt, nrp, ld, ld, Wr, nrp, s);
  L += 3;
  if (!ctx->P) LAKER_CUDA(ctx, cudaMalloc(&ctx->P, (size_t)(ctx->r1 - ctx->r0) * ld * 8));
  LAKER_CUDA(ctx, cudaMemsetAsync(ctx->P, 0, (size_t)(ctx->r1 - ctx->r0) * ld * 8, s));
  GemmArgs p{};
  p.M = ctx->r1 - ctx->r0; p.N = n; p.K = nrp;
  p.A = Wr + ctx->r0 * nrp; p.lda = nrp; p.B = Qr; p.ldb = nrp; p.C = ctx->P; p.ldc = ld;
  p.alpha = 1.0; p.diag = ainv; p.diag_offset = -ctx->r0; p.tri = 1; p.tri_off = ctx->r0;
  launch_dgemm(p, false, s);
  p.A = Qr + ctx->r0 * nrp; p.B = Wr; p.diag = 0.0; p.tri = 2;
  launch_dgemm(p, false, s);
  L += 2;
  if (n % 2 == 1) {  // the last double2 store of each row spilled one past n: restore zero padding
    LAKER_CUDA(ctx, cudaMemset2DAsync(ctx->P + n, ld * 8, 0, 8, ctx->r1 - ctx->r0, s));
  }
  LAKER_CUDA(ctx, cudaGetLastError());
  return LAKER_OK;
}

laker_status ensure_dense_p(laker_ctx ctx) {
  if (ctx->P || !ctx->p_factored) return LAKER_OK;
  if (ctx->f_local && ctx->world > 1)
    return set_err(ctx, LAKER_ERR_NOT_READY, "dense P rows: the sharded context keeps only its part of the factors");
  LAKER_TRY(form_dense_p(ctx, ctx->Qt, ctx->Mf, ctx->f_ldq, ctx->f_nrp, ctx->f_ainv));
  LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return LAKER_OK;
}

laker_status fit_learned(laker_ctx ctx, const laker_fit_opts &o, laker_fit_report *rep) {
  const int64_t n = ctx->n, ld = ctx->ld;
  int64_t nr = o.n_dirs;
  if (nr <= 0) nr = std::min<int64_t>(n, std::max<int64_t>((int64_t)std::ceil(8.0 * std::sqrt((double)n)),
                                                            (int64_t)std::ceil(n / 4.0)));
  if (nr > n * 64) return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "fit: n_dirs too large");
  const int64_t nrp = (nr + 127) / 128 * 128;
  const double gamma = o.gamma, eps = o.eps;
  const int32_t max_iters = o.max_iters > 0 ? o.max_iters : 200;
  const double fp_tol = o.fp_tol > 0 ? o.fp_tol : 1e-8;
  const double rho_floor = o.rho_floor > 0 ? o.rho_floor : 1e-3;
  cudaStream_t s = ctx->stream;
  int64_t &L = ctx->stats.kernel_launches;
  DevMem mem{{}, s};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);

  double *Zt, *Ut, *Cg, *G, *L1, *L2, *L3, *R, *Rt, *T, *X, *S, *qf, *cd, *b, *bo, *db, *scal;
  int *flag;
  CccpScalars *sc;
  const size_t big = (size_t)nrp * ld, sq = (size_t)nrp * nrp;
  LAKER_CUDA(ctx, mem.alloc(&Zt, big));
  LAKER_CUDA(ctx, mem.alloc(&Ut, big));
  LAKER_CUDA(ctx, mem.alloc(&Cg, sq));
  LAKER_CUDA(ctx, mem.alloc(&G, sq));
  LAKER_CUDA(ctx, mem.alloc(&L1, sq));
  LAKER_CUDA(ctx, mem.alloc(&L2, sq));
  LAKER_CUDA(ctx, mem.alloc(&L3, sq));
  LAKER_CUDA(ctx, mem.alloc(&R, sq));
  LAKER_CUDA(ctx, mem.alloc(&Rt, sq));
  LAKER_CUDA(ctx, mem.alloc(&T, 2 * sq));  // rows [nrp, 2 nrp): R^T for the augmented Cholesky
  LAKER_CUDA(ctx, mem.alloc(&X, sq));
  LAKER_CUDA(ctx, mem.alloc(&S, sq));
  LAKER_CUDA(ctx, mem.alloc(&qf, nrp));
  LAKER_CUDA(ctx, mem.alloc(&cd, nrp));
  LAKER_CUDA(ctx, mem.alloc(&b, nrp));
  LAKER_CUDA(ctx, mem.alloc(&bo, nrp));
  LAKER_CUDA(ctx, mem.alloc(&db, nrp));
  LAKER_CUDA(ctx, mem.alloc(&scal, 8));
  LAKER_CUDA(ctx, mem.alloc(&flag, 2));  // [0] factorization failed, [1] R6 trigger test
  LAKER_CUDA(ctx, mem.alloc(&sc, 1));
  LAKER_CUDA(ctx, cudaMemsetAsync(Zt, 0, big * 8, s));
  LAKER_CUDA(ctx, cudaMemsetAsync(Ut, 0, big * 8, s));  // padding columns [n, ld) must stay zero
  LAKER_CUDA(ctx, cudaMemsetAsync(flag, 0, sizeof(int), s));
  LAKER_CUDA(ctx, cudaMemsetAsync(b, 0, nrp * 8, s));
  const bool debug = std::getenv("LAKER_DEBUG_FIT") != nullptr;
  const bool dump = debug && std::getenv("LAKER_DEBUG_FIT")[0] == '2';
  auto dbg = [&](const char *name, const double *p, int64_t rows, int64_t cols, int64_t ldm) {
    if (!dump) return;
    std::vector<double> h((size_t)rows * ldm);
    cudaMemcpyAsync(h.data(), p, h.size() * 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    int64_t nan = 0;
    double mx = 0.0, fro = 0.0;
    for (int64_t r = 0; r < rows; ++r)
      for (int64_t c = 0; c < cols; ++c) {
        const double v = h[r * ldm + c];
        if (!std::isfinite(v)) ++nan;
        else { mx = std::max(mx, std::fabs(v)); fro += v * v; }
      }
    std::fprintf(stderr, "[fit] %-8s %lldx%lld nonfinite=%lld max=%.6e fro=%.6e first=%.6e err=%s\n", name,
                 (long long)rows, (long long)cols, (long long)nan, mx, std::sqrt(fro), h[0],
                 cudaGetErrorString(cudaGetLastError()));
  };

  cudaEvent_t tk_prev = nullptr;
  auto tick = [&](const char *what) {  // LAKER_DEBUG_FIT: device time of each fit phase
    if (!debug) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    cudaEventSynchronize(e);
    if (tk_prev) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tk_prev, e);
      std::fprintf(stderr, "[fit] phase %-12s %9.3f ms\n", what, ms);
      cudaEventDestroy(tk_prev);
    }
    tk_prev = e;
  };
  tick("start");

  // ---- 1. directions: Zt (N_r x n, row k = z_k), U^T = Zt K^T + lambda Zt
  if (o.Z) {
    cudaPointerAttributes at{};
    cudaMemcpyKind kind = cudaMemcpyHostToDevice;
    if (cudaPointerGetAttributes(&at, o.Z) == cudaSuccess &&
        (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged))
      kind = cudaMemcpyDeviceToDevice;
    cudaGetLastError();
    LAKER_CUDA(ctx, cudaMemcpy2DAsync(Zt, ld * 8, o.Z, n * 8, n * 8, nr, kind, s));
  } else {
    philox_normal_kernel<<<4 * ctx->num_sms, 256, 0, s>>>(Zt, ld, n, nr, o.seed);
    ++L;
  }
  // columns [cb, ce) of U^T = Zt K^T + lambda Zt into C (leading dimension ldc).  K is
  // symmetric, so K^T's columns [cb, ce) are K's rows [cb, ce): the stored local rows, or,
  // when K is not stored (ON_THE_FLY: LAKER at C5), rows assembled
  // chunk by chunk into a scratch buffer of <= 4 GiB by the assembly kernels of the
  // ctx's mode (EXACT: correctly rounded, bitwise the stored K) and consumed by the GEMM
  auto directions = [&](int64_t cb, int64_t ce, double *C, int64_t ldc) -> laker_status {
    GemmArgs g{};
    g.M = nrp; g.K = ld;
    g.A = Zt; g.lda = ld; g.ldb = ld;
    g.ldc = ldc; g.alpha = 1.0; g.beta = ctx->lambda; g.ldcin = ld;
    if (ctx->storage == LAKER_STORE_MATERIALIZED) {
      g.N = ce - cb; g.B = ctx->K; g.C = C; g.Cin = Zt + cb;
      launch_dgemm(g, false, s);
      ++L;
      return LAKER_OK;
    }
    int64_t cap = std::max<int64_t>(128, ((int64_t)4 << 30) / (ld * 8) / 128 * 128);
    if (const char *env = std::getenv("LAKER_FIT_OTF_CHUNK")) cap = std::max<int64_t>(1, std::atoll(env));  // tests
    const int64_t cw = std::min(ce - cb, cap);
    double *Kc;
    LAKER_CUDA(ctx, mem.alloc(&Kc, (size_t)cw * ld));
    LAKER_CUDA(ctx, cudaMemsetAsync(Kc, 0, (size_t)cw * ld * 8, s));  // padding columns [n, ld) stay zero
    for (int64_t c0 = cb; c0 < ce; c0 += cw) {
      const int64_t c1 = std::min(ce, c0 + cw);
      if (ctx->mode == LAKER_MODE_EXACT)
        launch_assemble_exact_rows(ctx->E, n, ctx->d, ctx->scale, c0, c1, Kc, ld, ctx->flags, ctx->emax, s);
      else
        launch_assemble_fast(ctx->E, n, ctx->d, ctx->scale, c0, c1, Kc, ld, ctx->flags, s);
      g.N = c1 - c0; g.B = Kc; g.C = C + (c0 - cb); g.Cin = Zt + c0;
      launch_dgemm(g, false, s);
      L += 2;
    }
    return LAKER_OK;
  };
  if (!ctx->comm) {
    LAKER_TRY(directions(0, n, Ut, ld));
  } else {
    // row-sharded K: this rank forms the columns [r0, r1) of U^T = Zt K^T + lambda Zt,
    // the W column blocks are all-gathered and the rest of the fit runs replicated
    // (identical kernels on identical data on every rank).
    const int64_t nloc = ctx->r1 - ctx->r0;
    double *Uloc, *Urecv;
    LAKER_CUDA(ctx, mem.alloc(&Uloc, (size_t)nrp * nloc));
    LAKER_CUDA(ctx, mem.alloc(&Urecv, (size_t)nrp * nloc * ctx->world));
    LAKER_TRY(directions(ctx->r0, ctx->r1, Uloc, nloc));
    LAKER_NCCL(ctx, ncclAllGather(Uloc, Urecv, (size_t)nrp * nloc, ncclDouble, ctx->comm, s));
    LAKER_CUDA(ctx, cudaMemsetAsync(Ut, 0, big * 8, s));
    for (int w = 0; w < ctx->world; ++w)
      LAKER_CUDA(ctx, cudaMemcpy2DAsync(Ut + (size_t)w * nloc, ld * 8, Urecv + (size_t)w * nrp * nloc, nloc * 8,
                                        nloc * 8, nrp, cudaMemcpyDeviceToDevice, s));
    ++L;
  }
  normalize_rows_kernel<<<(unsigned)nr, 256, 0, s>>>(Ut, ld, n);
  ++L;
  dbg("Ubar", Ut, nrp, ld, ld);

  tick("directions");
  // ---- 2. shifted CholeskyQR3 of Ubar (rows of Ut): Ut <- Q^T, R = R3 R2 R1
  auto gram = [&](double *dst) {  // SYRK: lower triangle on the tensor cores, mirrored
    GemmArgs g{};
    g.M = nrp; g.N = nrp; g.K = ld;
    g.A = Ut; g.lda = ld; g.B = Ut; g.ldb = ld; g.C = dst; g.ldc = nrp; g.alpha = 1.0; g.tri = 1;
    launch_dgemm(g, false, s);
    launch_mirror_lower(dst, nrp, nrp, s);
    L += 2;
  };
  gram(Cg);  // C = Ubar^T Ubar (kept for the Frobenius change)
  copy_diag_kernel<<<cdiv(nr, 256), 256, 0, s>>>(Cg, nrp, nr, cd);
  ++L;
  LAKER_CUDA(ctx, cudaMemcpyAsync(G, Cg, sq * 8, cudaMemcpyDeviceToDevice, s));
  const double u = 0x1p-53;
  const double shift = 11.0 * ((double)n * nr + (double)nr * (nr + 1)) * u * (double)nr;  // ||Ubar||_2^2 <= N_r
  add_diag_kernel<<<cdiv(nr, 256), 256, 0, s>>>(G, nrp, 0, nr, shift);
  if (nrp > nr) add_diag_kernel<<<cdiv(nrp - nr, 256), 256, 0, s>>>(G, nrp, nr, nrp, 1.0);
  L += 2;
  double *Ls[3] = {L1, L2, L3};
  for (int pass = 0; pass < 3; ++pass) {
    if (pass > 0) {
      gram(G);
      if (nrp > nr) {
        add_diag_kernel<<<cdiv(nrp - nr, 256), 256, 0, s>>>(G, nrp, nr, nrp, 1.0);
        ++L;
      }
    }
    cholesky_lower(G, nrp, nrp, flag, s, &L);
    LAKER_CUDA(ctx, cudaMemcpyAsync(Ls[pass], G, sq * 8, cudaMemcpyDeviceToDevice, s));
    trsm_lower_left(Ls[pass], nrp, nrp, Ut, ld, ld, s, &L);
  }
  // L_tot = L1 L2 L3 (R = L_tot^T)
  {
    // products of lower-triangular factors are lower triangular: only the tiles on or below
    // the diagonal are formed (tri = 1; the strict upper parts are zeroed first -- the same
    // lower entries, exact zeros above)
    LAKER_CUDA(ctx, cudaMemsetAsync(X, 0, sq * 8, s));
    LAKER_CUDA(ctx, cudaMemsetAsync(Rt, 0, sq * 8, s));
    GemmArgs g{};
    g.M = nrp; g.N = nrp; g.K = nrp; g.A = L1; g.lda = nrp; g.B = L2; g.ldb = nrp; g.C = X; g.ldc = nrp;
    g.alpha = 1.0;
    g.tri = 1;
    launch_dgemm(g, true, s);
    g.A = X; g.B = L3; g.C = Rt;
    launch_dgemm(g, true, s);
    L += 2;
    launch_transpose(Rt, nrp, nrp, nrp, R, nrp, s);  // R upper, positive diagonal
    ++L;
  }
  dbg("Cg", Cg, nrp, nrp, nrp);
  dbg("R", R, nrp, nrp, nrp);
  dbg("Qt", Ut, nrp, ld, ld);
  int hflag = 0;
  LAKER_CUDA(ctx, cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  if (hflag) return set_err(ctx, LAKER_ERR_NOT_POSITIVE_DEFINITE, "fit: CholeskyQR of the directions failed");

  tick("cholqr3");
  // ---- 3. CCCP iteration on (a, b)
  CccpScalars hs{};
  hs.a = 1.0;
  hs.gamma = gamma;
  hs.eps = eps;
  hs.nn = (double)n;
  hs.nr = (double)nr;
  double a = 1.0, change = INFINITY, rho_used = 0.0;
  int32_t it = 0;
  bool converged = false;
  for (it = 0; it < max_iters;) {
    // T = a I + (R diag(sqrt b)) (R diag(sqrt b))^T
    scale_cols_sqrt_kernel<<<dim3(cdiv(nrp, 256), (unsigned)nrp), 256, 0, s>>>(R, S, nrp, nrp, b);
    GemmArgs g{};
    g.M = nrp; g.N = nrp; g.K = nrp; g.A = S; g.lda = nrp; g.B = S; g.ldb = nrp; g.C = T; g.ldc = nrp;
    g.alpha = 1.0; g.diag = a; g.tri = 1;  // the Cholesky reads the lower triangle only
    launch_dgemm(g, false, s);
    // rho trigger of reading R6: lambda_min(Sigma_t) < 1e-6.  lambda_min(Sigma_t) = a_t when
    // N_r < n (O4'); when N_r >= n, Sigma_t = Q T_t Q^T with Q square, so lambda_min(Sigma_t) =
    // lambda_min(T_t) (the oracle's eigvalsh(T)[0]), decided here by whether T_t - 1e-6 I (the
    // leading nr x nr block; the identity padding is lifted) has a Cholesky factor
    double lmin = a;
    if (o.rho < 0.0 && nr >= n) {
      LAKER_CUDA(ctx, cudaMemcpyAsync(X, T, sq * 8, cudaMemcpyDeviceToDevice, s));
      add_diag_kernel<<<cdiv(nr, 256), 256, 0, s>>>(X, nrp, 0, nr, -1e-6);
      if (nrp > nr) add_diag_kernel<<<cdiv(nrp - nr, 256), 256, 0, s>>>(X, nrp, nr, nrp, 1.0);
      LAKER_CUDA(ctx, cudaMemsetAsync(flag + 1, 0, sizeof(int), s));
      cholesky_lower(X, nrp, nrp, flag + 1, s, &L);
      int lflag = 0;
      LAKER_CUDA(ctx, cudaMemcpyAsync(&lflag, flag + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
      LAKER_CUDA(ctx, cudaStreamSynchronize(s));
      lmin = lflag ? 0.0 : 1.0;  // only the comparison with 1e-6 enters host_rho
      L += 2;
    }
    const double rho_t = o.rho >= 0.0 ? o.rho : host_rho(nr, n, gamma, lmin, rho_floor);
    hs.rho = rho_t;
    hs.a = a;
    LAKER_CUDA(ctx, cudaMemcpyAsync(sc, &hs, sizeof(hs), cudaMemcpyHostToDevice, s));
    // q_k = || L_t^{-1} r_k ||^2 (T_t = L_t L_t^T, r_k column k of R): the Cholesky of
    // [[T_t, *], [R^T, *]] over its first N_r columns leaves R^T L_t^{-T} = (L_t^{-1} R)^T in
    // rows [nrp, 2 nrp) -- the triangular solve done inside the factorization's panel
    // steps instead of a separate blocked solve (one launch chain instead of two)
    LAKER_CUDA(ctx, cudaMemcpyAsync(T + sq, Rt, sq * 8, cudaMemcpyDeviceToDevice, s));
    cholesky_lower_aug(T, nrp, nrp, 2 * nrp, flag, s, &L);
    row_sumsq_kernel<<<(unsigned)cdiv(nr, 8), 256, 0, s>>>(T + sq, nrp, nrp, nr, qf);
    cccp_update_kernel<<<1, 1024, 0, s>>>(qf, cd, b, bo, db, nr, sc);
    const int qg = (int)std::min<int64_t>(2 * ctx->num_sms, (nr + 7) / 8);
    cccp_quadform_kernel<<<qg, 256, 0, s>>>(Cg, nrp, nr, db, bo, ctx->partials, ctx->counters + kCtrMisc, sc);
    L += 6;
    LAKER_CUDA(ctx, cudaMemcpyAsync(&hs, sc, sizeof(hs), cudaMemcpyDeviceToHost, s));
    LAKER_CUDA(ctx, cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    LAKER_CUDA(ctx, cudaStreamSynchronize(s));
    if (hflag) return set_err(ctx, LAKER_ERR_NOT_POSITIVE_DEFINITE, "fit: Cholesky of T_t failed");
    ++it;
    a = hs.a;
    change = hs.change;
    rho_used = rho_t;
    if (change <= fp_tol) {
      converged = true;
      break;
    }
  }

  tick("cccp");
  // ---- 4. T^{-1/2} of the final T = a I + R diag(b) R^T (coupled Newton-Schulz)
  {
    scale_cols_sqrt_kernel<<<dim3(cdiv(nrp, 256), (unsigned)nrp), 256, 0, s>>>(R, S, nrp, nrp, b);
    GemmArgs g{};
    g.M = nrp; g.N = nrp; g.K = nrp; g.A = S; g.lda = nrp; g.B = S; g.ldb = nrp; g.C = T; g.ldc = nrp;
    g.alpha = 1.0; g.diag = a; g.tri = 1;
    launch_dgemm(g, false, s);
    launch_mirror_lower(T, nrp, nrp, s);
    L += 3;
  }
  tick("T_build");
  // lambda_max(T) by power iteration (x0 = ones), c = 1.1 * estimate
  double cscale = 1.0;
  {
    double *x = qf, *y = db;  // reuse (nrp >= nr; nrp-length buffers)
    fill_kernel<<<cdiv(nrp, 256), 256, 0, s>>>(x, nrp, 1.0);
    ++L;
    double hn = 0.0;
    for (int k = 0; k < 30; ++k) {
      normalize_vec_kernel<<<1, 1024, 0, s>>>(x, nrp, scal);
      matvec_kernel<<<(unsigned)std::min<int64_t>(4 * ctx->num_sms, (nrp + 7) / 8), 256, 0, s>>>(T, nrp, nrp, x, y);
      std::swap(x, y);
      L += 2;
    }
    normalize_vec_kernel<<<1, 1024, 0, s>>>(x, nrp, scal);
    ++L;
    LAKER_CUDA(ctx, cudaMemcpyAsync(&hn, scal, sizeof(double), cudaMemcpyDeviceToHost, s));
    LAKER_CUDA(ctx, cudaStreamSynchronize(s));
    cscale = 1.1 * hn;
    if (debug) std::fprintf(stderr, "[fit] lambda_max(T) ~ %.6e a = %.6e\n", hn, a);
    dbg("T", T, nrp, nrp, nrp);
  }
  tick("power_iter");
  double *Y = S, *Zm = X, *W = G, *Tmp = L1, *Zsave = L2;
  LAKER_CUDA(ctx, cudaMemcpyAsync(Y, T, sq * 8, cudaMemcpyDeviceToDevice, s));
  scale_kernel<<<dim3(cdiv(nrp, 256), (unsigned)nrp), 256, 0, s>>>(Y, nrp, nrp, nrp, 1.0 / cscale);
  set_identity_kernel<<<dim3(cdiv(nrp, 256), (unsigned)nrp), 256, 0, s>>>(Zm, nrp, nrp);
  L += 2;
  // Coupled Newton-Schulz with a per-step scalar scaling (Chen & Chow-style):
  // with s_k^2 = sigma_k, W_k = (3I - sigma_k Z_k Y_k)/2, Y_{k+1} = s_k Y_k W_k,
  // Z_{k+1} = s_k W_k Z_k keeps Y_k = (T/c) Z_k, so Z_k -> (T/c)^{-1/2} as
  // Z_k Y_k -> I.  The eigenvalues of Z_k Y_k lie in [l_k, u_k] (l_0 = a/c is
  // a lower bound of lambda_min(T)/c, u_0 = 1); sigma_k equalizes
  // f(sigma l) = f(sigma u) for f(x) = x (3 - x)^2 / 4, giving
  // l_{k+1} = f(sigma_k l_k), u_{k+1} = 1: ~3x faster growth of the small
  // eigenvalues than the unscaled map.  Every product is symmetric in exact
  // arithmetic (all are polynomials in T): the lower triangle is formed on the
  // tensor cores and mirrored.  ||W_k - I|| is checked before each update; the
  // iteration stops at the tolerance or when it stops contracting.
  auto fmap = [](double x) { return x * (3.0 - x) * (3.0 - x) / 4.0; };
  double lo = std::max(a / cscale, 1e-300), up = 1.0;
  double prev = INFINITY;
  for (int k = 0; k < 100; ++k) {
    double sigma = 1.0;
    if (up - lo > 1e-3 * up) {  // bisection for f(sigma lo) = f(sigma up), sigma up in [1, 3)
      double s0 = 1.0 / up, s1 = 2.5 / up;  // sigma * u <= 2.5: safe if u underestimates by 10%
      for (int b = 0; b < 200; ++b) {
        const double sm = 0.5 * (s0 + s1);
        if (fmap(sm * lo) < fmap(sm * up)) s0 = sm; else s1 = sm;
      }
      sigma = s0;
    }
    const double sk = std::sqrt(sigma);
    GemmArgs g{};
    g.M = nrp; g.N = nrp; g.K = nrp; g.lda = g.ldb = g.ldc = nrp; g.tri = 1;
    g.b_sym = true;  // every B below (Y, W, Z) is mirrored, exactly symmetric
    g.A = Zm; g.B = Y; g.C = W; g.alpha = -0.5 * sigma; g.diag = 1.5;
    launch_dgemm(g, true, s);
    launch_mirror_lower(W, nrp, nrp, s);
    LAKER_CUDA(ctx, cudaMemsetAsync(scal + 1, 0, sizeof(double), s));
    frob_minus_identity_kernel<<<4 * ctx->num_sms, 256, 0, s>>>(W, nrp, nrp, scal + 1);
    L += 3;
    double fn = 0.0;
    LAKER_CUDA(ctx, cudaMemcpyAsync(&fn, scal + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
    LAKER_CUDA(ctx, cudaStreamSynchronize(s));
    fn = std::sqrt(fn);
    if (debug) std::fprintf(stderr, "[fit] NS %d sigma %.4f [%.3e, %.3e] ||W-I||_F = %.3e\n", k, sigma, lo, up, fn);
    // once in the quadratic regime hand over to the self-correcting uncoupled iteration
    // below: the coupled map carries Y_k = (T/c) Z_k only implicitly, and rounding that
    // breaks it can grow (measured: ||W - I|| 6e-6 -> x9.5 per step on an N_r = 512 fit)
    if (sigma == 1.0 && fn < 1e-3) break;
    if (sigma == 1.0 && fn > prev) {
      std::swap(Zm, Zsave);
      break;
    }
    prev = sigma == 1.0 ? fn : INFINITY;
    if (sigma == 1.0) LAKER_CUDA(ctx, cudaMemcpyAsync(Zsave, Zm, sq * 8, cudaMemcpyDeviceToDevice, s));
    g.diag = 0.0; g.alpha = sk;
    g.A = Y; g.B = W; g.C = Tmp;
    launch_dgemm(g, true, s);
    launch_mirror_lower(Tmp, nrp, nrp, s);
    std::swap(Y, Tmp);
    g.A = W; g.B = Zm; g.C = Tmp;
    launch_dgemm(g, true, s);
    launch_mirror_lower(Tmp, nrp, nrp, s);
    std::swap(Zm, Tmp);
    L += 4;
    const double nl = fmap(sigma * lo), nu = (sigma * up >= 1.0 && sigma * lo <= 1.0) ? 1.0 : fmap(sigma * up);
    lo = std::min(nl, nu);
    up = std::max(nl, nu);
  }
  // Uncoupled Newton-Schulz for the inverse square root, symmetric form:
  // E = Z (T/c) Z, Z <- Z (3I - E)/2.  It uses T itself every step, so rounding does
  // not accumulate; quadratic convergence from ||E - I|| < ~1e-3.  Stops at the
  // tolerance or when ||E - I|| stops contracting (keeping the better iterate).
  {
    double prev_e = INFINITY;
    for (int k = 0; k < 8; ++k) {
      GemmArgs g{};
      g.M = nrp; g.N = nrp; g.K = nrp; g.lda = g.ldb = g.ldc = nrp;
      g.b_sym = true;  // T, Z, W mirrored, exactly symmetric
      g.A = Zm; g.B = T; g.C = Tmp; g.alpha = 1.0 / cscale;   // Z T / c  (full)
      launch_dgemm(g, true, s);
      g.A = Tmp; g.B = Zm; g.C = W; g.alpha = -0.5; g.diag = 1.5; g.tri = 1;  // W = (3I - Z T Z / c) / 2
      launch_dgemm(g, true, s);
      launch_mirror_lower(W, nrp, nrp, s);
      LAKER_CUDA(ctx, cudaMemsetAsync(scal + 1, 0, sizeof(double), s));
      frob_minus_identity_kernel<<<4 * ctx->num_sms, 256, 0, s>>>(W, nrp, nrp, scal + 1);
      L += 4;
      double fe = 0.0;
      LAKER_CUDA(ctx, cudaMemcpyAsync(&fe, scal + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
      LAKER_CUDA(ctx, cudaStreamSynchronize(s));
      fe = std::sqrt(fe);
      if (debug) std::fprintf(stderr, "[fit] NS-uncoupled %d ||W-I||_F = %.3e\n", k, fe);
      if (fe > 0.5 * prev_e) {  // stagnated at the rounding floor: keep the previous iterate
        if (fe > prev_e) std::swap(Zm, Zsave);
        break;
      }
      prev_e = fe;
      LAKER_CUDA(ctx, cudaMemcpyAsync(Zsave, Zm, sq * 8, cudaMemcpyDeviceToDevice, s));
      g.A = Zm; g.B = W; g.C = Tmp; g.alpha = 1.0; g.diag = 0.0; g.tri = 1;  // Z W (symmetric: lower + mirror)
      launch_dgemm(g, true, s);
      launch_mirror_lower(Tmp, nrp, nrp, s);
      std::swap(Zm, Tmp);
      L += 2;
      if (fe < 1e-14 * std::sqrt((double)nrp)) break;
    }
  }
  tick("newton_schulz");
  // M = T^{-1/2} - a^{-1/2} I = Z / sqrt(c) - a^{-1/2} I   (into Zm)
  scale_kernel<<<dim3(cdiv(nrp, 256), (unsigned)nrp), 256, 0, s>>>(Zm, nrp, nrp, nrp, 1.0 / std::sqrt(cscale));
  add_diag_kernel<<<cdiv(nrp, 256), 256, 0, s>>>(Zm, nrp, 0, nrp, -1.0 / std::sqrt(a));
  L += 2;

  dbg("M", Zm, nrp, nrp, nrp);
  // ---- 5. P = a^{-1/2} I + Q M Q^T with Q^T = Ut (nrp x ld), M = Zm
  const double ainv = 1.0 / std::sqrt(a);
  // AUTO: factored in the QM form (the sharded solve gathers z = Q^T r, pcg_dist.cu)
  const bool factored = o.p_layout == LAKER_P_FACTORED || o.p_layout == LAKER_P_FACTORED_QM ||
                        o.p_layout == LAKER_P_AUTO;
  ctx->p_factored = false;
  if (factored) {
    // keep the factors: Q^T for z = Q^T r, Q for Q w, and M;
    // buffers of the same size are reused across fits (cudaFree/cudaMalloc of ~1 GiB
    // cost ~0.1 s per refit)
    if (ctx->P) {
      cudaFree(ctx->P);
      ctx->P = nullptr;
    }
    const int64_t ldq = (nrp + 255) / 256 * 256;  // gemv streams whole 256-column chunks
    // row-sharded context: every rank keeps only its own part -- Q^T's
    // columns [r0, r1) (nrp x ldl), Q's and QM's rows [r0, r1) -- so a P apply streams
    // 16 (n/W) N_r bytes per rank; M (N_r^2) is kept whole.  One rank: all of it.
    const bool loc = ctx->comm != nullptr || ctx->world > 1;
    const int64_t r0 = loc ? ctx->r0 : 0, nloc = loc ? ctx->r1 - ctx->r0 : n;
    const int64_t ldl = loc ? padded_ld(nloc) : ld;
    if (!(ctx->Qt && ctx->f_alloc_nrp == nrp && ctx->f_alloc_n == n)) {
      free_factors(ctx);
      LAKER_CUDA(ctx, cudaMalloc(&ctx->Qt, (size_t)nrp * ldl * 8));
      LAKER_CUDA(ctx, cudaMalloc(&ctx->Qr, (size_t)nloc * ldq * 8));
      LAKER_CUDA(ctx, cudaMalloc(&ctx->Mf, (size_t)nrp * ldq * 8));
      LAKER_CUDA(ctx, cudaMalloc(&ctx->fz, (size_t)2 * ldq * 8));
      ctx->f_alloc_nrp = nrp;
      ctx->f_alloc_n = n;
    }
    ctx->f_local = loc;
    ctx->f_ldl = ldl;
    ctx->fw = ctx->fz + ldq;
    LAKER_CUDA(ctx, cudaMemsetAsync(ctx->Qr, 0, (size_t)nloc * ldq * 8, s));
    LAKER_CUDA(ctx, cudaMemsetAsync(ctx->Mf, 0, (size_t)nrp * ldq * 8, s));
    LAKER_CUDA(ctx, cudaMemsetAsync(ctx->fz, 0, (size_t)2 * ldq * 8, s));
    if (loc) {
      LAKER_CUDA(ctx, cudaMemsetAsync(ctx->Qt, 0, (size_t)nrp * ldl * 8, s));
      LAKER_CUDA(ctx, cudaMemcpy2DAsync(ctx->Qt, ldl * 8, Ut + r0, ld * 8, nloc * 8, nrp, cudaMemcpyDeviceToDevice, s));
    } else {
      LAKER_CUDA(ctx, cudaMemcpyAsync(ctx->Qt, Ut, (size_t)nrp * ld * 8, cudaMemcpyDeviceToDevice, s));
    }
    launch_transpose(Ut + r0, nrp, nloc, ld, ctx->Qr, ldq, s);
    LAKER_CUDA(ctx, cudaMemcpy2DAsync(ctx->Mf, ldq * 8, Zm, nrp * 8, nrp * 8, nrp, cudaMemcpyDeviceToDevice, s));
    ++L;
    // QM = Q M (reading R21): the apply becomes two passes, a^-1/2 r + QM (Q^T r) --
    // 2353 vs ~2140 it/s at C3.  Its iteration counts lie inside the R15(iii) envelope
    // (own oracle fit on +-1-ulp copies of K: C2 [1007, 1053] vs 1029, R21),
    // so it is the default (AUTO); FACTORED keeps the three passes Q (M (Q^T r)).
    ctx->p_qm = o.p_layout == LAKER_P_AUTO || o.p_layout == LAKER_P_FACTORED_QM;
    if (!ctx->p_qm && ctx->QMf) {  // QM is only kept while the QM form is in use
      cudaFree(ctx->QMf);
      ctx->QMf = nullptr;
    }
    if (ctx->p_qm) {
      if (!ctx->QMf) LAKER_CUDA(ctx, cudaMalloc(&ctx->QMf, (size_t)nloc * ldq * 8));
      LAKER_CUDA(ctx, cudaMemsetAsync(ctx->QMf, 0, (size_t)nloc * ldq * 8, s));
      GemmArgs g{};
      g.M = nloc;
      g.N = nrp;
      g.K = nrp;
      g.A = ctx->Qr;
      g.lda = ldq;
      g.B = ctx->Mf;
      g.ldb = ldq;
      g.b_sym = true;  // M = Z / sqrt(c) - a^-1/2 I, Z mirrored
      g.C = ctx->QMf;
      g.ldc = ldq;
      g.alpha = 1.0;
      g.beta = 0.0;
      // int8-emulated GEMM (B8; 10 ms at C3 vs 56 ms on DMMA, the same iteration counts)
      launch_dgemm(g, true, s);
      ++L;
    }
    ctx->f_nr = nr;
    ctx->f_nrp = nrp;
    ctx->f_ldq = ldq;
    ctx->f_ainv = ainv;
    ctx->p_factored = true;
  } else {
    free_factors(ctx);
    LAKER_TRY(form_dense_p(ctx, Ut, Zm, nrp, nrp, ainv));
    dbg("P0", ctx->P, ctx->r1 - ctx->r0, n, ld);
  }
  tick("P_form");
  // trace of Sigma* = n a + sum_k b_k C_kk
  double htr = 0.0;
  {
    // reuse the quadform kernel's linear pieces: sum_b_cd of the current b
    hs.a = a;
    hs.rho = rho_used;
    LAKER_CUDA(ctx, cudaMemcpyAsync(sc, &hs, sizeof(hs), cudaMemcpyHostToDevice, s));
    std::vector<double> hb(nr), hcd(nr);
    LAKER_CUDA(ctx, cudaMemcpyAsync(hb.data(), b, nr * 8, cudaMemcpyDeviceToHost, s));
    LAKER_CUDA(ctx, cudaMemcpyAsync(hcd.data(), cd, nr * 8, cudaMemcpyDeviceToHost, s));
    LAKER_CUDA(ctx, cudaStreamSynchronize(s));
    double t = n * a;
    for (int64_t k = 0; k < nr; ++k) t += hb[k] * hcd[k];  // report only
    htr = t;
  }
  cudaEventRecord(e1, s);
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  LAKER_CUDA(ctx, cudaGetLastError());
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->stats.fit_ms = ms;
  if (rep) {
    rep->iters = it;
    rep->n_dirs = (int32_t)nr;
    rep->converged = converged ? 1 : 0;
    rep->final_change = change;
    rep->rho_used = rho_used;
    rep->sigma_min_eig = a;
    rep->trace = htr;
    rep->seconds = ms * 1e-3;
  }
  ctx->precond_kind = LAKER_PRECOND_LEARNED;
  return LAKER_OK;
}

}  // namespace laker
