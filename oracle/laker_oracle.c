/*
 * laker_oracle.c -- plain, slow, fp64 CPU oracle for the LAKER hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2604_25138_b200/csrc); the CUDA path never loads it.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, line numbers "P:n"):
 *   orc_assemble     K_ij = exp(scale * <e_i, e_j>)       P:141-147 (Eq. sc-exp-kernel), Alg.1 l.3
 *   orc_cross_kernel k(x, x_i) = exp(scale * <e(x), e_i>) P:164-172 (Eq. sc-radio-map-reconstruction)
 *   orc_predict      r(x) = sum_i k(x, x_i) alpha_i       P:164-172, Alg.1 l.24
 *   orc_apply        q = (lambda I + K) p                 P:517-519 (matvec remark)
 *   orc_jacobi_diag  d_i = 1 / (lambda + K_ii)            P:727, P:757-758 (Jacobi PCG baseline)
 *   orc_pcg          Alg. 1 "Preconditioned Conjugate Gradient", P:306-321 (and P:589-626), verbatim
 *   orc_factored_apply / orc_pcg_factored
 *                    theta = P r with P = Sigma*^{-1/2} held as a^{-1/2} I + Q M Q^T
 *                    (Eq. preconditioner-Sigmma P:273-278 in the structured form
 *                    of DESIGN.md O4': Sigma* = a I + Q (T - a I) Q^T, Q^T Q = I,
 *                    so Sigma*^{-1/2} = a^{-1/2} I + Q (T^{-1/2} - a^{-1/2} I) Q^T)
 *
 * Rounding policy (readings R17/R18): every inner product is Dot2
 * (Ogita, Rump & Oishi, "Accurate sum and dot product", SIAM J. Sci. Comput.
 * 2005, Alg. 5.3) evaluated sequentially in index order; every kernel entry is
 * RN(exp(RN(scale * RN(dot)))) with a correctly rounded exp obtained from
 * libquadmath's binary128 expq rounded once to binary64; vector updates are
 * single fma; division and sqrt are IEEE.  Compile with -ffp-contract=off and
 * never with -ffast-math (oracle/Makefile).
 *
 * The CCCP fit and the direct (Cholesky) reference solve are in oracle/fit.py
 * (numpy/LAPACK primitives as steps, no blocking or fusion).
 */
#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------ Dot2 */
/* TwoSum (Knuth): s + e == a + b exactly. */
static inline void two_sum(double a, double b, double *s, double *e) {
  double x = a + b;
  double z = x - a;
  *e = (a - (x - z)) + (b - z);
  *s = x;
}
/* TwoProduct with fma: p + e == a * b exactly. */
static inline void two_prod(double a, double b, double *p, double *e) {
  double x = a * b;
  *e = fma(a, b, -x);
  *p = x;
}

typedef struct { double s, c; } dot2_t;

static inline void dot2_add(dot2_t *A, double a, double b) {
  double p, pe, s, se;
  two_prod(a, b, &p, &pe);
  two_sum(A->s, p, &s, &se);
  A->s = s;
  A->c = A->c + (pe + se);
}
static inline double dot2_result(dot2_t A) { return A.s + A.c; }

static double dot2(int64_t n, const double *x, int64_t incx, const double *y, int64_t incy) {
  dot2_t A = {0.0, 0.0};
  for (int64_t k = 0; k < n; ++k) dot2_add(&A, x[k * incx], y[k * incy]);
  return dot2_result(A);
}

ORC_API double orc_dot2(int64_t n, const double *x, const double *y) { return dot2(n, x, 1, y, 1); }

/* ------------------------------------------------------- correctly rounded exp */
#define ORC_EXP_OVERFLOW_ARG 709.782712893383973096 /* ln(DBL_MAX) */

ORC_API double orc_exp_cr(double x) {
  /* binary128 exp has < 1 ulp(binary128) error; one rounding to binary64 is
     then correct unless exp(x) lies within 2^-112 relative of a binary64
     midpoint (probability ~2^-59 per argument). */
  __float128 q = expq((__float128)x);
  return (double)q;
}

/* one kernel entry: RN(exp(RN(scale * Dot2(e_i, e_j)))) -- P:144 with scale (R1) */
static inline double kernel_entry(int32_t d, const double *ei, const double *ej, double scale,
                                  int64_t *n_overflow) {
  double dot = dot2(d, ei, 1, ej, 1);
  double arg = scale * dot;
  if (arg > ORC_EXP_OVERFLOW_ARG) {
    __atomic_fetch_add(n_overflow, 1, __ATOMIC_RELAXED);
  }
  return orc_exp_cr(arg);
}

/* K (n x n row-major) = exp(scale * E E^T), upper triangle computed, mirrored. */
ORC_API int64_t orc_assemble(int64_t n, int32_t d, const double *E, double scale, double *K) {
  int64_t n_overflow = 0;
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = i; j < n; ++j) {
      double v = kernel_entry(d, E + i * d, E + j * d, scale, &n_overflow);
      K[i * n + j] = v;
      K[j * n + i] = v;
    }
  }
  return n_overflow;
}

/* Rows [r0, r1) of K, row-major (r1 - r0) x n.  Same entries as orc_assemble. */
ORC_API int64_t orc_assemble_rows(int64_t n, int32_t d, const double *E, double scale,
                                  int64_t r0, int64_t r1, double *Krows) {
  int64_t n_overflow = 0;
#pragma omp parallel for schedule(static)
  for (int64_t i = r0; i < r1; ++i)
    for (int64_t j = 0; j < n; ++j)
      Krows[(i - r0) * n + j] = kernel_entry(d, E + i * d, E + j * d, scale, &n_overflow);
  return n_overflow;
}

/* Kx (m x n row-major): Kx_mi = exp(scale * <eq_m, e_i>) -- P:164-172 */
ORC_API int64_t orc_cross_kernel(int64_t m, int64_t n, int32_t d, const double *Eq, const double *E,
                                 double scale, double *Kx) {
  int64_t n_overflow = 0;
#pragma omp parallel for schedule(static)
  for (int64_t a = 0; a < m; ++a)
    for (int64_t i = 0; i < n; ++i)
      Kx[a * n + i] = kernel_entry(d, Eq + a * d, E + i * d, scale, &n_overflow);
  return n_overflow;
}

/* r_hat_m = RN(sum_i k(x_m, x_i) alpha_i), Dot2 over i in order -- P:164-172 */
ORC_API int64_t orc_predict(int64_t m, int64_t n, int32_t d, const double *Eq, const double *E,
                            double scale, const double *alpha, double *out) {
  int64_t n_overflow = 0;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t a = 0; a < m; ++a) {
    dot2_t A = {0.0, 0.0};
    for (int64_t i = 0; i < n; ++i)
      dot2_add(&A, kernel_entry(d, Eq + a * d, E + i * d, scale, &n_overflow), alpha[i]);
    out[a] = dot2_result(A);
  }
  return n_overflow;
}

/* ------------------------------------------------------------------ operator */
/* q_i = RN(lambda p_i + sum_j K_ij p_j): one Dot2 over the n+1 terms, the
   lambda term first (reading R17).  Rows [r0, r1) of K given as Krows. */
static void apply_rows(int64_t n, int64_t r0, int64_t r1, const double *Krows, double lambda,
                       const double *p, double *q) {
#pragma omp parallel for schedule(static)
  for (int64_t i = r0; i < r1; ++i) {
    dot2_t A = {0.0, 0.0};
    dot2_add(&A, lambda, p[i]);
    const double *row = Krows + (i - r0) * n;
    for (int64_t j = 0; j < n; ++j) dot2_add(&A, row[j], p[j]);
    q[i - r0] = dot2_result(A);
  }
}

ORC_API void orc_apply(int64_t n, const double *K, double lambda, const double *p, double *q) {
  apply_rows(n, 0, n, K, lambda, p, q);
}

/* Dense P apply theta_i = RN(sum_j P_ij r_j), Dot2 in j order. */
static void dense_apply(int64_t n, const double *P, const double *r, double *theta) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) theta[i] = dot2(n, P + i * n, 1, r, 1);
}

ORC_API void orc_dense_apply(int64_t n, const double *P, const double *r, double *theta) {
  dense_apply(n, P, r, theta);
}

/* Jacobi: d_i = RN(1 / RN(lambda + K_ii)), K_ii the kernel entry of (i, i). */
ORC_API int64_t orc_jacobi_diag(int64_t n, int32_t d, const double *E, double scale, double lambda,
                                double *dvec) {
  int64_t n_overflow = 0;
  for (int64_t i = 0; i < n; ++i) {
    double kii = kernel_entry(d, E + i * d, E + i * d, scale, &n_overflow);
    dvec[i] = 1.0 / (lambda + kii);
  }
  return n_overflow;
}

/* ------------------------------------------------------- factored P apply */
/* P = ainv I + Q M Q^T: Q n x m row-major, M m x m row-major (O4').
   z_k = RN(sum_i Q_ik r_i), w_k = RN(sum_j M_kj z_j),
   theta_i = RN(ainv r_i + sum_k Q_ik w_k), each a Dot2 in index order. */
typedef struct { int64_t m; const double *Q, *M; double ainv; const double *QM; const double *Qt; } orc_factored;

/* Q^T (m x n row-major): a copy of Q with the storage order swapped, so that z_k reads
   column k of Q contiguously.  The Dot2 of z_k runs over the same numbers in the same
   index order i = 0..n-1 either way; only the memory access pattern differs (the PCG
   drivers below transpose once per solve). */
static double *transpose_copy(int64_t n, int64_t m, const double *Q) {
  double *Qt = malloc(sizeof(double) * (size_t)(n * m > 0 ? n * m : 1));
  if (!Qt) return NULL;
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < m; ++k)
    for (int64_t i = 0; i < n; ++i) Qt[k * n + i] = Q[i * m + k];
  return Qt;
}

static void factored_apply(int64_t n, const orc_factored *F, const double *r, double *theta) {
  const int64_t m = F->m;
  double *z = malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  double *w = malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < m; ++k)
    z[k] = F->Qt ? dot2(n, F->Qt + k * n, 1, r, 1) : dot2(n, F->Q + k, m, r, 1);
  if (F->QM) {
    /* QM form: P r = ainv r + (Q M)(Q^T r) -- the same product associated as
       Q (M z) -> (Q M) z with the n x m product QM given (R21):
       theta_i = Dot2([ainv, QM_i.], [r_i, z]). */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      dot2_t A = {0.0, 0.0};
      dot2_add(&A, F->ainv, r[i]);
      const double *q = F->QM + i * m;
      for (int64_t k = 0; k < m; ++k) dot2_add(&A, q[k], z[k]);
      theta[i] = dot2_result(A);
    }
    free(z);
    free(w);
    return;
  }
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < m; ++k) w[k] = dot2(m, F->M + k * m, 1, z, 1);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    dot2_t A = {0.0, 0.0};
    dot2_add(&A, F->ainv, r[i]);
    const double *q = F->Q + i * m;
    for (int64_t k = 0; k < m; ++k) dot2_add(&A, q[k], w[k]);
    theta[i] = dot2_result(A);
  }
  free(z);
  free(w);
}

ORC_API void orc_factored_apply(int64_t n, int64_t m, const double *Q, const double *M, double ainv,
                                const double *r, double *theta) {
  orc_factored F = {m, Q, M, ainv, NULL, NULL};
  factored_apply(n, &F, r, theta);
}

/* theta = ainv r + QM (Q^T r) (QM = Q M, n x m row-major; R21). */
ORC_API void orc_factored_qm_apply(int64_t n, int64_t m, const double *Q, const double *QM, double ainv,
                                   const double *r, double *theta) {
  orc_factored F = {m, Q, NULL, ainv, QM, NULL};
  factored_apply(n, &F, r, theta);
}

/* ----------------------------------------------------------------------- PCG */
enum { ORC_P_NONE = 0, ORC_P_JACOBI = 1, ORC_P_DENSE = 2, ORC_P_FACTORED = 3 };
enum { ORC_TERM_RESIDUAL_TOL = 0, ORC_TERM_MAX_ITERS = 1, ORC_TERM_ZERO_RHS = 2,
       ORC_TERM_BREAKDOWN = 3, ORC_TERM_INDEFINITE = 4 };

typedef struct {
  int32_t iters;          /* number of operator applies (R12) */
  int32_t termination;    /* ORC_TERM_* */
  double rel_residual;    /* recursive ||r|| / ||y|| at exit */
  double true_rel_residual; /* ||y - (lambda I + K) alpha|| / ||y|| recomputed at exit */
} orc_pcg_report;

static void precond_apply(int pkind, int64_t n, const double *P, const orc_factored *F, const double *r,
                          double *theta) {
  if (pkind == ORC_P_NONE) {
    memcpy(theta, r, (size_t)n * sizeof(double));
  } else if (pkind == ORC_P_JACOBI) {
    for (int64_t i = 0; i < n; ++i) theta[i] = P[i] * r[i];
  } else if (pkind == ORC_P_FACTORED) {
    factored_apply(n, F, r, theta);
  } else {
    dense_apply(n, P, r, theta);
  }
}

/*
 * Alg. 1, P:306-321:
 *   alpha^0 = 0, r^0 = y, theta^0 = P r^0, p^0 = theta^0
 *   loop: delta = r.theta / p.(lambda I + K)p ; alpha += delta p ; r -= delta (lambda I+K) p
 *         if ||r|| / ||y|| <= tol: break
 *         theta = P r ; beta = r_new.theta_new / r_old.theta_old ; p = theta + beta p
 * P: NULL for NONE, diag (n) for JACOBI, dense n x n row-major for DENSE.
 * history (optional, >= max_iters): ||r^{k+1}|| / ||y|| per iteration.
 */
static int pcg_impl(int64_t n, const double *K, double lambda, const double *y, int pkind,
                    const double *P, const orc_factored *F, double tol, int32_t max_iters, double *alpha,
                    orc_pcg_report *rep, double *history) {
  double *r = malloc(sizeof(double) * n), *th = malloc(sizeof(double) * n);
  double *p = malloc(sizeof(double) * n), *q = malloc(sizeof(double) * n);
  int status = 0;
  memset(rep, 0, sizeof(*rep));
  for (int64_t i = 0; i < n; ++i) { alpha[i] = 0.0; r[i] = y[i]; }
  double ynorm = sqrt(dot2(n, y, 1, y, 1));
  if (ynorm == 0.0) {
    rep->termination = ORC_TERM_ZERO_RHS;
    goto done;
  }
  precond_apply(pkind, n, P, F, r, th);
  memcpy(p, th, sizeof(double) * n);
  double rho = dot2(n, r, 1, th, 1);
  if (!(rho > 0.0)) { rep->termination = ORC_TERM_INDEFINITE; status = 1; goto done; }
  rep->termination = ORC_TERM_MAX_ITERS;
  for (int32_t k = 0; k < max_iters; ++k) {
    apply_rows(n, 0, n, K, lambda, p, q);
    double pq = dot2(n, p, 1, q, 1);
    if (!(pq > 0.0)) { rep->termination = ORC_TERM_BREAKDOWN; status = 1; break; }
    double delta = rho / pq;
    for (int64_t i = 0; i < n; ++i) {
      alpha[i] = fma(delta, p[i], alpha[i]);
      r[i] = fma(-delta, q[i], r[i]);
    }
    double rel = sqrt(dot2(n, r, 1, r, 1)) / ynorm;
    rep->iters = k + 1;
    rep->rel_residual = rel;
    if (history) history[k] = rel;
    if (rel <= tol) { rep->termination = ORC_TERM_RESIDUAL_TOL; break; }
    precond_apply(pkind, n, P, F, r, th);
    double rho_new = dot2(n, r, 1, th, 1);
    if (!(rho_new > 0.0)) { rep->termination = ORC_TERM_INDEFINITE; status = 1; break; }
    double beta = rho_new / rho;
    for (int64_t i = 0; i < n; ++i) p[i] = fma(beta, p[i], th[i]);
    rho = rho_new;
  }
  /* true residual, recomputed once (Eq. residual) */
  apply_rows(n, 0, n, K, lambda, alpha, q);
  {
    dot2_t A = {0.0, 0.0};
    for (int64_t i = 0; i < n; ++i) {
      double t = y[i] - q[i];
      dot2_add(&A, t, t);
    }
    rep->true_rel_residual = sqrt(dot2_result(A)) / ynorm;
  }
done:
  free(r); free(th); free(p); free(q);
  return status;
}

ORC_API int orc_pcg(int64_t n, const double *K, double lambda, const double *y, int pkind,
                    const double *P, double tol, int32_t max_iters, double *alpha,
                    orc_pcg_report *rep, double *history) {
  if (pkind == ORC_P_FACTORED) return -1; /* use orc_pcg_factored */
  return pcg_impl(n, K, lambda, y, pkind, P, NULL, tol, max_iters, alpha, rep, history);
}

/* PCG with the factored P = ainv I + Q M Q^T (Q n x m, M m x m, row-major). */
ORC_API int orc_pcg_factored(int64_t n, const double *K, double lambda, const double *y, int64_t m,
                             const double *Q, const double *M, double ainv, double tol, int32_t max_iters,
                             double *alpha, orc_pcg_report *rep, double *history) {
  orc_factored F = {m, Q, M, ainv, NULL, transpose_copy(n, m, Q)};
  int st = pcg_impl(n, K, lambda, y, ORC_P_FACTORED, NULL, &F, tol, max_iters, alpha, rep, history);
  free((void *)F.Qt);
  return st;
}

/* PCG with the factored P applied in QM form (orc_factored_qm_apply). */
ORC_API int orc_pcg_factored_qm(int64_t n, const double *K, double lambda, const double *y, int64_t m,
                                const double *Q, const double *QM, double ainv, double tol, int32_t max_iters,
                                double *alpha, orc_pcg_report *rep, double *history) {
  orc_factored F = {m, Q, NULL, ainv, QM, transpose_copy(n, m, Q)};
  int st = pcg_impl(n, K, lambda, y, ORC_P_FACTORED, NULL, &F, tol, max_iters, alpha, rep, history);
  free((void *)F.Qt);
  return st;
}

/* Thread count actually used by the parallel loops (for cpu_baseline.cores). */
#ifdef _OPENMP
#include <omp.h>
ORC_API int orc_num_threads(void) { return omp_get_max_threads(); }
#else
ORC_API int orc_num_threads(void) { return 1; }
#endif
