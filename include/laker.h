/*
 * laker.h -- C ABI of liblaker.so, the B200 (sm_100a) hot path of LAKER
 * (arXiv 2604.25138, "Accelerating Regularized Attention Kernel Regression
 * for Spectrum Cartography").  Citations "P:n" are lines of the paper's LaTeX
 * (PAPER.md); readings "Rn" are listed in DESIGN.md §3.
 *
 * The four calls follow Alg. 1:
 *   laker_assemble_kernel    Kernel Construction        (Alg.1 l.1-3,  P:289-291)
 *   laker_fit_preconditioner Regression Learning (CCCP)  (Alg.1 l.4-14)
 *   laker_pcg_solve          Preconditioned CG           (Alg.1 l.15-22)
 *   laker_predict            Radio Map Reconstruction    (Alg.1 l.23-25)
 * plus the block-CG variant of the multi-RHS solve (C4), laker_block_cg_solve
 * (O'Leary 1980, B14).
 *
 * Conventions (all calls):
 *  - Every call returns laker_status; no exception or abort crosses the ABI.
 *    On failure laker_last_error(ctx) holds a one-line reason.
 *  - Pointer arguments may be HOST or DEVICE memory (detected with
 *    cudaPointerGetAttributes); host buffers are staged through the context's
 *    stream.  The caller owns every pointer; none is retained after a call.
 *  - fp64 everywhere.  Matrices are row-major unless stated; multi-RHS blocks
 *    (Y, alpha) are column-major n x nrhs.
 *  - Calls are ordered on the context's CUDA stream (the caller's stream given
 *    to laker_create, or a context-owned one).  Calls that fill host reports
 *    synchronize that stream before returning.
 *  - A context is not thread-safe: one context per (process, device).
 *  - Multi-GPU (world > 1): every rank calls every function in the same
 *    order with identical scalar arguments (they are collective); rank r owns
 *    rows [r*n/W, (r+1)*n/W) of K and P (row-block sharding); vectors are
 *    replicated on return.
 *  - No CPU fallback exists: without a usable CUDA device laker_create fails.
 */
#ifndef LAKER_H_
#define LAKER_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct laker_ctx_s *laker_ctx;

typedef enum {
  LAKER_OK = 0,
  LAKER_ERR_INVALID_ARGUMENT = 1,
  LAKER_ERR_DIMENSION_MISMATCH = 2,
  LAKER_ERR_NOT_READY = 3,                 /* e.g. solve before assemble */
  LAKER_ERR_CUDA = 4,
  LAKER_ERR_NCCL = 5,
  LAKER_ERR_OUT_OF_MEMORY = 6,
  LAKER_ERR_NOT_POSITIVE_DEFINITE = 7,     /* fit: Cholesky pivot <= 0 */
  LAKER_ERR_INDEFINITE_PRECONDITIONER = 8, /* PCG: r.theta <= 0 */
  LAKER_ERR_BREAKDOWN_ZERO_CURVATURE = 9,  /* PCG: p.(lambda I + K)p <= 0 */
  LAKER_ERR_OVERFLOW = 10,                 /* scale*<e_i,e_j> > ln(DBL_MAX) (exp overflow) */
  LAKER_ERR_INTERNAL = 11
} laker_status;

enum { LAKER_STORE_MATERIALIZED = 0, LAKER_STORE_ON_THE_FLY = 1 };
/* EXACT: correctly rounded kernel entries (Dot2 inner product + correctly
   rounded exp, R18) -- bitwise equal to the oracle.  FAST: fp64 DMMA tensor-
   core inner products + CUDA exp (<= 1 ulp per entry). */
enum { LAKER_MODE_FAST = 0, LAKER_MODE_EXACT = 1 };
enum { LAKER_PRECOND_NONE = 0, LAKER_PRECOND_JACOBI = 1, LAKER_PRECOND_LEARNED = 2,
       LAKER_PRECOND_EXTERNAL_DENSE = 3 };
enum { LAKER_TERM_RESIDUAL_TOL = 0, LAKER_TERM_MAX_ITERS = 1, LAKER_TERM_ZERO_RHS = 2,
       LAKER_TERM_BREAKDOWN = 3, LAKER_TERM_INDEFINITE = 4 };

/* ---------------------------------------------------------------- lifecycle */
/* Rank 0 only: an NCCL unique id (ncclGetUniqueId) to broadcast to the other
   ranks (e.g. with torch.distributed).  Not needed when world == 1. */
laker_status laker_get_unique_id(unsigned char id[128]);

/* Create a context on CUDA device `device`.  world >= 1, 0 <= rank < world.
   nccl_id: the 128-byte id from rank 0 (ncclCommInitRank over `world` ranks).
   With world == 1 it may be NULL (single-GPU path) or an id from
   laker_get_unique_id, which creates a 1-rank communicator and runs the
   row-sharded collective code path (used to test it on one GPU).  With
   world > 1 and NULL the context is a detached shard: row-sharded assembly,
   predict and the row hooks work, calls that need collectives (LEARNED fit,
   solve, apply) return NOT_READY (used to test the sharded layouts).
   cuda_stream: a cudaStream_t to order all work on, or NULL for a
   context-owned non-blocking stream.  *out is NULL on failure. */
laker_status laker_create(laker_ctx *out, int device, int rank, int world,
                          const unsigned char *nccl_id, void *cuda_stream);
laker_status laker_destroy(laker_ctx ctx);
const char *laker_status_string(laker_status s);
const char *laker_last_error(laker_ctx ctx);

/* ------------------------------------------------------------ (1) assembly */
/* K = exp(scale * E E^T) elementwise (Eq. sc-exp-kernel; Alg.1 l.3,
   P:291).  E: n x d row-major, identical on every rank; it is COPIED into the
   context (kept for Jacobi, on-the-fly applies and predict).  scale: 1/sqrt(d)
   for the BASELINE configs, 1 for the paper's own kernel (R1).  lambda > 0 is
   stored for the operator lambda I + K; it is never added to K.
   storage MATERIALIZED: rank r stores rows [r n/W, (r+1) n/W) of K in HBM
   (upper-triangle tiles computed once and mirrored, so K is bitwise symmetric).
   When every entry of K lies on the grid 2^(eK-55) of its largest binade (all
   BASELINE configs), the upper-triangle tiles (one rank) or the rank's tiles of the
   sharded plan (n/W a multiple of 256) are also stored as 8 int8 digit slices per
   entry (n^2/(2W) x 8 bytes more) and every K apply runs exactly on the tcgen05
   int8 tensor cores (B13, §8: shards exchange exact int64 row sums by a
   reduce-scatter; stats.k_tensor_core), bitwise the fp64 Dot2 result; otherwise the
   fp64 symmetric kernel is used (LAKER_SYMV_TC=0 forces it, for A/B tests).
   storage ON_THE_FLY: only E is kept; every operator apply recomputes the
   entries tile by tile (P:517-519 matvec-only access).
   Errors: INVALID_ARGUMENT (n < 1, d < 1, lambda <= 0, n % world != 0, bad
   enum), OVERFLOW (some entry overflowed; K is still written), OUT_OF_MEMORY. */
laker_status laker_assemble_kernel(laker_ctx ctx, int64_t n, int32_t d, const double *E,
                                   double scale, double lambda, int storage, int mode);

/* --------------------------------------------------------- (2) preconditioner */
typedef struct {
  int32_t kind;      /* NONE | JACOBI | LEARNED */
  int32_t n_dirs;    /* N_r; 0 -> min(n, max(ceil(8 sqrt n), ceil(n/4))) */
  double gamma;      /* CCCP regularization gamma (0.1) */
  double eps;        /* safeguard epsilon of F_gamma (1e-12, R8) */
  double rho;        /* shrinkage rho; < 0 -> schedule of R6 */
  double rho_floor;  /* eps_rho (1e-3) */
  int32_t max_iters; /* CCCP steps cap (200, R8) */
  double fp_tol;     /* stop when ||Sigma_{t+1}-Sigma_t||_F/||Sigma_t||_F <= fp_tol (1e-8, R8) */
  const double *Z;   /* n x N_r column-major N(0,1) draws z_k (Eq. random_directions,
                        P:239), host or device; NULL -> device Philox stream `seed` */
  uint64_t seed;
  int32_t p_layout;  /* how P = Sigma*^{-1/2} is stored and applied (LAKER_P_*):
                        AUTO (0): FACTORED_QM (one rank or sharded; the sharded
                        apply gathers z = Q^T r, N_r doubles) */
} laker_fit_opts;

/* P = a^{-1/2} I + Q M Q^T with Q (n x N_r, orthonormal columns, the thin QR of
   Ubar) and M = T^{-1/2} - a^{-1/2} I (N_r x N_r) is exact (O4').
   DENSE: the n x n rows are formed (bitwise symmetric, B4) and each apply
   streams them (8 n^2 bytes, or 4 n^2 through the symmetric GEMV).
   FACTORED: Q^T, Q and M are kept and each apply is theta = a^{-1/2} r +
   Q (M (Q^T r)) -- three Dot2 GEMV passes, 16 n N_r + 8 N_r^2 bytes (SURVEY
   §8(f) NEXT-1); no n x n matrix is formed.
   FACTORED_QM (the AUTO choice): the same operator associated as
   theta = a^{-1/2} r + (Q M)(Q^T r) with the n x N_r product QM formed once
   at fit time (R21) -- two Dot2 GEMV passes, 16 n N_r bytes.  The
   multi-RHS solve applies the same form, so T18 holds in either. */
enum { LAKER_P_AUTO = 0, LAKER_P_DENSE = 1, LAKER_P_FACTORED = 2, LAKER_P_FACTORED_QM = 3 };

typedef struct {
  int32_t iters, n_dirs, converged;
  double final_change;  /* last relative Frobenius change of Sigma */
  double rho_used;
  double sigma_min_eig; /* lambda_min(Sigma*) (= a exactly when N_r < n) */
  double trace;         /* tr Sigma* (= n by construction, Theorem 1) */
  double seconds;
} laker_fit_report;

/* Alg.1 l.5-14 then P = Sigma*^{-1/2} (Eq. preconditioner-Sigmma).
   JACOBI: P = diag(lambda I + K)^{-1}.  NONE: P = I.
   LEARNED: u_k = (lambda I + K) z_k, ubar_k = u_k/||u_k||; CCCP
   with shrinkage and trace normalization in the exact structured
   form Sigma_t = a_t I + Ubar diag(b_t) Ubar^T (O4'); P kept as
   p_layout says (dense rows are row-sharded like K).  With ON_THE_FLY storage
   (LAKER at C5) the directions GEMM consumes K's rows
   assembled chunk by chunk into a transient buffer of <= 4 GiB (EXACT: the same
   correctly rounded entries as MATERIALIZED); K is still never stored.
   report: host, may be NULL.
   Errors: NOT_READY (no kernel), NOT_POSITIVE_DEFINITE, INVALID_ARGUMENT. */
laker_status laker_fit_preconditioner(laker_ctx ctx, const laker_fit_opts *opts,
                                      laker_fit_report *report);

/* ----------------------------------------------------------------- (3) solve */
typedef struct {
  double tol;         /* stop when ||r^k||_2 / ||y||_2 <= tol, 0 < tol < 1 */
  int32_t max_iters;  /* 0 -> 10 n */
  int32_t instrument; /* 1: time each operator / preconditioner launch with CUDA events */
} laker_solve_opts;

typedef struct {
  int32_t iters;            /* operator applies performed (R12) */
  int32_t termination;      /* LAKER_TERM_* */
  double rel_residual;      /* recursive ||r|| / ||y|| at exit */
  double true_rel_residual; /* ||y - (lambda I + K) alpha|| / ||y||, recomputed once */
  double seconds;           /* device time of the PCG loop (CUDA events) */
  /* extreme eigenvalues of the preconditioned operator P^(1/2) (lambda I + K) P^(1/2)
     estimated from the CG coefficients (the Lanczos tridiagonal T_k with
     T_jj = 1/delta_j + beta_{j-1}/delta_{j-1}, T_j,j+1 = sqrt(beta_j)/delta_j;
     Saad, Iterative Methods, 2nd ed., Sec. 6.7.3); their ratio estimates
     kappa(P A) (the quantity of Table I / P:853-858).  0 for the block solve. */
  double lanczos_lmin, lanczos_lmax;
} laker_solve_report;

/* Solve (lambda I + K) alpha = Y by Alg. 1's PCG:
   alpha^0 = 0, r^0 = y, theta^0 = P r^0, p^0 = theta^0; per iteration one
   operator apply q = (lambda I + K) p and one preconditioner apply theta = P r;
   delta = r.theta / p.q, beta = r'.theta' / r.theta; every inner product is a
   Dot2 reduction; alpha, r, p updates are single fma (R17).
   Y: n x nrhs column-major (host or device); alpha: n x nrhs output, complete
   on every rank.  nrhs > 1 runs nrhs independent recurrences sharing each
   operator / preconditioner pass (R13).  reports: host array [nrhs] or NULL.
   history: host [max_iters] relative residuals of column 0, or NULL.
   Reaching max_iters is not an error (termination MAX_ITERS).  Breakdown
   returns BREAKDOWN_ZERO_CURVATURE / INDEFINITE_PRECONDITIONER with the last
   iterate in alpha.  y = 0 gives alpha = 0, iters = 0, ZERO_RHS. */
laker_status laker_pcg_solve(laker_ctx ctx, int32_t nrhs, const double *Y, double *alpha,
                             const laker_solve_opts *opts, laker_solve_report *reports,
                             double *history);

/* Block-CG variant of the multi-RHS solve (C4): O'Leary's block PCG
   (Linear Algebra Appl. 29, 1980) -- the nrhs columns of Y share one block Krylov space:
   X0 = 0, R0 = Y, Z0 = P R0, D0 = Z0; per iteration Q = (lambda I + K) D,
   alpha = (D^T Q)^{-1} (Z^T R), X += D alpha, R -= Q alpha, Z = P R,
   beta = (Z_old^T R_old)^{-1} (Z^T R), D = Z + D beta, with the operator / preconditioner
   products of laker_pcg_solve's block solve and the nrhs x nrhs Gram matrices and SPD
   solves on the device; stops when every column has ||R_c|| / ||Y_c|| <= tol (R12's
   test, column-wise).  Not Alg. 1 column by column: compared with the oracle's block PCG
   (oracle.block_pcg) within a tolerance, never bitwise.  block (dividing nrhs; 0 = nrhs):
   the columns form nrhs / block independent groups of `block` columns, each its own block
   recurrence (the Gram matrices masked to their block x block diagonal blocks), all groups
   sharing every pass over K and P -- one group of 64 right-hand sides can lose rank and
   break down (C4), groups of 8 do not.  One rank, MATERIALIZED K, 1 <= nrhs <= 64.  Y, alpha, reports (all columns report the shared iteration count)
   and history (column 0) as laker_pcg_solve.  Errors: INVALID_ARGUMENT, NOT_READY;
   BREAKDOWN_ZERO_CURVATURE when D^T (lambda I + K) D, INDEFINITE_PRECONDITIONER when
   Z^T R is not numerically positive definite (last iterate in alpha). */
laker_status laker_block_cg_solve(laker_ctx ctx, int32_t nrhs, int32_t block, const double *Y, double *alpha,
                                  const laker_solve_opts *opts, laker_solve_report *reports,
                                  double *history);

/* --------------------------------------------------------------- (4) predict */
/* r_hat(x_m) = sum_i exp(scale <eq_m, e_i>) alpha_i (Eq. sc-radio-map-
   reconstruction; Alg.1 l.24), entries recomputed on the
   fly.  Eq: m x d row-major; alpha: n (host or device); out: m.  Rank r
   computes rows [r*ceil(m/W), ...) of out and leaves the others untouched.
   mode EXACT: correctly rounded entries + Dot2 row sums (bitwise = oracle). */
laker_status laker_predict(laker_ctx ctx, int64_t m, const double *Eq, const double *alpha,
                           double *out, int mode);

/* ------------------------------------------------- test / diagnostic hooks */
/* Replace / read the local K rows ((n/W) x n row-major). */
laker_status laker_load_kernel_rows(laker_ctx ctx, const double *K_rows);
laker_status laker_get_kernel_rows(laker_ctx ctx, double *K_rows);
/* kind EXTERNAL_DENSE: data = local P rows ((n/W) x n); JACOBI: data = diag (n),
   or NULL to derive it from the assembled K; NONE: data ignored. */
laker_status laker_set_preconditioner(laker_ctx ctx, int kind, const double *data);
laker_status laker_get_preconditioner_rows(laker_ctx ctx, double *P_rows);
/* LEARNED P in factored form: Q (n x n_dirs row-major), M (n_dirs x n_dirs
   row-major) and the scalar a^{-1/2} (host), so that P = a^{-1/2} I + Q M Q^T;
   any pointer may be NULL.  NOT_READY if the context holds no factored P.  A
   row-sharded context keeps only its part of the factors: Q is then its rows
   [r n/W, (r+1) n/W) (n/W x n_dirs); M is whole. */
laker_status laker_get_preconditioner_factors(laker_ctx ctx, double *Q, double *M, double *a_inv_sqrt);
/* The product QM = Q M (n x n_dirs row-major, host or device) the factored apply uses
   (R21: theta = a^{-1/2} r + QM (Q^T r), two Dot2 passes; a row-sharded
   context: its n/W rows).  NOT_READY if the
   context holds no factored P in QM form (a fit with p_layout FACTORED keeps three
   passes), INVALID_ARGUMENT for NULL. */
laker_status laker_get_preconditioner_qm(laker_ctx ctx, double *QM);
/* y = (lambda I + K) x, x and y length n (y complete on every rank). */
laker_status laker_apply_operator(laker_ctx ctx, const double *x, double *y);

/* Diagnostic: C (M x N int32, row-major) = A (M x K int8) B (N x K int8)^T on the
   tcgen05 int8 tensor cores (csrc/igemm.cu), all DEVICE pointers, K % 16 == 0,
   synchronous.  The building block of the fp64 emulation (Ozaki scheme). */
laker_status laker_debug_igemm_s8(const int8_t *A, const int8_t *B, int32_t *C, int64_t M, int64_t N, int64_t K);

/* Diagnostic: C (M x N) = A (M x K) B (N x K)^T in fp64 emulated on the int8
   tensor cores (Ozaki scheme, csrc/ozaki.cu; `slices` int8 digit slices per
   input, 0 = default 8), fp64 row-major DEVICE pointers, synchronous.  `kernel`:
   -1 the library's choice, 0 the level-streaming kernel, any other value the
   level-group kernel on chunk-interleaved slices (bitwise the same result; the
   choice exists for that test). */
laker_status laker_debug_ozaki_gemm(const double *A, const double *B, double *C, int64_t M, int64_t N, int64_t K,
                                    int32_t slices, int32_t kernel);

/* Test hooks of the row-sharded symmetric K apply (pcg_dist.cu, symv.cu).
   laker_debug_dist_tiles (host only, no GPU): the tile lists rank `rank` of `world`
   streams for an n x n symmetric matrix in br x tc tiles -- counts[0..2] = local
   block-rows L, tiles T, column tiles; toff [L+1], jt [T], cr_lo / cr_hi [n/tc] (any
   output NULL to query the counts).  INVALID_ARGUMENT unless n/world is a multiple of br
   (2 br for even world > 1).
   laker_debug_dist_symv_partials: on a context whose K uses the sharded symmetric apply
   (EXACT assembly, n/W % 256 == 0; a detached shard works), x (n) -> pairs (2 n: the
   unrounded (s, c) pair of this rank's partial sum of every row); rowmax (n: max_j |K_ij|
   of all rows) replaces the all-gathered row maxima a detached shard cannot form (NULL:
   keep).  laker_debug_dist_symv_combine: own (2 n/W: this rank's pairs of its rows) and
   recv (2 (W/2) n/W: the pairs of its rows from ranks w-1, ..., w-W/2) -> q_loc (n/W) =
   the rows of (lambda I + K) x, and pq_pair (2, may be NULL) = the unrounded x_loc.q_loc.
   All vectors host or device, synchronous. */
laker_status laker_debug_dist_tiles(int64_t n, int32_t br, int32_t tc, int32_t rank, int32_t world, int64_t *counts,
                                    int64_t *toff, int32_t *jt, int32_t *cr_lo, int32_t *cr_hi);
laker_status laker_debug_dist_symv_partials(laker_ctx ctx, const double *x, const double *rowmax, double *pairs);
laker_status laker_debug_dist_symv_combine(laker_ctx ctx, const double *x, const double *own, const double *recv,
                                           double *q_loc, double *pq_pair);
/* Test hook of the exact tensor-core K apply (B13; symv_tc.cu): on a context whose
   K uses it (stats.k_tensor_core; one rank, or a shard of the sharded plan -- detached
   shards included), x (n) -> groups (8 n int64, [g][i]): this rank's exact level-group sums
   G_g of every row i (tri.cuh), before any cross-rank sum; the shards' groups add up, as
   integers, to the one-rank groups.  rowmax (n, may be NULL) replaces the row maxima a
   detached shard cannot all-gather (it fixes K's slice exponent).  Synchronous. */
laker_status laker_debug_tc_groups(laker_ctx ctx, const double *x, const double *rowmax, int64_t *groups);

typedef struct {
  int64_t n, local_rows, ld;     /* problem size, rows held, padded row stride (doubles) */
  int32_t rank, world, precond_kind, storage, mode;
  uint64_t exp_inconclusive;     /* entries whose correctly-rounded test failed twice (R18) */
  uint64_t exp_overflow;
  /* instrumented solve (laker_solve_opts.instrument): summed CUDA-event times */
  double op_ms, prec_ms;         /* total ms in operator / dense-preconditioner passes */
  int64_t op_launches, prec_launches;
  double assemble_ms, fit_ms, solve_ms, predict_ms; /* last call of each (events) */
  int64_t kernel_launches;       /* kernels this context launched since creation */
  int32_t symmetric_k, symmetric_p; /* 1: K / dense P found bitwise symmetric on one rank, so the
                                       PCG applies stream only their block upper triangle (symv) */
  int32_t p_factored, n_dirs;    /* LEARNED P held as Q, M, a (LAKER_P_FACTORED): 1 applied in three
                                    passes Q (M (Q^T r)), 2 in the QM form (R21); its N_r */
  int32_t k_tensor_core, pad0;   /* 1: the symmetric K apply runs exactly on the int8 tensor cores
                                    (K held as 8 digit slices, csrc/symv_tc.cu); 0: fp64 kernel */
} laker_stats;
laker_status laker_get_stats(laker_ctx ctx, laker_stats *out);

#ifdef __cplusplus
}
#endif
#endif /* LAKER_H_ */
