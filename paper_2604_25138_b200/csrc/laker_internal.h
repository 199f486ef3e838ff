// Internal declarations of liblaker.so (not part of the ABI; see include/laker.h).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/laker.h"
#include "dot2.cuh"

namespace laker {

// Row stride of the materialized K and P: a multiple of 256 doubles (2 KiB)
// so every bulk-copied row segment is 16-byte aligned and whole-chunk sized.
constexpr int64_t kLdAlign = 256;
__host__ __device__ inline int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ inline int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }
inline int64_t padded_ld(int64_t n) { return (n + kLdAlign - 1) / kLdAlign * kLdAlign; }

// Device-resident PCG scalars (one struct per right-hand side).
struct PcgState {
  double rho;      // r.theta of the current iterate
  double delta;    // step length of the current iteration
  double beta;
  double ynorm;    // ||y||_2
  double rel;      // ||r|| / ||y|| after the last update
  double tol;
  int32_t iters;
  int32_t max_iters;
  int32_t done;    // 1 once terminated (later kernels of a captured chunk are no-ops)
  int32_t term;    // LAKER_TERM_*
  double *dh, *bh; // nullable: per-iteration delta_k / beta_k (Lanczos coefficients of the solve)
};

// every write of the step length / direction coefficient goes through these, so the
// solve keeps its CG coefficients for the Lanczos eigenvalue estimates (pcg.cu)
__device__ __forceinline__ void pcg_set_delta(PcgState *st, double d) {
  st->delta = d;
  if (st->dh) st->dh[st->iters] = d;
}
__device__ __forceinline__ void pcg_set_beta(PcgState *st, double b) {
  st->beta = b;
  if (st->bh && st->iters > 0) st->bh[st->iters - 1] = b;
}

// Ticket counters for the "last CTA reduces" epilogues, one per reduction
// site, reset by the last CTA.
enum { kCtrGemv = 0, kCtrUpdate = 1, kCtrInit = 2, kCtrMisc = 3, kCtrBar = 4, kCtrBarGen = 5, kNumCtr = 8 };

// Software grid barrier for kernels whose CTAs are all co-resident (persistent grids sized
// to the SMs): the calling threads of a CTA (`nthr` of them, named barrier `bar_id`) meet,
// thread 0 arrives on count and waits for the generation to move.  count / gen are zero /
// arbitrary at rest (the last arriver resets count).
__device__ __forceinline__ void grid_barrier(unsigned int *count, unsigned int *gen, int bar_id, int nthr) {
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthr) : "memory");
  if (threadIdx.x == 0) {
    const unsigned int g = *(volatile unsigned int *)gen;
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      *count = 0u;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*(volatile unsigned int *)gen == g) __nanosleep(20);
    }
    __threadfence();
  }
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthr) : "memory");
}

// The PCG step that follows an operator apply, fused into the apply's finalize (symv.cu):
// delta = rho / p.q, alpha += delta p, r -= delta q, ||r||^2 (and r.theta, Jacobi) and the
// termination test of pcg_update_kernel (pcg_kernels.cuh) -- the same fma / Dot2 operations.
struct FusedUpdate {
  int on;
  int pk;
  const double *p;       // the direction (x of the apply)
  double *alpha, *r, *theta;
  const double *dvec;    // Jacobi diagonal
  double *hist;
  unsigned int *bar;     // [2] grid barrier count, generation
  dd_pair *partials2;    // >= gridDim x 2
  unsigned int *counter2;
};

struct Buf {
  void *p = nullptr;
  size_t bytes = 0;
};

struct SymvPlan;  // symv.cu
struct SymvTc;    // symv_tc.cu: K as int8 digit slices for the exact tensor-core apply

// digit slices of a row-major fp64 matrix for the Ozaki products (otf_tc.cu)
struct OzSlices {
  int8_t *s = nullptr;   // rows x (S Kp), forward slice order
  int32_t *e = nullptr;  // rows
  int64_t rows = 0, Kp = 0;
  int S = 0;
};

}  // namespace laker

struct laker_ctx_s {
  int device = 0, rank = 0, world = 1;
  cudaStream_t stream = nullptr;
  bool owns_stream = false;
  ncclComm_t comm = nullptr;
  std::string last_error;

  // problem
  int64_t n = 0;
  int32_t d = 0;
  double scale = 1.0, lambda = 0.0;
  int storage = 0, mode = 1;
  int64_t r0 = 0, r1 = 0, ld = 0;   // local rows [r0, r1), padded stride
  bool assembled = false;

  double *E = nullptr;              // n x d
  double *K = nullptr;              // (r1-r0) x ld
  double *P = nullptr;              // (r1-r0) x ld (dense learned / external)
  double *Pdiag = nullptr;          // n (Jacobi)
  int precond_kind = LAKER_PRECOND_NONE;

  // workspace
  unsigned int *counters = nullptr;        // kNumCtr
  laker::dd_pair *partials = nullptr;      // per-CTA pairs (>= 2 x grid)
  unsigned long long *flags = nullptr;     // [0] exp inconclusive, [1] exp overflow
  int gemv_grid = 0, num_sms = 0;

  // symmetric (upper-triangle) GEMV, single rank: used for K / P only after a
  // device check found them bitwise symmetric (symv.cu)
  laker::SymvPlan *symv = nullptr;
  // the exact tensor-core form of the symmetric K apply (one rank, K's slices exact)
  laker::SymvTc *symv_tc = nullptr;
  bool k_tc = false;
  // tile partition of the symmetric on-the-fly operator (otf_sym.cu), built at assembly
  laker::SymvPlan *otf_sym = nullptr;
  // per-column factors {scale 2^(e_j), w_j} of the FAST tcgen05 on-the-fly kernels (otf_tc2.cu)
  double2 *cf = nullptr;
  int64_t cf_len = 0;
  // max_k |e_ik| per row of E (offsets of the EXACT entry kernels), set at assembly
  double *emax = nullptr;
  int64_t emax_len = 0;
  bool k_sym = false, p_sym = false;
  // factored LEARNED P = f_ainv I + Q M Q^T (fit.cu; applied in pcg.cu)
  bool p_factored = false;
  // one rank: Qt = nrp x ld (row k = q_k), Qr / QMf = n x f_ldq; sharded (f_local): Qt holds
  // the columns [r0, r1) (nrp x f_ldl), Qr / QMf the rows [r0, r1); M is always whole
  double *Qt = nullptr;             // nrp x ld   (row k = q_k, zero padded)
  double *Qr = nullptr;             // n x f_ldq  (row i = Q_i., zero padded)
  double *QMf = nullptr;            // n x f_ldq  QM = Q M (R21: theta = a^-1/2 r + QM (Q^T r))
  bool f_local = false;
  int64_t f_ldl = 0;
  bool p_qm = false;                // the factored apply uses QMf (two passes)
  double *Mf = nullptr;             // nrp x f_ldq
  double *fz = nullptr, *fw = nullptr;  // f_ldq workspaces (z = Q^T r, w = M z), zero padded
  int64_t f_nr = 0, f_nrp = 0, f_ldq = 0;
  int64_t f_alloc_nrp = 0, f_alloc_n = 0;  // sizes the factor buffers were allocated for (reused)
  size_t E_bytes = 0, K_bytes = 0;         // allocations kept across assemble calls of the same size
  double f_ainv = 0.0;

  // FAST on-the-fly: digit slices of E for the tcgen05 QK^T (otf_tc.cu), built lazily
  laker::OzSlices ozE;
  bool ozE_valid = false;

  laker_stats stats{};
};

namespace laker {

// error helpers (api.cu)
laker_status set_err(laker_ctx ctx, laker_status s, const std::string &msg);
laker_status cuda_err(laker_ctx ctx, cudaError_t e, const char *what);

#define LAKER_TRY(expr)            \
  do {                             \
    laker_status _s = (expr);      \
    if (_s != LAKER_OK) return _s; \
  } while (0)

#define LAKER_CUDA(ctx, call)                                      \
  do {                                                             \
    cudaError_t _e = (call);                                       \
    if (_e != cudaSuccess) return ::laker::cuda_err(ctx, _e, #call); \
  } while (0)

// ------------------------------------------------------------------ gemv.cu
// y_i = RN(lambda x_{row0+i} + sum_j A_ij x_j) for the `rows` local rows of A
// (row stride ld, n logical columns, zero padded), Dot2 rows, bulk-TMA staged.
// Also reduces dot(x[row0 .. row0+rows), y) over all CTAs into a pair and runs
// `epi` on it in the last CTA.
enum GemvEpi { kEpiNone = 0, kEpiDelta = 1, kEpiBeta = 2, kEpiStoreDot = 3, kEpiStorePair = 4 };
struct GemvArgs {
  const double *A;
  int64_t ld;
  int64_t rows;
  int64_t ncols;
  const double *x;        // full vector, length >= ld (zero padded)
  int64_t row0;           // global index of local row 0 (for the lambda term and the dot)
  double *y;              // local output (rows)
  double lambda;          // 0 -> no diagonal term
  PcgState *state;        // nullable; done != 0 -> no-op; epilogue target
  dd_pair *partials;      // >= gridDim
  unsigned int *counter;  // ticket
  double *dot_out;        // kEpiStoreDot target
  dd_pair *pair_out;      // kEpiStorePair target (unrounded Dot2 pair, for the rank-order combine)
  int epi;
  bool evict_first;       // stream A with an L2 evict-first policy
  // non-square applies (factored P): when set, the diagonal term lambda xd_i and the
  // epilogue dot use xd (global row index row0 + i) instead of the streamed x
  const double *xd;
  // symv: per-CTA maxima of |x| written by the kernel that produced x (nxparts of them);
  // null -> launch_symv computes them
  const double *xparts;
  int nxparts;
  // symv on a row-sharded plan: the unrounded pair of every row i < n (pcg_dist.cu)
  dd_pair *ypair;
  // symv on one rank inside the PCG (epi = kEpiDelta): the update step fused in
  FusedUpdate upd;
  // symv (which = 0): the exact int8 tensor-core tile pass instead of the fp64 one
  SymvTc *tc;
  // gemv with epi = kEpiBeta (the preconditioner's last pass, one rank): the direction
  // update p = fma(beta, p, theta) of pcg_pupdate_kernel fused in after a grid barrier
  // (persistent grid, one CTA per SM); the per-CTA max |p| go to pu_pmax[blockIdx]; with
  // pu_budget the iteration budget is closed after it (MAX_ITERS)
  double *pu_p;
  double *pu_pmax;
  int pu_budget;
  unsigned int *pu_bar;
};
void launch_gemv(const GemvArgs &a, int grid, cudaStream_t s);
void gemv_init();
int gemv_max_grid(int num_sms);
size_t gemv_smem_bytes();

// ----------------------------------------------------------------- symv.cu
// Symmetric Dot2 GEMV over the block upper triangle (half the bytes of gemv.cu),
// same outputs and epilogues, bitwise equal rows.  which = 0 (K) / 1 (P).
// world > 1: the row-sharded plan of rank `rank` (tri_plan_dist); the matrix holds the
// rank's n / W rows and launch_symv writes GemvArgs::ypair instead of y
cudaError_t symv_plan(SymvPlan *&p, int64_t n, int64_t ld, int num_sms, int rank = 0, int world = 1,
                      bool dist = false);
bool tri_is_dist(const SymvPlan *p);
double *symv_rowmax_ptr(SymvPlan *p, int which);
void symv_free(SymvPlan *&p);
bool symv_bind(SymvPlan *p, int which, const double *A);
void symv_rowmax(SymvPlan *p, int which, const double *A, cudaStream_t s);
void launch_symv(const SymvPlan *p, int which, const GemvArgs &g, cudaStream_t s);
void launch_symv_check(const double *A, int64_t n, int64_t ld, int *flag, cudaStream_t s);
void symv_init();
// ------------------------------------------------------------- symv_tc.cu
void symv_tc_init();
void symv_tc_free(SymvTc *&p);
// slice K (n x n, stride ld, bitwise symmetric) into 8 int8 digit slices with one global
// exponent; false if not every entry is exact in that form
bool symv_tc_prepare(SymvTc *&p, const double *K, int64_t n, int64_t ld, const double *rowmax, cudaStream_t s,
                     int rank = 0, int world = 1);
// the [W][8][cs] exact level-group accumulators (cs: rows per chunk) and {eK, F} of the last apply
long long *symv_tc_groups(SymvTc *p, int64_t *cs);
const int *symv_tc_exponents(const SymvTc *p);
// ------------------------------------------------------------- otf_sym.cu
void otf_sym_init();
cudaError_t otf_sym_prepare(laker_ctx ctx);
bool launch_operator_otf_sym(laker_ctx ctx, const double *p, double *q, PcgState *st, int epi, double *dot_out,
                             cudaStream_t s);
size_t symv_smem_bytes();
// set ctx->k_sym / p_sym: bitwise-symmetry check of the (whole, single-rank) matrix
// symmetric_rows: the rows are bitwise symmetric by construction (sharded contexts
// cannot check it)
laker_status refresh_symmetry(laker_ctx ctx, int which, bool symmetric_rows = false);

// -------------------------------------------------------------- assemble.cu
// emax: max_k |e_ik| per row of E (launch_rowabsmax), the offsets of the compensated dots
void launch_assemble_exact_sym(const double *E, int64_t n, int32_t d, double scale, double *K,
                               int64_t ld, unsigned long long *flags, const double *emax, cudaStream_t s);
void launch_assemble_exact_rows(const double *E, int64_t n, int32_t d, double scale, int64_t r0,
                                int64_t r1, double *K, int64_t ld, unsigned long long *flags,
                                const double *emax, cudaStream_t s);
void launch_rowabsmax(const double *X, int64_t rows, int32_t d, double *out, cudaStream_t s);
void launch_assemble_fast(const double *E, int64_t n, int32_t d, double scale, int64_t r0,
                          int64_t r1, double *K, int64_t ld, unsigned long long *flags,
                          cudaStream_t s);
void launch_jacobi_diag(const double *E, int64_t n, int32_t d, double scale, double lambda,
                        double *dvec, unsigned long long *flags, cudaStream_t s);

// --------------------------------------------------------------- predict.cu
// out[a] = RN(sum_i exp(scale <Eq_a, E_i>) w_i (+ lambda * xdiag[a]))  for a in [0, m)
void launch_kernel_matvec_exact(const double *Eq, int64_t m, const double *E, int64_t n, int32_t d,
                                double scale, const double *w, double lambda, const double *xdiag,
                                double *out, unsigned long long *flags, const int32_t *done,
                                cudaStream_t s, const double *emq, const double *emE);

// -------------------------------------------------------------- otf_fast.cu
// FAST (DMMA + CUDA exp) version of launch_kernel_matvec_exact; d <= 128.
void launch_kernel_matvec_fast(const double *Eq, int64_t m, const double *E, int64_t n, int32_t d, double scale,
                               const double *w, double lambda, const double *xdiag, double *out,
                               const int32_t *done, cudaStream_t s);
void otf_fast_init();
// mode dispatch with the context: FAST and d <= 128 -> tcgen05 QK^T (otf_tc.cu) with the
// E slices cached in ctx (rows of Eq = rows [eq_row0, eq_row0 + m) of E when Eq_is_E),
// else otf_fast.cu (DMMA) / the EXACT kernel.  LAKER_OTF_TC=0 selects DMMA.
cudaError_t launch_kernel_matvec_ctx(laker_ctx ctx, int mode, const double *Eq, int64_t m, bool Eq_is_E,
                                     int64_t eq_row0, const double *w, double lambda, const double *xdiag,
                                     double *out, const int32_t *done, cudaStream_t s);
// mode dispatch for the on-the-fly matvec (EXACT: correctly rounded entries + Dot2)
inline void launch_kernel_matvec(int mode, const double *Eq, int64_t m, const double *E, int64_t n, int32_t d,
                                 double scale, const double *w, double lambda, const double *xdiag, double *out,
                                 unsigned long long *flags, const int32_t *done, cudaStream_t s,
                                 const double *emq, const double *emE) {
  if (mode == LAKER_MODE_FAST && d <= 128)
    launch_kernel_matvec_fast(Eq, m, E, n, d, scale, w, lambda, xdiag, out, done, s);
  else
    launch_kernel_matvec_exact(Eq, m, E, n, d, scale, w, lambda, xdiag, out, flags, done, s, emq, emE);
}

// ----------------------------------------------------------------- dgemm.cu
struct GemmArgs {
  int64_t M, N, K;        // K % 16 == 0; N even (or ldc/ldcin padded)
  const double *A;        // M x K row-major
  int64_t lda;
  const double *B;        // b_kn ? K x N : N x K (row-major)
  int64_t ldb;
  double *C;
  int64_t ldc;
  double alpha, beta;     // C = alpha A op(B) + beta Cin (+ diag on row - col == diag_offset)
  const double *Cin;
  int64_t ldcin;
  double diag;
  int64_t diag_offset;
  bool lower_only;        // skip CTA tiles strictly above the block diagonal
  bool dmma_only = false; // keep the product on the fp64 (DMMA) path, never the int8 emulation
  int oz_slices = 0;      // int8 digit slices of the emulation when it is used (0: ozaki_S())
  bool b_sym = false;     // B is exactly symmetric (mirrored): the emulation slices op(B) by B's rows
  int tri;                // 0 all; 1 only entries with row + tri_off >= col; 2 only row + tri_off < col
  int64_t tri_off;        // (tiles with no kept entry are skipped; masked entries are not written)
  // internal (launch_dgemm's split-K for skinny products): CTA z covers k in
  // [z kchunk, (z+1) kchunk) and writes its raw partial to ws[z] (M x N)
  double *ws;
  int64_t kchunk;
};
// copy the strict lower triangle of the n x n matrix A onto its upper triangle
void launch_mirror_lower(double *A, int64_t lda, int64_t n, cudaStream_t s);
void dgemm_init();
void launch_dgemm(const GemmArgs &g, bool b_kn, cudaStream_t s);

// ---------------------------------------------------------------- igemm.cu
// int8 tensor-core GEMM (tcgen05 kind::i8) with an Ozaki epilogue:
// x = v 2^(shift + ea[row] + eb[col]) then W = x | W += x | C = alpha (W + x) + beta Cin + diag
enum { kIgemmStoreS32 = 0, kIgemmAccInit = 1, kIgemmAccAdd = 2, kIgemmFinal = 3 };
struct IgemmEpi {
  int mode;
  int64_t M, N;
  int32_t *Ci;
  int64_t ldci;
  double *W;
  int64_t ldw;
  bool has_w;
  const int32_t *ea, *eb;
  int shift;
  double *C;
  int64_t ldc;
  const double *Cin;
  int64_t ldcin;
  double alpha, beta, diag;
  int64_t diag_offset;
  int tri;
  int64_t tri_off;
};
void igemm_init();
cudaError_t launch_igemm_epi(const int8_t *A, int64_t lda, const int8_t *B, int64_t ldb, int64_t K,
                             const IgemmEpi &e, cudaStream_t s);

// ---------------------------------------------------------------- ozaki.cu
// C = alpha A op(B) + beta Cin + diag (GemmArgs semantics, tri honoured; lower_only as
// tri = 1, no entry above the diagonal written) in fp64 emulated on the int8 tensor cores: rows scaled by powers of two,
// split into S signed 7-bit digit slices, all slice products with s + t <= S - 1
// (0-based) accumulated exactly in int32 per digit level, levels summed in fp64.
cudaError_t launch_ozaki_gemm(const GemmArgs &g, bool b_kn, int S, cudaStream_t s, int kernel = -1);
// route a GemmArgs to the Ozaki path when it is large enough to pay
bool ozaki_eligible(const GemmArgs &g);
void launch_ozaki_split(const double *X, int64_t ld, int64_t rows, int64_t K, int trans, int S, int rev,
                        int8_t *out, int32_t *e, int64_t Kp, cudaStream_t s, unsigned long long *mx_buf = nullptr,
                        int il = 0);

// --------------------------------------------------------------- otf_tc.cu
// FAST on-the-fly kernel matvec on the tcgen05 int8 tensor cores: the QK^T dot
// products of exp(scale <eq_a, e_i>) in Ozaki digit levels (S slices, d <= 128),
// scale + exp + weight + row-sum epilogue fused (same contract as otf_fast.cu).
cudaError_t oz_slices_make(OzSlices &o, const double *X, int64_t rows, int32_t d, int S, cudaStream_t s);
void oz_slices_free(OzSlices &o, cudaStream_t s);
cudaError_t launch_otf_tc(const OzSlices &A, int64_t a0, int64_t m, const OzSlices &B, int64_t n, double scale,
                          const double *w, double lambda, const double *xdiag, double *out, const int32_t *done,
                          cudaStream_t s);
void otf_tc_init();
cudaError_t max_rownorm2(const double *E, int64_t n, int d, double *out, cudaStream_t s);

// ------------------------------------------------------------- otf_tc2.cu (d <= 64, K = 64 slices)
void otf_tc2_init();
cudaError_t launch_otf_tc2_rect(const OzSlices &A, int64_t a0, int64_t m, const OzSlices &B, int64_t n, double scale,
                                const double *w, double2 *cf, double lambda, const double *xdiag, double *out,
                                const int32_t *done, cudaStream_t s);


// ---------------------------------------------------------- ozaki_skinny.cu
// multi-RHS products C (M x N<=64) = alpha A op(B) + beta Cin with A pre-sliced (tcgen05)
cudaError_t oz_slices_make_general(OzSlices &o, const double *X, int64_t ld, int64_t rows, int64_t K, int trans, int S,
                                   cudaStream_t s, unsigned long long *mx_buf = nullptr);
cudaError_t launch_oz_skinny(const OzSlices &A, const OzSlices &B, int64_t N, double alpha, double beta,
                             const double *Cin, int64_t ldcin, double *C, int64_t ldc, double *part, int max_splits,
                             int num_sms, cudaStream_t s);
void oz_skinny_init();
int oz_skinny_max_slices();

// ------------------------------------------------------------- dense_la.cu
// In-place lower Cholesky of the n x n SPD matrix A (row-major, lda; n % 64 == 0);
// strict upper triangle zeroed.  *flag (device) set to 1 on a pivot <= 0.
void cholesky_lower(double *A, int64_t lda, int64_t n, int *flag, cudaStream_t s, int64_t *launches);
void cholesky_lower_aug(double *A, int64_t lda, int64_t n, int64_t m, int *flag, cudaStream_t s,
                        int64_t *launches);
// B <- L^{-1} B  (L n x n lower, n % 64 == 0; B n x ncols row-major, ldb).
void trsm_lower_left(const double *L, int64_t ldl, int64_t n, double *B, int64_t ldb, int64_t ncols,
                     cudaStream_t s, int64_t *launches);
void launch_transpose(const double *A, int64_t rows, int64_t cols, int64_t lda, double *B, int64_t ldb,
                      cudaStream_t s);

// ------------------------------------------------------------------- fit.cu
laker_status fit_learned(laker_ctx ctx, const laker_fit_opts &o, laker_fit_report *rep);
// dense P rows [r0, r1) into ctx->P from the factors (nrp x ld Q^T, M with row stride ldm)
laker_status form_dense_p(laker_ctx ctx, const double *Ut, const double *Mm, int64_t ldm, int64_t nrp,
                          double ainv);
// form (once) and cache the dense rows of a factored P (block / sharded solvers, hooks)
laker_status ensure_dense_p(laker_ctx ctx);
void free_factors(laker_ctx ctx);

// ------------------------------------------------------------------- pcg.cu
laker_status pcg_solve_device(laker_ctx ctx, const double *y, double *alpha, const laker_solve_opts &o,
                              laker_solve_report *rep, double *history);
laker_status apply_operator_device(laker_ctx ctx, const double *x, double *y);
void lanczos_extremes(const std::vector<double> &dl, const std::vector<double> &bt, int k, double &lmin,
                      double &lmax);

// -------------------------------------------------------------- pcg_dist.cu
// Row-sharded PCG over NCCL (ctx->comm != nullptr): identical recurrence,
// scalars combined from per-rank unrounded Dot2 pairs in rank order.
laker_status pcg_solve_dist(laker_ctx ctx, const double *y, double *alpha, const laker_solve_opts &o,
                            laker_solve_report *rep, double *history);
laker_status apply_operator_dist(laker_ctx ctx, const double *x, double *y);

// ------------------------------------------------------------- pcg_block.cu
// nrhs independent recurrences sharing GEMM-shaped applies (multi-RHS, C4).
laker_status pcg_solve_block(laker_ctx ctx, int32_t m, const double *Y, double *alpha,
                             const laker_solve_opts &o, laker_solve_report *reps, double *history, int block_cg = 0);
// the row-sharded version (ctx->comm): K / P / vectors by row blocks, rank-order combines
laker_status pcg_solve_block_dist(laker_ctx ctx, int32_t m, const double *Y, double *alpha,
                                  const laker_solve_opts &o, laker_solve_report *reps, double *history);
// wait for an event / the stream while watching the communicator for asynchronous NCCL
// errors (on one: ncclCommAbort, ctx->comm = null, LAKER_ERR_NCCL) -- pcg_dist.cu
laker_status dist_wait(laker_ctx ctx, cudaEvent_t ev);
laker_status dist_sync(laker_ctx ctx, cudaStream_t s);
laker_status nccl_err(laker_ctx ctx, ncclResult_t r, const char *what);

#define LAKER_NCCL(ctx, call)                                        \
  do {                                                               \
    ncclResult_t _r = (call);                                        \
    if (_r != ncclSuccess) return ::laker::nccl_err(ctx, _r, #call);  \
  } while (0)

}  // namespace laker
