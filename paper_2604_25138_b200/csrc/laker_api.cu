// The C ABI of liblaker.so (include/laker.h): argument checks, host/device
// staging, context lifecycle, and dispatch to the kernels.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "laker_internal.h"

using laker::set_err;

namespace laker {

laker_status set_err(laker_ctx ctx, laker_status s, const std::string &msg) {
  if (ctx) ctx->last_error = msg;
  return s;
}

laker_status cuda_err(laker_ctx ctx, cudaError_t e, const char *what) {
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  return set_err(ctx, e == cudaErrorMemoryAllocation ? LAKER_ERR_OUT_OF_MEMORY : LAKER_ERR_CUDA, m);
}

// The symmetric GEMV (symv.cu) is selected for K (which = 0) or P (which = 1) on a
// single rank for a materialized matrix that a device check finds bitwise symmetric.
// Row-sharded (world > 1), where no rank sees the whole matrix, it is selected for K
// only when the rows are symmetric by construction (EXACT assembly: K_ij and K_ji are
// the same correctly rounded operations, assemble.cu) and n / W is a multiple of 256;
// each rank then streams its tiles of tri_plan_dist and the row maxima of all n rows
// are all-gathered.  LAKER_SYMV=0 disables it (A/B measurements).
laker_status refresh_symmetry(laker_ctx ctx, int which, bool symmetric_rows) {
  bool &flag = which == 0 ? ctx->k_sym : ctx->p_sym;
  flag = false;
  if (which == 0) ctx->k_tc = false;
  const double *A = which == 0 ? ctx->K : ctx->P;
  if (!A || ctx->storage != LAKER_STORE_MATERIALIZED) return LAKER_OK;
  const char *env = std::getenv("LAKER_SYMV");
  if (env && env[0] == '0') return LAKER_OK;
  if (ctx->world > 1 || ctx->comm) {
    const int64_t nloc = ctx->n / ctx->world;
    if (which != 0 || !symmetric_rows || nloc % 256 != 0) return LAKER_OK;
    LAKER_CUDA(ctx, symv_plan(ctx->symv, ctx->n, ctx->ld, ctx->num_sms, ctx->rank, ctx->world, true));
    if (!symv_bind(ctx->symv, 0, A)) return LAKER_OK;
    symv_rowmax(ctx->symv, 0, A, ctx->stream);
    ctx->stats.kernel_launches++;
    if (ctx->comm) {
      double *rm = symv_rowmax_ptr(ctx->symv, 0);
      LAKER_NCCL(ctx, ncclAllGather(rm + ctx->r0, rm, nloc, ncclDouble, ctx->comm, ctx->stream));
    }
    LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    flag = true;
    // the exact tensor-core tiles (B13) on this rank's tiles of the sharded plan, used only
    // if every rank's entries are exact in the slice form (all ranks take the same path);
    // a detached shard (no communicator, tests) decides alone
    const char *tenv = std::getenv("LAKER_SYMV_TC");
    if (!(tenv && tenv[0] == '0') && ctx->comm) {
      int ok = symv_tc_prepare(ctx->symv_tc, A, ctx->n, ctx->ld, symv_rowmax_ptr(ctx->symv, 0), ctx->stream, ctx->rank,
                               ctx->world) ? 1 : 0;
      cudaGetLastError();
      int *dok = reinterpret_cast<int *>(ctx->flags + 2);
      LAKER_CUDA(ctx, cudaMemcpyAsync(dok, &ok, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
      LAKER_NCCL(ctx, ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, ctx->comm, ctx->stream));
      LAKER_CUDA(ctx, cudaMemcpyAsync(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
      ctx->k_tc = ok == 1;
      ctx->stats.kernel_launches += 2;
    } else if (!(tenv && tenv[0] == '0')) {
      ctx->k_tc = symv_tc_prepare(ctx->symv_tc, A, ctx->n, ctx->ld, symv_rowmax_ptr(ctx->symv, 0), ctx->stream,
                                  ctx->rank, ctx->world);
      cudaGetLastError();
      ctx->stats.kernel_launches += 2;
    }
    return LAKER_OK;
  }
  LAKER_CUDA(ctx, symv_plan(ctx->symv, ctx->n, ctx->ld, ctx->num_sms));
  int *dflag = reinterpret_cast<int *>(ctx->flags + 2);
  LAKER_CUDA(ctx, cudaMemsetAsync(dflag, 0, sizeof(int), ctx->stream));
  launch_symv_check(A, ctx->n, ctx->ld, dflag, ctx->stream);
  ctx->stats.kernel_launches++;
  int h = 1;
  LAKER_CUDA(ctx, cudaMemcpyAsync(&h, dflag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (h == 0) {
    flag = symv_bind(ctx->symv, which, A);
    if (flag) {
      symv_rowmax(ctx->symv, which, A, ctx->stream);
      ctx->stats.kernel_launches++;
      LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    }
  }
  if (which == 0) {
    // the exact int8 tensor-core form (symv_tc.cu) when every entry of K is exact in 8
    // digit slices with one exponent; LAKER_SYMV_TC=0 keeps the fp64 kernel (A/B)
    const char *tenv = std::getenv("LAKER_SYMV_TC");
    if (flag && !(tenv && tenv[0] == '0')) {
      ctx->k_tc = symv_tc_prepare(ctx->symv_tc, A, ctx->n, ctx->ld, symv_rowmax_ptr(ctx->symv, 0), ctx->stream, 0, 1);
      ctx->stats.kernel_launches += 2;
      cudaGetLastError();
    }
  }
  return LAKER_OK;
}

}  // namespace laker

namespace {

bool is_device_ptr(const void *p) {
  if (p == nullptr) return false;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// A caller buffer viewed on the device: host buffers are staged through a
// temporary device allocation on the context stream.
struct DevView {
  laker_ctx ctx = nullptr;
  double *dptr = nullptr;
  double *hptr = nullptr;  // host pointer to copy back (outputs)
  size_t bytes = 0;
  bool owned = false;
  ~DevView() {
    if (owned && dptr) cudaFreeAsync(dptr, ctx->stream);
  }
};

laker_status view_in(laker_ctx ctx, const double *p, size_t count, DevView &v) {
  v.ctx = ctx;
  v.bytes = count * sizeof(double);
  if (is_device_ptr(p)) {
    v.dptr = const_cast<double *>(p);
    return LAKER_OK;
  }
  LAKER_CUDA(ctx, cudaMallocAsync(&v.dptr, std::max<size_t>(v.bytes, 8), ctx->stream));
  v.owned = true;
  if (v.bytes) LAKER_CUDA(ctx, cudaMemcpyAsync(v.dptr, p, v.bytes, cudaMemcpyHostToDevice, ctx->stream));
  return LAKER_OK;
}

laker_status view_out(laker_ctx ctx, double *p, size_t count, DevView &v) {
  v.ctx = ctx;
  v.bytes = count * sizeof(double);
  if (is_device_ptr(p)) {
    v.dptr = p;
    return LAKER_OK;
  }
  LAKER_CUDA(ctx, cudaMallocAsync(&v.dptr, std::max<size_t>(v.bytes, 8), ctx->stream));
  v.owned = true;
  v.hptr = p;
  return LAKER_OK;
}

laker_status flush_out(laker_ctx ctx, DevView &v) {
  if (v.hptr && v.bytes) {
    LAKER_CUDA(ctx, cudaMemcpyAsync(v.hptr, v.dptr, v.bytes, cudaMemcpyDeviceToHost, ctx->stream));
    LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  }
  return LAKER_OK;
}

void free_dev(laker_ctx ctx, double *&p) {
  if (p) cudaFree(p);
  p = nullptr;
  (void)ctx;
}

laker_status ensure_jacobi(laker_ctx ctx) {
  if (ctx->Pdiag) return LAKER_OK;
  LAKER_CUDA(ctx, cudaMalloc(&ctx->Pdiag, ctx->n * sizeof(double)));
  laker::launch_jacobi_diag(ctx->E, ctx->n, ctx->d, ctx->scale, ctx->lambda, ctx->Pdiag, ctx->flags,
                            ctx->stream);
  ctx->stats.kernel_launches++;
  LAKER_CUDA(ctx, cudaGetLastError());
  return LAKER_OK;
}

#define CHECK_CTX(ctx) \
  if (!(ctx)) return LAKER_ERR_INVALID_ARGUMENT

}  // namespace

extern "C" {

const char *laker_status_string(laker_status s) {
  switch (s) {
    case LAKER_OK: return "ok";
    case LAKER_ERR_INVALID_ARGUMENT: return "invalid argument";
    case LAKER_ERR_DIMENSION_MISMATCH: return "dimension mismatch";
    case LAKER_ERR_NOT_READY: return "not ready";
    case LAKER_ERR_CUDA: return "CUDA error";
    case LAKER_ERR_NCCL: return "NCCL error";
    case LAKER_ERR_OUT_OF_MEMORY: return "out of memory";
    case LAKER_ERR_NOT_POSITIVE_DEFINITE: return "not positive definite";
    case LAKER_ERR_INDEFINITE_PRECONDITIONER: return "indefinite preconditioner";
    case LAKER_ERR_BREAKDOWN_ZERO_CURVATURE: return "breakdown (zero curvature)";
    case LAKER_ERR_OVERFLOW: return "exp overflow in kernel entries";
    default: return "internal error";
  }
}

const char *laker_last_error(laker_ctx ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

laker_status laker_get_unique_id(unsigned char id[128]) {
  if (!id) return LAKER_ERR_INVALID_ARGUMENT;
  ncclUniqueId u;
  if (ncclGetUniqueId(&u) != ncclSuccess) return LAKER_ERR_NCCL;
  std::memcpy(id, u.internal, 128);
  return LAKER_OK;
}

laker_status laker_create(laker_ctx *out, int device, int rank, int world, const unsigned char *nccl_id,
                          void *cuda_stream) {
  if (!out) return LAKER_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  // world > 1 without an id: a detached shard (row-sharded assembly / predict / hooks
  // only, no collectives) -- used to test the sharded layouts on one GPU.
  if (world < 1 || rank < 0 || rank >= world) return LAKER_ERR_INVALID_ARGUMENT;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return LAKER_ERR_CUDA;  // no CPU fallback
  }
  if (device < 0 || device >= ndev) return LAKER_ERR_INVALID_ARGUMENT;
  if (cudaSetDevice(device) != cudaSuccess) return LAKER_ERR_CUDA;
  auto *c = new laker_ctx_s();
  c->device = device;
  c->rank = rank;
  c->world = world;
  if (cuda_stream) {
    c->stream = static_cast<cudaStream_t>(cuda_stream);
  } else {
    // blocking stream: ordered with the legacy default stream torch uses
    if (cudaStreamCreate(&c->stream) != cudaSuccess) {
      delete c;
      return LAKER_ERR_CUDA;
    }
    c->owns_stream = true;
  }
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  {
    // keep freed stream-ordered allocations in the pool (the fit and the Ozaki GEMMs
    // allocate GiB-sized scratch per call; returning it to the OS at every sync is slow)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  c->gemv_grid = laker::gemv_max_grid(c->num_sms);
  laker::gemv_init();
  laker::symv_init();
  laker::symv_tc_init();
  laker::otf_sym_init();
  laker::otf_tc2_init();
  laker::dgemm_init();
  laker::igemm_init();
  laker::otf_tc_init();
  laker::oz_skinny_init();
  laker::otf_fast_init();
  const size_t npart = 4096;
  if (cudaMalloc(&c->counters, laker::kNumCtr * sizeof(unsigned int)) != cudaSuccess ||
      cudaMalloc(&c->partials, npart * sizeof(laker::dd_pair)) != cudaSuccess ||
      cudaMalloc(&c->flags, 4 * sizeof(unsigned long long)) != cudaSuccess) {
    delete c;
    return LAKER_ERR_OUT_OF_MEMORY;
  }
  cudaMemset(c->counters, 0, laker::kNumCtr * sizeof(unsigned int));
  cudaMemset(c->flags, 0, 4 * sizeof(unsigned long long));
  if (nccl_id) {  // world > 1, or a 1-rank communicator (exercises the collective path)
    ncclUniqueId u;
    std::memcpy(u.internal, nccl_id, 128);
    if (ncclCommInitRank(&c->comm, world, u, rank) != ncclSuccess) {
      delete c;
      return LAKER_ERR_NCCL;
    }
  }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    delete c;
    return LAKER_ERR_CUDA;
  }
  c->stats.rank = rank;
  c->stats.world = world;
  *out = c;
  return LAKER_OK;
}

laker_status laker_destroy(laker_ctx ctx) {
  CHECK_CTX(ctx);
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  free_dev(ctx, ctx->E);
  free_dev(ctx, ctx->K);
  free_dev(ctx, ctx->P);
  free_dev(ctx, ctx->Pdiag);
  laker::free_factors(ctx);
  laker::oz_slices_free(ctx->ozE, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  cudaFree(ctx->counters);
  cudaFree(ctx->partials);
  cudaFree(ctx->flags);
  laker::symv_free(ctx->symv);
  laker::symv_tc_free(ctx->symv_tc);
  laker::symv_free(ctx->otf_sym);
  if (ctx->cf) cudaFree(ctx->cf);
  if (ctx->emax) cudaFree(ctx->emax);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->owns_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return LAKER_OK;
}

laker_status laker_assemble_kernel(laker_ctx ctx, int64_t n, int32_t d, const double *E, double scale,
                                   double lambda, int storage, int mode) {
  CHECK_CTX(ctx);
  if (n < 1 || d < 1 || !E || !(lambda > 0.0) || !std::isfinite(scale) || n % ctx->world != 0 ||
      (storage != LAKER_STORE_MATERIALIZED && storage != LAKER_STORE_ON_THE_FLY) ||
      (mode != LAKER_MODE_FAST && mode != LAKER_MODE_EXACT))
    return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "assemble: need n>=1, d>=1, lambda>0, n % world == 0, valid enums");
  cudaSetDevice(ctx->device);
  // E and K buffers of the same size are kept (a refit/re-solve loop re-assembles
  // every step; cudaFree + cudaMalloc of 2 GiB costs ~10 ms); the factored-P
  // buffers are kept too (invalidated here, refilled by the next fit)
  const int64_t rows_new = n / ctx->world;
  const size_t e_bytes = (size_t)n * d * sizeof(double);
  const size_t k_bytes = storage == LAKER_STORE_MATERIALIZED ? (size_t)rows_new * laker::padded_ld(n) * sizeof(double) : 0;
  if (ctx->E_bytes != e_bytes) {
    free_dev(ctx, ctx->E);
    ctx->E_bytes = 0;
  }
  if (ctx->K_bytes != k_bytes) {
    free_dev(ctx, ctx->K);
    ctx->K_bytes = 0;
  }
  free_dev(ctx, ctx->P);
  free_dev(ctx, ctx->Pdiag);
  if (ctx->f_alloc_n != n) laker::free_factors(ctx);
  ctx->p_factored = false;
  ctx->assembled = false;
  ctx->k_sym = ctx->p_sym = false;
  ctx->precond_kind = LAKER_PRECOND_NONE;
  ctx->n = n;
  ctx->d = d;
  ctx->scale = scale;
  ctx->lambda = lambda;
  ctx->storage = storage;
  ctx->mode = mode;
  ctx->ld = laker::padded_ld(n);
  ctx->r0 = n / ctx->world * ctx->rank;
  ctx->r1 = ctx->r0 + n / ctx->world;
  const int64_t rows = ctx->r1 - ctx->r0;
  cudaStream_t s = ctx->stream;
  if (!ctx->E) {
    LAKER_CUDA(ctx, cudaMalloc(&ctx->E, e_bytes));
    ctx->E_bytes = e_bytes;
  }
  if (is_device_ptr(E))
    LAKER_CUDA(ctx, cudaMemcpyAsync(ctx->E, E, (size_t)n * d * sizeof(double), cudaMemcpyDeviceToDevice, s));
  else
    LAKER_CUDA(ctx, cudaMemcpyAsync(ctx->E, E, (size_t)n * d * sizeof(double), cudaMemcpyHostToDevice, s));
  LAKER_CUDA(ctx, cudaMemsetAsync(ctx->flags, 0, 2 * sizeof(unsigned long long), s));
  if (ctx->emax_len != n) {
    if (ctx->emax) cudaFree(ctx->emax);
    ctx->emax = nullptr;
    ctx->emax_len = 0;
    LAKER_CUDA(ctx, cudaMalloc(&ctx->emax, (size_t)n * sizeof(double)));
    ctx->emax_len = n;
  }
  laker::launch_rowabsmax(ctx->E, n, d, ctx->emax, s);
  // digit slices of E for the tcgen05 QK^T paths (FAST assembly, on-the-fly operator,
  // predict); those paths use a branch-free exp, so they are enabled only when
  // scale max ||e_i||^2 (a Cauchy-Schwarz bound of every argument) cannot overflow
  ctx->ozE_valid = false;
  if (d <= 128) {
    double mx2 = 0.0;
    LAKER_CUDA(ctx, laker::max_rownorm2(ctx->E, n, d, &mx2, s));
    const char *tcenv = std::getenv("LAKER_OTF_TC");
    if (std::fabs(scale) * mx2 < 700.0 && !(tcenv && tcenv[0] == '0') &&
        laker::oz_slices_make(ctx->ozE, ctx->E, n, d, 7, s) == cudaSuccess)
      ctx->ozE_valid = true;
    const int64_t cfl = (n + 127) / 128 * 128;
    if (ctx->ozE_valid && ctx->cf_len != cfl) {
      if (ctx->cf) cudaFree(ctx->cf);
      ctx->cf = nullptr;
      ctx->cf_len = 0;
      LAKER_CUDA(ctx, cudaMalloc(&ctx->cf, (size_t)cfl * sizeof(double2)));
      ctx->cf_len = cfl;
    }
    ctx->stats.kernel_launches += 3;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  if (storage == LAKER_STORE_MATERIALIZED) {
    if (!ctx->K) {
      LAKER_CUDA(ctx, cudaMalloc(&ctx->K, k_bytes));
      ctx->K_bytes = k_bytes;
    }
    LAKER_CUDA(ctx, cudaMemsetAsync(ctx->K, 0, (size_t)rows * ctx->ld * sizeof(double), s));
    const bool whole = (rows == n);
    if (mode == LAKER_MODE_EXACT) {
      if (whole)
        laker::launch_assemble_exact_sym(ctx->E, n, d, scale, ctx->K, ctx->ld, ctx->flags, ctx->emax, s);
      else
        laker::launch_assemble_exact_rows(ctx->E, n, d, scale, ctx->r0, ctx->r1, ctx->K, ctx->ld, ctx->flags,
                                          ctx->emax, s);
    } else {
      laker::launch_assemble_fast(ctx->E, n, d, scale, ctx->r0, ctx->r1, ctx->K, ctx->ld, ctx->flags, s);
    }
    ctx->stats.kernel_launches++;
    LAKER_CUDA(ctx, cudaGetLastError());
  }
  cudaEventRecord(e1, s);
  unsigned long long hf[2] = {0, 0};
  LAKER_CUDA(ctx, cudaMemcpyAsync(hf, ctx->flags, sizeof(hf), cudaMemcpyDeviceToHost, s));
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->stats.assemble_ms = ms;
  ctx->stats.exp_inconclusive += hf[0];
  ctx->stats.exp_overflow += hf[1];
  ctx->assembled = true;
  LAKER_CUDA(ctx, laker::otf_sym_prepare(ctx));
  if (hf[1] > 0) return set_err(ctx, LAKER_ERR_OVERFLOW, "scale*<e_i,e_j> exceeded ln(DBL_MAX)");
  LAKER_TRY(laker::refresh_symmetry(ctx, 0, mode == LAKER_MODE_EXACT));
  return LAKER_OK;
}

laker_status laker_fit_preconditioner(laker_ctx ctx, const laker_fit_opts *opts, laker_fit_report *report) {
  CHECK_CTX(ctx);
  if (!opts) return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "fit: opts is NULL");
  if (!ctx->assembled) return set_err(ctx, LAKER_ERR_NOT_READY, "fit: assemble the kernel first");
  cudaSetDevice(ctx->device);
  if (report) std::memset(report, 0, sizeof(*report));
  switch (opts->kind) {
    case LAKER_PRECOND_NONE:
      free_dev(ctx, ctx->P);
      laker::free_factors(ctx);
      ctx->p_sym = false;
      ctx->precond_kind = LAKER_PRECOND_NONE;
      return LAKER_OK;
    case LAKER_PRECOND_JACOBI:
      laker::free_factors(ctx);
      LAKER_TRY(ensure_jacobi(ctx));
      ctx->precond_kind = LAKER_PRECOND_JACOBI;
      LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
      return LAKER_OK;
    case LAKER_PRECOND_LEARNED:
      if (ctx->world > 1 && !ctx->comm)
        return set_err(ctx, LAKER_ERR_NOT_READY, "fit: detached shard (no NCCL communicator)");
      {
        ctx->p_sym = false;
        if (opts->p_layout < LAKER_P_AUTO || opts->p_layout > LAKER_P_FACTORED_QM)
          return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "fit: bad p_layout");
        laker_status st = laker::fit_learned(ctx, *opts, report);
        if (st != LAKER_OK) return st;
        LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        return ctx->p_factored ? LAKER_OK : laker::refresh_symmetry(ctx, 1);
      }
    default:
      return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "fit: unknown kind");
  }
}

laker_status laker_block_cg_solve(laker_ctx ctx, int32_t nrhs, int32_t block, const double *Y, double *alpha,
                                  const laker_solve_opts *opts, laker_solve_report *reports, double *history) {
  CHECK_CTX(ctx);
  if (!ctx->assembled) return set_err(ctx, LAKER_ERR_NOT_READY, "block CG: assemble the kernel first");
  if (ctx->comm || ctx->world > 1) return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "block CG: one rank only");
  if (ctx->storage != LAKER_STORE_MATERIALIZED) return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "block CG needs MATERIALIZED");
  if (nrhs < 1 || nrhs > 64 || !Y || !alpha || !opts || !(opts->tol > 0.0 && opts->tol < 1.0) || opts->max_iters < 0)
    return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "block CG: need 1 <= nrhs <= 64, Y, alpha, 0 < tol < 1");
  if (block < 0 || block > nrhs || (block > 0 && nrhs % block != 0))
    return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "block CG: block must divide nrhs (0: one block of nrhs)");
  cudaSetDevice(ctx->device);
  const int64_t n = ctx->n;
  DevView yv, av;
  LAKER_TRY(view_in(ctx, Y, (size_t)n * nrhs, yv));
  LAKER_TRY(view_out(ctx, alpha, (size_t)n * nrhs, av));
  laker_status sb = laker::pcg_solve_block(ctx, nrhs, yv.dptr, av.dptr, *opts, reports, history,
                                             block > 0 ? block : nrhs);
  if (sb == LAKER_OK || sb == LAKER_ERR_BREAKDOWN_ZERO_CURVATURE || sb == LAKER_ERR_INDEFINITE_PRECONDITIONER) {
    LAKER_TRY(flush_out(ctx, av));
    LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  }
  return sb;
}

laker_status laker_pcg_solve(laker_ctx ctx, int32_t nrhs, const double *Y, double *alpha,
                             const laker_solve_opts *opts, laker_solve_report *reports, double *history) {
  CHECK_CTX(ctx);
  if (!ctx->assembled) return set_err(ctx, LAKER_ERR_NOT_READY, "solve: assemble the kernel first");
  if (ctx->world > 1 && !ctx->comm) return set_err(ctx, LAKER_ERR_NOT_READY, "solve: detached shard (no NCCL communicator)");
  if (nrhs < 1 || !Y || !alpha || !opts || !(opts->tol > 0.0 && opts->tol < 1.0) || opts->max_iters < 0)
    return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "solve: need nrhs >= 1, Y, alpha, 0 < tol < 1");
  cudaSetDevice(ctx->device);
  const int64_t n = ctx->n;
  DevView yv, av;
  LAKER_TRY(view_in(ctx, Y, (size_t)n * nrhs, yv));
  LAKER_TRY(view_out(ctx, alpha, (size_t)n * nrhs, av));
  laker_status st = LAKER_OK;
  double total = 0.0;
  if (nrhs > 1 && !ctx->comm && ctx->storage == LAKER_STORE_MATERIALIZED && nrhs <= 256) {
    // block solve: one GEMM-shaped pass over K (and P) per iteration for all columns
    laker_status sb = laker::pcg_solve_block(ctx, nrhs, yv.dptr, av.dptr, *opts, reports, history);
    if (sb == LAKER_OK || sb == LAKER_ERR_BREAKDOWN_ZERO_CURVATURE || sb == LAKER_ERR_INDEFINITE_PRECONDITIONER) {
      LAKER_TRY(flush_out(ctx, av));
      LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    }
    return sb;
  }
  for (int32_t j = 0; j < nrhs; ++j) {
    laker_solve_report rep{};
    laker_status sj =
        ctx->comm ? laker::pcg_solve_dist(ctx, yv.dptr + (size_t)j * n, av.dptr + (size_t)j * n, *opts, &rep,
                                          j == 0 ? history : nullptr)
                  : laker::pcg_solve_device(ctx, yv.dptr + (size_t)j * n, av.dptr + (size_t)j * n, *opts, &rep,
                                            j == 0 ? history : nullptr);
    total += rep.seconds;
    if (reports) reports[j] = rep;
    if (sj != LAKER_OK && st == LAKER_OK) st = sj;
    if (sj == LAKER_ERR_CUDA || sj == LAKER_ERR_OUT_OF_MEMORY || sj == LAKER_ERR_INVALID_ARGUMENT ||
        sj == LAKER_ERR_NOT_READY)
      return sj;
  }
  ctx->stats.solve_ms = total * 1e3;
  LAKER_TRY(flush_out(ctx, av));
  LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return st;
}

laker_status laker_predict(laker_ctx ctx, int64_t m, const double *Eq, const double *alpha, double *out,
                           int mode) {
  CHECK_CTX(ctx);
  if (!ctx->assembled) return set_err(ctx, LAKER_ERR_NOT_READY, "predict: assemble the kernel first");
  if (m < 0 || (m > 0 && (!Eq || !out)) || !alpha || (mode != LAKER_MODE_FAST && mode != LAKER_MODE_EXACT))
    return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "predict: bad arguments");
  if (m == 0) return LAKER_OK;
  cudaSetDevice(ctx->device);
  const int64_t per = (m + ctx->world - 1) / ctx->world;
  const int64_t a0 = std::min<int64_t>(m, per * ctx->rank), a1 = std::min<int64_t>(m, a0 + per);
  DevView ev, alv, ov;
  LAKER_TRY(view_in(ctx, Eq, (size_t)m * ctx->d, ev));
  LAKER_TRY(view_in(ctx, alpha, (size_t)ctx->n, alv));
  LAKER_TRY(view_out(ctx, out, (size_t)m, ov));
  if (ov.hptr) {  // keep untouched rows of a host output as they were
    LAKER_CUDA(ctx, cudaMemcpyAsync(ov.dptr, out, (size_t)m * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  }
  LAKER_CUDA(ctx, cudaMemsetAsync(ctx->flags, 0, 2 * sizeof(unsigned long long), ctx->stream));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, ctx->stream);
  if (a1 > a0)
    LAKER_CUDA(ctx, laker::launch_kernel_matvec_ctx(ctx, mode, ev.dptr + a0 * ctx->d, a1 - a0, false, 0, alv.dptr,
                                                    0.0, nullptr, ov.dptr + a0, nullptr, ctx->stream));
  ctx->stats.kernel_launches++;
  LAKER_CUDA(ctx, cudaGetLastError());
  cudaEventRecord(e1, ctx->stream);
  unsigned long long hf[2] = {0, 0};
  LAKER_CUDA(ctx, cudaMemcpyAsync(hf, ctx->flags, sizeof(hf), cudaMemcpyDeviceToHost, ctx->stream));
  LAKER_TRY(flush_out(ctx, ov));
  LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->stats.predict_ms = ms;
  ctx->stats.exp_inconclusive += hf[0];
  ctx->stats.exp_overflow += hf[1];
  if (hf[1] > 0) return set_err(ctx, LAKER_ERR_OVERFLOW, "predict: exp overflow");
  return LAKER_OK;
}

laker_status laker_load_kernel_rows(laker_ctx ctx, const double *K_rows) {
  CHECK_CTX(ctx);
  if (!ctx->assembled || ctx->storage != LAKER_STORE_MATERIALIZED)
    return set_err(ctx, LAKER_ERR_NOT_READY, "load_kernel_rows: needs a materialized kernel");
  if (!K_rows) return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "load_kernel_rows: NULL");
  cudaSetDevice(ctx->device);
  const int64_t rows = ctx->r1 - ctx->r0;
  LAKER_CUDA(ctx, cudaMemcpy2DAsync(ctx->K, ctx->ld * sizeof(double), K_rows, ctx->n * sizeof(double),
                                    ctx->n * sizeof(double), rows, cudaMemcpyDefault, ctx->stream));
  LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  free_dev(ctx, ctx->Pdiag);  // Jacobi diagonal derived from E no longer matches
  if (ctx->precond_kind == LAKER_PRECOND_JACOBI) ctx->precond_kind = LAKER_PRECOND_NONE;
  return laker::refresh_symmetry(ctx, 0, false);
}

laker_status laker_get_kernel_rows(laker_ctx ctx, double *K_rows) {
  CHECK_CTX(ctx);
  if (!ctx->assembled || ctx->storage != LAKER_STORE_MATERIALIZED)
    return set_err(ctx, LAKER_ERR_NOT_READY, "get_kernel_rows: needs a materialized kernel");
  if (!K_rows) return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "get_kernel_rows: NULL");
  cudaSetDevice(ctx->device);
  const int64_t rows = ctx->r1 - ctx->r0;
  LAKER_CUDA(ctx, cudaMemcpy2DAsync(K_rows, ctx->n * sizeof(double), ctx->K, ctx->ld * sizeof(double),
                                    ctx->n * sizeof(double), rows, cudaMemcpyDefault, ctx->stream));
  LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return LAKER_OK;
}

laker_status laker_set_preconditioner(laker_ctx ctx, int kind, const double *data) {
  CHECK_CTX(ctx);
  if (!ctx->assembled) return set_err(ctx, LAKER_ERR_NOT_READY, "set_preconditioner: assemble first");
  cudaSetDevice(ctx->device);
  const int64_t rows = ctx->r1 - ctx->r0;
  if (kind != LAKER_PRECOND_NONE && kind != LAKER_PRECOND_JACOBI && kind != LAKER_PRECOND_EXTERNAL_DENSE)
    return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "set_preconditioner: kind must be NONE, JACOBI or EXTERNAL_DENSE");
  laker::free_factors(ctx);
  if (kind == LAKER_PRECOND_NONE) {
    ctx->precond_kind = kind;
    return LAKER_OK;
  }
  if (kind == LAKER_PRECOND_JACOBI) {
    if (data) {
      if (!ctx->Pdiag) LAKER_CUDA(ctx, cudaMalloc(&ctx->Pdiag, ctx->n * sizeof(double)));
      LAKER_CUDA(ctx, cudaMemcpyAsync(ctx->Pdiag, data, ctx->n * sizeof(double), cudaMemcpyDefault, ctx->stream));
    } else {
      LAKER_TRY(ensure_jacobi(ctx));
    }
    LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    ctx->precond_kind = kind;
    return LAKER_OK;
  }
  if (kind == LAKER_PRECOND_EXTERNAL_DENSE) {
    if (!data) return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "set_preconditioner: dense P rows needed");
    if (!ctx->P) {
      LAKER_CUDA(ctx, cudaMalloc(&ctx->P, (size_t)rows * ctx->ld * sizeof(double)));
      LAKER_CUDA(ctx, cudaMemsetAsync(ctx->P, 0, (size_t)rows * ctx->ld * sizeof(double), ctx->stream));
    }
    LAKER_CUDA(ctx, cudaMemcpy2DAsync(ctx->P, ctx->ld * sizeof(double), data, ctx->n * sizeof(double),
                                      ctx->n * sizeof(double), rows, cudaMemcpyDefault, ctx->stream));
    LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    ctx->precond_kind = kind;
    return laker::refresh_symmetry(ctx, 1);
  }
  return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "set_preconditioner: kind must be NONE, JACOBI or EXTERNAL_DENSE");
}

laker_status laker_get_preconditioner_rows(laker_ctx ctx, double *P_rows) {
  CHECK_CTX(ctx);
  if (!ctx->P && !ctx->p_factored) return set_err(ctx, LAKER_ERR_NOT_READY, "no dense preconditioner");
  if (!P_rows) return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "NULL");
  cudaSetDevice(ctx->device);
  LAKER_TRY(laker::ensure_dense_p(ctx));  // factored P: the rows are formed from the factors
  const int64_t rows = ctx->r1 - ctx->r0;
  LAKER_CUDA(ctx, cudaMemcpy2DAsync(P_rows, ctx->n * sizeof(double), ctx->P, ctx->ld * sizeof(double),
                                    ctx->n * sizeof(double), rows, cudaMemcpyDefault, ctx->stream));
  LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return LAKER_OK;
}

laker_status laker_get_preconditioner_factors(laker_ctx ctx, double *Q, double *M, double *a_inv_sqrt) {
  CHECK_CTX(ctx);
  if (!ctx->p_factored) return set_err(ctx, LAKER_ERR_NOT_READY, "no factored preconditioner");
  cudaSetDevice(ctx->device);
  const int64_t n = ctx->f_local ? ctx->r1 - ctx->r0 : ctx->n, nr = ctx->f_nr;  // sharded: own rows of Q
  if (Q)
    LAKER_CUDA(ctx, cudaMemcpy2DAsync(Q, nr * sizeof(double), ctx->Qr, ctx->f_ldq * sizeof(double),
                                      nr * sizeof(double), n, cudaMemcpyDefault, ctx->stream));
  if (M)
    LAKER_CUDA(ctx, cudaMemcpy2DAsync(M, nr * sizeof(double), ctx->Mf, ctx->f_ldq * sizeof(double),
                                      nr * sizeof(double), nr, cudaMemcpyDefault, ctx->stream));
  if (a_inv_sqrt) *a_inv_sqrt = ctx->f_ainv;
  LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return LAKER_OK;
}

laker_status laker_apply_operator(laker_ctx ctx, const double *x, double *y) {
  CHECK_CTX(ctx);
  if (!ctx->assembled) return set_err(ctx, LAKER_ERR_NOT_READY, "apply: assemble first");
  if (ctx->world > 1 && !ctx->comm) return set_err(ctx, LAKER_ERR_NOT_READY, "apply: detached shard (no NCCL communicator)");
  if (!x || !y) return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "apply: NULL");
  cudaSetDevice(ctx->device);
  DevView xv, yv;
  LAKER_TRY(view_in(ctx, x, (size_t)ctx->n, xv));
  LAKER_TRY(view_out(ctx, y, (size_t)ctx->n, yv));
  if (ctx->comm)
    LAKER_TRY(laker::apply_operator_dist(ctx, xv.dptr, yv.dptr));
  else
    LAKER_TRY(laker::apply_operator_device(ctx, xv.dptr, yv.dptr));
  LAKER_TRY(flush_out(ctx, yv));
  LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return LAKER_OK;
}

laker_status laker_get_preconditioner_qm(laker_ctx ctx, double *QM) {
  CHECK_CTX(ctx);
  if (!ctx->p_factored || !ctx->p_qm) return set_err(ctx, LAKER_ERR_NOT_READY, "no QM-form factored preconditioner");
  if (!QM) return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "get_preconditioner_qm: NULL");
  cudaSetDevice(ctx->device);
  const int64_t n = ctx->f_local ? ctx->r1 - ctx->r0 : ctx->n, nr = ctx->f_nr;  // sharded: own rows of QM
  LAKER_CUDA(ctx, cudaMemcpy2DAsync(QM, nr * sizeof(double), ctx->QMf, ctx->f_ldq * sizeof(double),
                                    nr * sizeof(double), n, cudaMemcpyDefault, ctx->stream));
  LAKER_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return LAKER_OK;
}

laker_status laker_get_stats(laker_ctx ctx, laker_stats *out) {
  CHECK_CTX(ctx);
  if (!out) return LAKER_ERR_INVALID_ARGUMENT;
  ctx->stats.n = ctx->n;
  ctx->stats.local_rows = ctx->r1 - ctx->r0;
  ctx->stats.ld = ctx->ld;
  ctx->stats.rank = ctx->rank;
  ctx->stats.world = ctx->world;
  ctx->stats.precond_kind = ctx->precond_kind;
  ctx->stats.storage = ctx->storage;
  ctx->stats.mode = ctx->mode;
  ctx->stats.symmetric_k = ctx->k_sym ? 1 : 0;
  ctx->stats.k_tensor_core = ctx->k_sym && ctx->k_tc ? 1 : 0;
  ctx->stats.symmetric_p = ctx->p_sym ? 1 : 0;
  ctx->stats.p_factored = ctx->p_factored ? (ctx->p_qm ? 2 : 1) : 0;
  ctx->stats.n_dirs = (int32_t)ctx->f_nr;
  *out = ctx->stats;
  return LAKER_OK;
}

}  // extern "C"
