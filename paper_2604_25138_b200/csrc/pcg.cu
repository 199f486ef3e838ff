// Preconditioned conjugate gradient, Alg. 1 l.15-22,
// run entirely on the device.  One iteration is
//   (a) q = (lambda I + K) p               -- gemv.cu (epilogue: delta = rho / p.q)
//   (b) alpha += delta p ; r -= delta q    -- update kernel (epilogue: ||r||/||y||,
//       termination test; for P = I / Jacobi also theta and beta)
//   (c) theta = P r                        -- gemv.cu on the dense P (epilogue: beta)
//   (d) p = theta + beta p                 -- update kernel
// with every inner product a Dot2 reduction (fixed-order last-CTA epilogues)
// and every vector update a single fma (R17), i.e. the same IEEE operations as
// the oracle's orc_pcg.  Scalars live in a device PcgState; a kernel that finds
// state->done set returns at once, so `chunk` iterations are captured into one
// CUDA graph and the host only polls the state between graph launches.


#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "pcg_kernels.cuh"

namespace laker {

// extreme eigenvalues of the Lanczos tridiagonal of k CG steps (delta_0..k-1,
// beta_0..k-2) by Sturm-sequence bisection
void lanczos_extremes(const std::vector<double> &dl, const std::vector<double> &bt, int k, double &lmin,
                      double &lmax) {
  lmin = lmax = 0.0;
  if (k <= 0) return;
  std::vector<double> a(k), b2(k > 1 ? k - 1 : 1, 0.0);
  for (int j = 0; j < k; ++j) a[j] = 1.0 / dl[j] + (j > 0 ? bt[j - 1] / dl[j - 1] : 0.0);
  for (int j = 0; j + 1 < k; ++j) b2[j] = bt[j] / (dl[j] * dl[j]);  // (sqrt(beta_j)/delta_j)^2
  double lo = INFINITY, hi = -INFINITY;
  for (int j = 0; j < k; ++j) {
    const double r = (j > 0 ? std::sqrt(b2[j - 1]) : 0.0) + (j + 1 < k ? std::sqrt(b2[j]) : 0.0);
    lo = std::min(lo, a[j] - r);
    hi = std::max(hi, a[j] + r);
  }
  auto count_below = [&](double x) {  // eigenvalues < x
    int c = 0;
    double q = a[0] - x;
    if (q < 0) ++c;
    for (int j = 1; j < k; ++j) {
      if (q == 0.0) q = 1e-300;
      q = (a[j] - x) - b2[j - 1] / q;
      if (q < 0) ++c;
    }
    return c;
  };
  auto kth = [&](int idx) {  // idx-th smallest (0-based)
    double l = lo, h = hi;
    for (int it = 0; it < 200 && h - l > 1e-15 * std::max(std::fabs(l), std::fabs(h)); ++it) {
      const double mid = 0.5 * (l + h);
      if (count_below(mid) > idx) h = mid; else l = mid;
    }
    return 0.5 * (l + h);
  };
  lmin = kth(0);
  lmax = kth(k - 1);
}

// The operator apply used by the solver: q = (lambda I + K) p.
static void launch_operator(laker_ctx ctx, const double *p, double *q, PcgState *st, int epi, double *dot_out,
                            const double *pmax = nullptr, int npmax = 0, const FusedUpdate *upd = nullptr) {
  if (ctx->storage == LAKER_STORE_MATERIALIZED) {
    GemvArgs a{};
    a.A = ctx->K;
    a.ld = ctx->ld;
    a.rows = ctx->r1 - ctx->r0;
    a.ncols = ctx->n;
    a.x = p;
    a.row0 = ctx->r0;
    a.y = q;
    a.lambda = ctx->lambda;
    a.state = st;
    a.partials = ctx->partials;
    a.counter = ctx->counters + kCtrGemv;
    a.dot_out = dot_out;
    a.epi = epi;
    a.evict_first = true;
    if (ctx->k_sym) {
      a.xparts = pmax;
      a.nxparts = npmax;
      if (upd) a.upd = *upd;
      a.tc = ctx->k_tc ? ctx->symv_tc : nullptr;
      launch_symv(ctx->symv, 0, a, ctx->stream);
      ctx->stats.kernel_launches++;
    } else {
      launch_gemv(a, ctx->gemv_grid, ctx->stream);
    }
  } else if (launch_operator_otf_sym(ctx, p, q, st, epi, dot_out, ctx->stream)) {
    ctx->stats.kernel_launches++;  // tile kernel + finalize (with the epilogue)
  } else {
    launch_kernel_matvec_ctx(ctx, ctx->mode, ctx->E + ctx->r0 * ctx->d, ctx->r1 - ctx->r0, true, ctx->r0, p,
                             ctx->lambda, p + ctx->r0, q, st ? &st->done : nullptr, ctx->stream);
    if (epi == kEpiDelta) {
      const int g = (int)std::min<int64_t>(2 * ctx->num_sms, (ctx->n + kVecThreads - 1) / kVecThreads);
      dot_delta_kernel<<<g, kVecThreads, 0, ctx->stream>>>(ctx->n, p, q, st, ctx->partials,
                                                          ctx->counters + kCtrMisc);
      ctx->stats.kernel_launches++;
    }
  }
  ctx->stats.kernel_launches++;
}

// pu_p != null (epi = kEpiBeta, factored P): the last pass also forms p = theta + beta p
// (gemv.cu fused direction update) and the per-CTA max |p| into pu_pmax
static void launch_precond(laker_ctx ctx, const double *r, double *theta, PcgState *st, int epi, double *dot_out,
                           double *pu_p = nullptr, double *pu_pmax = nullptr) {
  if (ctx->p_factored) {
    // theta = a^{-1/2} r + Q (M (Q^T r)): three Dot2 GEMV passes (NEXT-1); the last
    // one carries the a^{-1/2} r_i term and the r.theta epilogue
    const int64_t nrp = ctx->f_nrp, ldq = ctx->f_ldq;
    GemvArgs z{};
    z.A = ctx->Qt; z.ld = ctx->ld; z.rows = nrp; z.ncols = ctx->n; z.x = r; z.row0 = 0; z.y = ctx->fz;
    z.state = st; z.partials = ctx->partials; z.counter = ctx->counters + kCtrGemv; z.epi = kEpiNone;
    z.evict_first = true;
    launch_gemv(z, ctx->gemv_grid, ctx->stream);
    if (ctx->p_qm) {  // R21: theta = a^-1/2 r + QM z
      GemvArgs t = z;
      t.A = ctx->QMf + ctx->r0 * ldq; t.ld = ldq; t.rows = ctx->r1 - ctx->r0; t.ncols = nrp; t.x = ctx->fz;
      t.row0 = ctx->r0; t.y = theta; t.lambda = ctx->f_ainv; t.xd = r; t.epi = epi; t.dot_out = dot_out;
      t.pu_p = pu_p; t.pu_pmax = pu_pmax; t.pu_budget = 1; t.pu_bar = ctx->counters + kCtrBar;
      launch_gemv(t, ctx->gemv_grid, ctx->stream);
      ctx->stats.kernel_launches += 2;
      return;
    }
    GemvArgs w = z;
    w.A = ctx->Mf; w.ld = ldq; w.rows = nrp; w.ncols = nrp; w.x = ctx->fz; w.y = ctx->fw;
    w.evict_first = false;  // keep M in L2 across iterations
    launch_gemv(w, ctx->gemv_grid, ctx->stream);
    GemvArgs t = z;
    t.A = ctx->Qr + ctx->r0 * ldq; t.ld = ldq; t.rows = ctx->r1 - ctx->r0; t.ncols = nrp; t.x = ctx->fw; t.row0 = ctx->r0;
    t.y = theta; t.lambda = ctx->f_ainv; t.xd = r; t.epi = epi; t.dot_out = dot_out;
    t.pu_p = pu_p; t.pu_pmax = pu_pmax; t.pu_budget = 1; t.pu_bar = ctx->counters + kCtrBar;
    launch_gemv(t, ctx->gemv_grid, ctx->stream);
    ctx->stats.kernel_launches += 3;
    return;
  }
  GemvArgs a{};
  a.A = ctx->P;
  a.ld = ctx->ld;
  a.rows = ctx->r1 - ctx->r0;
  a.ncols = ctx->n;
  a.x = r;
  a.row0 = ctx->r0;
  a.y = theta;
  a.lambda = 0.0;
  a.state = st;
  a.partials = ctx->partials;
  a.counter = ctx->counters + kCtrGemv;
  a.dot_out = dot_out;
  a.epi = epi;
  a.evict_first = true;
  if (ctx->p_sym) {
    launch_symv(ctx->symv, 1, a, ctx->stream);
    ctx->stats.kernel_launches++;
  } else {
    launch_gemv(a, ctx->gemv_grid, ctx->stream);
  }
  ctx->stats.kernel_launches++;
}

laker_status apply_operator_device(laker_ctx ctx, const double *x, double *y) {
  // x must be padded to ld with zeros: stage it.
  double *xp = nullptr;
  LAKER_CUDA(ctx, cudaMallocAsync(&xp, ctx->ld * sizeof(double), ctx->stream));
  LAKER_CUDA(ctx, cudaMemsetAsync(xp, 0, ctx->ld * sizeof(double), ctx->stream));
  LAKER_CUDA(ctx, cudaMemcpyAsync(xp, x, ctx->n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  launch_operator(ctx, xp, y + ctx->r0, nullptr, kEpiNone, nullptr);
  LAKER_CUDA(ctx, cudaGetLastError());
  LAKER_CUDA(ctx, cudaFreeAsync(xp, ctx->stream));
  return LAKER_OK;
}

laker_status pcg_solve_device(laker_ctx ctx, const double *y, double *alpha_out, const laker_solve_opts &o,
                              laker_solve_report *rep, double *history) {
  if (ctx->world != 1) return set_err(ctx, LAKER_ERR_INVALID_ARGUMENT, "multi-rank PCG not built in this version");
  const bool tdbg = std::getenv("LAKER_DEBUG_SOLVE") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  auto tmark = [&](const char *what) {
    if (!tdbg) return;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    std::fprintf(stderr, "[solve] %-14s %9.3f ms\n", what, ms);
  };
  const int64_t n = ctx->n, ld = ctx->ld;
  const int pk = ctx->precond_kind;
  const bool dense = (pk == LAKER_PRECOND_LEARNED || pk == LAKER_PRECOND_EXTERNAL_DENSE);
  if (dense && !ctx->P && !ctx->p_factored) return set_err(ctx, LAKER_ERR_NOT_READY, "dense preconditioner not set");
  if (pk == LAKER_PRECOND_JACOBI && !ctx->Pdiag) return set_err(ctx, LAKER_ERR_NOT_READY, "Jacobi diagonal not set");
  const int32_t max_iters = o.max_iters > 0 ? o.max_iters : (int32_t)std::min<int64_t>(10 * n, 1 << 30);
  cudaStream_t s = ctx->stream;

  Workspace w;
  const size_t vb = (size_t)ld * sizeof(double);
  LAKER_CUDA(ctx, cudaMallocAsync(&w.alpha, 6 * vb + (2 + 256) * sizeof(double), s));
  w.r = w.alpha + ld;
  w.theta = w.r + ld;
  w.p = w.theta + ld;
  w.q = w.p + ld;
  w.y = w.q + ld;
  w.scal = w.y + ld;
  double *pmax = w.scal + 2;  // per-CTA max |p| from the vector kernels (vg <= 148 entries), for symv
  LAKER_CUDA(ctx, cudaMemsetAsync(w.alpha, 0, 6 * vb + (2 + 256) * sizeof(double), s));
  LAKER_CUDA(ctx, cudaMallocAsync(&w.hist, (size_t)3 * max_iters * sizeof(double), s));
  double *dh = w.hist + max_iters, *bh = dh + max_iters;  // CG coefficients (Lanczos estimates)
  LAKER_CUDA(ctx, cudaMallocAsync(&w.st, sizeof(PcgState), s));
  LAKER_CUDA(ctx, cudaMemcpyAsync(w.y, y, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  PcgState h0{};
  h0.tol = o.tol;
  h0.max_iters = max_iters;
  h0.dh = dh;
  h0.bh = bh;
  LAKER_CUDA(ctx, cudaMemcpyAsync(w.st, &h0, sizeof(PcgState), cudaMemcpyHostToDevice, s));

  // vector kernels: ~4 elements per thread (n = 16384 -> 16 CTAs) keeps the last-CTA reduction short
  const int vg = (int)std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms, (n + 4 * kVecThreads - 1) / (4 * kVecThreads)));
  cudaEvent_t ev0, ev1;
  cudaEventCreate(&ev0);
  cudaEventCreate(&ev1);
  cudaEventRecord(ev0, s);
  tmark("ev0");

  pcg_init_kernel<<<vg, kVecThreads, 0, s>>>(n, w.y, w.alpha, w.r, w.st, ctx->partials, ctx->counters + kCtrInit);
  if (dense) launch_precond(ctx, w.r, w.theta, w.st, kEpiStoreDot, &w.st->rho);
  pcg_first_dir_kernel<<<vg, kVecThreads, 0, s>>>(n, pk, ctx->Pdiag, w.r, w.theta, w.p, w.st, ctx->partials,
                                                  ctx->counters + kCtrInit, pmax);
  ctx->stats.kernel_launches += 2;
  LAKER_CUDA(ctx, cudaGetLastError());

  const double *theta_src = (pk == LAKER_PRECOND_NONE) ? w.r : w.theta;
  // iterations per captured graph (32 per chunk at C3 measured the same as 8, tools/iter_gap.py)
  const int chunk = n >= 8192 ? 8 : (n >= 2048 ? 32 : 64);
  const bool instr = o.instrument != 0;
  std::vector<cudaEvent_t> evs;
  // instrumented: two event sets, one per captured graph, so the speculative loop below
  // reads a finished chunk's events while the next chunk (the other graph) runs
  const int nsets = instr ? 2 : 1;
  if (instr) {
    evs.resize(4 * chunk * nsets);
    for (auto &e : evs) cudaEventCreate(&e);
  }
  // the update step (alpha, r, ||r||, termination) rides in the symmetric apply's finalize
  // (a grid barrier for delta instead of a kernel boundary; symv.cu)
  const bool fuse_upd = ctx->k_sym && ctx->storage == LAKER_STORE_MATERIALIZED;
  // the direction update rides in the factored preconditioner's last pass (gemv.cu)
  const bool fuse_pu = dense && ctx->p_factored;
  // symv offsets: max |p| over the per-CTA maxima of whichever kernel formed p last
  // (pcg_first_dir_kernel: vg CTAs at init, the fused pass: <= gemv_grid CTAs; pmax is
  // zeroed at solve start, vg <= that grid)
  const int npmax = fuse_pu ? std::max(vg, ctx->gemv_grid) : vg;
  FusedUpdate fu{};
  fu.on = 1; fu.pk = pk; fu.p = w.p; fu.alpha = w.alpha; fu.r = w.r; fu.theta = w.theta; fu.dvec = ctx->Pdiag;
  fu.hist = w.hist; fu.bar = ctx->counters + kCtrBar; fu.partials2 = ctx->partials + 2048;
  fu.counter2 = ctx->counters + kCtrUpdate;
  auto record_iteration = [&](int j, int set) {
    cudaEvent_t *ev = instr ? &evs[4 * (set * chunk + j)] : nullptr;
    if (instr) cudaEventRecordWithFlags(ev[0], s, cudaEventRecordExternal);
    launch_operator(ctx, w.p, w.q, w.st, kEpiDelta, nullptr, pmax, npmax, fuse_upd ? &fu : nullptr);
    if (instr) cudaEventRecordWithFlags(ev[1], s, cudaEventRecordExternal);
    if (!fuse_upd)
      pcg_update_kernel<<<dim3(vg), dim3(kVecThreads), 0, s>>>(n, pk, (const double *)ctx->Pdiag, (const double *)w.p, (const double *)w.q, w.alpha, w.r, w.theta, w.st, w.hist, ctx->partials, ctx->counters + kCtrUpdate);
    if (dense) {
      if (instr) cudaEventRecordWithFlags(ev[2], s, cudaEventRecordExternal);
      launch_precond(ctx, w.r, w.theta, w.st, kEpiBeta, nullptr, fuse_pu ? w.p : nullptr, fuse_pu ? pmax : nullptr);
      if (instr) cudaEventRecordWithFlags(ev[3], s, cudaEventRecordExternal);
    }
    if (!fuse_pu) {
      pcg_pupdate_kernel<<<dim3(vg), dim3(kVecThreads), 0, s>>>(n, theta_src, w.p, w.st, dense ? 1 : 0, pmax);
      ctx->stats.kernel_launches++;
    }
    if (!fuse_upd) ctx->stats.kernel_launches++;
  };

  // capture one chunk into a graph (two when instrumented: one per event set)
  cudaGraph_t graph[2] = {nullptr, nullptr};
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  const int64_t launches_before = ctx->stats.kernel_launches;
  int64_t per_chunk = 0;
  for (int set = 0; set < nsets; ++set) {
    LAKER_CUDA(ctx, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int j = 0; j < chunk; ++j) record_iteration(j, set);
    LAKER_CUDA(ctx, cudaStreamEndCapture(s, &graph[set]));
    per_chunk = (ctx->stats.kernel_launches - launches_before) / (set + 1);
    LAKER_CUDA(ctx, cudaGraphInstantiate(&gexec[set], graph[set], 0));
  }
  ctx->stats.kernel_launches = launches_before;
  tmark("instantiated");

  // One chunk is always queued ahead of the host's check of the previous one, so the
  // GPU never idles for the state read-back + relaunch; a chunk queued after the solve
  // finished runs as early-exiting no-op kernels (every kernel tests st->done).  The
  // instrumented run alternates its two graphs and reads each finished chunk's events
  // while the next one runs.
  PcgState *hs = nullptr, *hs2 = nullptr;
  LAKER_CUDA(ctx, cudaMallocHost(&hs, 2 * sizeof(PcgState)));
  hs2 = hs + 1;
  LAKER_CUDA(ctx, cudaMemcpyAsync(hs, w.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  int32_t iters_prev = hs->iters;
  auto read_events = [&](int set, const PcgState *st_after) {
    const int ran = st_after->iters - iters_prev;  // iterations whose operator pass did real work
    for (int j = 0; j < std::min(ran, chunk); ++j) {
      const cudaEvent_t *ev = &evs[4 * (set * chunk + j)];
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[0], ev[1]);
      ctx->stats.op_ms += ms;
      ctx->stats.op_launches++;
      if (dense && (j < ran - 1 || !st_after->done || st_after->term != LAKER_TERM_RESIDUAL_TOL)) {
        cudaEventElapsedTime(&ms, ev[2], ev[3]);
        ctx->stats.prec_ms += ms;
        ctx->stats.prec_launches++;
      }
    }
    iters_prev = st_after->iters;
  };
  if (!hs->done) {
    cudaEvent_t ce[2];
    cudaEventCreateWithFlags(&ce[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ce[1], cudaEventDisableTiming);
    PcgState *slot[2] = {hs, hs2};
    int cur = 0;
    LAKER_CUDA(ctx, cudaGraphLaunch(gexec[0], s));
    ctx->stats.kernel_launches += per_chunk;
    LAKER_CUDA(ctx, cudaMemcpyAsync(slot[0], w.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    cudaEventRecord(ce[0], s);
    for (;;) {
      LAKER_CUDA(ctx, cudaGraphLaunch(gexec[(cur ^ 1) % nsets], s));  // speculative next chunk
      ctx->stats.kernel_launches += per_chunk;
      LAKER_CUDA(ctx, cudaMemcpyAsync(slot[cur ^ 1], w.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
      cudaEventRecord(ce[cur ^ 1], s);
      LAKER_CUDA(ctx, cudaEventSynchronize(ce[cur]));
      if (instr) read_events(cur, slot[cur]);
      if (slot[cur]->done) break;
      cur ^= 1;
    }
    LAKER_CUDA(ctx, cudaStreamSynchronize(s));
    *hs = *slot[cur ^ 1];  // the state after the last queued chunk (== final state)
    cudaEventDestroy(ce[0]);
    cudaEventDestroy(ce[1]);
  }
  cudaEventRecord(ev1, s);
  tmark("loop done");

  // true residual (one extra operator apply, outside the timed loop)
  launch_operator(ctx, w.alpha, w.q, nullptr, kEpiNone, nullptr);
  true_residual_kernel<<<vg, kVecThreads, 0, s>>>(n, w.y, w.q, w.st, w.scal, ctx->partials,
                                                  ctx->counters + kCtrMisc);
  ctx->stats.kernel_launches++;
  LAKER_CUDA(ctx, cudaMemcpyAsync(alpha_out, w.alpha, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  double true_rel = 0.0;
  LAKER_CUDA(ctx, cudaMemcpyAsync(&true_rel, w.scal, sizeof(double), cudaMemcpyDeviceToHost, s));
  LAKER_CUDA(ctx, cudaMemcpyAsync(hs, w.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
  if (history && hs->iters > 0) {
    LAKER_CUDA(ctx, cudaStreamSynchronize(s));
    LAKER_CUDA(ctx, cudaMemcpyAsync(history, w.hist, (size_t)hs->iters * sizeof(double), cudaMemcpyDeviceToHost, s));
  }
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev0, ev1);
  ctx->stats.solve_ms = ms;
  tmark("post sync");
  if (rep && hs->iters > 0) {
    std::vector<double> hd(hs->iters), hb(hs->iters);
    cudaMemcpy(hd.data(), dh, hs->iters * sizeof(double), cudaMemcpyDeviceToHost);
    cudaMemcpy(hb.data(), bh, hs->iters * sizeof(double), cudaMemcpyDeviceToHost);
    lanczos_extremes(hd, hb, hs->iters, rep->lanczos_lmin, rep->lanczos_lmax);
  }
  if (rep) {
    rep->iters = hs->iters;
    rep->termination = hs->term;
    rep->rel_residual = hs->iters > 0 ? hs->rel : (hs->term == LAKER_TERM_ZERO_RHS ? 0.0 : 1.0);
    rep->true_rel_residual = true_rel;
    rep->seconds = ms * 1e-3;
  }
  const int term = hs->term;
  tmark("lanczos");
  cudaFreeHost(hs);
  for (auto &e : evs) cudaEventDestroy(e);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  for (int set = 0; set < nsets; ++set) {
    cudaGraphExecDestroy(gexec[set]);
    cudaGraphDestroy(graph[set]);
  }
  cudaFreeAsync(w.alpha, s);
  cudaFreeAsync(w.hist, s);
  tmark("destroyed");
  cudaFreeAsync(w.st, s);
  LAKER_CUDA(ctx, cudaStreamSynchronize(s));
  if (term == LAKER_TERM_BREAKDOWN) return set_err(ctx, LAKER_ERR_BREAKDOWN_ZERO_CURVATURE, "p.(lambda I + K)p <= 0");
  if (term == LAKER_TERM_INDEFINITE) return set_err(ctx, LAKER_ERR_INDEFINITE_PRECONDITIONER, "r.theta <= 0");
  return LAKER_OK;
}

}  // namespace laker
