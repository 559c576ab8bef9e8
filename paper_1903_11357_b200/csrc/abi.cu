// abi.cu — the remaining C-ABI entry points (include/dgas.h): rhs, spmv, apply, pcg (device-resident
// loop: one CUDA graph whose WHILE conditional node runs PCG iterations until the device-side
// convergence test clears the condition), info, history, diagnostics.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>

#include "internal.h"

// Local-solve kernel choice and the panel kernel's launch geometry (local_panel.cu). Shared memory
// per CTA leaves room for one coarse-solve CTA per SM (the coarse chain runs concurrently on a side
// stream).
static int panel_configure(dgas_ctx ctx) {
  const bool ok = panel_supported(ctx->p) && ctx->max_sub_cells > 1;
  ctx->local_kernel = ok ? 2 : 1;
  if (const char* e = std::getenv("DGAS_LOCAL_KERNEL")) {
    const int v = std::atoi(e);
    if (v == 1 || (v == 2 && ok)) ctx->local_kernel = v;
  }
  if (ctx->local_kernel != 2) return 0;
  int dev = 0, nsm = 148, smem_sm = 233472, optin = 232448;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // CTAs per SM: the fewest that hold every subdomain in one wave, with 256 consumer threads per
  // subdomain (short chain steps) up to 3 per SM; beyond that the kernel is HBM-bound and runs 7
  // 128-thread CTAs per SM (measured on B200, tools/ab.sh: cfg4 local 0.361 -> 0.336 ms, cfg3
  // 0.562 -> 0.462 ms against the envelope kernel; 1-3 CTAs/SM with L2 reuse of the backward sweep
  // are latency-bound, 0.78-0.90 ms)
  int cps = (ctx->nsub + nsm - 1) / nsm;
  if (cps > 3) cps = 7;
  if (const char* e = std::getenv("DGAS_LOCAL_CPS")) cps = std::max(1, std::min(8, std::atoi(e)));  // tests, sweeps
  ctx->panel_cps = cps;
  size_t reserve = 8 * 1024;
  if (ctx->coarse_mode == 2) reserve += (size_t)std::max(ctx->nd.maxN, ctx->nd.maxF + ctx->nd.maxU) * 8 + 1024;
  size_t per_cta = ((size_t)smem_sm - std::min((size_t)smem_sm / 2, reserve)) / cps - 1024;
  per_cta = std::min(per_cta, (size_t)optin);
  const size_t base = panel_base_bytes(ctx->max_sub_cells, ctx->np, cps > 3) + 128;
  // ring: S (a power of two) slots of about `target` bytes that together fill the budget; CC columns
  // per slot (even, at least panel_min_cc, at most the widest panel)
  size_t target = 8 * 1024;
  if (const char* e = std::getenv("DGAS_PANEL_SLOT_KB")) target = (size_t)std::atoi(e) * 1024;
  const int maxW = ctx->max_urow + ctx->np;
  if (const char* e = std::getenv("DGAS_PANEL_F32")) ctx->panel_f32 = std::atoi(e) != 0;
  const int al = panel_al(ctx->panel_f32), esz = ctx->panel_f32 ? 4 : 8;
  const int cc_min = panel_min_cc(ctx->np, ctx->panel_f32), cc_max = std::max(cc_min, (maxW + al - 1) / al * al);
  ctx->panel_slots = 0;
  if (per_cta > base) {
    const size_t B = per_cta - base;
    int S = 2;
    while (S < 64 && B / (2 * S) >= target) S *= 2;
    for (; S >= 2; S /= 2) {
      int CC = (int)std::min<size_t>(cc_max, (B / S) / (esz * ctx->np)) / al * al;
      if (CC < cc_min) continue;
      const uint32_t sb = (uint32_t)(((((int64_t)CC * ctx->np + al - 1) / al * al) * esz + 127) / 128 * 128);
      while (S < 64 && (size_t)2 * S * sb <= B) S *= 2;  // CC capped at the widest panel: more slots
      ctx->panel_slots = S;
      ctx->panel_slot_bytes = sb;
      ctx->panel_cc = CC;
      break;
    }
  }
  if (ctx->panel_slots < 2) { ctx->local_kernel = 1; return 0; }  // subdomain too large: envelope kernel
  ctx->panel_keep = 1;
  if (const char* e = std::getenv("DGAS_PANEL_KEEP")) ctx->panel_keep = std::atoi(e) != 0;
  int st = panel_setup(ctx, ctx->sub_ptr_h, ctx->first_h);
  if (st) return st;
  return panel_set_smem(ctx);
}

static int finish_setup_buffers(dgas_ctx ctx) {
  if (ctx->d_pbuf) return 0;
  double* pb[2] = {ctx->d_p[0], ctx->d_p[1]};
  DGAS_CUDA(cudaMalloc((void**)&ctx->d_r2, ctx->N * sizeof(double)));
  DGAS_CUDA(cudaMemsetAsync(ctx->d_r2, 0, ctx->N * sizeof(double), ctx->stream));
  double* rb[2] = {ctx->d_r, ctx->d_r2};
  DGAS_CUDA(cudaMalloc((void**)&ctx->d_pbuf, sizeof pb));
  DGAS_CUDA(cudaMalloc((void**)&ctx->d_rbuf, sizeof rb));
  DGAS_CUDA(cudaMemcpyAsync(ctx->d_pbuf, pb, sizeof pb, cudaMemcpyHostToDevice, ctx->stream));
  DGAS_CUDA(cudaMemcpyAsync(ctx->d_rbuf, rb, sizeof rb, cudaMemcpyHostToDevice, ctx->stream));
  DGAS_CUDA(cudaMalloc((void**)&ctx->d_perm_dev, ctx->nc * sizeof(int)));
  DGAS_CUDA(cudaMemcpyAsync(ctx->d_perm_dev, ctx->perm.data(), ctx->nc * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  DGAS_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
  DGAS_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream2, cudaStreamNonBlocking));
  int prio_lo = 0, prio_hi = 0;
  DGAS_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  for (int i = 0; i < 3; ++i) {
    // the coarse chain is latency-bound: give its fork stream the highest priority so its small
    // kernels are scheduled ahead of pending local-solve CTAs
    DGAS_CUDA(cudaStreamCreateWithPriority(&ctx->side[i], cudaStreamNonBlocking, prio_hi));
    DGAS_CUDA(cudaEventCreateWithFlags(&ctx->ev_fork[i], cudaEventDisableTiming));
    DGAS_CUDA(cudaEventCreateWithFlags(&ctx->ev_join[i], cudaEventDisableTiming));
  }
  {
    // restriction: about 4 warp steps (32 / L pieces each) per warp; 1..8 warps per coarse element in one
    // CTA, then more CTAs per coarse element (cpj) while the grid stays within the partials buffer
    const int64_t per_warp = 4 * pack_ppw(ctx->np);  // pieces per warp step (n_p lanes per piece)
    const int64_t need = (ctx->nov + ctx->ncoarse * per_warp - 1) / (ctx->ncoarse * per_warp);  // warps per J
    int w = 1;
    while (w < 8 && w < need) w *= 2;
    ctx->restrict_wpj = w;
    int64_t cpj = w == 8 ? (need + 7) / 8 : 1;
    cpj = std::min<int64_t>(cpj, std::max<int64_t>(1, ctx->partial_cap / 2 / std::max(1, ctx->ncoarse) - 1));
    cpj = std::min<int64_t>(cpj, 64);
    if (const char* e = std::getenv("DGAS_RESTRICT_CPJ")) cpj = std::max(1, std::atoi(e));
    ctx->restrict_cpj = (int)cpj;
    if (cpj > 1) {
      DGAS_CUDA(cudaMalloc((void**)&ctx->d_rpart, (size_t)ctx->ncoarse * cpj * ctx->nq * sizeof(double)));
      DGAS_CUDA(cudaMalloc((void**)&ctx->d_jcnt, (size_t)ctx->ncoarse * sizeof(unsigned)));
      DGAS_CUDA(cudaMemsetAsync(ctx->d_jcnt, 0, (size_t)ctx->ncoarse * sizeof(unsigned), ctx->stream));
    }
  }
  if (ctx->coarse_mode == 2) {
    if (const char* e = std::getenv("DGAS_ND_GRID")) ctx->nd_grid = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("DGAS_ND_L2")) ctx->nd_l2 = std::atoi(e) != 0;
    if (const char* e = std::getenv("DGAS_ND_TOL")) ctx->nd_tol = std::atof(e);
    int st2 = nd_set_smem(ctx);
    if (st2) return st2;
    if ((st2 = nd_calibrate(ctx))) return st2;
  }

  if (const char* e = std::getenv("DGAS_UNROLL")) ctx->unroll = std::max(1, std::min(8, std::atoi(e)));
  {
    // chunked restriction: pieces of each coarse element in chunks of <= 8 warp steps (32/n_p pieces
    // per step); persistent grid of 4 x 256-thread CTAs per SM
    const char* e = std::getenv("DGAS_RESTRICT");
    if (!(e && std::atoi(e) == 1)) {
      std::vector<int> cov_ptr(ctx->ncoarse + 1);
      DGAS_CUDA(cudaMemcpy(cov_ptr.data(), ctx->d_cov_ptr, (ctx->ncoarse + 1) * sizeof(int), cudaMemcpyDeviceToHost));
      int steps = 8;  // warp steps per chunk (measured: 8 vs 4: cfg3 +2.2%, cfg4 neutral; 2 slower)
      if (const char* e3 = std::getenv("DGAS_RESTRICT_STEPS")) steps = std::max(1, std::atoi(e3));
      const int per = steps * pack_ppw(ctx->np);
      std::vector<int4> ch;
      std::vector<int> jp(ctx->ncoarse + 1, 0);
      for (int J = 0; J < ctx->ncoarse; ++J) {
        // at most 64 chunks per coarse element (its last warp adds the chunk partials serially; the
        // paper regime has thousands of pieces per element)
        const int npc = cov_ptr[J + 1] - cov_ptr[J];
        const int ppw = pack_ppw(ctx->np);
        const int cs = std::max(per, (npc + 63) / 64 + ppw - 1) / ppw * ppw;
        int t = 0;
        for (int k = cov_ptr[J]; k < cov_ptr[J + 1]; k += cs, ++t)
          ch.push_back(make_int4(J, k, std::min(cov_ptr[J + 1], k + cs), t));
        jp[J + 1] = (int)ch.size();
      }
      ctx->nchunk = (int)ch.size();
      DGAS_CUDA(cudaMalloc((void**)&ctx->d_chunks, std::max<size_t>(1, ch.size()) * sizeof(int4)));
      DGAS_CUDA(cudaMemcpy(ctx->d_chunks, ch.data(), ch.size() * sizeof(int4), cudaMemcpyHostToDevice));
      DGAS_CUDA(cudaMalloc((void**)&ctx->d_jchunk_ptr, jp.size() * sizeof(int)));
      DGAS_CUDA(cudaMemcpy(ctx->d_jchunk_ptr, jp.data(), jp.size() * sizeof(int), cudaMemcpyHostToDevice));
      DGAS_CUDA(cudaMalloc((void**)&ctx->d_cpart, std::max<size_t>(1, ch.size()) * ctx->nq * sizeof(double)));
      DGAS_CUDA(cudaMalloc((void**)&ctx->d_jcnt2, ctx->ncoarse * sizeof(unsigned)));
      DGAS_CUDA(cudaMemset(ctx->d_jcnt2, 0, ctx->ncoarse * sizeof(unsigned)));
      int dev = 0, nsm = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      int per_sm = std::min(4, restrict_ctas_per_sm(ctx));  // one wave (the kernel is persistent)
      if (const char* e2 = std::getenv("DGAS_RESTRICT_CTAS_PER_SM")) per_sm = std::max(1, std::atoi(e2));
      const int warps = restrict_chunk_threads() / 32;
      ctx->rc_grid = std::max(1, std::min(per_sm * nsm, (ctx->nchunk + warps - 1) / warps));
      // the last-CTA sum of r.r reads one partial per CTA: within the partials buffer
      ctx->rc_grid = std::min(ctx->rc_grid, std::max(1, ctx->partial_cap / 2 - 1));
    }
  }
  {
    // persistent prolongation: one wave of 256-thread CTAs, at most 4 per SM (DGAS_PROLONG_CTAS_PER_SM)
    int dev = 0, nsm = 148, per = std::min(4, prolong_ctas_per_sm(ctx));
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (const char* e = std::getenv("DGAS_PROLONG_CTAS_PER_SM")) per = std::max(1, std::atoi(e));
    ctx->prolong_grid = per * nsm;
  }
  ctx->n_coarse_ctas = ctx->coarse_dense ? (int)std::min<int64_t>(592, std::max<int64_t>(1, ctx->N0 / 32)) : 1;
  if (ctx->coarse_mode == 0) {  // calibrated refinement of the dense coarse solve (R30, Z30)
    if (const char* e = std::getenv("DGAS_ND_TOL")) ctx->nd_tol = std::atof(e);
    int st2 = dense_calibrate(ctx);
    if (st2) return st2;
  }
  {
    // TMA ring of the local-solve CTAs: unit = CC columns of a row-block (about the average row-block
    // for n_p = 15), S slots; 128-thread CTAs target ~55 KB (3-4 CTAs/SM), 256-thread ~110 KB.
    // Invariant (else the forward/backward refill protocol would deadlock): a row-block spans at most
    // S - 1 units, because the slots of a block are refilled only after that block's barrier.
    ctx->ring_slots = 0;
    {
      // Ring of the warp-specialised local solve: fixed slots of CC columns; S from the per-CTA budget.
      // The budget targets enough resident CTAs for all subdomains at once when possible.
      int dev = 0, nsm = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      const int T = local_threads(ctx->p);
      const int per_sm = (ctx->nsub + nsm - 1) / nsm;
      size_t budget = per_sm <= 1 ? 200 * 1024 : per_sm <= 2 ? 105 * 1024 : per_sm <= 3 ? 70 * 1024
                      : per_sm <= 4 ? 55 * 1024 : per_sm <= 5 ? 44 * 1024 : per_sm <= 6 ? 36 * 1024 : 31 * 1024;
      if (T == 256) budget = std::max<size_t>(budget, 100 * 1024);
      size_t target = T == 128 ? 12 * 1024 : 24 * 1024;  // measured best on B200 (tools/ab.sh)
      if (const char* e = std::getenv("DGAS_APPLY_BUDGET_KB")) budget = (size_t)std::atoi(e) * 1024;
      if (const char* e = std::getenv("DGAS_APPLY_SLOT_KB")) target = (size_t)std::atoi(e) * 1024;
      const int maxW = std::max(2, (ctx->max_urow + 1) / 2 * 2);
      const size_t base = apply_smem_bytes(ctx);
      int CC = std::min(maxW, std::max(2, (int)(target / (8 * ctx->np)) / 2 * 2));
      for (; CC >= 2; CC -= 2) {
        uint32_t sb = (uint32_t)(((((int64_t)CC * ctx->np + 1) / 2 * 2) * 8 + 127) / 128 * 128);
        int S = (int)std::min<size_t>(64, (budget - std::min(budget, base)) / sb);
        if (S >= 2) { ctx->ring_slots = S; ctx->slot_bytes = sb; ctx->ring_rows = CC; break; }
      }
    }
    if (ctx->ring_slots < 2) { ctx->detail = "subdomain row-block too large for shared memory"; return DGAS_E_INVALID_ARG; }
    {
      // L2 reuse across the forward/backward turnaround: the units just below each subdomain's ring-
      // resident tail are streamed evict-last (budget shared by all subdomains; vectors keep the rest)
      double mb = 0;  // measured: no gain at 24-96 MB on cfg3/4/5 (tools/ab.sh), kept as a knob
      if (const char* e = std::getenv("DGAS_LOCAL_REUSE_MB")) mb = std::atof(e);
      ctx->local_reuse = (int)std::min<double>(1 << 20, mb * 1048576.0 / ((double)ctx->nsub * ctx->slot_bytes));
    }
    int st = apply_set_smem(ctx, apply_smem_bytes(ctx));
    if (st) return st;
    if ((st = panel_configure(ctx))) return st;
    if (ctx->local_kernel == 2 && (st = local_warp_setup(ctx))) return st;
    if ((st = local_inv_setup(ctx))) return st;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    // consumer groups: two independent 128-thread groups for n_p >= 10 (95 registers, so 2 CTAs/SM;
    // measured: cfg3 765 -> 812 it/s, cfg4 1444 -> 1530, cfg5 p5q5 1848 -> 2335, p6q6 1315 -> 1470);
    // one 256-thread group below (no gain at n_p <= 6)
    int ng = ctx->np >= 10 ? 2 : 1;
    if (const char* e = std::getenv("DGAS_SPMV_GROUPS")) ng = std::atoi(e) == 2 ? 2 : 1;
    if (spmv_groups_ok(ctx->p) < ng) ng = 1;
    if (ng == 2 && (int64_t)ctx->max_deg * ctx->np > spmv_gather_cap(ctx->p, 2)) ng = 1;
    ctx->spmv_groups = ng;
    int per_sm = ng == 2 ? 2 : 3;  // measured best on B200 (tools/ab.sh): 3 CTAs/SM, 2-cell batches, ~64 KB rings
    if (const char* e = std::getenv("DGAS_SPMV_CTAS_PER_SM")) per_sm = std::max(1, std::atoi(e));
    ctx->spmv_grid = std::min(ctx->nc, per_sm * nsm);
    // SpMV ring: one slot per batch of G consecutive row-blocks of a CTA's cell range
    {
      // cells per batch: ~24 KB of row-blocks per bulk copy (per-batch consumer overhead dominates
      // below that, tools/ab.sh), at most the thread-limited maximum
      int G = spmv_batch_cells(ctx->p, ng);
      if (!std::getenv("DGAS_SPMV_G")) {
        const double avg_row = (double)ctx->a_off_h[ctx->nc] * 8.0 / ctx->nc;
        G = std::max(1, std::min(G, (int)std::lround(24576.0 / avg_row)));
      }
      while (G > 1 && (int64_t)G * ctx->max_deg * ctx->np > spmv_gather_cap(ctx->p, ng)) --G;
      ctx->spmv_G = G;
      if ((int64_t)G * ctx->max_deg * ctx->np > spmv_gather_cap(ctx->p, ng)) { ctx->detail = "cell degree too large for the SpMV kernel"; return DGAS_E_INVALID_ARG; }
      const int chunk = (ctx->nc + ctx->spmv_grid - 1) / ctx->spmv_grid;
      int64_t mx = 0;
      for (int c0 = 0; c0 < ctx->nc; c0 += chunk) {
        const int c1 = std::min(ctx->nc, c0 + chunk);
        for (int k0 = c0; k0 < c1; k0 += G) mx = std::max(mx, ctx->a_off_h[std::min(c1, k0 + G)] - ctx->a_off_h[k0]);
      }
      ctx->spmv_slot_bytes = (uint32_t)((mx * 8 + 127) / 128 * 128);
      int64_t budget = 64 * 1024;
      if (const char* e = std::getenv("DGAS_SPMV_BUDGET_KB")) budget = (int64_t)std::atoi(e) * 1024;
      ctx->spmv_slots = (int)std::max<int64_t>(2, std::min<int64_t>(16, budget / ctx->spmv_slot_bytes));
    }
    st = spmv_set_smem(ctx, spmv_smem_bytes(ctx));
    if (st) return st;
    // byte-ring SpMV (spmv_ring.cu) unless DGAS_SPMV_KERNEL=3 or the mesh exceeds its degree limit
    ctx->spmv_kernel = 3;
    {
      const char* e = std::getenv("DGAS_SPMV_KERNEL");
      if (!(e && std::atoi(e) == 3)) {
        const int rc = spmv_ring_configure(ctx, nsm);
        if (rc < 0) return DGAS_E_CUDA;
        if (rc == 0) ctx->spmv_kernel = 4;
        // separate direction-update pass when the vectors are large (config 3, 21 MB each: the fused
        // gather of z and p_old costs more than one extra stream; measured +3.9% PCG it/s there,
        // neutral on config 4, -1..2% on small configs)
        ctx->spmv_psplit = ctx->N * 8 > 12 * 1024 * 1024;
        if (const char* e2 = std::getenv("DGAS_SPMV_PSPLIT")) ctx->spmv_psplit = std::atoi(e2) != 0;
      }
    }
  }
  DGAS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (std::getenv("DGAS_DEDUP_STATS")) {  // diagnostic: bitwise-identical row-blocks / local factors
    std::vector<double> A((size_t)ctx->a_off_h[ctx->nc]);
    DGAS_CUDA(cudaMemcpy(A.data(), ctx->d_A, A.size() * 8, cudaMemcpyDeviceToHost));
    auto fnv = [](const double* p, int64_t n) {
      uint64_t h = 1469598103934665603ULL;
      const unsigned char* b = reinterpret_cast<const unsigned char*>(p);
      for (int64_t i = 0; i < n * 8; ++i) { h ^= b[i]; h *= 1099511628211ULL; }
      return h ^ (uint64_t)n;
    };
    std::map<uint64_t, int> rows;
    for (int c = 0; c < ctx->nc; ++c) rows[fnv(A.data() + ctx->a_off_h[c], ctx->a_off_h[c + 1] - ctx->a_off_h[c])]++;
    std::map<uint64_t, int> subs;
    if (ctx->local_kernel == 2 || ctx->local_kernel == 4) {
      std::vector<int64_t> po(ctx->nc + 1);
      DGAS_CUDA(cudaMemcpy(po.data(), ctx->d_p_off, (ctx->nc + 1) * 8, cudaMemcpyDeviceToHost));
      std::vector<double> Pp((size_t)ctx->p_total);
      DGAS_CUDA(cudaMemcpy(Pp.data(), ctx->d_P, Pp.size() * 8, cudaMemcpyDeviceToHost));
      for (int s2 = 0; s2 < ctx->nsub; ++s2) {
        const int64_t a0 = po[ctx->sub_ptr_h[s2]], a1 = po[ctx->sub_ptr_h[s2 + 1]];
        subs[fnv(Pp.data() + a0, a1 - a0)]++;
      }
    }
    fprintf(stderr, "dgas: dedup stats: %d cells, %zu distinct row-blocks; %d subdomains, %zu distinct local factors\n",
            ctx->nc, rows.size(), ctx->nsub, subs.size());
  }
  {
    int st3 = dedup_setup(ctx);  // exact de-duplication of bitwise-identical operator data (dedup.cu)
    if (st3) return st3;
  }
  return 0;
}

int dgas_post_setup(dgas_ctx ctx) { return finish_setup_buffers(ctx); }

extern "C" int dgas_rhs(dgas_ctx ctx, int f_kind, double* b, void* stream) {
  if (!ctx || !b || f_kind < 0 || f_kind > 2) return DGAS_E_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  int st = finish_setup_buffers(ctx);
  if (st) return st;
  {
    cudaStream_t keep = ctx->stream;
    ctx->stream = s;
    st = launch_rhs(ctx, f_kind, ctx->d_t1);
    ctx->stream = keep;
    if (st) return st;
  }
  launch_perm(ctx, ctx->d_t1, b, 0, s);
  DGAS_CUDA(cudaGetLastError());
  return DGAS_OK;
}

extern "C" int dgas_spmv(dgas_ctx ctx, const double* x, double* y, void* stream) {
  if (!ctx || !x || !y) return DGAS_E_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  int st = finish_setup_buffers(ctx);
  if (st) return st;
  launch_perm(ctx, x, ctx->d_t1, 1, s);
  launch_spmv(ctx, 0, ctx->d_t1, ctx->d_t2, nullptr, s);
  launch_perm(ctx, ctx->d_t2, y, 0, s);
  DGAS_CUDA(cudaGetLastError());
  return DGAS_OK;
}

// internal-order apply on context buffers: t1 (r) -> t2 (z)
static void apply_internal(dgas_ctx ctx, cudaStream_t s) {
  launch_restrict(ctx, 0, nullptr, ctx->d_t1, s);
  launch_apply(ctx, 0, nullptr, ctx->d_t1, ctx->d_t2, s);
  launch_prolong(ctx, 0, nullptr, nullptr, ctx->d_t2, s, 0, 0);
}

extern "C" int dgas_apply(dgas_ctx ctx, const double* r, double* z, void* stream) {
  if (!ctx || !r || !z) return DGAS_E_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  int st = finish_setup_buffers(ctx);
  if (st) return st;
  launch_perm(ctx, r, ctx->d_t1, 1, s);
  apply_internal(ctx, s);
  launch_perm(ctx, ctx->d_t2, z, 0, s);
  DGAS_CUDA(cudaGetLastError());
  return DGAS_OK;
}

extern "C" int dgas_set_precond(dgas_ctx ctx, int mode) {
  if (!ctx || mode < DGAS_PRECOND_TWO_LEVEL || mode > DGAS_PRECOND_NONE) return DGAS_E_INVALID_ARG;
  if (mode == ctx->precond) return DGAS_OK;
  int st = finish_setup_buffers(ctx);
  if (st) return st;
  // the PCG graph bakes the kernel sequence in: rebuild it on the next solve
  if (ctx->graph_exec) { cudaGraphExecDestroy(ctx->graph_exec); ctx->graph_exec = nullptr; }
  if (ctx->graph) { cudaGraphDestroy(ctx->graph); ctx->graph = nullptr; }
  ctx->precond = mode;
  if (mode == DGAS_PRECOND_ONE_LEVEL || mode == DGAS_PRECOND_NONE) {
    DGAS_CUDA(cudaMemset(ctx->d_z0, 0, (size_t)ctx->N0 * sizeof(double)));
    DGAS_CUDA(cudaDeviceSynchronize());
  }
  return DGAS_OK;
}

// Internal-order hooks used by bench.py's kernel timing (same kernels as inside the PCG graph).
extern "C" int dgas_bench_kernels(dgas_ctx ctx, int which, int reps, void* stream) {
  if (!ctx || reps < 1) return DGAS_E_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  int st = finish_setup_buffers(ctx);
  if (st) return st;
  for (int k = 0; k < reps; ++k) {
    if (which == 0) launch_spmv(ctx, 0, ctx->d_t1, ctx->d_t2, nullptr, s);
    else if (which == 1) apply_internal(ctx, s);
    else if (which == 2) launch_apply(ctx, 0, nullptr, ctx->d_t1, ctx->d_t2, s);
    else if (which == 3) launch_local_only(ctx, ctx->d_t1, ctx->d_t2, s);
    else if (which == 4) launch_coarse_only(ctx, s);
    else return DGAS_E_INVALID_ARG;
  }
  DGAS_CUDA(cudaGetLastError());
  return DGAS_OK;
}

static int build_graph_impl(dgas_ctx ctx, int maxit);

static int build_graph(dgas_ctx ctx, int maxit) {
  int st = build_graph_impl(ctx, maxit);
  ctx->side_sel = 0;
  if (st) {
    // leave no capture open and no half-built graph behind
    cudaGraph_t g = nullptr;
    cudaStreamCaptureStatus cs;
    if (cudaStreamIsCapturing(ctx->cap_stream2, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) cudaStreamEndCapture(ctx->cap_stream2, &g);
    for (int i = 0; i < 3; ++i)
      if (cudaStreamIsCapturing(ctx->side[i], &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) cudaStreamEndCapture(ctx->side[i], &g);
    if (cudaStreamIsCapturing(ctx->cap_stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
      cudaStreamEndCapture(ctx->cap_stream, &g);
      if (g) cudaGraphDestroy(g);
    }
    if (ctx->graph_exec) { cudaGraphExecDestroy(ctx->graph_exec); ctx->graph_exec = nullptr; }
    if (ctx->graph) { cudaGraphDestroy(ctx->graph); ctx->graph = nullptr; }
    cudaGetLastError();
  }
  return st;
}

static int build_graph_impl(dgas_ctx ctx, int maxit) {
  if (ctx->graph_exec && maxit <= ctx->hist_cap) return 0;
  if (ctx->graph_exec) { cudaGraphExecDestroy(ctx->graph_exec); ctx->graph_exec = nullptr; }
  if (ctx->graph) { cudaGraphDestroy(ctx->graph); ctx->graph = nullptr; }
  if (maxit > ctx->hist_cap) {
    if (ctx->d_alpha) cudaFree(ctx->d_alpha);
    if (ctx->d_beta) cudaFree(ctx->d_beta);
    int cap = std::max(maxit, 8192);
    DGAS_CUDA(cudaMalloc((void**)&ctx->d_alpha, cap * sizeof(double)));
    DGAS_CUDA(cudaMalloc((void**)&ctx->d_beta, cap * sizeof(double)));
    ctx->hist_cap = cap;
  }
  cudaStream_t cs = ctx->cap_stream, cs2 = ctx->cap_stream2;
  PcgState* st = ctx->d_state;
  DGAS_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
  cudaStreamCaptureStatus cst;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  DGAS_CUDA(cudaStreamGetCaptureInfo(cs, &cst, nullptr, &g, &deps, &ndeps));
  cudaGraphConditionalHandle h;
  DGAS_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  // init: r = b - A x0, r0 = Q^T r, z = P^-1 r, gamma_0 = r.z
  ctx->side_sel = 1;
  launch_spmv(ctx, 0, ctx->d_x, ctx->d_q, nullptr, cs);
  launch_restrict(ctx, 2, st, nullptr, cs);
  launch_apply(ctx, 1, st, nullptr, ctx->d_z, cs);
  launch_prolong(ctx, 1, st, nullptr, ctx->d_z, cs, h, 1);
  DGAS_CUDA(cudaStreamGetCaptureInfo(cs, &cst, nullptr, &g, &deps, &ndeps));
  cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cnode;
  DGAS_CUDA(cudaGraphAddNode(&cnode, g, deps, ndeps, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  DGAS_CUDA(cudaStreamUpdateCaptureDependencies(cs, &cnode, 1, cudaStreamSetCaptureDependencies));
  DGAS_CUDA(cudaStreamBeginCaptureToGraph(cs2, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  ctx->side_sel = 2;
  // the body holds `unroll` iterations: every kernel returns at once when the state says done, so the
  // copies after convergence cost one launch each, and the per-body cost of the WHILE node is shared
  for (int u = 0; u < ctx->unroll; ++u) {
    launch_spmv(ctx, 1, nullptr, ctx->d_q, st, cs2);
    if (!apply_fuses_restrict(ctx)) launch_restrict(ctx, 1, st, nullptr, cs2);
    launch_apply(ctx, 2, st, nullptr, ctx->d_z, cs2);
    launch_prolong(ctx, 2, st, nullptr, ctx->d_z, cs2, h, 1);
  }
  DGAS_CUDA(cudaGetLastError());
  DGAS_CUDA(cudaStreamEndCapture(cs2, &body));
  ctx->side_sel = 0;
  launch_lanczos(ctx, cs);
  DGAS_CUDA(cudaStreamEndCapture(cs, &g));
  ctx->graph = g;
  DGAS_CUDA(cudaGraphInstantiate(&ctx->graph_exec, g, 0));
  return 0;
}

// Profiling path (DGAS_EAGER=1): the same kernels launched from the host, 8 iterations between host
// checks of the state (kernels return at once after convergence). ncu then sees every iteration kernel
// as its own launch, which it does not inside the graph's conditional WHILE node.
static int pcg_eager(dgas_ctx ctx, double rtol, int maxit, cudaStream_t s) {
  if (maxit > ctx->hist_cap) {
    if (ctx->d_alpha) cudaFree(ctx->d_alpha);
    if (ctx->d_beta) cudaFree(ctx->d_beta);
    int cap = std::max(maxit, 8192);
    DGAS_CUDA(cudaMalloc((void**)&ctx->d_alpha, cap * sizeof(double)));
    DGAS_CUDA(cudaMalloc((void**)&ctx->d_beta, cap * sizeof(double)));
    ctx->hist_cap = cap;
    if (ctx->graph_exec) { cudaGraphExecDestroy(ctx->graph_exec); ctx->graph_exec = nullptr; }
    if (ctx->graph) { cudaGraphDestroy(ctx->graph); ctx->graph = nullptr; }
  }
  PcgState* st = ctx->d_state;
  launch_init_state(ctx, st, maxit, rtol, s);
  ctx->side_sel = 0;
  launch_spmv(ctx, 0, ctx->d_x, ctx->d_q, nullptr, s);
  launch_restrict(ctx, 2, st, nullptr, s);
  launch_apply(ctx, 1, st, nullptr, ctx->d_z, s);
  launch_prolong(ctx, 1, st, nullptr, ctx->d_z, s, 0, 0);
  // DGAS_EAGER_TIMING=1: CUDA events around each phase of every iteration on the launching stream
  // (in-situ kernel times, L2 state as in a real solve), averaged and printed to stderr at the end
  static const bool timing = std::getenv("DGAS_EAGER_TIMING") != nullptr;
  cudaEvent_t ev[8][5];
  double acc[4] = {0, 0, 0, 0};
  int nacc = 0;
  if (timing)
    for (auto& row : ev)
      for (auto& e : row) DGAS_CUDA(cudaEventCreate(&e));
  for (;;) {
    for (int u = 0; u < 8; ++u) {
      if (timing) cudaEventRecord(ev[u][0], s);
      launch_spmv(ctx, 1, nullptr, ctx->d_q, st, s);
      if (timing) cudaEventRecord(ev[u][1], s);
      if (!apply_fuses_restrict(ctx)) launch_restrict(ctx, 1, st, nullptr, s);
      if (timing) cudaEventRecord(ev[u][2], s);
      launch_apply(ctx, 2, st, nullptr, ctx->d_z, s);
      if (timing) cudaEventRecord(ev[u][3], s);
      launch_prolong(ctx, 2, st, nullptr, ctx->d_z, s, 0, 0);
      if (timing) cudaEventRecord(ev[u][4], s);
    }
    DGAS_CUDA(cudaMemcpyAsync(ctx->h_state, st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    DGAS_CUDA(cudaStreamSynchronize(s));
    if (timing && !ctx->h_state->done) {
      for (int u = 0; u < 8; ++u)
        for (int k = 0; k < 4; ++k) {
          float ms = 0;
          cudaEventElapsedTime(&ms, ev[u][k], ev[u][k + 1]);
          acc[k] += ms;
        }
      nacc += 8;
    }
    if (ctx->h_state->done) break;
  }
  if (timing) {
    if (nacc)
      fprintf(stderr, "eager timing (%d iterations): spmv %.1f us, restrict %.1f us, apply %.1f us, prolong %.1f us\n",
              nacc, acc[0] * 1e3 / nacc, acc[1] * 1e3 / nacc, acc[2] * 1e3 / nacc, acc[3] * 1e3 / nacc);
    for (auto& row : ev)
      for (auto& e : row) cudaEventDestroy(e);
  }
  launch_lanczos(ctx, s);
  DGAS_CUDA(cudaGetLastError());
  return 0;
}

static int pcg_device(dgas_ctx ctx, double rtol, int maxit, int* iters, double* cond, cudaStream_t s) {
  const bool eager = std::getenv("DGAS_EAGER") != nullptr;  // per call (tests switch it)
  if (eager) {
    int st = pcg_eager(ctx, rtol, maxit, s);
    if (st) return st;
    DGAS_CUDA(cudaMemcpyAsync(ctx->h_state, ctx->d_state, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    DGAS_CUDA(cudaMemcpyAsync(ctx->h_scal, ctx->d_lanczos, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
    return 0;
  }
  int st = build_graph(ctx, maxit);
  if (st) return st;
  launch_init_state(ctx, ctx->d_state, maxit, rtol, s);
  DGAS_CUDA(cudaGraphLaunch(ctx->graph_exec, s));
  DGAS_CUDA(cudaMemcpyAsync(ctx->h_state, ctx->d_state, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
  DGAS_CUDA(cudaMemcpyAsync(ctx->h_scal, ctx->d_lanczos, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
  return 0;
}

static int pcg_finish(dgas_ctx ctx, int* iters, double* cond) {
  const PcgState& h = *ctx->h_state;
  ctx->last_iters = h.it;
  ctx->last_status = h.status;
  ctx->last_lmin = ctx->h_scal[0];
  ctx->last_lmax = ctx->h_scal[1];
  ctx->last_cond = h.it > 0 ? ctx->h_scal[2] : 1.0;
  ctx->last_relres = h.bb > 0 ? std::sqrt(h.rr / h.bb) : 0.0;
  if (iters) *iters = h.it;
  if (cond) *cond = ctx->last_cond;
  if (h.status == DGAS_E_BREAKDOWN) ctx->detail = "PCG breakdown (p.Ap <= 0, r.z <= 0 or non-finite)";
  return h.status;
}

extern "C" int dgas_pcg(dgas_ctx ctx, const double* b, double* x, double rtol, int maxit, int* iters,
                        double* lanczos_cond, void* stream) {
  if (!ctx || !b || !x || !(rtol > 0) || maxit < 1) return DGAS_E_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  int st = finish_setup_buffers(ctx);
  if (st) return st;
  launch_perm(ctx, b, ctx->d_b, 1, s);
  launch_perm(ctx, x, ctx->d_x, 1, s);
  if ((st = pcg_device(ctx, rtol, maxit, iters, lanczos_cond, s))) return st;
  launch_perm(ctx, ctx->d_x, x, 0, s);
  DGAS_CUDA(cudaGetLastError());
  DGAS_CUDA(cudaStreamSynchronize(s));
  return pcg_finish(ctx, iters, lanczos_cond);
}

extern "C" int dgas_pcg_host(dgas_ctx ctx, const double* b_host, double* x_host, double rtol, int maxit, int* iters,
                             double* lanczos_cond, void* stream) {
  if (!ctx || !b_host || !x_host || !(rtol > 0) || maxit < 1) return DGAS_E_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  int st = finish_setup_buffers(ctx);
  if (st) return st;
  const size_t bytes = ctx->N * sizeof(double);
  DGAS_CUDA(cudaMemcpyAsync(ctx->d_t1, b_host, bytes, cudaMemcpyHostToDevice, s));
  DGAS_CUDA(cudaMemcpyAsync(ctx->d_t2, x_host, bytes, cudaMemcpyHostToDevice, s));
  launch_perm(ctx, ctx->d_t1, ctx->d_b, 1, s);
  launch_perm(ctx, ctx->d_t2, ctx->d_x, 1, s);
  if ((st = pcg_device(ctx, rtol, maxit, iters, lanczos_cond, s))) return st;
  launch_perm(ctx, ctx->d_x, ctx->d_t2, 0, s);
  DGAS_CUDA(cudaMemcpyAsync(x_host, ctx->d_t2, bytes, cudaMemcpyDeviceToHost, s));
  DGAS_CUDA(cudaGetLastError());
  DGAS_CUDA(cudaStreamSynchronize(s));
  return pcg_finish(ctx, iters, lanczos_cond);
}

extern "C" int dgas_history(dgas_ctx ctx, double* alphas, double* betas, int cap) {
  if (!ctx || !alphas || !betas || cap < 0) return DGAS_E_INVALID_ARG;
  if (!ctx->d_alpha) return 0;
  int n = std::min(cap, ctx->last_iters);
  if (n > 0) {
    DGAS_CUDA(cudaMemcpy(alphas, ctx->d_alpha, n * sizeof(double), cudaMemcpyDeviceToHost));
    int nb = std::min(cap, std::max(0, ctx->last_iters - 1));
    if (ctx->last_status == DGAS_NOT_CONVERGED) nb = std::min(cap, ctx->last_iters);
    if (nb > 0) DGAS_CUDA(cudaMemcpy(betas, ctx->d_beta, nb * sizeof(double), cudaMemcpyDeviceToHost));
  }
  return n;
}

extern "C" int dgas_info(dgas_ctx ctx, dgas_info_t* info) {
  if (!ctx || !info) return DGAS_E_INVALID_ARG;
  std::memset(info, 0, sizeof *info);
  const int64_t np = ctx->np, nq = ctx->nq, N = ctx->N;
  info->N = N; info->N0 = ctx->N0; info->n_cells = ctx->nc; info->n_p = ctx->np; info->n_q = ctx->nq;
  info->n_subdomains = ctx->nsub; info->n_coarse = ctx->ncoarse; info->n_faces = ctx->nface;
  info->n_overlaps = ctx->nov; info->coarse_dense = ctx->coarse_dense; info->coarse_band = ctx->coarse_bw;
  info->nnz_blocks = ctx->nnzb;
  info->bytes_A = ctx->nnzb * np * np * 8;
  info->bytes_U = ctx->u_total * 8;
  info->bytes_Dinv = (int64_t)ctx->nc * np * np * 8;
  info->bytes_G = (int64_t)ctx->nov * np * nq * 8;
  info->bytes_coarse = ctx->coarse_mode == 2 ? ctx->nd.bytes : ctx->coarse_dense ? ctx->N0 * ctx->ldX * 8
                                         : (int64_t)ctx->nT * (ctx->bt + 1) * CT * CT * 8 + (int64_t)ctx->nT * CT * CT * 8;
  // algorithmic bytes: every operator entry read once, vectors once each
  info->alg_bytes_spmv = info->bytes_A + (2 * N) * 8 + (int64_t)ctx->nnzb * 4;  // full-storage bytes (reference)
  const int64_t dinv_tri = (int64_t)ctx->nc * (np * (np + 1) / 2) * 8;
  // refinement steps of the ND coarse solve re-read the factors and read the A0 pair blocks once more
  const int refine = ctx->coarse_mode == 2 ? ctx->nd.refine : ctx->coarse_mode == 0 ? ctx->dense_refine : 0;
  const int64_t a0b = ctx->n_pairs * nq * nq * 8;
  const int64_t coarse_alg = info->bytes_coarse * (1 + refine) + refine * a0b;
  const int64_t local_b = ctx->local_kernel == 3 ? ctx->inv_bytes : info->bytes_U + dinv_tri;
  info->alg_bytes_apply = local_b + coarse_alg + 2 * info->bytes_G + 3 * N * 8;
  info->alg_bytes_iter = info->bytes_A + local_b + coarse_alg + 2 * info->bytes_G + 16 * N * 8;
  info->last_iters = ctx->last_iters; info->last_status = ctx->last_status;
  info->last_cond = ctx->last_cond; info->last_lmin = ctx->last_lmin; info->last_lmax = ctx->last_lmax;
  info->last_relres = ctx->last_relres;
  info->coarse_mode = ctx->coarse_mode;
  info->coarse_refine = refine;
  info->unroll = ctx->unroll;
  info->local_kernel = ctx->local_kernel;
  info->local_ctas_per_sm = ctx->local_kernel == 2 ? ctx->panel_cps : 0;
  info->bytes_local = ctx->local_kernel == 3 ? ctx->inv_bytes : info->bytes_U + dinv_tri;
  info->local_inv_err = ctx->inv_err;
  info->dedup_A_bytes = ctx->d_a_dd ? ctx->a_bytes_stored : 0;
  info->dedup_local_bytes = ctx->p_bytes_stored;
  info->coarse_solve_relerr = ctx->coarse_mode == 2 ? ctx->nd.calib_err : ctx->coarse_mode == 0 ? ctx->dense_err : 0.0;
  int coarse_launches = 1 + 3 * (ctx->coarse_mode == 0 ? ctx->dense_refine : 0);
  if (ctx->coarse_mode == 2) {
    coarse_launches = 0;
    for (int L = 0; L < ctx->nd.nlev; ++L) {
      coarse_launches += ctx->nd.h_wf_ptr[L + 1] > ctx->nd.h_wf_ptr[L];
      coarse_launches += ctx->nd.h_wb_ptr[L + 1] > ctx->nd.h_wb_ptr[L];
    }
    coarse_launches = coarse_launches * (1 + ctx->nd.refine) + 2 * ctx->nd.refine;  // + residual, axpy per step
  }
  // body: spmv, restrict, coarse (side stream), local, prolong; solve: 2 perm in, init_state,
  // init (spmv, restrict, coarse, local, prolong), lanczos, perm out
  info->launches_per_iter = 4 + coarse_launches + (ctx->spmv_kernel == 4 && ctx->spmv_psplit ? 1 : 0);
  info->launches_per_solve = 3 + (4 + coarse_launches) + 2;
  return DGAS_OK;
}

extern "C" int dgas_debug_block(dgas_ctx ctx, int32_t i, int32_t j, double* out) {
  if (!ctx || !out || i < 0 || j < 0 || i >= ctx->nc || j >= ctx->nc) return DGAS_E_INVALID_ARG;
  const int np = ctx->np;
  std::memset(out, 0, sizeof(double) * np * np);
  int ci = ctx->iperm[i], cj = ctx->iperm[j];
  int lo = ctx->nbr_ptr_h[ci], hi = ctx->nbr_ptr_h[ci + 1];
  int deg = hi - lo, sl = -1;
  for (int k = lo; k < hi; ++k) if (ctx->nbr_h[k] == cj) sl = k - lo;
  if (sl < 0) return 0;
  const int64_t off = ctx->d_a_dd ? ctx->a_dd_h[ci] : ctx->a_off_h[ci];
  std::vector<double> row((size_t)np * deg * np);
  DGAS_CUDA(cudaMemcpy(row.data(), ctx->d_A + off, row.size() * sizeof(double), cudaMemcpyDeviceToHost));
  for (int a = 0; a < np; ++a)
    for (int b = 0; b < np; ++b) out[a * np + b] = row[((size_t)sl * np + b) * np + a];
  return 1;
}

extern "C" int dgas_debug_basis(dgas_ctx ctx, int32_t i, double* out) {
  if (!ctx || !out || i < 0 || i >= ctx->nc) return DGAS_E_INVALID_ARG;
  const int np = ctx->np;
  DGAS_CUDA(cudaMemcpy(out, ctx->d_C + (size_t)ctx->iperm[i] * np * np, sizeof(double) * np * np, cudaMemcpyDeviceToHost));
  return DGAS_OK;
}

extern "C" int dgas_debug_A0(dgas_ctx ctx, double* out) {
  if (!ctx || !out) return DGAS_E_INVALID_ARG;
  // A0 = Q^T A Q as assembled (eq:A0): the coupled-pair blocks, before any scaling or factorisation
  const int64_t N0 = ctx->N0, nq = ctx->nq, np_ = ctx->n_pairs;
  std::vector<int> pair((size_t)2 * np_);
  std::vector<double> blk((size_t)np_ * nq * nq);
  DGAS_CUDA(cudaMemcpy(pair.data(), ctx->d_pair, pair.size() * sizeof(int), cudaMemcpyDeviceToHost));
  DGAS_CUDA(cudaMemcpy(blk.data(), ctx->d_A0b, blk.size() * sizeof(double), cudaMemcpyDeviceToHost));
  std::fill(out, out + N0 * N0, 0.0);
  for (int64_t k = 0; k < np_; ++k)
    for (int a = 0; a < nq; ++a)
      for (int c = 0; c < nq; ++c)
        out[((int64_t)pair[2 * k] * nq + a) * N0 + (int64_t)pair[2 * k + 1] * nq + c] = blk[((size_t)k * nq + a) * nq + c];
  return DGAS_OK;
}

extern "C" const char* dgas_strerror(int status) {
  switch (status) {
    case DGAS_OK: return "ok";
    case DGAS_NOT_CONVERGED: return "PCG did not converge within maxit";
    case DGAS_E_INVALID_ARG: return "invalid argument";
    case DGAS_E_MESH: return "invalid mesh or coarse description";
    case DGAS_E_NOT_SPD: return "matrix not SPD (Cholesky pivot <= 0)";
    case DGAS_E_BREAKDOWN: return "PCG breakdown";
    case DGAS_E_CUDA: return "CUDA error";
    case DGAS_E_NOMEM: return "out of device memory";
  }
  return "unknown status";
}

extern "C" const char* dgas_error_detail(dgas_ctx ctx) { return ctx ? ctx->detail.c_str() : "null context"; }
