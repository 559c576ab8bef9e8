// shard.cu — the subdomain-sharded multi-GPU ASPCG iteration ("massively
// parallel", the method is defined for any decomposition): one process per GPU, each owning a
// contiguous range of subdomains (cells are numbered subdomain-major, so the range is a contiguous
// block of cells and dofs). Every rank holds the whole replicated setup (A, factors, Q, the coarse
// factor: at most a few GB per GPU for the BASELINE configs), and per iteration works only on its own
// rows / subdomains / cells:
//   * I1 SpMV of the own rows (the byte-ring kernel on the sub-range), after a halo exchange of p on
//     the cells that border another rank (pack -> all-gather -> unpack);
//   * I2 x, r update of the own dofs and partial r.r; I3 partial Q^T r over the own cells' pieces;
//     one all-reduce of [Q^T r | r.r];
//   * I4 the coarse solve replicated on every rank (same summed r0 -> same z0, no broadcast);
//   * I5 local solves of the own subdomains (the single-GPU kernels on a subdomain sub-range), I6
//     prolongation on the own cells and partial r.z (all-reduced), I7 p = z + beta p on the own dofs.
// Collectives are the caller's (torch.distributed over NCCL or gloo, dgas.ShardedSolver): the entry
// points below only compute, asynchronously on the caller's stream, from and into caller buffers.
// All dot products are deterministic (fixed grid, per-CTA partials summed in order).
#include <cmath>

#include "internal.h"

#define SH_T 256
#define SH_GRID 296  // 2 x 148 CTAs for the dot products

struct ShState {
  double rz_old, rz, pq, alpha, beta;
  int it, status;
};

__global__ void k_sh_dot(int64_t i0, int64_t i1, const double* a, const double* b, double* partials) {
  __shared__ double red[SH_T / 32];
  double v = 0;
  for (int64_t i = i0 + blockIdx.x * (int64_t)SH_T + threadIdx.x; i < i1; i += (int64_t)gridDim.x * SH_T)
    v += a[i] * b[i];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int k = 0; k < SH_T / 32; ++k) s += red[k];
    partials[blockIdx.x] = s;
  }
}
__global__ void k_sh_sum(int n, const double* partials, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0;
    for (int k = 0; k < n; ++k) s += partials[k];
    *out = s;
  }
}

// partial Q^T r over the pieces of the own cells [c0, c1) (warp per coarse element, restriction order)
__global__ void k_sh_restrict(int ncoarse, int np, int nq, int c0, int c1, const int* __restrict__ cov_ptr,
                              const int2* __restrict__ rrec, const double* __restrict__ G, const double* r,
                              double* r0) {
  const int J = blockIdx.x * (SH_T / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (J >= ncoarse) return;
  for (int b = 0; b < nq; ++b) {
    double v = 0;
    for (int k = cov_ptr[J] + lane; k < cov_ptr[J + 1]; k += 32) {
      const int2 rec = rrec[k];
      const int cell = rec.x, piece = rec.y & 0x7fffffff;
      if (cell < c0 || cell >= c1) continue;
      const double* g = G + (size_t)piece * np * nq + b;
      for (int a = 0; a < np; ++a) v += g[a * nq] * r[(size_t)cell * np + a];
    }
    v = warp_sum(v);
    if (lane == 0) r0[(size_t)J * nq + b] = v;
  }
}

// z[c] += sum over the pieces o of c of G_o z0[J(o)] on the own cells (thread per dof)
__global__ void k_sh_prolong(int np, int nq, int c0, int c1, const int* __restrict__ fov_ptr,
                             const int* __restrict__ fov, const int* __restrict__ ov_coarse,
                             const double* __restrict__ G, const double* __restrict__ z0, double* z) {
  const int64_t g = (int64_t)c0 * np + blockIdx.x * (int64_t)SH_T + threadIdx.x;
  if (g >= (int64_t)c1 * np) return;
  const int c = (int)(g / np), a = (int)(g % np);
  double v = 0;
  for (int k = fov_ptr[c]; k < fov_ptr[c + 1]; ++k) {
    const int o = fov[k], J = ov_coarse[o];
    const double* gr = G + (size_t)o * np * nq + (size_t)a * nq;
    for (int b = 0; b < nq; ++b) v += gr[b] * z0[(size_t)J * nq + b];
  }
  z[g] += v;
}

__global__ void k_sh_begin(int64_t N, const double* b, double* x, double* r) {
  for (int64_t i = blockIdx.x * (int64_t)SH_T + threadIdx.x; i < N; i += (int64_t)gridDim.x * SH_T) {
    x[i] = 0.0;
    r[i] = b[i];
  }
}

// alpha = rz / pq (pq summed over ranks); x += alpha p, r -= alpha q on [i0, i1)
__global__ void k_sh_update(int64_t i0, int64_t i1, const double* pq_sum, ShState* S, double* alpha_hist,
                            const double* p, const double* q, double* x, double* r) {
  const double pq = *pq_sum;
  const double alpha = S->rz / pq;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    S->pq = pq;
    S->alpha = alpha;
    alpha_hist[S->it] = alpha;
    if (!(pq > 0) || !isfinite(alpha)) S->status = DGAS_E_BREAKDOWN;
  }
  for (int64_t i = i0 + blockIdx.x * (int64_t)SH_T + threadIdx.x; i < i1; i += (int64_t)gridDim.x * SH_T) {
    x[i] += alpha * p[i];
    r[i] -= alpha * q[i];
  }
}

// p = z + beta p on [i0, i1) with beta = rz / rz_old from the summed r.z (first call: p = z)
__global__ void k_sh_direction(int64_t i0, int64_t i1, const double* rz_sum, const ShState* S, const double* z,
                               double* p, int first) {
  const double beta = first ? 0.0 : *rz_sum / S->rz;
  for (int64_t i = i0 + blockIdx.x * (int64_t)SH_T + threadIdx.x; i < i1; i += (int64_t)gridDim.x * SH_T)
    p[i] = first ? z[i] : z[i] + beta * p[i];
}
__global__ void k_sh_dir_state(const double* rz_sum, ShState* S, double* beta_hist, int first) {
  const double rz = *rz_sum;
  if (!first) {
    const double beta = rz / S->rz;
    S->beta = beta;
    beta_hist[S->it - 1] = beta;
  }
  if (!(rz > 0) || !isfinite(rz)) S->status = DGAS_E_BREAKDOWN;
  S->rz = rz;
}
__global__ void k_sh_pack(int np, int nsend, const int* __restrict__ send, const double* p, double* hbuf) {
  const int e = blockIdx.x * SH_T + threadIdx.x;
  if (e >= nsend * np) return;
  hbuf[e] = p[(size_t)send[e / np] * np + e % np];
}
// p on the border cells of every other rank, from the all-gathered halo buffers [R][cap]
__global__ void k_sh_unpack(int np, int R, int me, int cap, const int* __restrict__ send_ptr,
                            const int* __restrict__ send, const double* hall, double* p) {
  const int rr = blockIdx.y;
  if (rr == me) return;
  const int n = send_ptr[rr + 1] - send_ptr[rr];
  for (int e = blockIdx.x * SH_T + threadIdx.x; e < n * np; e += gridDim.x * SH_T)
    p[(size_t)send[send_ptr[rr] + e / np] * np + e % np] = hall[(size_t)rr * cap + e];
}
__global__ void k_sh_it(ShState* S, int inc) {
  if (threadIdx.x == 0) S->it += inc;
}
__global__ void k_sh_scatter(int64_t i0, int64_t i1, const int* __restrict__ perm, int np, const double* xin,
                             double* xout) {
  // internal dof i (cell ci = i / np) -> caller dof perm[ci] * np + a; own range only, others zero
  for (int64_t i = i0 + blockIdx.x * (int64_t)SH_T + threadIdx.x; i < i1; i += (int64_t)gridDim.x * SH_T)
    xout[(size_t)perm[i / np] * np + i % np] = xin[i];
}
__global__ void k_sh_lanczos_state(PcgState* st, int iters) {
  if (threadIdx.x == 0) st->it = iters;
}

// ------------------------------------------------------------------ host side
static int sh_blocks(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(2 * 148 * 4, (n + SH_T - 1) / SH_T)); }

extern "C" int dgas_shard(dgas_ctx ctx, int32_t rank, int32_t nranks, int64_t* info) {
  if (!ctx || nranks < 1 || rank < 0 || rank >= nranks || !info) return DGAS_E_INVALID_ARG;
  int st = dgas_post_setup(ctx);
  if (st) return st;
  if (nranks > ctx->nsub) { ctx->detail = "more ranks than subdomains"; return DGAS_E_INVALID_ARG; }
  ShardPlan& P = ctx->sh;
  P = ShardPlan();
  P.rank = rank; P.nranks = nranks;
  const std::vector<int>& sp = ctx->sub_ptr_h;
  // contiguous subdomain ranges balanced by cell count (every rank at least one subdomain)
  P.s_begin.assign(nranks + 1, 0);
  P.s_begin[nranks] = ctx->nsub;
  for (int r = 1; r < nranks; ++r) {
    const int64_t target = (int64_t)ctx->nc * r / nranks;
    int s = P.s_begin[r - 1] + 1;
    while (s < ctx->nsub - (nranks - r) && sp[s] < target) ++s;
    P.s_begin[r] = s;
  }
  P.c_begin.resize(nranks + 1);
  for (int r = 0; r <= nranks; ++r) P.c_begin[r] = sp[P.s_begin[r]];
  // border cells of every rank (a face neighbour on another rank): the halo it sends
  std::vector<int> nptr(ctx->nc + 1), nbr;
  DGAS_CUDA(cudaMemcpy(nptr.data(), ctx->d_nbr_ptr, (ctx->nc + 1) * sizeof(int), cudaMemcpyDeviceToHost));
  nbr.resize(nptr[ctx->nc]);
  DGAS_CUDA(cudaMemcpy(nbr.data(), ctx->d_nbr, nbr.size() * sizeof(int), cudaMemcpyDeviceToHost));
  std::vector<int> owner(ctx->nc);
  for (int r = 0; r < nranks; ++r)
    for (int c = P.c_begin[r]; c < P.c_begin[r + 1]; ++c) owner[c] = r;
  std::vector<int> send_ptr(nranks + 1, 0), send;
  for (int r = 0; r < nranks; ++r) {
    for (int c = P.c_begin[r]; c < P.c_begin[r + 1]; ++c) {
      bool border = false;
      for (int k = nptr[c]; k < nptr[c + 1] && !border; ++k) border = owner[nbr[k]] != r;
      if (border) send.push_back(c);
    }
    send_ptr[r + 1] = (int)send.size();
  }
  int cap = 1;
  for (int r = 0; r < nranks; ++r) cap = std::max(cap, (send_ptr[r + 1] - send_ptr[r]) * ctx->np);
  P.cap = cap;
  P.nsend_own = send_ptr[rank + 1] - send_ptr[rank];
  P.send_off = send_ptr[rank];
  if (ctx->spmv_kernel != 4) { ctx->detail = "sharded solve needs the byte-ring SpMV (cell degree <= 16)"; return DGAS_E_INVALID_ARG; }
  if ((st = dev_upload(ctx, &P.d_send_ptr, send_ptr)) || (st = dev_upload(ctx, &P.d_send, send))) return st;
  if ((st = dev_alloc(ctx, &P.d_partials, (size_t)SH_GRID + 8))) return st;
  DGAS_CUDA(cudaMalloc((void**)&P.d_state, sizeof(ShState)));
  DGAS_CUDA(cudaMemset(P.d_state, 0, sizeof(ShState)));
  if (ctx->hist_cap < 8192) {
    if (ctx->d_alpha) cudaFree(ctx->d_alpha);
    if (ctx->d_beta) cudaFree(ctx->d_beta);
    DGAS_CUDA(cudaMalloc((void**)&ctx->d_alpha, 8192 * sizeof(double)));
    DGAS_CUDA(cudaMalloc((void**)&ctx->d_beta, 8192 * sizeof(double)));
    ctx->hist_cap = 8192;
  }
  P.active = 1;
  const int64_t np = ctx->np;
  info[0] = P.c_begin[rank] * np; info[1] = P.c_begin[rank + 1] * np; info[2] = cap; info[3] = ctx->N;
  info[4] = ctx->N0; info[5] = P.s_begin[rank + 1] - P.s_begin[rank];
  return DGAS_OK;
}

static void sh_dot(dgas_ctx ctx, int64_t i0, int64_t i1, const double* a, const double* b, double* out, cudaStream_t s) {
  k_sh_dot<<<SH_GRID, SH_T, 0, s>>>(i0, i1, a, b, ctx->sh.d_partials);
  k_sh_sum<<<1, 32, 0, s>>>(SH_GRID, ctx->sh.d_partials, out);
}

static int sh_check(dgas_ctx ctx) {
  if (!ctx || !ctx->sh.active) return DGAS_E_INVALID_ARG;
  return 0;
}

// red0 = [Q^T r | r.r | b.b] (own part) with r = b, x = 0
extern "C" int dgas_shard_begin(dgas_ctx ctx, const double* b, double* red0, void* stream) {
  if (sh_check(ctx) || !b || !red0) return DGAS_E_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  ShardPlan& P = ctx->sh;
  const int64_t np = ctx->np, i0 = P.c_begin[P.rank] * np, i1 = P.c_begin[P.rank + 1] * np;
  launch_perm(ctx, b, ctx->d_b, 1, s);
  k_sh_begin<<<sh_blocks(ctx->N), SH_T, 0, s>>>(ctx->N, ctx->d_b, ctx->d_x, ctx->d_r);
  DGAS_CUDA(cudaMemsetAsync(P.d_state, 0, sizeof(ShState), s));
  k_sh_restrict<<<(ctx->ncoarse + SH_T / 32 - 1) / (SH_T / 32), SH_T, 0, s>>>(
      ctx->ncoarse, ctx->np, ctx->nq, P.c_begin[P.rank], P.c_begin[P.rank + 1], ctx->d_cov_ptr, ctx->d_rrec, ctx->d_G,
      ctx->d_r, red0);
  sh_dot(ctx, i0, i1, ctx->d_r, ctx->d_r, red0 + ctx->N0, s);
  sh_dot(ctx, i0, i1, ctx->d_b, ctx->d_b, red0 + ctx->N0 + 1, s);
  DGAS_CUDA(cudaGetLastError());
  return DGAS_OK;
}

// z = local solves (own subdomains) + Q A0^-1 r0 (own cells), r0 = summed red0[0 .. N0); red1 = r.z (own)
extern "C" int dgas_shard_precond(dgas_ctx ctx, const double* red0, double* red1, void* stream) {
  if (sh_check(ctx) || !red0 || !red1) return DGAS_E_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  ShardPlan& P = ctx->sh;
  const int64_t np = ctx->np, i0 = P.c_begin[P.rank] * np, i1 = P.c_begin[P.rank + 1] * np;
  const int c0 = P.c_begin[P.rank], c1 = P.c_begin[P.rank + 1];
  DGAS_CUDA(cudaMemcpyAsync(ctx->d_r0, red0, ctx->N0 * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (ctx->precond == 0 || ctx->precond == 2) launch_coarse_only(ctx, s);  // replicated coarse solve
  if (ctx->precond == 0 || ctx->precond == 1) {
    launch_local_range(ctx, P.s_begin[P.rank], P.s_begin[P.rank + 1], ctx->d_r, ctx->d_z, s);
  } else {
    const int64_t n = i1 - i0;
    if (ctx->precond == 3) DGAS_CUDA(cudaMemcpyAsync(ctx->d_z + i0, ctx->d_r + i0, n * 8, cudaMemcpyDeviceToDevice, s));
    else DGAS_CUDA(cudaMemsetAsync(ctx->d_z + i0, 0, n * 8, s));
  }
  if (ctx->precond == 0 || ctx->precond == 2)
    k_sh_prolong<<<(unsigned)((i1 - i0 + SH_T - 1) / SH_T), SH_T, 0, s>>>(ctx->np, ctx->nq, c0, c1, ctx->d_fov_ptr,
                                                                          ctx->d_fov, ctx->d_ov_coarse, ctx->d_G,
                                                                          ctx->d_z0, ctx->d_z);
  sh_dot(ctx, i0, i1, ctx->d_r, ctx->d_z, red1, s);
  DGAS_CUDA(cudaGetLastError());
  return DGAS_OK;
}

// beta from the summed r.z (red1), p = z + beta p (own dofs), halo of p packed into hsend [cap]
extern "C" int dgas_shard_direction(dgas_ctx ctx, const double* red1, double* hsend, int32_t first, void* stream) {
  if (sh_check(ctx) || !red1 || !hsend) return DGAS_E_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  ShardPlan& P = ctx->sh;
  const int64_t np = ctx->np, i0 = P.c_begin[P.rank] * np, i1 = P.c_begin[P.rank + 1] * np;
  double* p = ctx->d_p[0];
  k_sh_direction<<<sh_blocks(i1 - i0), SH_T, 0, s>>>(i0, i1, red1, (const ShState*)P.d_state, ctx->d_z, p, first);
  k_sh_dir_state<<<1, 32, 0, s>>>(red1, (ShState*)P.d_state, ctx->d_beta, first);
  if (P.nsend_own > 0)
    k_sh_pack<<<(P.nsend_own * ctx->np + SH_T - 1) / SH_T, SH_T, 0, s>>>(ctx->np, P.nsend_own, P.d_send + P.send_off,
                                                                        p, hsend);
  DGAS_CUDA(cudaGetLastError());
  return DGAS_OK;
}

// halo unpack from hall [nranks][cap], q = A p on the own rows, red2 = p.q (own)
extern "C" int dgas_shard_spmv(dgas_ctx ctx, const double* hall, double* red2, void* stream) {
  if (sh_check(ctx) || !hall || !red2) return DGAS_E_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  ShardPlan& P = ctx->sh;
  const int64_t np = ctx->np, i0 = P.c_begin[P.rank] * np, i1 = P.c_begin[P.rank + 1] * np;
  double* p = ctx->d_p[0];
  if (P.nranks > 1)
    k_sh_unpack<<<dim3(std::max(1, (P.cap + SH_T - 1) / SH_T), P.nranks), SH_T, 0, s>>>(
        ctx->np, P.nranks, P.rank, P.cap, P.d_send_ptr, P.d_send, hall, p);
  launch_spmv_range(ctx, P.c_begin[P.rank], P.c_begin[P.rank + 1], p, ctx->d_q, s);
  sh_dot(ctx, i0, i1, p, ctx->d_q, red2, s);
  DGAS_CUDA(cudaGetLastError());
  return DGAS_OK;
}

// alpha from the summed p.q (red2); x, r update (own); red0 = [Q^T r | r.r] (own); iteration count + 1
extern "C" int dgas_shard_update(dgas_ctx ctx, const double* red2, double* red0, void* stream) {
  if (sh_check(ctx) || !red2 || !red0) return DGAS_E_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  ShardPlan& P = ctx->sh;
  const int64_t np = ctx->np, i0 = P.c_begin[P.rank] * np, i1 = P.c_begin[P.rank + 1] * np;
  k_sh_update<<<sh_blocks(i1 - i0), SH_T, 0, s>>>(i0, i1, red2, (ShState*)P.d_state, ctx->d_alpha, ctx->d_p[0],
                                                   ctx->d_q, ctx->d_x, ctx->d_r);
  k_sh_it<<<1, 32, 0, s>>>((ShState*)P.d_state, 1);
  k_sh_restrict<<<(ctx->ncoarse + SH_T / 32 - 1) / (SH_T / 32), SH_T, 0, s>>>(
      ctx->ncoarse, ctx->np, ctx->nq, P.c_begin[P.rank], P.c_begin[P.rank + 1], ctx->d_cov_ptr, ctx->d_rrec, ctx->d_G,
      ctx->d_r, red0);
  sh_dot(ctx, i0, i1, ctx->d_r, ctx->d_r, red0 + ctx->N0, s);
  DGAS_CUDA(cudaGetLastError());
  return DGAS_OK;
}

// x (caller order, length N): the own dofs of the iterate, zero elsewhere (the caller sums over ranks);
// Lanczos estimate (lmin, lmax, cond) of the first `iters` coefficients into lanczos[3]; status
extern "C" int dgas_shard_finish(dgas_ctx ctx, int32_t iters, double* x, double* lanczos, void* stream) {
  if (sh_check(ctx) || !x || !lanczos || iters < 0) return DGAS_E_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  ShardPlan& P = ctx->sh;
  const int64_t np = ctx->np, i0 = P.c_begin[P.rank] * np, i1 = P.c_begin[P.rank + 1] * np;
  DGAS_CUDA(cudaMemsetAsync(x, 0, ctx->N * sizeof(double), s));
  k_sh_scatter<<<sh_blocks(i1 - i0), SH_T, 0, s>>>(i0, i1, ctx->d_perm_dev, ctx->np, ctx->d_x, x);
  k_sh_lanczos_state<<<1, 32, 0, s>>>(ctx->d_state, iters);
  launch_lanczos(ctx, s);
  DGAS_CUDA(cudaMemcpyAsync(lanczos, ctx->d_lanczos, 3 * sizeof(double), cudaMemcpyDeviceToDevice, s));
  ShState h{};
  DGAS_CUDA(cudaMemcpyAsync(&h, P.d_state, sizeof(ShState), cudaMemcpyDeviceToHost, s));
  DGAS_CUDA(cudaStreamSynchronize(s));
  return h.status;
}

void shard_free(dgas_ctx ctx) {
  ShardPlan& P = ctx->sh;
  for (void* p : {(void*)P.d_send_ptr, (void*)P.d_send, (void*)P.d_partials, P.d_state})
    if (p) cudaFree(p);
  P = ShardPlan();
}
