// local_inv.cu — explicit local inverses Z_i = A_i^-1 for the local solves of the additive Schwarz
// preconditioner (exact local solvers; SURVEY.md §8(f) NEXT-4 "explicit
// packed A_i^-1: one read, no chain").
//
// The triangular sweeps of the exact local solve are a chain of 2 x (cells per subdomain) dependent
// steps. On the small configs (1, 2 and config 5 at p = 1) every factor sits in L2 and the chain
// latency is the whole cost (config 2: 52 us for 16 subdomains). There z_i = Z_i r_i is one GEMV per
// subdomain, split into row chunks over many CTAs: no chain at all. Z_i is built at setup by running
// the exact solve (the envelope/panel kernels) on unit vectors, column j of every Z_i in one launch,
// so Z_i is that solver's inverse to rounding. A setup check compares Z r against the exact solve on
// a random r and keeps Z only within 1e-12 relative (ill-conditioned A_i, e.g. rho jumps, fall back).
// Chosen automatically when sum_i n_i^2 * 8 bytes fits the L2 (DGAS_LOCAL_INV=0/1 overrides).
#include <cmath>

#include "internal.h"

#define INV_T 256
#define INV_ROWS 32  // rows of Z_i per work item (4 per warp)

// r = e_j inside every subdomain with n_i > j (r zeroed before)
__global__ void k_inv_unit(int np, int nsub, const int* __restrict__ sub_ptr, int j, double* r) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nsub) return;
  const int n = (sub_ptr[s + 1] - sub_ptr[s]) * np;
  if (j < n) r[(size_t)sub_ptr[s] * np + j] = 1.0;
}

// row j of Z_i (= column j, A_i symmetric) from the solve of A_i z = e_j
__global__ void k_inv_store(int np, const int* __restrict__ sub_ptr, const int64_t* __restrict__ zoff, int j,
                            const double* __restrict__ z, double* Z) {
  const int s = blockIdx.x;
  const int n = (sub_ptr[s + 1] - sub_ptr[s]) * np;
  if (j >= n) return;
  const double* zs = z + (size_t)sub_ptr[s] * np;
  for (int b = threadIdx.x; b < n; b += blockDim.x) Z[zoff[s] + (int64_t)j * n + b] = zs[b];
}

// z_i = Z_i r_i: work items (subdomain, first row), r_i staged in shared memory, warp per row
__global__ void __launch_bounds__(INV_T) k_local_inv(int mode, int np, const int2* __restrict__ items, int nitems,
                                                     const int* __restrict__ sub_ptr,
                                                     const int64_t* __restrict__ zoff, const double* __restrict__ Z,
                                                     const double* r_in, double* const* rbuf, double* z,
                                                     const PcgState* st, const double* qvec) {
  extern __shared__ double rs[];
  // mode 3: residual update fused (r = r_old - alpha q formed while staging, see apply_fuses_restrict)
  const double* r = r_in;
  double alpha = 0;
  const bool fuse = mode == 3;
  if (mode >= 1) {
    if (st->done) return;
    const int it0 = st->it;
    r = mode == 1 ? rbuf[0] : mode == 2 ? rbuf[(it0 + 1) & 1] : rbuf[it0 & 1];
    if (fuse) alpha = st->alpha;
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    if (it != (int)blockIdx.x) __syncthreads();
    const int2 wi = items[it];
    const int s = wi.x, row0 = wi.y;
    const int n = (sub_ptr[s + 1] - sub_ptr[s]) * np;
    const size_t off = (size_t)sub_ptr[s] * np;
    if (fuse) for (int k = threadIdx.x; k < n; k += INV_T) rs[k] = fma(-alpha, qvec[off + k], r[off + k]);
    else for (int k = threadIdx.x; k < n; k += INV_T) rs[k] = r[off + k];
    __syncthreads();
    const double* Zs = Z + zoff[s];
    const int r1 = min(n, row0 + INV_ROWS);
    for (int row = row0 + w; row < r1; row += INV_T / 32) {
      const double* zr = Zs + (int64_t)row * n;
      double v0 = 0, v1 = 0, v2 = 0, v3 = 0;
      int k = lane;
      for (; k + 96 < n; k += 128) {
        v0 += __ldg(zr + k) * rs[k];
        v1 += __ldg(zr + k + 32) * rs[k + 32];
        v2 += __ldg(zr + k + 64) * rs[k + 64];
        v3 += __ldg(zr + k + 96) * rs[k + 96];
      }
      for (; k < n; k += 32) v0 += __ldg(zr + k) * rs[k];
      const double v = warp_sum((v0 + v1) + (v2 + v3));
      if (lane == 0) z[off + row] = v;
    }
  }
}

__global__ void k_inv_testvec(int64_t n, double* v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t x = (uint64_t)i * 0x9e3779b97f4a7c15ULL + 0x1234567ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  x ^= x >> 31;
  v[i] = (double)(x >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

void launch_local_inv(dgas_ctx ctx, int mode, const PcgState* st, const double* r, double* z, cudaStream_t s) {
  const int grid = std::min(ctx->inv_nitems, ctx->inv_grid);
  k_local_inv<<<grid, INV_T, (size_t)ctx->inv_maxn * 8, s>>>(mode, ctx->np, ctx->d_inv_items, ctx->inv_nitems,
                                                             ctx->d_sub_ptr, ctx->d_inv_zoff, ctx->d_inv_Z, r,
                                                             ctx->d_rbuf, z, st, ctx->d_q);
}

// the work items of subdomains [sb, se) only (sharded solve, mode 0)
void launch_local_inv_range(dgas_ctx ctx, int sb, int se, const double* r, double* z, cudaStream_t s) {
  const int i0 = ctx->inv_item_ptr[sb], n = ctx->inv_item_ptr[se] - i0;
  if (n <= 0) return;
  k_local_inv<<<std::min(n, ctx->inv_grid), INV_T, (size_t)ctx->inv_maxn * 8, s>>>(
      0, ctx->np, ctx->d_inv_items + i0, n, ctx->d_sub_ptr, ctx->d_inv_zoff, ctx->d_inv_Z, r, ctx->d_rbuf, z, nullptr, nullptr);
}

// Build Z_i after the local-solve kernel is configured; switch local_kernel to 3 when accepted.
int local_inv_setup(dgas_ctx ctx) {
  if (ctx->max_sub_cells <= 1) return 0;  // one-cell subdomains: k_bjacobi already is the inverse
  const int np = ctx->np, nsub = ctx->nsub;
  const std::vector<int>& sp = ctx->sub_ptr_h;
  std::vector<int64_t> zoff(nsub + 1, 0);
  int maxn = 0;
  for (int s = 0; s < nsub; ++s) {
    const int n = (sp[s + 1] - sp[s]) * np;
    maxn = std::max(maxn, n);
    zoff[s + 1] = zoff[s] + (int64_t)n * n;
  }
  int dev = 0, l2 = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // measured (B200): config 5 p1q1, 75 MB of Z: local 48 -> 19 us; p2q1, 302 MB: 59 -> 68 us (HBM-bound GEMV
  // loses to the L2-resident factor sweeps) -> enabled up to the L2 size
  int want = zoff[nsub] * 8 <= (int64_t)l2 ? 1 : 0;
  bool forced = false;
  if (const char* e = std::getenv("DGAS_LOCAL_INV")) { want = std::atoi(e) != 0; forced = true; }
  if (!want) return 0;
  if ((size_t)maxn * 8 > 96 * 1024) return 0;  // r_i staged in shared memory
  std::vector<int2> items;
  ctx->inv_item_ptr.assign(nsub + 1, 0);
  for (int s = 0; s < nsub; ++s) {
    for (int r0 = 0; r0 < (sp[s + 1] - sp[s]) * np; r0 += INV_ROWS) items.push_back(make_int2(s, r0));
    ctx->inv_item_ptr[s + 1] = (int)items.size();
  }
  int st;
  if ((st = dev_upload(ctx, &ctx->d_inv_zoff, zoff)) || (st = dev_upload(ctx, &ctx->d_inv_items, items))) return st;
  if ((st = dev_alloc(ctx, &ctx->d_inv_Z, (size_t)std::max<int64_t>(1, zoff[nsub])))) return st;
  ctx->inv_nitems = (int)items.size();
  ctx->inv_maxn = maxn;
  ctx->inv_grid = 4 * nsm;
  ctx->inv_bytes = zoff[nsub] * 8;
  DGAS_CUDA(cudaFuncSetAttribute(k_local_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
  cudaStream_t s = ctx->stream;
  double *r = ctx->d_t1, *z = ctx->d_t2;
  for (int j = 0; j < maxn; ++j) {
    DGAS_CUDA(cudaMemsetAsync(r, 0, (size_t)ctx->N * 8, s));
    k_inv_unit<<<(nsub + 255) / 256, 256, 0, s>>>(np, nsub, ctx->d_sub_ptr, j, r);
    launch_local_only(ctx, r, z, s);
    k_inv_store<<<nsub, 128, 0, s>>>(np, ctx->d_sub_ptr, ctx->d_inv_zoff, j, z, ctx->d_inv_Z);
  }
  DGAS_CUDA(cudaGetLastError());
  // accept Z only where it reproduces the exact solve: one random r, relative 2-norm
  double* z2 = nullptr;
  DGAS_CUDA(cudaMalloc((void**)&z2, (size_t)ctx->N * 8));
  k_inv_testvec<<<(unsigned)((ctx->N + 255) / 256), 256, 0, s>>>(ctx->N, r);
  launch_local_only(ctx, r, z, s);
  launch_local_inv(ctx, 0, nullptr, r, z2, s);
  std::vector<double> h1(ctx->N), h2(ctx->N);
  DGAS_CUDA(cudaMemcpyAsync(h1.data(), z, (size_t)ctx->N * 8, cudaMemcpyDeviceToHost, s));
  DGAS_CUDA(cudaMemcpyAsync(h2.data(), z2, (size_t)ctx->N * 8, cudaMemcpyDeviceToHost, s));
  DGAS_CUDA(cudaStreamSynchronize(s));
  cudaFree(z2);
  double e = 0, nn = 0;
  for (int64_t i = 0; i < ctx->N; ++i) { e += (h1[i] - h2[i]) * (h1[i] - h2[i]); nn += h1[i] * h1[i]; }
  ctx->inv_err = std::sqrt(e / std::max(nn, 1e-300));
  if (std::getenv("DGAS_VERBOSE"))
    fprintf(stderr, "dgas: explicit local inverses %.1f MB, Z r vs exact solve %.3e%s\n", ctx->inv_bytes / 1e6,
            ctx->inv_err, ctx->inv_err <= 1e-12 || forced ? "" : " (rejected)");
  if (!(ctx->inv_err <= 1e-12) && !forced) {
    cudaFree(ctx->d_inv_Z); cudaFree(ctx->d_inv_zoff); cudaFree(ctx->d_inv_items);
    ctx->d_inv_Z = nullptr; ctx->d_inv_zoff = nullptr; ctx->d_inv_items = nullptr;
    ctx->inv_bytes = 0;
    return 0;
  }
  ctx->local_kernel = 3;
  return 0;
}
