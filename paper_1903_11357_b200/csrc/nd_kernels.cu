// nd_kernels.cu — multifrontal nested-dissection factorisation and solve of the coarse operator
// A0 = Q^T A Q (eq:A0) for large N0 (see nd_host.cu for the plan).
//   setup, per tree level (deepest first), one CTA per front:
//     S = [S_FF S_FU; S_UF S_UU] = A0 restricted to (F, F u U) + extend-add of the children's updates
//     X_F = S_FF^-1 (Cholesky, triangular inverse, L^-T L^-1),  B_F = S_UF L^-T,  M_F = B_F L^-1,
//     update_F = S_UU - B_F B_F^T  (passed to the parent)
//   solve, per level: forward u_F = t_U - M_F t_F (t = r0|_F + children's u), backward
//     x_F = X_F t_F - M_F^T x_U. Every level is one launch of GEMV rows (row chunks per CTA).
#include "internal.h"

#define ND_T 256
#define ND_ROWS 16  // rows of a front per CTA in the solve
#define ND_RW (ND_ROWS / (ND_T / 32))  // rows per warp, computed together

// Solve-phase operator loads (X_F, M_F, M_F^T) carry an L2 evict-last policy: the chain of level
// launches is latency-bound and runs beside the HBM-saturating local solves, so it should find its
// factors in L2 (the streamed SpMV / local-solve copies are evict-first). DGAS_ND_L2=0 disables it.
__device__ __forceinline__ double ld_keep(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t nd_policy(int keep) {
  uint64_t pol;
  if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// ------------------------------------------------------------------ setup: assemble front matrices
__global__ void __launch_bounds__(ND_T) k_nd_assemble(int nq, const int* __restrict__ fronts, const int* nF, const int* nU,
                                                      const int64_t* offS, const int64_t* offUpd, const int* asm_ptr,
                                                      const int4* asmv, const int* childptr, const int* childs,
                                                      const int* cmap_ptr, const int* cmap, const double* A0b,
                                                      const int* __restrict__ pair, const double* __restrict__ dsc,
                                                      const double* Upd, double* Sg) {
  const int f = fronts[blockIdx.x];
  const int n = nF[f] + nU[f], nFe = nF[f] / nq;
  double* S = Sg + offS[f];
  for (int64_t e = threadIdx.x; e < (int64_t)n * n; e += ND_T) S[e] = 0.0;
  __syncthreads();
  const int nq2 = nq * nq;
  for (int e = threadIdx.x; e < (asm_ptr[f + 1] - asm_ptr[f]) * nq2; e += ND_T) {
    const int4 a4 = asmv[asm_ptr[f] + e / nq2];
    const int ab = e % nq2, a = ab / nq, b = ab % nq;
    // symmetric diagonal scaling D^-1/2 A0 D^-1/2 (see nd_setup_run)
    const double v = A0b[(size_t)a4.x * nq2 + ab] * dsc[(size_t)pair[2 * a4.x] * nq + a] *
                     dsc[(size_t)pair[2 * a4.x + 1] * nq + b];
    S[(size_t)(a4.y * nq + a) * n + a4.z * nq + b] = v;
    if (a4.z >= nFe) S[(size_t)(a4.z * nq + b) * n + a4.y * nq + a] = v;
  }
  __syncthreads();
  for (int ci = childptr[f]; ci < childptr[f + 1]; ++ci) {
    const int c = childs[ci];
    const int nuc = nU[c];
    const double* Uc = Upd + offUpd[c];
    const int* mp = cmap + cmap_ptr[ci];
    for (int64_t e = threadIdx.x; e < (int64_t)nuc * nuc; e += ND_T) {
      const int a = (int)(e / nuc), b = (int)(e % nuc);
      const int la = mp[a / nq] * nq + a % nq, lb = mp[b / nq] * nq + b % nq;
      S[(size_t)la * n + lb] += Uc[e];
    }
    __syncthreads();
  }
}

// dsc[J nq + a] = diag(A0)^-1/2 (the diagonal entry of the (J, J) pair block)
__global__ void k_nd_diag(int ncoarse, int nq, const int* __restrict__ prow, const int* __restrict__ pair,
                          const double* __restrict__ A0b, double* dsc) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ncoarse * nq) return;
  const int J = g / nq, a = g % nq;
  double d = 1.0;
  for (int pr = prow[J]; pr < prow[J + 1]; ++pr)
    if (pair[2 * pr + 1] == J) d = A0b[((size_t)pr * nq + a) * nq + a];
  dsc[g] = d > 0 ? 1.0 / sqrt(d) : 1.0;  // a non-positive pivot is reported by the factorisation
}

// ------------------------------------------------------------------ setup: partial factorisation
__global__ void __launch_bounds__(ND_T) k_nd_factor(const int* __restrict__ fronts, const int* nF, const int* nU,
                                                    const int64_t* offS, const int64_t* offX, const int64_t* offM,
                                                    const int64_t* offUpd, double* Sg, double* Xg, double* Mg,
                                                    double* MTg, double* Upd, int* err) {
  const int f = fronts[blockIdx.x];
  const int nf = nF[f], nu = nU[f], n = nf + nu;
  double* S = Sg + offS[f];
  double* L = Xg + offX[f];  // Cholesky factor, later overwritten by X
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  for (int64_t e = threadIdx.x; e < (int64_t)nf * nf; e += ND_T) L[e] = S[(e / nf) * n + e % nf];
  __syncthreads();
  // right-looking Cholesky of S_FF (lower, in L)
  for (int j = 0; j < nf; ++j) {
    if (threadIdx.x == 0) {
      double d = L[(size_t)j * nf + j];
      if (!(d > 0)) { bad = 1; d = 1.0; }
      L[(size_t)j * nf + j] = sqrt(d);
    }
    __syncthreads();
    const double d = L[(size_t)j * nf + j];
    for (int i = j + 1 + threadIdx.x; i < nf; i += ND_T) L[(size_t)i * nf + j] /= d;
    __syncthreads();
    const int m = nf - j - 1;
    for (int64_t e = threadIdx.x; e < (int64_t)m * m; e += ND_T) {
      const int i = j + 1 + (int)(e / m), k = j + 1 + (int)(e % m);
      if (k <= i) L[(size_t)i * nf + k] -= L[(size_t)i * nf + j] * L[(size_t)k * nf + j];
    }
    __syncthreads();
  }
  if (bad && threadIdx.x == 0) atomicExch(&err[4], 1);
  // W = L^-1 into the S_FF block of S (no longer needed), column per thread
  for (int c = threadIdx.x; c < nf; c += ND_T) {
    for (int i = 0; i < c; ++i) S[(size_t)i * n + c] = 0.0;
    for (int i = c; i < nf; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = c; k < i; ++k) s -= L[(size_t)i * nf + k] * S[(size_t)k * n + c];
      S[(size_t)i * n + c] = s / L[(size_t)i * nf + i];
    }
  }
  __syncthreads();
  // X = W^T W (symmetric, full)
  double* X = L;
  for (int64_t e = threadIdx.x; e < (int64_t)nf * nf; e += ND_T) {
    const int i = (int)(e / nf), j = (int)(e % nf);
    double s = 0;
    for (int k = max(i, j); k < nf; ++k) s += S[(size_t)k * n + i] * S[(size_t)k * n + j];
    X[e] = s;
  }
  __syncthreads();
  // B = S_UF W^T = S_UF L^-T (nu x nf), held in the M^T buffer as B^T until M is formed. The Schur
  // update S_UU - B B^T is formed without the explicit inverse: S_UF X S_UF^T carried the
  // kappa(S_FF) eps error of X into every ancestor front (coarse-solve error on config 5 p = q = 6:
  // 1.8e-9 that way, 9e-12 this way).
  double* M = Mg + offM[f];
  double* MT = MTg + offM[f];
  for (int64_t e = threadIdx.x; e < (int64_t)nu * nf; e += ND_T) {
    const int r = (int)(e / nf), j = (int)(e % nf);
    const double* srow = S + (size_t)(nf + r) * n;
    double s = 0;
    for (int k = 0; k <= j; ++k) s += srow[k] * S[(size_t)j * n + k];  // W[j][k], k <= j
    MT[(size_t)j * nu + r] = s;
  }
  __syncthreads();
  // update = S_UU - B B^T  (nu x nu)
  double* Up = Upd + offUpd[f];
  for (int64_t e = threadIdx.x; e < (int64_t)nu * nu; e += ND_T) {
    const int r = (int)(e / nu), t = (int)(e % nu);
    double s = S[(size_t)(nf + r) * n + nf + t];
    for (int j = 0; j < nf; ++j) s -= MT[(size_t)j * nu + r] * MT[(size_t)j * nu + t];
    Up[e] = s;
  }
  // M = B W = S_UF S_FF^-1 (nu x nf) for the solve
  for (int64_t e = threadIdx.x; e < (int64_t)nu * nf; e += ND_T) {
    const int r = (int)(e / nf), j = (int)(e % nf);
    double s = 0;
    for (int k = j; k < nf; ++k) s += MT[(size_t)k * nu + r] * S[(size_t)k * n + j];  // W[k][j], k >= j
    M[e] = s;
  }
  __syncthreads();
  for (int64_t e = threadIdx.x; e < (int64_t)nu * nf; e += ND_T) {
    const int r = (int)(e / nf), j = (int)(e % nf);
    MT[(size_t)j * nu + r] = M[e];
  }
}

// ------------------------------------------------------------------ solve: forward level
// work item (front, first row of U); t assembled in shared memory by every CTA of the front
__global__ void __launch_bounds__(ND_T) k_nd_fwd(int nq, const int2* __restrict__ work, int nwork, const int* __restrict__ nF,
                                                 const int* __restrict__ nU, const int* __restrict__ offT,
                                                 const int* __restrict__ offu, const int* __restrict__ offFe,
                                                 const int* __restrict__ Fe, const int64_t* __restrict__ offM,
                                                 const int* __restrict__ childptr, const int* __restrict__ childs,
                                                 const int* __restrict__ cmap_ptr, const int* __restrict__ cmap,
                                                 const double* __restrict__ Mg, const double* __restrict__ dsc,
                                                 const double* r0, double* Tg, double* ug, const PcgState* st,
                                                 int mode, int keep) {
  extern __shared__ double t[];
  const uint64_t pol = nd_policy(keep);
  if (mode >= 1 && st->done) return;
  // grid-stride over the level's work items: a level runs in one wave of at most nd_grid CTAs, which
  // fit beside the local-solve CTAs the coarse chain runs concurrently with
  for (int wk = blockIdx.x; wk < nwork; wk += gridDim.x) {
  if (wk != (int)blockIdx.x) __syncthreads();  // t of the previous item fully consumed
  const int2 wi = work[wk];
  const int f = wi.x, row0 = wi.y;
  const int nf = nF[f], nu = nU[f];
  for (int k = threadIdx.x; k < nf; k += ND_T) {
    const size_t g = (size_t)Fe[offFe[f] + k / nq] * nq + k % nq;
    t[k] = r0[g] * dsc[g];
  }
  for (int k = nf + threadIdx.x; k < nf + nu; k += ND_T) t[k] = 0.0;
  __syncthreads();
  for (int ci = childptr[f]; ci < childptr[f + 1]; ++ci) {
    const int c = childs[ci];
    const double* uc = ug + offu[c];
    const int* mp = cmap + cmap_ptr[ci];
    for (int a = threadIdx.x; a < nU[c]; a += ND_T) t[mp[a / nq] * nq + a % nq] += uc[a];
    __syncthreads();
  }
  if (row0 == 0)
    for (int k = threadIdx.x; k < nf; k += ND_T) Tg[offT[f] + k] = t[k];
  // GEMV rows: each warp owns ND_RW rows and keeps ND_RW x 4 loads in flight per lane (a level is a
  // short dependent chain: memory latency, not bandwidth, sets its time)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* M = Mg + offM[f];
  const int rend = min(nu, row0 + ND_ROWS);
  const double* mr[ND_RW];
  double v[ND_RW];
#pragma unroll
  for (int i = 0; i < ND_RW; ++i) {
    const int r = row0 + w + (ND_T / 32) * i;
    mr[i] = M + (size_t)(r < rend ? r : row0) * nf;
    v[i] = 0.0;
  }
  for (int k0 = 0; k0 < nf; k0 += 128) {
    double tk[4], a[ND_RW][4];
    int kk[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = k0 + lane + 32 * u;
      kk[u] = min(k, nf - 1);
      tk[u] = k < nf ? t[k] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < ND_RW; ++i)
#pragma unroll
      for (int u = 0; u < 4; ++u) a[i][u] = ld_keep(mr[i] + kk[u], pol);
#pragma unroll
    for (int i = 0; i < ND_RW; ++i)
#pragma unroll
      for (int u = 0; u < 4; ++u) v[i] += a[i][u] * tk[u];
  }
#pragma unroll
  for (int i = 0; i < ND_RW; ++i) {
    const int r = row0 + w + (ND_T / 32) * i;
    const double vv = warp_sum(v[i]);
    if (lane == 0 && r < rend) ug[offu[f] + r] = t[nf + r] - vv;
  }
  }
}

// ------------------------------------------------------------------ solve: backward level
__global__ void __launch_bounds__(ND_T) k_nd_bwd(int nq, const int2* __restrict__ work, int nwork, const int* __restrict__ nF,
                                                 const int* __restrict__ nU, const int* __restrict__ offT,
                                                 const int* __restrict__ offFe, const int* __restrict__ Fe,
                                                 const int* __restrict__ offUe, const int* __restrict__ Ue,
                                                 const int64_t* __restrict__ offX, const int64_t* __restrict__ offM,
                                                 const double* __restrict__ Xg, const double* __restrict__ MTg,
                                                 const double* __restrict__ dsc, const double* Tg, double* z0,
                                                 const PcgState* st, int mode, int keep) {
  extern __shared__ double sh[];
  const uint64_t pol = nd_policy(keep);
  if (mode >= 1 && st->done) return;
  for (int wk = blockIdx.x; wk < nwork; wk += gridDim.x) {  // grid-stride (see k_nd_fwd)
  if (wk != (int)blockIdx.x) __syncthreads();
  const int2 wi = work[wk];
  const int f = wi.x, row0 = wi.y;
  const int nf = nF[f], nu = nU[f];
  double* tF = sh;
  double* xU = sh + nf;
  for (int k = threadIdx.x; k < nf; k += ND_T) tF[k] = Tg[offT[f] + k];
  for (int k = threadIdx.x; k < nu; k += ND_T) {
    const size_t g = (size_t)Ue[offUe[f] + k / nq] * nq + k % nq;
    xU[k] = -z0[g] / dsc[g];  // the scaled unknown of an ancestor front (negated: one dot product)
  }
  __syncthreads();
  // row j: x_F[j] = sum_k X[j][k] tF[k] + sum_k MT[j][k] (-x_U[k]) over the concatenated k in [0, nf + nu)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* X = Xg + offX[f];
  const double* MT = MTg + offM[f];
  const int rend = min(nf, row0 + ND_ROWS), nk = nf + nu;
  const double* xr[ND_RW];
  const double* mr[ND_RW];
  double v[ND_RW];
#pragma unroll
  for (int i = 0; i < ND_RW; ++i) {
    const int j = row0 + w + (ND_T / 32) * i, jj = j < rend ? j : row0;
    xr[i] = X + (size_t)jj * nf;
    mr[i] = MT + (size_t)jj * nu - nf;
    v[i] = 0.0;
  }
  for (int k0 = 0; k0 < nk; k0 += 128) {
    double sk[4], a[ND_RW][4];
    int kk[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = k0 + lane + 32 * u;
      kk[u] = min(k, nk - 1);
      sk[u] = k < nk ? sh[k] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < ND_RW; ++i)
#pragma unroll
      for (int u = 0; u < 4; ++u) a[i][u] = ld_keep((kk[u] < nf ? xr[i] : mr[i]) + kk[u], pol);
#pragma unroll
    for (int i = 0; i < ND_RW; ++i)
#pragma unroll
      for (int u = 0; u < 4; ++u) v[i] += a[i][u] * sk[u];
  }
#pragma unroll
  for (int i = 0; i < ND_RW; ++i) {
    const int j = row0 + w + (ND_T / 32) * i;
    const double vv = warp_sum(v[i]);
    if (lane == 0 && j < rend) {
      const size_t g = (size_t)Fe[offFe[f] + j / nq] * nq + j % nq;
      z0[g] = vv * dsc[g];
    }
  }
  }
}

// ------------------------------------------------------------------ host launchers
template <typename T>
static int up(dgas_ctx ctx, T** d, const std::vector<T>& h) {
  DGAS_CUDA(cudaMalloc((void**)d, std::max<size_t>(1, h.size()) * sizeof(T)));
  if (!h.empty()) DGAS_CUDA(cudaMemcpyAsync(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  return 0;
}

static int nd_v2_build(dgas_ctx ctx);

int nd_setup_run(dgas_ctx ctx) {
  NdPlan& P = ctx->nd;
  cudaStream_t s = ctx->stream;
  int st = 0;
  if ((st = up(ctx, &P.d_nF, P.h_nF)) || (st = up(ctx, &P.d_nU, P.h_nU)) || (st = up(ctx, &P.d_offX, P.h_offX)) ||
      (st = up(ctx, &P.d_offM, P.h_offM)) || (st = up(ctx, &P.d_offUpd, P.h_offUpd)) ||
      (st = up(ctx, &P.d_offS, P.h_offS)) || (st = up(ctx, &P.d_offT, P.h_offT)) || (st = up(ctx, &P.d_offu, P.h_offu)) ||
      (st = up(ctx, &P.d_offFe, P.h_offFe)) || (st = up(ctx, &P.d_offUe, P.h_offUe)) || (st = up(ctx, &P.d_Fe, P.h_Fe)) ||
      (st = up(ctx, &P.d_Ue, P.h_Ue)) || (st = up(ctx, &P.d_childptr, P.h_childptr)) ||
      (st = up(ctx, &P.d_childs, P.h_childs)) || (st = up(ctx, &P.d_cmap_ptr, P.h_cmap_ptr)) ||
      (st = up(ctx, &P.d_cmap, P.h_cmap)) || (st = up(ctx, &P.d_asm_ptr, P.h_asm_ptr)) || (st = up(ctx, &P.d_asm, P.h_asm)) ||
      (st = up(ctx, &P.d_lev_fronts, P.h_lev_fronts)) || (st = up(ctx, &P.d_prow, P.h_prow)))
    return st;
  const int nf = P.nf;
  // D^-1/2 of diag(A0): the fronts factor the symmetrically scaled D^-1/2 A0 D^-1/2, whose conditioning
  // does not carry the rho contrast (config 4: 1e8) into the explicit front inverses
  DGAS_CUDA(cudaMalloc((void**)&P.d_dsc, std::max<int64_t>(1, ctx->N0) * 8));
  k_nd_diag<<<(unsigned)((ctx->N0 + 255) / 256), 256, 0, s>>>(ctx->ncoarse, ctx->nq, P.d_prow, ctx->d_pair,
                                                             ctx->d_A0b, P.d_dsc);
  DGAS_CUDA(cudaMalloc((void**)&P.d_X, std::max<int64_t>(1, P.h_offX[nf]) * 8));
  DGAS_CUDA(cudaMalloc((void**)&P.d_M, std::max<int64_t>(1, P.h_offM[nf]) * 8));
  DGAS_CUDA(cudaMalloc((void**)&P.d_MT, std::max<int64_t>(1, P.h_offM[nf]) * 8));
  DGAS_CUDA(cudaMalloc((void**)&P.d_T, std::max<int>(1, P.h_offT[nf]) * 8));
  DGAS_CUDA(cudaMalloc((void**)&P.d_u, std::max<int>(1, P.h_offu[nf]) * 8));
  double *dS = nullptr, *dUpd = nullptr;
  DGAS_CUDA(cudaMalloc((void**)&dS, std::max<int64_t>(1, P.h_offS[nf]) * 8));
  DGAS_CUDA(cudaMalloc((void**)&dUpd, std::max<int64_t>(1, P.h_offUpd[nf]) * 8));
  for (int L = 0; L < P.nlev; ++L) {
    const int n = P.h_lev_ptr[L + 1] - P.h_lev_ptr[L];
    if (!n) continue;
    const int* fr = P.d_lev_fronts + P.h_lev_ptr[L];
    k_nd_assemble<<<n, ND_T, 0, s>>>(ctx->nq, fr, P.d_nF, P.d_nU, P.d_offS, P.d_offUpd, P.d_asm_ptr, P.d_asm, P.d_childptr,
                                     P.d_childs, P.d_cmap_ptr, P.d_cmap, ctx->d_A0b, ctx->d_pair, P.d_dsc, dUpd, dS);
    k_nd_factor<<<n, ND_T, 0, s>>>(fr, P.d_nF, P.d_nU, P.d_offS, P.d_offX, P.d_offM, P.d_offUpd, dS, P.d_X, P.d_M, P.d_MT,
                                   dUpd, ctx->d_err);
  }
  DGAS_CUDA(cudaGetLastError());
  // per-level work lists (front, first row) for the solve kernels
  std::vector<int2> wf, wb;
  P.h_wf_ptr.assign(P.nlev + 1, 0);
  P.h_wb_ptr.assign(P.nlev + 1, 0);
  for (int L = 0; L < P.nlev; ++L) {
    for (int k = P.h_lev_ptr[L]; k < P.h_lev_ptr[L + 1]; ++k) {
      const int f = P.h_lev_fronts[k];
      for (int r = 0; r < std::max(1, P.h_nU[f]); r += ND_ROWS) wf.push_back(make_int2(f, r));
      for (int r = 0; r < P.h_nF[f]; r += ND_ROWS) wb.push_back(make_int2(f, r));
    }
    P.h_wf_ptr[L + 1] = (int)wf.size();
    P.h_wb_ptr[L + 1] = (int)wb.size();
  }
  if (std::getenv("DGAS_VERBOSE")) {
    for (int L = 0; L < P.nlev; ++L) {
      int mf = 0, mu = 0;
      int64_t by = 0;
      for (int k = P.h_lev_ptr[L]; k < P.h_lev_ptr[L + 1]; ++k) {
        const int f = P.h_lev_fronts[k];
        mf = std::max(mf, P.h_nF[f]); mu = std::max(mu, P.h_nU[f]);
        by += ((int64_t)P.h_nF[f] * P.h_nF[f] + 2 * (int64_t)P.h_nF[f] * P.h_nU[f]) * 8;
      }
      fprintf(stderr, "dgas: ND level %d: %d fronts, max nF %d, max nU %d, %.2f MB, work fwd %d bwd %d\n", L,
              P.h_lev_ptr[L + 1] - P.h_lev_ptr[L], mf, mu, by / 1e6, P.h_wf_ptr[L + 1] - P.h_wf_ptr[L],
              P.h_wb_ptr[L + 1] - P.h_wb_ptr[L]);
    }
  }
  if ((st = up(ctx, &P.d_wf, wf)) || (st = up(ctx, &P.d_wb, wb))) return st;
  DGAS_CUDA(cudaMalloc((void**)&P.d_rb, (ctx->N0 + 1) * 8));
  DGAS_CUDA(cudaMalloc((void**)&P.d_zb, (ctx->N0 + 1) * 8));
  DGAS_CUDA(cudaStreamSynchronize(s));
  cudaFree(dS);
  cudaFree(dUpd);
  P.bytes = (P.h_offX[nf] + 2 * P.h_offM[nf]) * 8;
  P.v2 = 1;
  if (const char* e = std::getenv("DGAS_ND_V2")) P.v2 = std::atoi(e) != 0;
  P.pdl = 1;
  if (const char* e = std::getenv("DGAS_ND_PDL")) P.pdl = std::atoi(e) != 0;
  if (P.v2) {
    const int r = nd_v2_build(ctx);
    if (r < 0) return -r;
    if (r > 0) P.v2 = 0;
  }
  if (!P.v2) P.pdl = 0;
  return 0;
}


// ------------------------------------------------------------------ solve v2
// Same arithmetic as k_nd_fwd / k_nd_bwd (the t assembly adds r0 dsc, then child 1, then child 2),
// with fewer dependent memory rounds per level: one 64-byte descriptor per work item, the global
// indices of F and U precomputed (gF, gU), and for every position of t the child-u sources (tsrc).
// With programmatic dependent launch (DGAS_ND_PDL) a level's CTAs start while the previous level runs
// and load their static tables before griddepcontrol.wait.
struct __align__(16) NdItem {
  int f, row0, nf, nu;
  int offT, offu, gofs, sofs;
  long long offM, offX;
  int gUofs, pad0, pad1, pad2;
};

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

__global__ void __launch_bounds__(ND_T) k_nd_fwd2(const NdItem* __restrict__ items, int nwork, const int* __restrict__ gF,
                                                  const int2* __restrict__ tsrc, const double* __restrict__ Mg,
                                                  const double* __restrict__ dsc, const double* r0, double* Tg,
                                                  double* ug, const PcgState* st, int mode, int keep) {
  extern __shared__ double t[];
  pdl_launch();
  const uint64_t pol = nd_policy(keep);
  if (mode >= 1 && st->done) return;
  bool waited = false;
  for (int wk = blockIdx.x; wk < nwork; wk += gridDim.x) {
    if (wk != (int)blockIdx.x) __syncthreads();
    const NdItem it = items[wk];
    const int nf = it.nf, nu = it.nu, n = nf + nu;
    constexpr int KPT = 4;  // positions per thread held across the wait (n <= KPT * ND_T handled in one pass)
    int gk[KPT];
    int2 sk[KPT];
    for (int k0 = 0; k0 < n; k0 += KPT * ND_T) {
#pragma unroll
      for (int u = 0; u < KPT; ++u) {
        const int k = k0 + threadIdx.x + u * ND_T;
        gk[u] = k < nf ? gF[it.gofs + k] : -1;
        sk[u] = k < n ? tsrc[it.sofs + k] : make_int2(-1, -1);
      }
      if (!waited) { pdl_wait(); waited = true; }
#pragma unroll
      for (int u = 0; u < KPT; ++u) {
        const int k = k0 + threadIdx.x + u * ND_T;
        if (k < n) {
          double v = gk[u] >= 0 ? r0[gk[u]] * dsc[gk[u]] : 0.0;
          if (sk[u].x >= 0) v += ug[sk[u].x];
          if (sk[u].y >= 0) v += ug[sk[u].y];
          t[k] = v;
        }
      }
    }
    __syncthreads();
    if (it.row0 == 0)
      for (int k = threadIdx.x; k < nf; k += ND_T) Tg[it.offT + k] = t[k];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double* M = Mg + it.offM;
    const int row0 = it.row0, rend = min(nu, row0 + ND_ROWS);
    const double* mr[ND_RW];
    double v[ND_RW];
#pragma unroll
    for (int i = 0; i < ND_RW; ++i) {
      const int r = row0 + w + (ND_T / 32) * i;
      mr[i] = M + (size_t)(r < rend ? r : row0) * nf;
      v[i] = 0.0;
    }
    for (int k0 = 0; k0 < nf; k0 += 128) {
      double tk[4], a[ND_RW][4];
      int kk[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + lane + 32 * u;
        kk[u] = min(k, nf - 1);
        tk[u] = k < nf ? t[k] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < ND_RW; ++i)
#pragma unroll
        for (int u = 0; u < 4; ++u) a[i][u] = ld_keep(mr[i] + kk[u], pol);
#pragma unroll
      for (int i = 0; i < ND_RW; ++i)
#pragma unroll
        for (int u = 0; u < 4; ++u) v[i] += a[i][u] * tk[u];
    }
#pragma unroll
    for (int i = 0; i < ND_RW; ++i) {
      const int r = row0 + w + (ND_T / 32) * i;
      const double vv = warp_sum(v[i]);
      if (lane == 0 && r < rend) ug[it.offu + r] = t[nf + r] - vv;
    }
  }
  if (!waited) pdl_wait();
}

__global__ void __launch_bounds__(ND_T, 6) k_nd_bwd2(const NdItem* __restrict__ items, int nwork, const int* __restrict__ gF,
                                                  const int* __restrict__ gU, const double* __restrict__ Xg,
                                                  const double* __restrict__ MTg, const double* __restrict__ dsc,
                                                  const double* Tg, double* z0, const PcgState* st, int mode, int keep) {
  extern __shared__ double sh[];
  pdl_launch();
  const uint64_t pol = nd_policy(keep);
  if (mode >= 1 && st->done) return;
  bool waited = false;
  for (int wk = blockIdx.x; wk < nwork; wk += gridDim.x) {
    if (wk != (int)blockIdx.x) __syncthreads();
    const NdItem it = items[wk];
    const int nf = it.nf, nu = it.nu, nk = nf + nu;
    constexpr int KPT = 4;
    int gk[KPT];
    for (int k0 = 0; k0 < nk; k0 += KPT * ND_T) {
#pragma unroll
      for (int u = 0; u < KPT; ++u) {
        const int k = k0 + threadIdx.x + u * ND_T;
        gk[u] = (k >= nf && k < nk) ? gU[it.gUofs + k - nf] : -1;
      }
      if (!waited) { pdl_wait(); waited = true; }
#pragma unroll
      for (int u = 0; u < KPT; ++u) {
        const int k = k0 + threadIdx.x + u * ND_T;
        if (k < nf) sh[k] = Tg[it.offT + k];
        else if (k < nk) sh[k] = -z0[gk[u]] / dsc[gk[u]];  // scaled unknown of an ancestor front, negated
      }
    }
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double* X = Xg + it.offX;
    const double* MT = MTg + it.offM;
    const int row0 = it.row0, rend = min(nf, row0 + ND_ROWS);
    const double* xr[ND_RW];
    const double* mr[ND_RW];
    double v[ND_RW];
#pragma unroll
    for (int i = 0; i < ND_RW; ++i) {
      const int j = row0 + w + (ND_T / 32) * i, jj = j < rend ? j : row0;
      xr[i] = X + (size_t)jj * nf;
      mr[i] = MT + (size_t)jj * nu - nf;
      v[i] = 0.0;
    }
    for (int k0 = 0; k0 < nk; k0 += 128) {
      double sk[4], a[ND_RW][4];
      int kk[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + lane + 32 * u;
        kk[u] = min(k, nk - 1);
        sk[u] = k < nk ? sh[k] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < ND_RW; ++i)
#pragma unroll
        for (int u = 0; u < 4; ++u) a[i][u] = ld_keep((kk[u] < nf ? xr[i] : mr[i]) + kk[u], pol);
#pragma unroll
      for (int i = 0; i < ND_RW; ++i)
#pragma unroll
        for (int u = 0; u < 4; ++u) v[i] += a[i][u] * sk[u];
    }
#pragma unroll
    for (int i = 0; i < ND_RW; ++i) {
      const int j = row0 + w + (ND_T / 32) * i;
      const double vv = warp_sum(v[i]);
      if (lane == 0 && j < rend) {
        const int g = gF[it.gofs + j];
        z0[g] = vv * dsc[g];
      }
    }
  }
  if (!waited) pdl_wait();
}

// host tables of the v2 solve (after nd_setup_run's plan upload); 0 = built, 1 = not applicable
static int nd_v2_build(dgas_ctx ctx) {
  NdPlan& P = ctx->nd;
  const int nq = ctx->nq;
  std::vector<int> gF, gU, gofs(P.nf), gUofs(P.nf), sofs(P.nf);
  std::vector<int2> tsrc;
  for (int f = 0; f < P.nf; ++f) {
    const int nf = P.h_nF[f], nu = P.h_nU[f];
    gofs[f] = (int)gF.size();
    for (int k = 0; k < nf; ++k) gF.push_back(P.h_Fe[P.h_offFe[f] + k / nq] * nq + k % nq);
    gUofs[f] = (int)gU.size();
    for (int k = 0; k < nu; ++k) gU.push_back(P.h_Ue[P.h_offUe[f] + k / nq] * nq + k % nq);
    sofs[f] = (int)tsrc.size();
    std::vector<int2> src(nf + nu, make_int2(-1, -1));
    for (int ci = P.h_childptr[f]; ci < P.h_childptr[f + 1]; ++ci) {
      const int c = P.h_childs[ci];
      for (int a = 0; a < P.h_nU[c]; ++a) {
        const int pos = P.h_cmap[P.h_cmap_ptr[ci] + a / nq] * nq + a % nq;
        int2& sp = src[pos];
        if (sp.x < 0) sp.x = P.h_offu[c] + a;
        else if (sp.y < 0) sp.y = P.h_offu[c] + a;
        else return 1;  // more than two contributions to one position: keep the v1 kernels
      }
    }
    tsrc.insert(tsrc.end(), src.begin(), src.end());
  }
  auto item = [&](int f, int row0) {
    NdItem it{};
    it.f = f; it.row0 = row0; it.nf = P.h_nF[f]; it.nu = P.h_nU[f];
    it.offT = P.h_offT[f]; it.offu = P.h_offu[f]; it.gofs = gofs[f]; it.sofs = sofs[f];
    it.offM = P.h_offM[f]; it.offX = P.h_offX[f]; it.gUofs = gUofs[f];
    return it;
  };
  std::vector<NdItem> wf, wb;
  for (int L = 0; L < P.nlev; ++L)
    for (int k = P.h_lev_ptr[L]; k < P.h_lev_ptr[L + 1]; ++k) {
      const int f = P.h_lev_fronts[k];
      for (int r = 0; r < std::max(1, P.h_nU[f]); r += ND_ROWS) wf.push_back(item(f, r));
      for (int r = 0; r < P.h_nF[f]; r += ND_ROWS) wb.push_back(item(f, r));
    }
  int st;
  if ((st = up(ctx, &P.d_gF, gF)) || (st = up(ctx, &P.d_gU, gU)) || (st = up(ctx, &P.d_tsrc, tsrc))) return -st;
  NdItem *dwf = nullptr, *dwb = nullptr;
  if ((st = up(ctx, &dwf, wf)) || (st = up(ctx, &dwb, wb))) return -st;
  P.d_wf2 = dwf;
  P.d_wb2 = dwb;
  return 0;
}

template <typename K, typename... Args>
static void nd_launch(bool pdl, K kern, int grid, size_t smem, cudaStream_t s, Args... args) {
  if (!pdl) {
    kern<<<grid, ND_T, smem, s>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(ND_T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}

static void nd_solve_once_v2(dgas_ctx ctx, int mode, const PcgState* st, cudaStream_t s, const double* rin, double* zout) {
  NdPlan& P = ctx->nd;
  const size_t shf = (size_t)P.maxN * 8, shb = (size_t)(P.maxF + P.maxU) * 8;
  const NdItem* wf = static_cast<const NdItem*>(P.d_wf2);
  const NdItem* wb = static_cast<const NdItem*>(P.d_wb2);
  bool first = true;  // the first level of a chain waits for the restriction (another stream): plain launch
  for (int L = 0; L < P.nlev; ++L) {
    const int n = P.h_wf_ptr[L + 1] - P.h_wf_ptr[L];
    if (!n) continue;
    nd_launch(P.pdl && !first, k_nd_fwd2, std::min(n, ctx->nd_grid), shf, s, wf + P.h_wf_ptr[L], n,
              (const int*)P.d_gF, (const int2*)P.d_tsrc, (const double*)P.d_M, (const double*)P.d_dsc, rin, P.d_T,
              P.d_u, st, mode, ctx->nd_l2);
    first = false;
  }
  for (int L = P.nlev - 1; L >= 0; --L) {
    const int n = P.h_wb_ptr[L + 1] - P.h_wb_ptr[L];
    if (!n) continue;
    nd_launch(P.pdl && !first, k_nd_bwd2, std::min(n, ctx->nd_grid), shb, s, wb + P.h_wb_ptr[L], n,
              (const int*)P.d_gF, (const int*)P.d_gU, (const double*)P.d_X, (const double*)P.d_MT,
              (const double*)P.d_dsc, (const double*)P.d_T, zout, st, mode, ctx->nd_l2);
    first = false;
  }
}

// res = b - A0 z  (coarse block rows, warp per coarse element; A0 blocks per coupled pair)
__global__ void __launch_bounds__(ND_T) k_a0_resid(int ncoarse, int nq, const int* __restrict__ prow,
                                                   const int* __restrict__ pair, const double* __restrict__ A0b,
                                                   const double* b, const double* z, double* res, const PcgState* st,
                                                   int mode) {
  if (mode >= 1 && st->done) return;
  const int J = blockIdx.x * (ND_T / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (J >= ncoarse) return;
  for (int a = 0; a < nq; ++a) {
    double v = 0;
    for (int e = lane; e < (prow[J + 1] - prow[J]) * nq; e += 32) {
      const int pr = prow[J] + e / nq, bcol = e % nq;
      v += A0b[((size_t)pr * nq + a) * nq + bcol] * z[(size_t)pair[2 * pr + 1] * nq + bcol];
    }
    v = warp_sum(v);
    if (lane == 0) res[(size_t)J * nq + a] = b[(size_t)J * nq + a] - v;
  }
}

__global__ void k_axpy_add(int64_t n, const double* a, double* y, const PcgState* st, int mode) {
  if (mode >= 1 && st->done) return;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] += a[i];
}

static void nd_solve_once(dgas_ctx ctx, int mode, const PcgState* st, cudaStream_t s, const double* rin, double* zout);

void launch_a0_diag(dgas_ctx ctx, const int* prow, double* dsc, cudaStream_t s) {
  k_nd_diag<<<(unsigned)((ctx->N0 + 255) / 256), 256, 0, s>>>(ctx->ncoarse, ctx->nq, prow, ctx->d_pair, ctx->d_A0b, dsc);
}
void launch_a0_resid(dgas_ctx ctx, const int* prow, const double* b, const double* z, double* res, const PcgState* st,
                     int mode, cudaStream_t s) {
  const int nb = (ctx->ncoarse + ND_T / 32 - 1) / (ND_T / 32);
  k_a0_resid<<<nb, ND_T, 0, s>>>(ctx->ncoarse, ctx->nq, prow, ctx->d_pair, ctx->d_A0b, b, z, res, st, mode);
}
void launch_axpy_add(int64_t n, const double* a, double* y, const PcgState* st, int mode, cudaStream_t s) {
  k_axpy_add<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, a, y, st, mode);
}

void nd_solve_launch(dgas_ctx ctx, int mode, const PcgState* st, cudaStream_t s) {
  nd_solve_once(ctx, mode, st, s, ctx->d_r0, ctx->d_z0);
  for (int it = 0; it < ctx->nd.refine; ++it) {  // iterative refinement (R30)
    const int nb = (ctx->ncoarse + ND_T / 32 - 1) / (ND_T / 32);
    k_a0_resid<<<nb, ND_T, 0, s>>>(ctx->ncoarse, ctx->nq, ctx->nd.d_prow, ctx->d_pair, ctx->d_A0b, ctx->d_r0,
                                   ctx->d_z0, ctx->nd.d_rb, st, mode);
    nd_solve_once(ctx, mode, st, s, ctx->nd.d_rb, ctx->nd.d_zb);
    k_axpy_add<<<(unsigned)((ctx->N0 + 255) / 256), 256, 0, s>>>(ctx->N0, ctx->nd.d_zb, ctx->d_z0, st, mode);
  }
}

static void nd_solve_once(dgas_ctx ctx, int mode, const PcgState* st, cudaStream_t s, const double* rin, double* zout) {
  NdPlan& P = ctx->nd;
  if (P.v2) { nd_solve_once_v2(ctx, mode, st, s, rin, zout); return; }
  const size_t shf = (size_t)P.maxN * 8, shb = (size_t)(P.maxF + P.maxU) * 8;
  for (int L = 0; L < P.nlev; ++L) {
    const int n = P.h_wf_ptr[L + 1] - P.h_wf_ptr[L];
    if (n)
      k_nd_fwd<<<std::min(n, ctx->nd_grid), ND_T, shf, s>>>(ctx->nq, P.d_wf + P.h_wf_ptr[L], n, P.d_nF, P.d_nU, P.d_offT, P.d_offu, P.d_offFe,
                                    P.d_Fe, P.d_offM, P.d_childptr, P.d_childs, P.d_cmap_ptr, P.d_cmap, P.d_M, P.d_dsc,
                                    rin, P.d_T, P.d_u, st, mode, ctx->nd_l2);
  }
  for (int L = P.nlev - 1; L >= 0; --L) {
    const int n = P.h_wb_ptr[L + 1] - P.h_wb_ptr[L];
    if (n)
      k_nd_bwd<<<std::min(n, ctx->nd_grid), ND_T, shb, s>>>(ctx->nq, P.d_wb + P.h_wb_ptr[L], n, P.d_nF, P.d_nU, P.d_offT, P.d_offFe, P.d_Fe,
                                    P.d_offUe, P.d_Ue, P.d_offX, P.d_offM, P.d_X, P.d_MT, P.d_dsc, P.d_T, zout, st,
                                    mode, ctx->nd_l2);
  }
}

// deterministic test vector in [-1, 1) (splitmix of the index)
__global__ void k_nd_testvec(int64_t n, double* v) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t z = (uint64_t)i * 0x9e3779b97f4a7c15ULL + 0x632be59bd9b4e019ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  z ^= z >> 31;
  v[i] = (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

// Choose the iterative-refinement steps of the multifrontal coarse solve (R30):
// solve A0 z = A0 v for a fixed test vector v; while its relative error ||z - v|| / ||v|| exceeds
// nd_tol = 3e-11, add refinement steps as long as each one cuts the error by at least 4x (at most 2).
// Measured on config 4 (kappa(A0) = 8e8, 9e6 after diagonal scaling): LAPACK Cholesky 5.8e-11,
// explicit dense inverse 3.5e-6, this solve 2.9e-10, with one refinement step 2.4e-11. The step doubles
// the coarse chain, which then sticks out of the local solves on config 4 (2100 -> 1826 PCG it/s);
// configs 3 and 5 (4e-12, 1.2e-11) need none. A persistent dependency-driven single-launch solve and
// a 4-rows-per-warp GEMV were tried for this and measured slower (beside the local solves only one
// 256-thread CTA per SM fits, and both designs hold fewer loads in flight than this one).
// shared by both coarse paths: solve A0 z = A0 v (r0 = -A0 v, expect z = -v) with `refine` steps
static int coarse_calibrate_impl(dgas_ctx ctx, const int* prow, int* refine_out, double* err_out, double* err0_out,
                                 int* refine_ctl, void (*solve)(dgas_ctx, cudaStream_t)) {
  cudaStream_t s = ctx->stream;
  const int64_t n = ctx->N0;
  double *dv = nullptr, *dzero = nullptr;
  DGAS_CUDA(cudaMalloc((void**)&dv, n * 8));
  DGAS_CUDA(cudaMalloc((void**)&dzero, n * 8));
  DGAS_CUDA(cudaMemsetAsync(dzero, 0, n * 8, s));
  k_nd_testvec<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, dv);
  std::vector<double> hv(n), hz(n);
  DGAS_CUDA(cudaMemcpyAsync(hv.data(), dv, n * 8, cudaMemcpyDeviceToHost, s));
  auto measure = [&](int refine) -> double {
    *refine_ctl = refine;
    launch_a0_resid(ctx, prow, dzero, dv, ctx->d_r0, nullptr, 0, s);
    solve(ctx, s);
    if (cudaMemcpyAsync(hz.data(), ctx->d_z0, n * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess) return -1;
    if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
    double e = 0, vv = 0;
    for (int64_t i = 0; i < n; ++i) { e += (hz[i] + hv[i]) * (hz[i] + hv[i]); vv += hv[i] * hv[i]; }
    return std::sqrt(e / vv);
  };
  double err = measure(0);
  *err0_out = err;
  int best = 0;
  for (int r = 1; r <= 2 && err > ctx->nd_tol; ++r) {
    const double e = measure(r);
    if (!(e >= 0) || !(e < 0.25 * err)) break;
    err = e;
    best = r;
  }
  *refine_ctl = best;
  *refine_out = best;
  *err_out = err;
  cudaFree(dv);
  cudaFree(dzero);
  DGAS_CUDA(cudaMemsetAsync(ctx->d_z0, 0, n * 8, s));
  DGAS_CUDA(cudaGetLastError());
  return err >= 0 ? 0 : DGAS_E_CUDA;
}

static void nd_solve_plain(dgas_ctx ctx, cudaStream_t s) { nd_solve_launch(ctx, 0, nullptr, s); }
static void dense_solve_plain(dgas_ctx ctx, cudaStream_t s) { launch_coarse_dense(ctx, 0, nullptr, ctx->d_r0, ctx->d_z0, s); }

int nd_calibrate(dgas_ctx ctx) {
  NdPlan& P = ctx->nd;
  if (P.refine_env >= 0) return 0;
  int r = 0;
  int st = coarse_calibrate_impl(ctx, P.d_prow, &r, &P.calib_err, &P.calib_err0, &P.refine, nd_solve_plain);
  if (std::getenv("DGAS_VERBOSE"))
    fprintf(stderr, "dgas: ND coarse solve relerr %.3e unrefined, %.3e with %d refinement step(s)\n", P.calib_err0,
            P.calib_err, P.refine);
  return st;
}

int dense_calibrate(dgas_ctx ctx) {
  int r = 0;
  int st = coarse_calibrate_impl(ctx, ctx->d_prow, &r, &ctx->dense_err, &ctx->dense_err0, &ctx->dense_refine,
                                 dense_solve_plain);
  if (const char* e = std::getenv("DGAS_DENSE_REFINE")) ctx->dense_refine = std::max(0, std::atoi(e));
  if (std::getenv("DGAS_VERBOSE"))
    fprintf(stderr, "dgas: dense coarse solve relerr %.3e unrefined, %.3e with %d refinement step(s)\n",
            ctx->dense_err0, ctx->dense_err, ctx->dense_refine);
  return st;
}

int nd_set_smem(dgas_ctx ctx) {
  NdPlan& P = ctx->nd;
  const size_t shf = (size_t)P.maxN * 8, shb = (size_t)(P.maxF + P.maxU) * 8;
  int dev = 0, mx = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // The limit is a per-function (process-wide) attribute shared by every context: raise it to the
  // opt-in maximum rather than this context's front size, so a later context with smaller fronts
  // never lowers it under an earlier one's launches (or its instantiated PCG graph).
  cudaFuncAttributes ff{}, fb{};
  DGAS_CUDA(cudaFuncGetAttributes(&ff, k_nd_fwd));
  DGAS_CUDA(cudaFuncGetAttributes(&fb, k_nd_bwd));
  if (shf + ff.sharedSizeBytes > (size_t)mx || shb + fb.sharedSizeBytes > (size_t)mx) {
    ctx->detail = "nested-dissection front too large for shared memory";
    return DGAS_E_INVALID_ARG;
  }
  DGAS_CUDA(cudaFuncSetAttribute(k_nd_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, mx - (int)ff.sharedSizeBytes));
  DGAS_CUDA(cudaFuncSetAttribute(k_nd_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, mx - (int)fb.sharedSizeBytes));
  return 0;
}

void nd_free(dgas_ctx ctx) {
  NdPlan& P = ctx->nd;
  void* ptrs[] = {P.d_nF, P.d_nU, P.d_offX, P.d_offM, P.d_offUpd, P.d_offS, P.d_offT, P.d_offu, P.d_offFe, P.d_offUe,
                  P.d_Fe, P.d_Ue, P.d_childptr, P.d_childs, P.d_cmap_ptr, P.d_cmap, P.d_asm_ptr, P.d_asm,
                  P.d_lev_fronts, P.d_X, P.d_M, P.d_MT, P.d_T, P.d_u, P.d_wf, P.d_wb, P.d_prow, P.d_rb, P.d_zb,
                  P.d_dsc, P.d_wf2, P.d_wb2, P.d_gF, P.d_gU, P.d_tsrc};
  for (void* p : ptrs)
    if (p) cudaFree(p);
}
