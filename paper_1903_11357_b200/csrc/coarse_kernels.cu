// coarse_kernels.cu — GPU setup of the coarse correction:
//   * psi_J: degree-q bbox-Legendre products orthonormalised over D_J (R8), Gram summed over the
//     overlap pieces kappa ∩ D_J (signed fan from vertex 0, exact at degree 2q);
//   * G[(kappa,a),(J,b)] = int_{kappa ∩ D_J} phi_a psi_b (eq:R0T; Q = M_h^-1 G = G because the fine
//     basis is orthonormal), exact at degree p+q;
//   * A0 = Q^T A Q (eq:A0), gathered per coarse block pair in a fixed order (deterministic), into
//     CT x CT tile storage (lower tiles only, band-limited when N0 > 8192);
//   * tiled right-looking Cholesky of A0; for dense A0 also the explicit inverse X = L^-T L^-1
//     used by the per-iteration coarse solve (one parallel GEMV instead of a sequential sweep).
#include "internal.h"

#include "dense_cta.cuh"

__device__ inline void piece_point(int k, int m, const double* pxy, int t, const double* glx, const double* glw,
                                   double& x, double& y, double& w) {
  // signed fan triangle (v0, v_t, v_{t+1})
  const double* a = pxy;
  const double* b = pxy + 2 * t;
  const double* c = pxy + 2 * (t + 1);
  int i = k / m, j = k % m;
  double u = 0.5 * (1 + glx[gl_off(m) + i]);
  double v = (1 - u) * 0.5 * (1 + glx[gl_off(m) + j]);
  double j1x = b[0] - a[0], j1y = b[1] - a[1], j2x = c[0] - a[0], j2y = c[1] - a[1];
  double det = j1x * j2y - j2x * j1y;
  x = a[0] + u * j1x + v * j2x;
  y = a[1] + u * j1y + v * j2y;
  w = glw[gl_off(m) + i] * glw[gl_off(m) + j] * (1 - u) * 0.25 * det;
}

#define CCHUNK 64

// ------------------------------------------------------------------ coarse basis psi_J
__global__ void __launch_bounds__(128) k_coarse_basis(int q, const int* cov_ptr, const int* cov, const int* pptr,
                                                      const double* pxy, const int* ctri_ptr, const int* ctri,
                                                      const double* glx, const double* glw, double* Cc,
                                                      double* cbbox, int* err) {
  const int J = blockIdx.x, n = np_of(q), m = q + 1;
  __shared__ double bb[4];
  __shared__ double Gp[CCHUNK][DGAS_MAXNP];
  __shared__ double Wp[CCHUNK];
  __shared__ double M[DGAS_MAXNP * DGAS_MAXNP], T1[DGAS_MAXNP * DGAS_MAXNP], T2[DGAS_MAXNP * DGAS_MAXNP];
  if (threadIdx.x == 0) {
    double x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300;
    for (int k = cov_ptr[J]; k < cov_ptr[J + 1]; ++k) {
      int o = cov[k];
      for (int v = pptr[o]; v < pptr[o + 1]; ++v) {
        x0 = fmin(x0, pxy[2 * v]); x1 = fmax(x1, pxy[2 * v]); y0 = fmin(y0, pxy[2 * v + 1]); y1 = fmax(y1, pxy[2 * v + 1]);
      }
    }
    bb[0] = x0; bb[1] = x1; bb[2] = y0; bb[3] = y1;
    for (int k = 0; k < 4; ++k) cbbox[4 * J + k] = bb[k];
  }
  __syncthreads();
  const int t0 = ctri_ptr[J], ntri = ctri_ptr[J + 1] - t0;
  const int npts = ntri * m * m;
  double acc[8];
  for (int k = 0; k < 8; ++k) acc[k] = 0;
  for (int base = 0; base < npts; base += CCHUNK) {
    int k = base + threadIdx.x;
    if (threadIdx.x >= CCHUNK) {
    } else if (k < npts) {
      int tri = t0 + k / (m * m), r = k % (m * m);
      int o = ctri[2 * tri], t = ctri[2 * tri + 1];
      double x, y, w;
      piece_point(r, m, pxy + 2 * pptr[o], t, glx, glw, x, y, w);
      dev_raw(q, bb, x, y, Gp[threadIdx.x], nullptr, nullptr);
      Wp[threadIdx.x] = w;
    } else {
      Wp[threadIdx.x] = 0;
      for (int a = 0; a < n; ++a) Gp[threadIdx.x][a] = 0;
    }
    __syncthreads();
    int lim = min(CCHUNK, npts - base);
    for (int e = threadIdx.x, s = 0; e < n * n; e += blockDim.x, ++s) {
      int a = e / n, b = e % n;
      double v = 0;
      for (int l = 0; l < lim; ++l) v += Wp[l] * Gp[l][a] * Gp[l][b];
      acc[s] += v;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x, s = 0; e < n * n; e += blockDim.x, ++s) M[e] = acc[s];
  __syncthreads();
  int bad = cta_cholqr2(M, T1, T2, n, Cc + (size_t)J * n * n);
  if (bad && threadIdx.x == 0) atomicExch(&err[3], 1);
}

// ------------------------------------------------------------------ G per overlap piece
__global__ void __launch_bounds__(128) k_G(int p, int q, const int* ov_cell, const int* ov_coarse, const int* pptr,
                                           const double* pxy, const double* glx, const double* glw, const double* C,
                                           const double* bbox, const double* Cc, const double* cbbox, double* G) {
  // collapsed m-point rule is exact for total degree <= 2m-2: m = ceil((p+q)/2) + 1
  const int o = blockIdx.x, n = np_of(p), nqq = np_of(q), m = (p + q + 1) / 2 + 1;
  __shared__ double PH[CCHUNK][DGAS_MAXNP], PS[CCHUNK][DGAS_MAXNP];
  __shared__ double Wp[CCHUNK];
  const int cell = ov_cell[o], J = ov_coarse[o];
  const double* poly = pxy + 2 * pptr[o];
  const int nt = pptr[o + 1] - pptr[o] - 2;
  const int npts = nt * m * m;
  double acc[8];
  for (int k = 0; k < 8; ++k) acc[k] = 0;
  for (int base = 0; base < npts; base += CCHUNK) {
    int k = base + threadIdx.x;
    if (threadIdx.x >= CCHUNK) {
    } else if (k < npts) {
      int t = 1 + k / (m * m), r = k % (m * m);
      double x, y, w;
      piece_point(r, m, poly, t, glx, glw, x, y, w);
      dev_phi(p, n, C + (size_t)cell * n * n, bbox + 4 * cell, x, y, PH[threadIdx.x], nullptr, nullptr);
      dev_phi(q, nqq, Cc + (size_t)J * nqq * nqq, cbbox + 4 * J, x, y, PS[threadIdx.x], nullptr, nullptr);
      Wp[threadIdx.x] = w;
    } else {
      Wp[threadIdx.x] = 0;
      for (int a = 0; a < n; ++a) PH[threadIdx.x][a] = 0;
      for (int a = 0; a < nqq; ++a) PS[threadIdx.x][a] = 0;
    }
    __syncthreads();
    int lim = min(CCHUNK, npts - base);
    for (int e = threadIdx.x, s = 0; e < n * nqq; e += blockDim.x, ++s) {
      int a = e / nqq, b = e % nqq;
      double v = 0;
      for (int l = 0; l < lim; ++l) v += Wp[l] * PH[l][a] * PS[l][b];
      acc[s] += v;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x, s = 0; e < n * nqq; e += blockDim.x, ++s) G[(size_t)o * n * nqq + e] = acc[s];
}

// ------------------------------------------------------------------ A0 = Q^T A Q (tile storage)
__device__ inline double* tile_ptr(double* T, int bt, int I, int K) {
  return T + ((size_t)I * (bt + 1) + (K - I + bt)) * (CT * CT);
}

__global__ void __launch_bounds__(128) k_A0(int n, int nqq, int bt, const int* pair, const int* cptr,
                                            const int4* contrib, const int* nbr_ptr, const int64_t* a_off,
                                            const double* A, const double* G, double* A0t, double* A0b) {
  const int pr = blockIdx.x;
  const int J1 = pair[2 * pr], J2 = pair[2 * pr + 1];
  __shared__ double T[DGAS_MAXNP * DGAS_MAXNP];
  double acc[8];
  for (int k = 0; k < 8; ++k) acc[k] = 0;
  for (int k = cptr[pr]; k < cptr[pr + 1]; ++k) {
    int4 c4 = contrib[k];
    int cell = c4.x, sl = c4.y, o1 = c4.z, o2 = c4.w;
    const double* Ab = A + a_off[cell] + (size_t)sl * n * n;  // column-major block: (a, c) at c * n + a
    const double* G2 = G + (size_t)o2 * n * nqq;
    const double* G1 = G + (size_t)o1 * n * nqq;
    // T = A_ij G_o2  (n x nq)
    for (int e = threadIdx.x; e < n * nqq; e += blockDim.x) {
      int a = e / nqq, b = e % nqq;
      double v = 0;
      for (int c = 0; c < n; ++c) v += Ab[(size_t)c * n + a] * G2[c * nqq + b];
      T[e] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x, s = 0; e < nqq * nqq; e += blockDim.x, ++s) {
      int a = e / nqq, b = e % nqq;
      double v = 0;
      for (int c = 0; c < n; ++c) v += G1[c * nqq + a] * T[c * nqq + b];
      acc[s] += v;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x, s = 0; e < nqq * nqq; e += blockDim.x, ++s) {
    int a = e / nqq, b = e % nqq;
    if (A0b) A0b[(size_t)pr * nqq * nqq + e] = acc[s];
    if (!A0t) continue;
    int r = J1 * nqq + a, c = J2 * nqq + b;
    int I = r / CT, K = c / CT;
    if (K > I || I - K > bt) continue;
    tile_ptr(A0t, bt, I, K)[(r % CT) * CT + (c % CT)] = acc[s];
  }
}

// identity on the padded diagonal (N0 .. nT*CT)
__global__ void k_pad(int64_t N0, int nT, int bt, double* A0t) {
  int64_t r = N0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (int64_t)nT * CT) return;
  int I = (int)(r / CT);
  tile_ptr(A0t, bt, I, I)[(r % CT) * CT + (r % CT)] = 1.0;
}

// ------------------------------------------------------------------ tiled Cholesky
__global__ void __launch_bounds__(256) k_potrf(int K, int bt, double* A0t, double* Dinv0, int* err) {
  __shared__ double S[CT * CT], X[CT * CT];
  double* t = tile_ptr(A0t, bt, K, K);
  for (int e = threadIdx.x; e < CT * CT; e += blockDim.x) S[e] = t[e];
  __syncthreads();
  int bad = cta_chol(S, CT, CT);
  if (bad && threadIdx.x == 0) atomicExch(&err[4], 1 + K);
  cta_trinv(S, X, CT, CT);
  for (int e = threadIdx.x; e < CT * CT; e += blockDim.x) { t[e] = S[e]; Dinv0[(size_t)K * CT * CT + e] = X[e]; }
}

// L_IK = A_IK L_KK^-T for I = K+1 .. K+bt
__global__ void __launch_bounds__(256) k_trsm(int K, int nT, int bt, double* A0t, const double* Dinv0) {
  int I = K + 1 + blockIdx.x;
  if (I >= nT) return;
  __shared__ double S[CT * CT], Li[CT * CT];
  double* t = tile_ptr(A0t, bt, I, K);
  for (int e = threadIdx.x; e < CT * CT; e += blockDim.x) { S[e] = t[e]; Li[e] = Dinv0[(size_t)K * CT * CT + e]; }
  __syncthreads();
  for (int e = threadIdx.x; e < CT * CT; e += blockDim.x) {
    int a = e / CT, b = e % CT;
    double v = 0;
    for (int c = 0; c <= b; ++c) v += S[a * CT + c] * Li[b * CT + c];
    t[e] = v;
  }
}

// A_IJ -= L_IK L_JK^T for K < J <= I <= K+bt
__global__ void __launch_bounds__(256) k_syrk(int K, int nT, int bt, double* A0t) {
  int li = blockIdx.y, lj = blockIdx.x;  // I = K+1+li, J = K+1+lj, lj <= li
  if (lj > li) return;
  int I = K + 1 + li, J = K + 1 + lj;
  if (I >= nT) return;
  __shared__ double X[CT * (CT + 1)], Y[CT * (CT + 1)];
  const double* a = tile_ptr(A0t, bt, I, K);
  const double* b = tile_ptr(A0t, bt, J, K);
  for (int e = threadIdx.x; e < CT * CT; e += blockDim.x) { X[(e / CT) * (CT + 1) + e % CT] = a[e]; Y[(e / CT) * (CT + 1) + e % CT] = b[e]; }
  __syncthreads();
  double* t = tile_ptr(A0t, bt, I, J);
  for (int e = threadIdx.x; e < CT * CT; e += blockDim.x) {
    int r = e / CT, c = e % CT;
    double v = 0;
#pragma unroll 8
    for (int k = 0; k < CT; ++k) v += X[r * (CT + 1) + k] * Y[c * (CT + 1) + k];
    t[e] -= v;
  }
}

// ------------------------------------------------------------------ explicit inverse (dense A0)
// W = L^-1 by tile rows: W_II = Dinv_I, W_IJ = -Dinv_I sum_{K=J}^{I-1} L_IK W_KJ
__global__ void __launch_bounds__(256) k_trtri_row(int I, int bt, const double* A0t, const double* Dinv0, double* Wt) {
  int J = blockIdx.x;
  if (J > I) return;
  __shared__ double S[CT * (CT + 1)], X[CT * (CT + 1)], Acc[CT * CT];
  double* w = tile_ptr(Wt, bt, I, J);
  if (J == I) {
    for (int e = threadIdx.x; e < CT * CT; e += blockDim.x) w[e] = Dinv0[(size_t)I * CT * CT + e];
    return;
  }
  for (int e = threadIdx.x; e < CT * CT; e += blockDim.x) Acc[e] = 0;
  for (int K = J; K < I; ++K) {
    if (I - K > bt) continue;
    const double* l = tile_ptr((double*)A0t, bt, I, K);
    const double* x = tile_ptr(Wt, bt, K, J);
    __syncthreads();
    for (int e = threadIdx.x; e < CT * CT; e += blockDim.x) { S[(e / CT) * (CT + 1) + e % CT] = l[e]; X[(e % CT) * (CT + 1) + e / CT] = x[e]; }
    __syncthreads();
    for (int e = threadIdx.x; e < CT * CT; e += blockDim.x) {
      int r = e / CT, c = e % CT;
      double v = 0;
#pragma unroll 8
      for (int k = 0; k < CT; ++k) v += S[r * (CT + 1) + k] * X[c * (CT + 1) + k];
      Acc[e] += v;
    }
  }
  __syncthreads();
  const double* Di = Dinv0 + (size_t)I * CT * CT;
  for (int e = threadIdx.x; e < CT * CT; e += blockDim.x) {
    int r = e / CT, c = e % CT;
    double v = 0;
    for (int k = 0; k <= r; ++k) v += Di[r * CT + k] * Acc[k * CT + c];
    w[e] = -v;
  }
}

// X_IJ = sum_{K >= I} W_KI^T W_KJ (J <= I), written to the full row-major N0 x N0 matrix (both halves)
__global__ void __launch_bounds__(256) k_lauum(int nT, int bt, int64_t N0, int64_t ldX, const double* Wt, double* X) {
  int I = blockIdx.y, J = blockIdx.x;
  if (J > I) return;
  __shared__ double A[CT * (CT + 1)], B[CT * (CT + 1)];
  double acc[4] = {0, 0, 0, 0};
  for (int K = I; K < nT; ++K) {
    const double* a = tile_ptr((double*)Wt, bt, K, I);
    const double* b = tile_ptr((double*)Wt, bt, K, J);
    __syncthreads();
    for (int e = threadIdx.x; e < CT * CT; e += blockDim.x) { A[(e / CT) * (CT + 1) + e % CT] = a[e]; B[(e / CT) * (CT + 1) + e % CT] = b[e]; }
    __syncthreads();
    for (int e = threadIdx.x, s = 0; e < CT * CT; e += blockDim.x, ++s) {
      int r = e / CT, c = e % CT;
      double v = 0;
#pragma unroll 8
      for (int k = 0; k < CT; ++k) v += A[k * (CT + 1) + r] * B[k * (CT + 1) + c];
      acc[s] += v;
    }
  }
  for (int e = threadIdx.x, s = 0; e < CT * CT; e += blockDim.x, ++s) {
    int64_t r = (int64_t)I * CT + e / CT, c = (int64_t)J * CT + e % CT;
    if (r < N0 && c < N0) { X[r * ldX + c] = acc[s]; X[c * ldX + r] = acc[s]; }
  }
}

// dense path: factor the symmetrically scaled D^-1/2 A0 D^-1/2 (D = diag A0; config-4-like rho
// jumps put kappa(A0) at 8e8 and kappa of the scaled matrix at 9e6) and fold the scaling back into X
__global__ void k_scale_tiles(int64_t N0, int nT, int bt, const double* __restrict__ dsc, double* A0t) {
  const int I = blockIdx.x, K = I - bt + (int)blockIdx.y;
  if (K < 0) return;
  double* t = A0t + ((size_t)I * (bt + 1) + (K - I + bt)) * CT * CT;
  for (int e = threadIdx.x; e < CT * CT; e += blockDim.x) {
    const int64_t r = (int64_t)I * CT + e / CT, c = (int64_t)K * CT + e % CT;
    if (r < N0 && c < N0) t[e] *= dsc[r] * dsc[c];
  }
}
__global__ void k_scale_X(int64_t N0, int64_t ldX, const double* __restrict__ dsc, double* X) {
  const int64_t r = blockIdx.x;
  const double dr = dsc[r];
  for (int64_t c = threadIdx.x; c < N0; c += blockDim.x) X[r * ldX + c] *= dr * dsc[c];
}

// ------------------------------------------------------------------ launcher
int coarse_setup_run(dgas_ctx ctx) {
  cudaStream_t s = ctx->stream;
  const int n = ctx->np, nqq = ctx->nq;
  k_coarse_basis<<<ctx->ncoarse, 128, 0, s>>>(ctx->q, ctx->d_cov_ptr, ctx->d_cov, ctx->d_ov_pptr, ctx->d_ov_xy,
                                               ctx->d_ctri_ptr, ctx->d_ctri, ctx->d_glx, ctx->d_glw, ctx->d_Cc,
                                               ctx->d_cbbox, ctx->d_err);
  DGAS_CUDA(cudaGetLastError());
  k_G<<<ctx->nov, 128, 0, s>>>(ctx->p, ctx->q, ctx->d_ov_cell, ctx->d_ov_coarse, ctx->d_ov_pptr, ctx->d_ov_xy,
                                ctx->d_glx, ctx->d_glw, ctx->d_C, ctx->d_bbox, ctx->d_Cc, ctx->d_cbbox, ctx->d_G);
  DGAS_CUDA(cudaGetLastError());
  if (ctx->n_pairs > 0)
    k_A0<<<(unsigned)ctx->n_pairs, 128, 0, s>>>(n, nqq, ctx->bt, ctx->d_pair, ctx->d_contrib_ptr, ctx->d_contrib,
                                                 ctx->d_nbr_ptr, ctx->d_a_off, ctx->d_A, ctx->d_G,
                                                 ctx->coarse_mode == 2 ? nullptr : ctx->d_A0t, ctx->d_A0b);
  DGAS_CUDA(cudaGetLastError());
  if (ctx->coarse_mode == 2) {
    int st = nd_setup_run(ctx);
    if (st) return st;
    int herr[8];
    DGAS_CUDA(cudaMemcpyAsync(herr, ctx->d_err, sizeof herr, cudaMemcpyDeviceToHost, s));
    DGAS_CUDA(cudaStreamSynchronize(s));
    if (herr[3]) { ctx->detail = "coarse basis Gram not SPD"; return DGAS_E_MESH; }
    if (herr[4]) { ctx->detail = "coarse operator A0 not SPD (nested-dissection front)"; return DGAS_E_NOT_SPD; }
    return 0;
  }
  k_pad<<<1, CT, 0, s>>>(ctx->N0, ctx->nT, ctx->bt, ctx->d_A0t);
  const int nT = ctx->nT, bt = ctx->bt;
  if (ctx->coarse_dense) {
    launch_a0_diag(ctx, ctx->d_prow, ctx->d_dsc0, s);
    k_scale_tiles<<<dim3(nT, bt + 1), 256, 0, s>>>(ctx->N0, nT, bt, ctx->d_dsc0, ctx->d_A0t);
  }
  for (int K = 0; K < nT; ++K) {
    k_potrf<<<1, 256, 0, s>>>(K, bt, ctx->d_A0t, ctx->d_Dinv0, ctx->d_err);
    int nb = std::min(bt, nT - 1 - K);
    if (nb > 0) {
      k_trsm<<<nb, 256, 0, s>>>(K, nT, bt, ctx->d_A0t, ctx->d_Dinv0);
      k_syrk<<<dim3(nb, nb), 256, 0, s>>>(K, nT, bt, ctx->d_A0t);
    }
  }
  DGAS_CUDA(cudaGetLastError());
  if (ctx->coarse_dense) {
    for (int I = 0; I < nT; ++I) k_trtri_row<<<I + 1, 256, 0, s>>>(I, bt, ctx->d_A0t, ctx->d_Dinv0, ctx->d_W);
    k_lauum<<<dim3(nT, nT), 256, 0, s>>>(nT, bt, ctx->N0, ctx->ldX, ctx->d_W, ctx->d_X);
    k_scale_X<<<(unsigned)ctx->N0, 256, 0, s>>>(ctx->N0, ctx->ldX, ctx->d_dsc0, ctx->d_X);
    DGAS_CUDA(cudaGetLastError());
  }
  int herr[8];
  DGAS_CUDA(cudaMemcpyAsync(herr, ctx->d_err, sizeof herr, cudaMemcpyDeviceToHost, s));
  DGAS_CUDA(cudaStreamSynchronize(s));
  if (herr[3]) { ctx->detail = "coarse basis Gram not SPD"; return DGAS_E_MESH; }
  if (herr[4]) { ctx->detail = "coarse operator A0 not SPD (tile " + std::to_string(herr[4] - 1) + ")"; return DGAS_E_NOT_SPD; }
  return 0;
}
