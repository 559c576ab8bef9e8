// setup_kernels.cu — GPU setup: Gauss–Legendre table, per-cell orthonormal bases, SIPDG assembly
// (volume / face / deterministic row gather), right-hand side, and the envelope block Cholesky of
// every subdomain block A_i. Runs once per dgas_setup.
#include <cmath>

#include "internal.h"
#include "dense_cta.cuh"

// ------------------------------------------------------------------ Gauss–Legendre by Newton
__global__ void k_gauss_legendre(double* gx, double* gw) {
  int m = blockIdx.x + 1, i = threadIdx.x;
  if (i >= m) return;
  const double pi = 3.14159265358979323846;
  double x = cos(pi * (i + 0.75) / (m + 0.5));
  double dP = 1;
  for (int it = 0; it < 100; ++it) {
    double P0 = 1, P1 = x;
    for (int n = 1; n < m; ++n) { double P2 = ((2 * n + 1) * x * P1 - n * P0) / (n + 1); P0 = P1; P1 = P2; }
    if (m == 1) { P1 = x; P0 = 1; }
    dP = m * (x * P1 - P0) / (x * x - 1);
    double dx = P1 / dP;
    x -= dx;
    if (fabs(dx) < 1e-17) break;
  }
  {
    double P0 = 1, P1 = x;
    for (int n = 1; n < m; ++n) { double P2 = ((2 * n + 1) * x * P1 - n * P0) / (n + 1); P0 = P1; P1 = P2; }
    if (m == 1) { P1 = x; P0 = 1; }
    dP = m * (x * P1 - P0) / (x * x - 1);
  }
  // ascending order
  gx[gl_off(m) + (m - 1 - i)] = x;
  gw[gl_off(m) + (m - 1 - i)] = 2.0 / ((1 - x * x) * dP * dP);
}

// point k of the fan rule with m x m collapsed points per triangle (apex, v_t, v_{t+1})
__device__ inline void fan_point(int k, int m, const double* apex, const double* va, const double* vb,
                                 const double* glx, const double* glw, double& x, double& y, double& w) {
  int i = k / m, j = k % m;
  double u = 0.5 * (1 + glx[gl_off(m) + i]);
  double v = (1 - u) * 0.5 * (1 + glx[gl_off(m) + j]);
  double j1x = va[0] - apex[0], j1y = va[1] - apex[1], j2x = vb[0] - apex[0], j2y = vb[1] - apex[1];
  double det = j1x * j2y - j2x * j1y;
  x = apex[0] + u * j1x + v * j2x;
  y = apex[1] + u * j1y + v * j2y;
  w = glw[gl_off(m) + i] * glw[gl_off(m) + j] * (1 - u) * 0.25 * det;
}

#define MAXV 64
#define CHUNK 64

// ------------------------------------------------------------------ basis (R6)
__global__ void __launch_bounds__(128) k_basis(int p, const int* cptr, const double* cxy, const double* glx,
                                               const double* glw, double* Cout, double* bbox, double* hk, int* err) {
  const int c = blockIdx.x, n = np_of(p), m = p + 1;
  __shared__ double V[2 * MAXV];
  __shared__ double sh[8];  // bbox, apex
  __shared__ double Gp[CHUNK][DGAS_MAXNP];
  __shared__ double Wp[CHUNK];
  __shared__ double M[DGAS_MAXNP * DGAS_MAXNP], T1[DGAS_MAXNP * DGAS_MAXNP], T2[DGAS_MAXNP * DGAS_MAXNP];
  const int v0 = cptr[c], nv = cptr[c + 1] - v0;
  for (int k = threadIdx.x; k < 2 * nv; k += blockDim.x) V[k] = cxy[2 * v0 + k];
  __syncthreads();
  if (threadIdx.x == 0) {
    double x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300, ax = 0, ay = 0, h = 0;
    for (int k = 0; k < nv; ++k) {
      x0 = fmin(x0, V[2 * k]); x1 = fmax(x1, V[2 * k]); y0 = fmin(y0, V[2 * k + 1]); y1 = fmax(y1, V[2 * k + 1]);
      ax += V[2 * k]; ay += V[2 * k + 1];
      for (int l = k + 1; l < nv; ++l) h = fmax(h, hypot(V[2 * k] - V[2 * l], V[2 * k + 1] - V[2 * l + 1]));
    }
    sh[0] = x0; sh[1] = x1; sh[2] = y0; sh[3] = y1; sh[4] = ax / nv; sh[5] = ay / nv;
    hk[c] = h;  // h_kappa = diameter (R1)
    for (int k = 0; k < 4; ++k) bbox[4 * c + k] = sh[k];
  }
  __syncthreads();
  // Gram of the raw basis over the centroid fan (exact at degree 2p with m = p+1)
  const int npts = nv * m * m;
  double acc[8];
  for (int k = 0; k < 8; ++k) acc[k] = 0;
  for (int base = 0; base < npts; base += CHUNK) {
    int k = base + threadIdx.x;
    if (threadIdx.x >= CHUNK) {
    } else if (k < npts) {
      int t = k / (m * m), r = k % (m * m);
      double x, y, w;
      fan_point(r, m, &sh[4], &V[2 * t], &V[2 * ((t + 1) % nv)], glx, glw, x, y, w);
      dev_raw(p, sh, x, y, Gp[threadIdx.x], nullptr, nullptr);
      Wp[threadIdx.x] = w;
    } else {
      Wp[threadIdx.x] = 0;
      for (int a = 0; a < n; ++a) Gp[threadIdx.x][a] = 0;
    }
    __syncthreads();
    int lim = min(CHUNK, npts - base);
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
  int bad = cta_cholqr2(M, T1, T2, n, Cout + (size_t)c * n * n);
  if (bad && threadIdx.x == 0) atomicExch(err, 1);
}

// ------------------------------------------------------------------ assembly: volume blocks
__global__ void __launch_bounds__(128) k_volume(int p, const int* cptr, const double* cxy, const double* glx,
                                                const double* glw, const double* Cg, const double* bbox,
                                                const double* kappa, double* vol) {
  const int c = blockIdx.x, n = np_of(p), m = p + 1;
  __shared__ double V[2 * MAXV];
  __shared__ double sh[8];
  __shared__ double C[DGAS_MAXNP * DGAS_MAXNP];
  __shared__ double PX[CHUNK][DGAS_MAXNP], PY[CHUNK][DGAS_MAXNP];
  __shared__ double Wp[CHUNK];
  const int v0 = cptr[c], nv = cptr[c + 1] - v0;
  for (int k = threadIdx.x; k < 2 * nv; k += blockDim.x) V[k] = cxy[2 * v0 + k];
  for (int k = threadIdx.x; k < n * n; k += blockDim.x) C[k] = Cg[(size_t)c * n * n + k];
  if (threadIdx.x < 4) sh[threadIdx.x] = bbox[4 * c + threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    double ax = 0, ay = 0;
    for (int k = 0; k < nv; ++k) { ax += V[2 * k]; ay += V[2 * k + 1]; }
    sh[4] = ax / nv; sh[5] = ay / nv;
  }
  __syncthreads();
  const double rho = kappa[c];
  const int npts = nv * m * m;
  double acc[8];
  for (int k = 0; k < 8; ++k) acc[k] = 0;
  for (int base = 0; base < npts; base += CHUNK) {
    int k = base + threadIdx.x;
    if (threadIdx.x >= CHUNK) {
    } else if (k < npts) {
      int t = k / (m * m), r = k % (m * m);
      double x, y, w, phi[DGAS_MAXNP];
      fan_point(r, m, &sh[4], &V[2 * t], &V[2 * ((t + 1) % nv)], glx, glw, x, y, w);
      dev_phi(p, n, C, sh, x, y, phi, PX[threadIdx.x], PY[threadIdx.x]);
      Wp[threadIdx.x] = w;
    } else {
      Wp[threadIdx.x] = 0;
      for (int a = 0; a < n; ++a) PX[threadIdx.x][a] = PY[threadIdx.x][a] = 0;
    }
    __syncthreads();
    int lim = min(CHUNK, npts - base);
    for (int e = threadIdx.x, s = 0; e < n * n; e += blockDim.x, ++s) {
      int a = e / n, b = e % n;
      double v = 0;
      for (int l = 0; l < lim; ++l) v += Wp[l] * (PX[l][a] * PX[l][b] + PY[l][a] * PY[l][b]);
      acc[s] += v;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x, s = 0; e < n * n; e += blockDim.x, ++s) vol[(size_t)c * n * n + e] = rho * acc[s];
}

// ------------------------------------------------------------------ assembly: face blocks
// Face form of eq:Ah. Interior face, test side s, trial side t
// (eps_+ = 1, eps_- = -1, n from kappa+ to kappa-, W = <rho>/2 = omega rho+ = (1-omega) rho-):
//   B^{st}_{ab} = int_F sigma eps_s eps_t phi^t_b phi^s_a - W (eps_s d_n phi^t_b phi^s_a + eps_t d_n phi^s_a phi^t_b)
// Boundary face: int_F sigma phi_b phi_a - rho (d_n phi_b phi_a + d_n phi_a phi_b), n outward.
__global__ void __launch_bounds__(128) k_face(int p, double Cs, const int* fcells, const double* fxy,
                                              const double* glx, const double* glw, const double* Cg,
                                              const double* bbox, const double* kappa, const double* hk,
                                              double* fblk) {
  const int f = blockIdx.x, n = np_of(p), m = p + 1;
  __shared__ double PH[2][DGAS_MAXP + 1][DGAS_MAXNP], DN[2][DGAS_MAXP + 1][DGAS_MAXNP];
  __shared__ double Wq[DGAS_MAXP + 1];
  const int kp = fcells[2 * f], km = fcells[2 * f + 1];
  const double ax = fxy[4 * f], ay = fxy[4 * f + 1], bx = fxy[4 * f + 2], by = fxy[4 * f + 3];
  const double len = hypot(bx - ax, by - ay);
  const double nx = (by - ay) / len, ny = -(bx - ax) / len;
  const int nsides = km < 0 ? 1 : 2;
  // evaluate basis values and normal derivatives at the m Gauss points, for each side
  for (int e = threadIdx.x; e < nsides * m; e += blockDim.x) {
    int s = e / m, g = e % m;
    int cell = s == 0 ? kp : km;
    double t = 0.5 * (1 + glx[gl_off(m) + g]);
    double x = ax + t * (bx - ax), y = ay + t * (by - ay);
    double px[DGAS_MAXNP], py[DGAS_MAXNP];
    dev_phi(p, n, Cg + (size_t)cell * n * n, bbox + 4 * cell, x, y, PH[s][g], px, py);
    for (int a = 0; a < n; ++a) DN[s][g][a] = px[a] * nx + py[a] * ny;
    if (s == 0) Wq[g] = 0.5 * glw[gl_off(m) + g] * len;
  }
  __syncthreads();
  const double p2 = (double)p * p;
  double* out = fblk + (size_t)f * 4 * n * n;
  if (km < 0) {
    const double rho = kappa[kp];
    const double sigma = Cs * rho * p2 / hk[kp];
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      int a = e / n, b = e % n;
      double v = 0;
      for (int g = 0; g < m; ++g)
        v += Wq[g] * (sigma * PH[0][g][b] * PH[0][g][a] - rho * (DN[0][g][b] * PH[0][g][a] + DN[0][g][a] * PH[0][g][b]));
      out[e] = v;
    }
  } else {
    const double rp = kappa[kp], rm = kappa[km];
    const double rho_h = 2 * rp * rm / (rp + rm), h_h = 2 * hk[kp] * hk[km] / (hk[kp] + hk[km]);
    const double sigma = Cs * rho_h * p2 / h_h;  // eq:Sigma
    const double W = 0.5 * rho_h;
    for (int e = threadIdx.x; e < 4 * n * n; e += blockDim.x) {
      int blk = e / (n * n), r = e % (n * n), a = r / n, b = r % n;
      int s = blk >> 1, t = blk & 1;
      double es = s ? -1.0 : 1.0, et = t ? -1.0 : 1.0;
      double v = 0;
      for (int g = 0; g < m; ++g)
        v += Wq[g] * (sigma * es * et * PH[t][g][b] * PH[s][g][a] - W * (es * DN[t][g][b] * PH[s][g][a] + et * DN[s][g][a] * PH[t][g][b]));
      out[e] = v;
    }
  }
}

// ------------------------------------------------------------------ assembly: deterministic row gather
__global__ void __launch_bounds__(128) k_gather_rows(int n, const int* nbr_ptr, const int* nbr, const int64_t* a_off,
                                                     const int* cf_ptr, const int* cf, const int* fcells,
                                                     const double* vol, const double* fblk, double* A) {
  const int c = blockIdx.x;
  const int deg = nbr_ptr[c + 1] - nbr_ptr[c];
  const int W = deg * n;
  double* row = A + a_off[c];
  for (int e = threadIdx.x; e < n * W; e += blockDim.x) {
    int a = e / W, col = e % W, sl = col / n, b = col % n;
    int j = nbr[nbr_ptr[c] + sl];
    double v = 0;
    if (j == c) v = vol[(size_t)c * n * n + a * n + b];
    for (int k = cf_ptr[c]; k < cf_ptr[c + 1]; ++k) {
      int f = cf[k] >> 1, side = cf[k] & 1;
      int other = fcells[2 * f + (1 - side)];
      if (j == c) v += fblk[((size_t)f * 4 + side * 3) * n * n + a * n + b];
      else if (other == j) v += fblk[((size_t)f * 4 + side * 2 + (1 - side)) * n * n + a * n + b];
    }
    row[(size_t)col * n + a] = v;  // column-major row-block
  }
}

// ------------------------------------------------------------------ right-hand side (R10: m = p + 4)
__global__ void __launch_bounds__(128) k_rhs(int p, int f_kind, const int* cptr, const double* cxy, const double* glx,
                                             const double* glw, const double* Cg, const double* bbox, double* b) {
  const int c = blockIdx.x, n = np_of(p), m = p + 4;
  __shared__ double V[2 * MAXV];
  __shared__ double sh[8];
  __shared__ double PH[CHUNK][DGAS_MAXNP];
  __shared__ double Wf[CHUNK];
  const int v0 = cptr[c], nv = cptr[c + 1] - v0;
  for (int k = threadIdx.x; k < 2 * nv; k += blockDim.x) V[k] = cxy[2 * v0 + k];
  if (threadIdx.x < 4) sh[threadIdx.x] = bbox[4 * c + threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    double ax = 0, ay = 0;
    for (int k = 0; k < nv; ++k) { ax += V[2 * k]; ay += V[2 * k + 1]; }
    sh[4] = ax / nv; sh[5] = ay / nv;
  }
  __syncthreads();
  const double* C = Cg + (size_t)c * n * n;
  const int npts = nv * m * m;
  double acc = 0;
  const double pi = 3.14159265358979323846;
  for (int base = 0; base < npts; base += CHUNK) {
    int k = base + threadIdx.x;
    if (threadIdx.x >= CHUNK) {
    } else if (k < npts) {
      int t = k / (m * m), r = k % (m * m);
      double x, y, w;
      fan_point(r, m, &sh[4], &V[2 * t], &V[2 * ((t + 1) % nv)], glx, glw, x, y, w);
      double f = f_kind == 0 ? 2 * pi * pi * sin(pi * x) * sin(pi * y) : f_kind == 1 ? 1.0 : 2 * (x * (1 - x) + y * (1 - y));
      dev_phi(p, n, C, sh, x, y, PH[threadIdx.x], nullptr, nullptr);
      Wf[threadIdx.x] = w * f;
    } else {
      Wf[threadIdx.x] = 0;
      for (int a = 0; a < n; ++a) PH[threadIdx.x][a] = 0;
    }
    __syncthreads();
    if (threadIdx.x < n) {
      int lim = min(CHUNK, npts - base);
      for (int l = 0; l < lim; ++l) acc += Wf[l] * PH[l][threadIdx.x];
    }
    __syncthreads();
  }
  if (threadIdx.x < n) b[(size_t)c * n + threadIdx.x] = acc;
}

// ------------------------------------------------------------------ local envelope Cholesky
// A_i = L L^T in block-envelope (profile) storage: row-block k holds L_kj for j in [f_k, k) as an
// n x ((k - f_k) n) row-major panel; the fill of a profile Cholesky stays inside the envelope.
// After factorisation each row-block is scaled to U_kj = L_kk^-1 L_kj and Dinv_k = L_kk^-1.
__global__ void __launch_bounds__(256) k_local_factor(int n, const int* sub_ptr, const int* first, const int64_t* u_off,
                                                      const int* nbr_ptr, const int* nbr, const int64_t* a_off,
                                                      const double* A, double* U, double* Dinv, int* err) {
  const int s = blockIdx.x, s0 = sub_ptr[s], m = sub_ptr[s + 1] - s0;
  const int nn = n * n;
  __shared__ double S[DGAS_MAXNP * DGAS_MAXNP], Li[DGAS_MAXNP * DGAS_MAXNP];
  for (int k = 0; k < m; ++k) {
    const int gk = s0 + k, fk = first[gk];
    const int Wk = (k - fk) * n;
    double* Lk = U + u_off[gk];
    // A row of gk
    const int lo = nbr_ptr[gk], deg = nbr_ptr[gk + 1] - lo;
    const double* Ak = A + a_off[gk];
    for (int j = fk; j < k; ++j) {
      const int gj = s0 + j, fj = first[gj];
      const double* Lj = U + u_off[gj];
      int sl = -1;
      for (int t = 0; t < deg; ++t) if (nbr[lo + t] == gj) sl = t;
      const int l0 = max(fk, fj);
      for (int e = threadIdx.x; e < nn; e += blockDim.x) {
        int a = e / n, b = e % n;
        double v = sl >= 0 ? Ak[((size_t)sl * n + b) * n + a] : 0.0;
        for (int l = l0; l < j; ++l) {
          const double* x = Lk + (size_t)(l - fk) * n * n + a;   // L_kl[a][c] at x[c * n]
          const double* y = Lj + (size_t)(l - fj) * n * n + b;
          for (int c = 0; c < n; ++c) v -= x[c * n] * y[c * n];
        }
        S[e] = v;
      }
      for (int e = threadIdx.x; e < nn; e += blockDim.x) Li[e] = Dinv[(size_t)gj * nn + e];
      __syncthreads();
      // L_kj = S L_jj^-T : (a,b) = sum_{c<=b} S[a][c] Linv_jj[b][c]
      for (int e = threadIdx.x; e < nn; e += blockDim.x) {
        int a = e / n, b = e % n;
        double v = 0;
        for (int c = 0; c <= b; ++c) v += S[a * n + c] * Li[b * n + c];
        Lk[((size_t)(j - fk) * n + b) * n + a] = v;
      }
      __syncthreads();
    }
    // diagonal: S = A_kk - sum_l L_kl L_kl^T
    int slk = -1;
    for (int t = 0; t < deg; ++t) if (nbr[lo + t] == gk) slk = t;
    for (int e = threadIdx.x; e < nn; e += blockDim.x) {
      int a = e / n, b = e % n;
      double v = Ak[((size_t)slk * n + b) * n + a];
      for (int l = fk; l < k; ++l) {
        const double* x = Lk + (size_t)(l - fk) * n * n + a;
        const double* y = Lk + (size_t)(l - fk) * n * n + b;
        for (int c = 0; c < n; ++c) v -= x[c * n] * y[c * n];
      }
      S[e] = v;
    }
    __syncthreads();
    int bad = cta_chol(S, n, n);
    if (bad && threadIdx.x == 0) { atomicExch(&err[1], 1); atomicMin(&err[2], s); }
    cta_trinv(S, Li, n, n);
    for (int e = threadIdx.x; e < nn; e += blockDim.x) Dinv[(size_t)gk * nn + e] = Li[e];
    __syncthreads();
  }
  // scale row-blocks: U_kj = Linv_kk L_kj (column by column, in place)
  for (int k = 0; k < m; ++k) {
    const int gk = s0 + k, Wk = (k - first[gk]) * n;
    if (Wk == 0) continue;
    double* Lk = U + u_off[gk];
    for (int e = threadIdx.x; e < nn; e += blockDim.x) Li[e] = Dinv[(size_t)gk * nn + e];
    __syncthreads();
    for (int col = threadIdx.x; col < Wk; col += blockDim.x) {
      double v[DGAS_MAXNP];
      for (int a = 0; a < n; ++a) v[a] = Lk[(size_t)col * n + a];
      for (int a = n - 1; a >= 0; --a) {
        double t = 0;
        for (int c = 0; c <= a; ++c) t += Li[a * n + c] * v[c];
        Lk[(size_t)col * n + a] = t;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ launcher
int setup_kernels_run(dgas_ctx ctx) {
  cudaStream_t s = ctx->stream;
  const int p = ctx->p, n = ctx->np, nc = ctx->nc;
  k_gauss_legendre<<<16, 16, 0, s>>>(ctx->d_glx, ctx->d_glw);
  DGAS_CUDA(cudaMemsetAsync(ctx->d_err, 0, 8 * sizeof(int), s));
  {
    int init[8] = {0, 0, 0x7fffffff, 0, 0, 0, 0, 0};
    DGAS_CUDA(cudaMemcpyAsync(ctx->d_err, init, sizeof init, cudaMemcpyHostToDevice, s));
  }
  k_basis<<<nc, 128, 0, s>>>(p, ctx->d_cptr, ctx->d_xy, ctx->d_glx, ctx->d_glw, ctx->d_C, ctx->d_bbox, ctx->d_hk,
                              ctx->d_err);
  DGAS_CUDA(cudaGetLastError());
  k_volume<<<nc, 128, 0, s>>>(p, ctx->d_cptr, ctx->d_xy, ctx->d_glx, ctx->d_glw, ctx->d_C, ctx->d_bbox,
                               ctx->d_kappa, ctx->d_vol);
  DGAS_CUDA(cudaGetLastError());
  k_face<<<ctx->nface, 128, 0, s>>>(p, ctx->penalty, ctx->d_face_cells, ctx->d_face_xy, ctx->d_glx, ctx->d_glw,
                                     ctx->d_C, ctx->d_bbox, ctx->d_kappa, ctx->d_hk, ctx->d_fblk);
  DGAS_CUDA(cudaGetLastError());
  k_gather_rows<<<nc, 128, 0, s>>>(n, ctx->d_nbr_ptr, ctx->d_nbr, ctx->d_a_off, ctx->d_cf_ptr, ctx->d_cf,
                                    ctx->d_face_cells, ctx->d_vol, ctx->d_fblk, ctx->d_A);
  DGAS_CUDA(cudaGetLastError());
  k_local_factor<<<ctx->nsub, 256, 0, s>>>(n, ctx->d_sub_ptr, ctx->d_first, ctx->d_u_off, ctx->d_nbr_ptr, ctx->d_nbr,
                                            ctx->d_a_off, ctx->d_A, ctx->d_U, ctx->d_Dinv, ctx->d_err);
  DGAS_CUDA(cudaGetLastError());
  int herr[8];
  DGAS_CUDA(cudaMemcpyAsync(herr, ctx->d_err, sizeof herr, cudaMemcpyDeviceToHost, s));
  DGAS_CUDA(cudaStreamSynchronize(s));
  if (herr[0]) { ctx->detail = "basis Gram matrix not SPD (degenerate cell)"; return DGAS_E_MESH; }
  if (herr[1]) { ctx->detail = "local block A_i not SPD: subdomain " + std::to_string(herr[2]); return DGAS_E_NOT_SPD; }
  return 0;
}

int launch_rhs(dgas_ctx ctx, int f_kind, double* b) {
  k_rhs<<<ctx->nc, 128, 0, ctx->stream>>>(ctx->p, f_kind, ctx->d_cptr, ctx->d_xy, ctx->d_glx, ctx->d_glw, ctx->d_C,
                                           ctx->d_bbox, b);
  return cudaGetLastError() == cudaSuccess ? 0 : DGAS_E_CUDA;
}
