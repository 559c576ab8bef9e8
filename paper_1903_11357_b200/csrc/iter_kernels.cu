// iter_kernels.cu — per-iteration kernels of ASPCG with the additive Schwarz
// preconditioner P^-1 = Q A0^-1 Q^T + sum_i E_i A_i^-1 E_i^T (R8).
//
// One PCG iteration = 4 launches (all fp64, HBM-bound GEMV-class work, no tensor cores):
//   k_spmv     p = z + beta p_old (fused), q = A p, p.q  -> alpha          (I1, I7)
//   k_restrict x += alpha p, r -= alpha q, r.r -> convergence; r0 = Q^T r (I2, I3)
//   k_apply    [coarse CTAs] z0 = A0^-1 r0   ||   [subdomain CTAs] z_i = A_i^-1 r_i   (I4, I5)
//   k_prolong  z += Q z0, r.z -> beta, iteration bookkeeping, graph condition   (I6)
// Reductions are deterministic: per-CTA partials, the last CTA to arrive sums them in a fixed order.
#include <cfloat>

#include "internal.h"

// ------------------------------------------------------------------ deterministic last-block sum
template <int NT>
__device__ inline double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < NT / 32 ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
  }
  return t;  // valid in thread 0
}

// returns true in every thread of the last CTA; totals[k] = sum of partial k over all CTAs
template <int NT, int K>
__device__ inline bool last_block(const double* mine, double* partials, unsigned* cnt, double* totals, double* red) {
  __shared__ bool am_last;
  if (threadIdx.x == 0) {
    for (int k = 0; k < K; ++k) partials[(size_t)k * gridDim.x + blockIdx.x] = mine[k];
    __threadfence();
    unsigned t = atomicAdd(cnt, 1u);
    am_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  for (int k = 0; k < K; ++k) {
    double s = 0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += NT) s += __ldcg(partials + (size_t)k * gridDim.x + i);
    s = block_sum<NT>(s, red);
    if (threadIdx.x == 0) totals[k] = s;
  }
  if (threadIdx.x == 0) *cnt = 0;
  __syncthreads();
  return true;
}

// ------------------------------------------------------------------ SpMV (+ fused direction update)
// mode 0: y = A x.   mode 1 (PCG): p_new = z + beta p_old (beta = 0 at it = 0), q = A p_new, p.q.
// One warp per cell row; the row block is n x (deg n) row-major, lanes stride its columns.
#define SPMV_WARPS 8
template <int NP>
__global__ void __launch_bounds__(SPMV_WARPS * 32) k_spmv(int mode, int nc, const int* __restrict__ nbr_ptr,
                                                          const int* __restrict__ nbr, const int64_t* __restrict__ a_off,
                                                          const double* __restrict__ A, const double* x, double* y,
                                                          const double* z, double* const* pbuf, PcgState* st,
                                                          double* partials, double* alpha_hist) {
  constexpr int MAXT = (16 * NP + 31) / 32;
  __shared__ double red[SPMV_WARPS];
  __shared__ double wdot[SPMV_WARPS];
  int it = 0;
  double beta = 0;
  const double* pold = nullptr;
  double* pnew = nullptr;
  if (mode == 1) {
    if (st->done) return;
    it = st->it;
    beta = it > 0 ? st->beta : 0.0;
    pold = pbuf[it & 1];
    pnew = pbuf[(it + 1) & 1];
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * SPMV_WARPS + w;
  double mydot = 0;
  if (c < nc) {
    const int lo = nbr_ptr[c], deg = nbr_ptr[c + 1] - lo, W = deg * NP;
    const double* row = A + a_off[c];
    double pv[MAXT];
#pragma unroll
    for (int t = 0; t < MAXT; ++t) {
      int col = lane + 32 * t;
      pv[t] = 0;
      if (col < W) {
        int j = __ldg(nbr + lo + col / NP), b = col % NP;
        size_t id = (size_t)j * NP + b;
        pv[t] = mode == 1 ? (it > 0 ? z[id] + beta * pold[id] : z[id]) : x[id];
      }
    }
    double acc[NP];
#pragma unroll
    for (int a = 0; a < NP; ++a) {
      double v = 0;
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        int col = lane + 32 * t;
        if (col < W) v += __ldcs(row + (size_t)a * W + col) * pv[t];
      }
      acc[a] = v;
    }
#pragma unroll
    for (int a = 0; a < NP; ++a) acc[a] = warp_sum(acc[a]);
    double out = 0;
#pragma unroll
    for (int a = 0; a < NP; ++a) if (lane == a) out = acc[a];
    if (lane < NP) {
      size_t id = (size_t)c * NP + lane;
      y[id] = out;
      if (mode == 1) {
        double pn = it > 0 ? z[id] + beta * pold[id] : z[id];
        pnew[id] = pn;
        mydot = pn * out;
      }
    }
  }
  if (mode != 1) return;
  mydot = warp_sum(mydot);
  if (lane == 0) wdot[w] = mydot;
  __syncthreads();
  double tot[1] = {0};
  if (threadIdx.x == 0)
    for (int k = 0; k < SPMV_WARPS; ++k) tot[0] += wdot[k];
  double res[1];
  if (last_block<SPMV_WARPS * 32, 1>(tot, partials, &st->cnt[0], res, red)) {
    if (threadIdx.x == 0) {
      double pq = res[0];
      st->pq = pq;
      if (!(pq > 0) || !isfinite(pq)) { st->done = 1; st->status = DGAS_E_BREAKDOWN; }
      else { st->alpha = st->gamma / pq; alpha_hist[it] = st->alpha; }
    }
  }
}

// ------------------------------------------------------------------ update + restriction
// mode 0: r0 = Q^T r_in (no update).  mode 1 (PCG iteration): r_new = r_old - alpha q (owner pieces
// write r_new and x += alpha p_new), r.r -> convergence test, r0 = Q^T r_new.
// mode 2 (PCG init): r_new = b - q (q = A x0), r.r and b.b.
// One CTA per coarse element J, one warp per overlap piece.
#define RW 4
template <int NP, int NQ>
__global__ void __launch_bounds__(RW * 32) k_restrict(int mode, const int* __restrict__ cov_ptr, const int* __restrict__ cov,
                                                      const int* __restrict__ ov_cell, const int* __restrict__ fov_ptr,
                                                      const int* __restrict__ fov, const double* __restrict__ G,
                                                      const double* r_in, double* const* rbuf, const double* q,
                                                      double* const* pbuf, double* x, const double* b, double* r0,
                                                      PcgState* st, double* partials) {
  __shared__ double red[RW];
  __shared__ double part[RW][NQ];
  __shared__ double wsum[RW][2];
  int it = 0;
  double alpha = 0;
  const double* rold = r_in;
  double* rnew = nullptr;
  const double* pnew = nullptr;
  if (mode >= 1) {
    if (st->done) return;
    it = st->it;
    if (mode == 1) {
      alpha = st->alpha;
      rold = rbuf[it & 1];
      rnew = rbuf[(it + 1) & 1];
      pnew = pbuf[(it + 1) & 1];
    } else {
      rnew = rbuf[0];
    }
  }
  const int J = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double accq[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) accq[k] = 0;
  double rr = 0, bb = 0;
  for (int k = cov_ptr[J] + w; k < cov_ptr[J + 1]; k += RW) {
    const int o = cov[k], cell = ov_cell[o];
    const bool owner = fov[fov_ptr[cell]] == o;
    double rv = 0;
    if (lane < NP) {
      size_t id = (size_t)cell * NP + lane;
      if (mode == 0) rv = rold[id];
      else if (mode == 1) rv = rold[id] - alpha * q[id];
      else rv = b[id] - q[id];
      if (owner && mode >= 1) {
        rnew[id] = rv;
        rr += rv * rv;
        if (mode == 1) x[id] += alpha * pnew[id];
        else bb += b[id] * b[id];
      }
    }
    const double* Go = G + (size_t)o * NP * NQ;
#pragma unroll
    for (int c = 0; c < NQ; ++c) {
      double v = lane < NP ? Go[lane * NQ + c] * rv : 0.0;
      accq[c] += warp_sum(v);
    }
  }
  if (lane == 0)
    for (int c = 0; c < NQ; ++c) part[w][c] = accq[c];
  rr = warp_sum(rr); bb = warp_sum(bb);
  if (lane == 0) { wsum[w][0] = rr; wsum[w][1] = bb; }
  __syncthreads();
  if (threadIdx.x < NQ) {
    double v = 0;
    for (int k = 0; k < RW; ++k) v += part[k][threadIdx.x];
    r0[(size_t)J * NQ + threadIdx.x] = v;
  }
  if (mode == 0) return;
  double mine[2] = {0, 0};
  if (threadIdx.x == 0)
    for (int k = 0; k < RW; ++k) { mine[0] += wsum[k][0]; mine[1] += wsum[k][1]; }
  double tot[2];
  if (last_block<RW * 32, 2>(mine, partials, &st->cnt[1], tot, red)) {
    if (threadIdx.x == 0) {
      st->rr = tot[0];
      if (mode == 2) { st->bb = tot[1]; st->rtol2_bb *= tot[1]; }
      if (!isfinite(tot[0])) { st->done = 1; st->status = DGAS_E_BREAKDOWN; }
      else if (tot[0] <= st->rtol2_bb) { st->done = 1; st->status = DGAS_OK; if (mode == 1) st->it = it + 1; }
    }
  }
}

// ------------------------------------------------------------------ fused apply: coarse || local
// blocks [0, ncc): coarse solve (dense: rows of X = A0^-1; banded: one CTA runs the tile sweeps)
// blocks [ncc, ncc + nsub): exact local solve of subdomain s with the envelope factor:
//   s = D^-1 r (parallel), U y = s (forward, row-oriented), U^T u = y (backward, column-oriented),
//   z = D^-T u (parallel), where A_i = D U U^T D^T ... i.e. L = D^{-1}-scaled rows (see setup).
#define AT 256
template <int NP>
__global__ void __launch_bounds__(AT) k_apply(int mode, int ncc, int dense, int64_t N0, int nT, int bt,
                                              const double* __restrict__ X, const double* __restrict__ A0t,
                                              const double* __restrict__ Dinv0, const double* r0, double* z0,
                                              const int* __restrict__ sub_ptr, const int* __restrict__ first,
                                              const int64_t* __restrict__ u_off, const double* __restrict__ U,
                                              const double* __restrict__ Dinv, const double* r_in,
                                              double* const* rbuf, double* z, PcgState* st) {
  extern __shared__ double sm[];
  // mode 0: r = r_in (standalone apply); 1: PCG init (rbuf[0]); 2: PCG iteration (rbuf[(it+1)&1])
  const double* r = r_in;
  if (mode >= 1) {
    if (st->done) return;
    r = mode == 1 ? rbuf[0] : rbuf[(st->it + 1) & 1];
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if ((int)blockIdx.x < ncc) {
    if (dense) {
      // z0 = X r0, warp per row
      const int64_t rows_per = (N0 + ncc - 1) / ncc;
      const int64_t r_lo = blockIdx.x * rows_per, r_hi = min(N0, r_lo + rows_per);
      for (int64_t row = r_lo + w; row < r_hi; row += AT / 32) {
        const double* xr = X + row * N0;
        double v = 0;
        for (int64_t c = lane; c < N0; c += 32) v += __ldcs(xr + c) * __ldg(r0 + c);
        v = warp_sum(v);
        if (lane == 0) z0[row] = v;
      }
    } else if (blockIdx.x == 0) {
      // banded: forward L y = r0 then backward L^T x = y, by CT-row tiles (in place in z0)
      for (int64_t i = threadIdx.x; i < (int64_t)nT * CT; i += AT) z0[i] = i < N0 ? r0[i] : 0.0;
      __syncthreads();
      double* acc = sm;  // CT
      for (int I = 0; I < nT; ++I) {
        for (int a = w; a < CT; a += AT / 32) {
          double v = 0;
          for (int K = max(0, I - bt); K < I; ++K) {
            const double* t = A0t + ((size_t)I * (bt + 1) + (K - I + bt)) * CT * CT + a * CT;
            v += t[lane] * z0[(size_t)K * CT + lane];
          }
          v = warp_sum(v);
          if (lane == 0) acc[a] = z0[(size_t)I * CT + a] - v;
        }
        __syncthreads();
        if (threadIdx.x < CT) {
          const double* D = Dinv0 + (size_t)I * CT * CT + threadIdx.x * CT;
          double v = 0;
          for (int c = 0; c <= (int)threadIdx.x; ++c) v += D[c] * acc[c];
          z0[(size_t)I * CT + threadIdx.x] = v;
        }
        __syncthreads();
      }
      for (int I = nT - 1; I >= 0; --I) {
        if (threadIdx.x < CT) {
          // x_I = D_I^T y_I
          const int a = threadIdx.x;
          double v = 0;
          for (int c = a; c < CT; ++c) v += Dinv0[(size_t)I * CT * CT + c * CT + a] * z0[(size_t)I * CT + c];
          acc[a] = v;
        }
        __syncthreads();
        if (threadIdx.x < CT) z0[(size_t)I * CT + threadIdx.x] = acc[threadIdx.x];
        __syncthreads();
        // y_K -= L_IK^T x_I for K in [I-bt, I)
        const int K0 = max(0, I - bt);
        for (int e = threadIdx.x; e < (I - K0) * CT; e += AT) {
          int K = K0 + e / CT, col = e % CT;
          const double* t = A0t + ((size_t)I * (bt + 1) + (K - I + bt)) * CT * CT + col;
          double v = 0;
          for (int a = 0; a < CT; ++a) v += t[a * CT] * acc[a];
          z0[(size_t)K * CT + col] -= v;
        }
        __syncthreads();
      }
    }
    return;
  }
  // ---------------- local solve of subdomain s
  const int s = blockIdx.x - ncc;
  const int s0 = sub_ptr[s], m = sub_ptr[s + 1] - s0;
  double* y = sm;
  const double* rs = r + (size_t)s0 * NP;
  for (int e = threadIdx.x; e < m * NP; e += AT) {
    const int k = e / NP, a = e % NP;
    const double* D = Dinv + ((size_t)(s0 + k) * NP + a) * NP;
    double v = 0;
    for (int c = 0; c <= a; ++c) v += D[c] * rs[k * NP + c];
    y[e] = v;
  }
  __syncthreads();
  for (int k = 1; k < m; ++k) {
    const int fk = first[s0 + k], W = (k - fk) * NP;
    if (W > 0) {
      const double* Uk = U + u_off[s0 + k];
      const double* yw = y + fk * NP;
      for (int a = w; a < NP; a += AT / 32) {
        double v = 0;
        for (int col = lane; col < W; col += 32) v += __ldcs(Uk + a * W + col) * yw[col];
        v = warp_sum(v);
        if (lane == 0) y[k * NP + a] -= v;
      }
    }
    __syncthreads();
  }
  for (int k = m - 1; k > 0; --k) {
    const int fk = first[s0 + k], W = (k - fk) * NP;
    if (W > 0) {
      const double* Uk = U + u_off[s0 + k];
      const double* uk = y + k * NP;
      for (int col = threadIdx.x; col < W; col += AT) {
        double v = 0;
#pragma unroll
        for (int a = 0; a < NP; ++a) v += Uk[a * W + col] * uk[a];
        y[fk * NP + col] -= v;
      }
    }
    __syncthreads();
  }
  double* zs = z + (size_t)s0 * NP;
  for (int e = threadIdx.x; e < m * NP; e += AT) {
    const int k = e / NP, a = e % NP;
    const double* D = Dinv + (size_t)(s0 + k) * NP * NP;
    double v = 0;
    for (int c = a; c < NP; ++c) v += D[c * NP + a] * y[k * NP + c];
    zs[e] = v;
  }
}

// ------------------------------------------------------------------ prolongation + r.z
// z_kappa += sum_{pieces o of kappa} G_o z0_J(o).  mode 0: apply only.  mode 1: PCG init (gamma_0).
// mode 2: PCG iteration (beta = gamma_new / gamma, history, it++, maxit, graph condition).
#define PW 8
template <int NP, int NQ>
__global__ void __launch_bounds__(PW * 32) k_prolong(int mode, int nc, const int* __restrict__ fov_ptr,
                                                     const int* __restrict__ fov, const int* __restrict__ ov_coarse,
                                                     const double* __restrict__ G, const double* z0, double* z,
                                                     double* const* rbuf, PcgState* st, double* partials,
                                                     double* beta_hist, cudaGraphConditionalHandle h, int use_h) {
  __shared__ double red[PW];
  __shared__ double wd[PW];
  int it = 0;
  const double* r = nullptr;
  if (mode >= 1) {
    if (st->done) {
      if (use_h && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(h, 0);
      return;
    }
    it = st->it;
    r = rbuf[mode == 1 ? 0 : ((it + 1) & 1)];
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * PW + w;
  double d = 0;
  if (c < nc && lane < NP) {
    size_t id = (size_t)c * NP + lane;
    double v = z[id];
    for (int k = fov_ptr[c]; k < fov_ptr[c + 1]; ++k) {
      const int o = fov[k], J = ov_coarse[o];
      const double* Go = G + ((size_t)o * NP + lane) * NQ;
#pragma unroll
      for (int b = 0; b < NQ; ++b) v += Go[b] * z0[(size_t)J * NQ + b];
    }
    z[id] = v;
    if (mode >= 1) d = r[id] * v;
  }
  if (mode == 0) return;
  d = warp_sum(d);
  if (lane == 0) wd[w] = d;
  __syncthreads();
  double mine[1] = {0};
  if (threadIdx.x == 0)
    for (int k = 0; k < PW; ++k) mine[0] += wd[k];
  double tot[1];
  if (last_block<PW * 32, 1>(mine, partials, &st->cnt[2], tot, red)) {
    if (threadIdx.x == 0) {
      const double g = tot[0];
      if (!(g > 0) || !isfinite(g)) { st->done = 1; st->status = DGAS_E_BREAKDOWN; }
      else if (mode == 1) { st->gamma = g; st->beta = 0; }
      else {
        st->beta = g / st->gamma;
        beta_hist[it] = st->beta;
        st->gamma = g;
        st->it = it + 1;
        if (st->it >= st->maxit) { st->done = 1; st->status = DGAS_NOT_CONVERGED; }
      }
      if (use_h) cudaGraphSetConditional(h, st->done ? 0u : 1u);
    }
  }
}

// ------------------------------------------------------------------ misc kernels
__global__ void k_perm(int64_t nc, int np, const int* perm, const double* in, double* out, int to_internal) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nc * np) return;
  int64_t c = i / np, a = i % np;
  // to_internal: out[c (internal)] = in[perm[c] (caller)]
  if (to_internal) out[i] = in[(int64_t)perm[c] * np + a];
  else out[(int64_t)perm[c] * np + a] = in[i];
}

__global__ void k_init_state(PcgState* st, int maxit, double rtol) {
  st->it = 0; st->done = 0; st->status = 0; st->maxit = maxit;
  st->rtol2_bb = rtol * rtol; st->bb = 0; st->gamma = 0; st->pq = 0; st->alpha = 0; st->beta = 0; st->rr = 0;
  for (int k = 0; k < 4; ++k) st->cnt[k] = 0;
}

// Lanczos tridiagonal T_m from the CG coefficients (R12), extreme eigenvalues by Sturm multisection.
__device__ inline int sturm(int m, const double* al, const double* be, double x) {
  int cnt = 0;
  double qv = 1.0 / al[0] - x;
  if (qv < 0) cnt++;
  for (int i = 1; i < m; ++i) {
    double d = 1.0 / al[i] + be[i - 1] / al[i - 1];
    double e2 = be[i - 1] / (al[i - 1] * al[i - 1]);
    if (qv == 0) qv = 1e-300;
    qv = d - x - e2 / qv;
    if (qv < 0) cnt++;
  }
  return cnt;
}
__global__ void __launch_bounds__(256) k_lanczos(const PcgState* st, const double* al, const double* be, double* out) {
  const int m = st->it;
  __shared__ double lo_s, hi_s;
  __shared__ int cnts[256];
  if (m < 1) { if (threadIdx.x == 0) { out[0] = out[1] = out[2] = 0; } return; }
  if (threadIdx.x == 0) {
    double lo = 1e300, hi = -1e300;
    for (int j = 0; j < m; ++j) {
      double d = 1.0 / al[j] + (j > 0 ? be[j - 1] / al[j - 1] : 0.0);
      double r = (j > 0 ? sqrt(be[j - 1]) / al[j - 1] : 0.0) + (j + 1 < m ? sqrt(be[j]) / al[j] : 0.0);
      lo = fmin(lo, d - r); hi = fmax(hi, d + r);
    }
    lo_s = lo; hi_s = hi;
  }
  __syncthreads();
  const double glo = lo_s, ghi = hi_s;
  for (int which = 0; which < 2; ++which) {
    const int k = which == 0 ? 0 : m - 1;  // k-th smallest
    double lo = glo, hi = ghi;
    for (int round = 0; round < 40; ++round) {
      if (!(hi - lo > 1e-15 * fmax(fabs(lo), fabs(hi)))) break;
      double x = lo + (hi - lo) * (threadIdx.x + 1) / 257.0;
      cnts[threadIdx.x] = sturm(m, al, be, x);
      __syncthreads();
      // first point with count > k bounds the eigenvalue from above
      __shared__ double nlo, nhi;
      if (threadIdx.x == 0) {
        int j = 0;
        while (j < 256 && cnts[j] <= k) ++j;
        nlo = j == 0 ? lo : lo + (hi - lo) * j / 257.0;
        nhi = j == 256 ? hi : lo + (hi - lo) * (j + 1) / 257.0;
      }
      __syncthreads();
      lo = nlo; hi = nhi;
      __syncthreads();
    }
    if (threadIdx.x == 0) out[which] = 0.5 * (lo + hi);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[2] = out[1] / out[0];
}

// ------------------------------------------------------------------ launchers
#define DISPATCH_P(P, ...)                       \
  switch (P) {                                   \
    case 1: { constexpr int NP_ = 3; __VA_ARGS__; } break;  \
    case 2: { constexpr int NP_ = 6; __VA_ARGS__; } break;  \
    case 3: { constexpr int NP_ = 10; __VA_ARGS__; } break; \
    case 4: { constexpr int NP_ = 15; __VA_ARGS__; } break; \
    case 5: { constexpr int NP_ = 21; __VA_ARGS__; } break; \
    case 6: { constexpr int NP_ = 28; __VA_ARGS__; } break; \
  }
#define DISPATCH_Q(Q, ...)                       \
  switch (Q) {                                   \
    case 1: { constexpr int NQ_ = 3; __VA_ARGS__; } break;  \
    case 2: { constexpr int NQ_ = 6; __VA_ARGS__; } break;  \
    case 3: { constexpr int NQ_ = 10; __VA_ARGS__; } break; \
    case 4: { constexpr int NQ_ = 15; __VA_ARGS__; } break; \
    case 5: { constexpr int NQ_ = 21; __VA_ARGS__; } break; \
    case 6: { constexpr int NQ_ = 28; __VA_ARGS__; } break; \
  }

void launch_perm(dgas_ctx ctx, const double* in, double* out, int to_internal, cudaStream_t s) {
  int64_t n = ctx->N;
  k_perm<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ctx->nc, ctx->np, ctx->d_perm_dev, in, out, to_internal);
}

void launch_spmv(dgas_ctx ctx, int mode, const double* x, double* y, PcgState* st, cudaStream_t s) {
  unsigned grid = (ctx->nc + SPMV_WARPS - 1) / SPMV_WARPS;
  DISPATCH_P(ctx->p, (k_spmv<NP_><<<grid, SPMV_WARPS * 32, 0, s>>>(mode, ctx->nc, ctx->d_nbr_ptr, ctx->d_nbr,
                                                                    ctx->d_a_off, ctx->d_A, x, y, ctx->d_z,
                                                                    ctx->d_pbuf, st, ctx->d_partials, ctx->d_alpha)));
}

void launch_restrict(dgas_ctx ctx, int mode, PcgState* st, const double* r, cudaStream_t s) {
  DISPATCH_P(ctx->p, DISPATCH_Q(ctx->q, (k_restrict<NP_, NQ_><<<ctx->ncoarse, RW * 32, 0, s>>>(
                                            mode, ctx->d_cov_ptr, ctx->d_cov, ctx->d_ov_cell, ctx->d_fov_ptr,
                                            ctx->d_fov, ctx->d_G, r, ctx->d_rbuf, ctx->d_q, ctx->d_pbuf, ctx->d_x,
                                            ctx->d_b, ctx->d_r0, st, ctx->d_partials))));
}

void launch_apply(dgas_ctx ctx, int mode, PcgState* st, const double* r, double* z, cudaStream_t s) {
  size_t smem = (size_t)std::max(ctx->max_sub_cells * ctx->np, CT) * sizeof(double);
  DISPATCH_P(ctx->p, (k_apply<NP_><<<ctx->n_coarse_ctas + ctx->nsub, AT, smem, s>>>(
                         mode, ctx->n_coarse_ctas, ctx->coarse_dense, ctx->N0, ctx->nT, ctx->bt, ctx->d_X, ctx->d_A0t,
                         ctx->d_Dinv0, ctx->d_r0, ctx->d_z0, ctx->d_sub_ptr, ctx->d_first, ctx->d_u_off, ctx->d_U,
                         ctx->d_Dinv, r, ctx->d_rbuf, z, st)));
}

void launch_prolong(dgas_ctx ctx, int mode, PcgState* st, const double* r, double* z, cudaStream_t s,
                    cudaGraphConditionalHandle h, int use_handle) {
  (void)r;
  unsigned grid = (ctx->nc + PW - 1) / PW;
  DISPATCH_P(ctx->p, DISPATCH_Q(ctx->q, (k_prolong<NP_, NQ_><<<grid, PW * 32, 0, s>>>(
                                            mode, ctx->nc, ctx->d_fov_ptr, ctx->d_fov, ctx->d_ov_coarse, ctx->d_G,
                                            ctx->d_z0, z, ctx->d_rbuf, st, ctx->d_partials, ctx->d_beta, h,
                                            use_handle))));
}

void launch_init_state(dgas_ctx ctx, PcgState* st, int maxit, double rtol, cudaStream_t s) {
  (void)ctx;
  k_init_state<<<1, 1, 0, s>>>(st, maxit, rtol);
}

void launch_lanczos(dgas_ctx ctx, cudaStream_t s) {
  k_lanczos<<<1, 256, 0, s>>>(ctx->d_state, ctx->d_alpha, ctx->d_beta, ctx->d_lanczos);
}

int apply_set_smem(dgas_ctx ctx, size_t smem) {
  cudaError_t e = cudaSuccess;
  DISPATCH_P(ctx->p, (e = cudaFuncSetAttribute(k_apply<NP_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)));
  if (e != cudaSuccess) { ctx->detail = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e); return DGAS_E_CUDA; }
  return 0;
}
