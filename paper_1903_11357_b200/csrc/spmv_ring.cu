// spmv_ring.cu — q = A p for the block-sparse SIPDG matrix (eq:Ah), fused with the
// PCG direction update p = z + beta p_old and the dot product p.q (ASPCG).
//
// Design (HBM-bound GEMV-class work, 2 flops per 8-byte entry): each persistent CTA owns a
// contiguous range of cell rows. A producer lane streams the cells' column-major row-blocks
// (n_p x deg n_p, contiguous, 16-byte padded) with one cp.async.bulk per cell into a BYTE ring:
// blocks are packed back to back (a block never straddles the ring end), so the ring holds as many
// blocks as fit, not a fixed number of worst-case slots, and ~100 KB per CTA stay in flight.
// Consumer warps take the CTA's cells round-robin (cell i -> warp i mod NW) and work independently:
// no CTA or group barrier per batch, only a per-cell mbarrier (full: bytes landed; empty: the
// warp is done, the producer may reuse the bytes). Each warp gathers the neighbour values of its
// NEXT cell (index load one cell further ahead) while it multiplies the current one; lane
// (a, h) = (row, column slice) reads A[col n_p + a] (consecutive lanes -> consecutive words).
#include "internal.h"
#define TMA_HOST_BACKOFF
#include "tma.cuh"

#include <algorithm>
#include <map>

#define SR_NW 8    // consumer warps per CTA
#define SR_NB 32   // cells in flight per CTA (mbarrier pairs)
#define CLS_MAXDEG 6  // k_spmv_cls: neighbours per cell incl. itself (Cartesian meshes: 5)
#define CLS_DEPTH 4   // k_spmv_cls: gathers in flight per warp (cells ahead)

template <int NP>
struct SrCfg {
  static constexpr int LPR = 32 / NP > 0 ? 32 / NP : 1;   // lanes per row (column slices)
  static constexpr int LANES = NP * LPR <= 32 ? NP * LPR : 32;
  static constexpr int ROWS_PER_PASS = NP <= 32 ? NP : 32;
  static constexpr int E = (16 * NP + 31) / 32;           // gathered entries per lane (deg <= 16)
  static constexpr int XS = 32 * E;                        // gathered values per warp
};

// smem layout (must match spmv_ring_smem): full | empty | vst | pst | ao[chunk+1] | nptr[chunk+1] | xs | ring
struct SrLayout {
  size_t off_ao, off_np, off_xs, off_ring;
  __host__ __device__ SrLayout(int chunk, int xs_per_warp) {
    off_ao = (size_t)4 * SR_NB * 8;
    off_np = off_ao + (size_t)(chunk + 1) * 8;
    off_xs = (off_np + (size_t)(chunk + 1) * 4 + 15) & ~(size_t)15;
    off_ring = (off_xs + (size_t)SR_NW * xs_per_warp * 8 + 127) & ~(size_t)127;
  }
};

template <int NP>
__global__ void __launch_bounds__((SR_NW + 1) * 32) k_spmv_ring(
    int mode, int nc, int chunk, const int* __restrict__ nbr_ptr, const int* __restrict__ nbr,
    const int64_t* __restrict__ a_off, const double* __restrict__ A, const double* x, double* y, const double* z,
    double* const* pbuf, PcgState* st, double* partials, double* alpha_hist, uint32_t ring_bytes, int G,
    const int64_t* __restrict__ a_dd) {
  constexpr int LPR = SrCfg<NP>::LPR, E = SrCfg<NP>::E, XS = SrCfg<NP>::XS;
  constexpr int NTT = (SR_NW + 1) * 32;
  extern __shared__ __align__(128) double sm[];
  __shared__ double red[NTT / 32];
  __shared__ double wdot[NTT / 32];
  int it = 0;
  double beta = 0;
  const double* pold = nullptr;
  double* pnew = nullptr;
  // mode 3 (PCG, p_new precomputed by k_pupdate): gather p_new, no p write; else as mode 1
  const bool pcg = mode == 1 || mode == 3;
  if (pcg) {
    if (st->done) return;
    it = st->it;
    beta = it > 0 ? st->beta : 0.0;
    pold = pbuf[it & 1];
    pnew = pbuf[(it + 1) & 1];
    if (mode == 3) x = pnew;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c0 = min(nc, blockIdx.x * chunk), c1 = min(nc, c0 + chunk), n = c1 - c0;
  const SrLayout Ly(chunk, XS);
  unsigned char* smb = reinterpret_cast<unsigned char*>(sm);
  uint64_t* full = reinterpret_cast<uint64_t*>(smb);
  uint64_t* empty = full + SR_NB;
  uint64_t* vst = empty + SR_NB;                      // virtual start of each in-flight block
  uint64_t* pst = vst + SR_NB;                        // its physical ring offset
  int64_t* ao = reinterpret_cast<int64_t*>(smb + Ly.off_ao);  // a_off[c0 .. c1]
  int* nptr = reinterpret_cast<int*>(smb + Ly.off_np);        // nbr_ptr[c0 .. c1]
  double* xs_all = reinterpret_cast<double*>(smb + Ly.off_xs);  // [SR_NW][XS] gathered values
  unsigned char* ring = smb + Ly.off_ring;
  for (int k = threadIdx.x; k <= n; k += NTT) { ao[k] = a_off[c0 + k]; nptr[k] = nbr_ptr[c0 + k]; }
  if (threadIdx.x == 0) {
    for (int t = 0; t < SR_NB; ++t) { mbar_init(&full[t], 1); mbar_init(&empty[t], G); }
    fence_mbar_init();
  }
  __syncthreads();
  double mydot = 0;
  if (w == SR_NW) {
    // ---------------- producer lane: cell i at virtual bytes [V_i, V_i + len_i), physical V_i mod RB
    if (lane == 0) {
      const uint64_t pol = l2_evict_first();
      const uint64_t RB = ring_bytes;
      uint64_t V = 0, Pp = 0;  // virtual and physical write positions
      int tail = 0;
      const int ng = (n + G - 1) / G;
      for (int gi = 0; gi < ng; ++gi) {  // group gi = cells [gi G, gi G + G): one bulk copy
        const int64_t o0 = ao[gi * G], o1 = ao[min(n, gi * G + G)];
        const uint32_t len = (uint32_t)((o1 - o0) * 8);
        if (Pp + len > RB) { V += RB - Pp; Pp = 0; }  // do not straddle the ring end
        // free space: every byte before the oldest unreleased group's start is free
        while (gi - tail >= SR_NB || (tail < gi && V + len > vst[tail % SR_NB] + RB)) {
          mbar_wait_producer(&empty[tail % SR_NB], (uint32_t)((tail / SR_NB) & 1));
          ++tail;
        }
        vst[gi % SR_NB] = V;
        pst[gi % SR_NB] = Pp;
        // de-duplicated storage (G = 1): the cell's row-block lives at a_dd[cell] in the compact store
        bulk_load(ring + Pp, A + (a_dd ? a_dd[c0 + gi] : o0), len, &full[gi % SR_NB], pol);
        V += len;
        Pp += len;
      }
    }
  } else {
    // ---------------- consumer warp w: cells i = w, w + NW, ...
    double* xs = xs_all + w * XS;
    auto colval = [&](int64_t id) -> double {
      return mode == 1 ? (it > 0 ? z[id] + beta * pold[id] : z[id]) : x[id];
    };
    // gather pipeline: idx of cell i + 2 NW, values of cell i + NW
    int idxA[E], idxB[E];  // idxB: indices of the cell whose values are in vB (kept for clarity)
    double vB[E];
    auto load_idx = [&](int i, int* idx) {
      if (i >= n) {
#pragma unroll
        for (int t = 0; t < E; ++t) idx[t] = -1;
        return;
      }
      const int lo = nptr[i], W = (nptr[i + 1] - lo) * NP;
#pragma unroll
      for (int t = 0; t < E; ++t) {
        const int e = lane + 32 * t;
        idx[t] = e < W ? __ldg(nbr + lo + e / NP) * NP + e % NP : -1;
      }
    };
    auto load_val = [&](const int* idx, double* v) {
#pragma unroll
      for (int t = 0; t < E; ++t) v[t] = idx[t] >= 0 ? colval(idx[t]) : 0.0;
    };
    {
      int idx0[E];
      load_idx(w, idx0);
      double v0[E];
      load_val(idx0, v0);
#pragma unroll
      for (int t = 0; t < E; ++t) xs[lane + 32 * t] = v0[t];
      load_idx(w + SR_NW, idxB);
      load_val(idxB, vB);
      load_idx(w + 2 * SR_NW, idxA);
    }
    __syncwarp();
    const int a = lane % NP, h = lane / NP;  // row, column slice (h < LPR)
    for (int i = w; i < n; i += SR_NW) {
      const int c = c0 + i;
      const int W = (nptr[i + 1] - nptr[i]) * NP;
      // own p_new (mode 1), loaded before the wait so its latency overlaps
      double pn = 0;
      if (pcg && h == 0 && lane < NP) {
        const size_t id = (size_t)c * NP + a;
        pn = mode == 3 ? x[id] : it > 0 ? z[id] + beta * pold[id] : z[id];
      }
      const int gi = i / G, gs = gi % SR_NB;
      mbar_wait(&full[gs], (uint32_t)((gi / SR_NB) & 1));
      const double* Ab = reinterpret_cast<const double*>(ring + pst[gs]) + (ao[i] - ao[gi * G]);
      double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
      if (h < LPR) {
        int col = h;
        for (; col + 3 * LPR < W; col += 4 * LPR) {
          s0 += Ab[col * NP + a] * xs[col];
          s1 += Ab[(col + LPR) * NP + a] * xs[col + LPR];
          s2 += Ab[(col + 2 * LPR) * NP + a] * xs[col + 2 * LPR];
          s3 += Ab[(col + 3 * LPR) * NP + a] * xs[col + 3 * LPR];
        }
        for (; col < W; col += LPR) s0 += Ab[col * NP + a] * xs[col];
      }
      double v = (s0 + s1) + (s2 + s3);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[gs]);  // this cell's bytes consumed (G arrivals free the group)
      // row sums: lane a (h = 0) adds the partials of lanes a + NP h2
      double tot = v;
#pragma unroll
      for (int h2 = 1; h2 < LPR; ++h2) {
        const double o = __shfl_sync(0xffffffffu, v, (a + NP * h2) & 31);
        tot += o;
      }
      if (h == 0 && lane < NP) {
        const size_t id = (size_t)c * NP + a;
        y[id] = tot;
        if (pcg) {
          if (mode == 1) pnew[id] = pn;
          mydot += pn * tot;
        }
      }
      // publish the next cell's gathered values (xs is not read again for cell i), advance the pipeline
      __syncwarp();
#pragma unroll
      for (int t = 0; t < E; ++t) xs[lane + 32 * t] = vB[t];
      load_val(idxA, vB);
#pragma unroll
      for (int t = 0; t < E; ++t) idxB[t] = idxA[t];
      load_idx(i + 3 * SR_NW, idxA);
      __syncwarp();
    }
  }
  if (!pcg) return;
  mydot = warp_sum(mydot);
  if (lane == 0) wdot[w] = mydot;
  __syncthreads();
  double tot[1] = {0};
  if (threadIdx.x == 0)
    for (int k = 0; k < NTT / 32; ++k) tot[0] += wdot[k];
  double res[1];
  __shared__ bool am_last;
  // deterministic last-CTA sum of the per-CTA partials (same protocol as iter_kernels.cu)
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = tot[0];
    __threadfence();
    am_last = atomicAdd(&st->cnt[0], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double sacc = 0;
  for (int k = threadIdx.x; k < (int)gridDim.x; k += NTT) sacc += __ldcg(partials + k);
  sacc = warp_sum(sacc);
  if (lane == 0) red[w] = sacc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double pq = 0;
    for (int k = 0; k < NTT / 32; ++k) pq += red[k];
    res[0] = pq;
    st->cnt[0] = 0;
    st->pq = pq;
    if (!(pq > 0) || !isfinite(pq)) { st->done = 1; st->status = DGAS_E_BREAKDOWN; }
    else { st->alpha = st->gamma / pq; alpha_hist[it] = st->alpha; }
  }
}

// ------------------------------------------------------------------------------------------------
// k_spmv_dd — the same q = A p (+ PCG fusion: p = z + beta p_old, p.q, alpha) when A is stored
// de-duplicated (dedup.cu: config 3 has 1225 distinct row-blocks, 4.8 MB, L2-resident): no TMA ring
// (one bulk copy per cell was the bottleneck, 0.40 ms), each warp reads its cell's row-block straight
// from the compact store through the L2 (__ldg), lanes (row a, column slice h) as in k_spmv_ring, the
// neighbour values gathered one cell ahead. Persistent CTAs of 8 warps over contiguous cell ranges.
template <int NP>
__global__ void __launch_bounds__(SR_NW * 32) k_spmv_dd(
    int mode, int nc, int chunk, const int* __restrict__ nbr_ptr, const int* __restrict__ nbr,
    const int64_t* __restrict__ a_dd, const double* __restrict__ A, const double* x, double* y, const double* z,
    double* const* pbuf, PcgState* st, double* partials, double* alpha_hist) {
  constexpr int LPR = SrCfg<NP>::LPR, E = SrCfg<NP>::E, XS = SrCfg<NP>::XS;
  constexpr int NTT = SR_NW * 32;
  __shared__ double red[NTT / 32];
  __shared__ double wdot[NTT / 32];
  __shared__ double xs_all[SR_NW * XS];
  int it = 0;
  double beta = 0;
  const double* pold = nullptr;
  double* pnew = nullptr;
  const bool pcg = mode == 1 || mode == 3;
  if (pcg) {
    if (st->done) return;
    it = st->it;
    beta = it > 0 ? st->beta : 0.0;
    pold = pbuf[it & 1];
    pnew = pbuf[(it + 1) & 1];
    if (mode == 3) x = pnew;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c0 = min(nc, blockIdx.x * chunk), c1 = min(nc, c0 + chunk), n = c1 - c0;
  double* xs = xs_all + w * XS;
  auto colval = [&](int64_t id) -> double {
    return mode == 1 ? (it > 0 ? z[id] + beta * pold[id] : z[id]) : x[id];
  };
  double mydot = 0;
  const int a = lane % NP, h = lane / NP;
  double vN[E];
  auto load = [&](int i, double* v) {  // gathered neighbour values of cell i (index load + value load)
    if (i >= n) {
#pragma unroll
      for (int t = 0; t < E; ++t) v[t] = 0.0;
      return;
    }
    const int lo = nbr_ptr[c0 + i], W = (nbr_ptr[c0 + i + 1] - lo) * NP;
#pragma unroll
    for (int t = 0; t < E; ++t) {
      const int e = lane + 32 * t;
      v[t] = e < W ? colval((int64_t)__ldg(nbr + lo + e / NP) * NP + e % NP) : 0.0;
    }
  };
  load(w, vN);
  for (int i = w; i < n; i += SR_NW) {
    const int c = c0 + i;
    __syncwarp();
#pragma unroll
    for (int t = 0; t < E; ++t) xs[lane + 32 * t] = vN[t];
    __syncwarp();
    load(i + SR_NW, vN);  // next cell's gather overlaps this cell's products
    const int W = (nbr_ptr[c + 1] - nbr_ptr[c]) * NP;
    const double* Ab = A + a_dd[c] + a;
    double pn = 0;
    if (pcg && h == 0 && lane < NP) {
      const size_t id = (size_t)c * NP + a;
      pn = mode == 3 ? x[id] : it > 0 ? z[id] + beta * pold[id] : z[id];
    }
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    if (h < LPR) {
      int col = h;
      for (; col + 3 * LPR < W; col += 4 * LPR) {
        s0 += __ldg(Ab + col * NP) * xs[col];
        s1 += __ldg(Ab + (col + LPR) * NP) * xs[col + LPR];
        s2 += __ldg(Ab + (col + 2 * LPR) * NP) * xs[col + 2 * LPR];
        s3 += __ldg(Ab + (col + 3 * LPR) * NP) * xs[col + 3 * LPR];
      }
      for (; col < W; col += LPR) s0 += __ldg(Ab + col * NP) * xs[col];
    }
    const double v = (s0 + s1) + (s2 + s3);
    double tot = v;
#pragma unroll
    for (int h2 = 1; h2 < LPR; ++h2) tot += __shfl_sync(0xffffffffu, v, (a + NP * h2) & 31);
    if (h == 0 && lane < NP) {
      const size_t id = (size_t)c * NP + a;
      y[id] = tot;
      if (pcg) {
        if (mode == 1) pnew[id] = pn;
        mydot += pn * tot;
      }
    }
  }
  if (!pcg) return;
  mydot = warp_sum(mydot);
  if (lane == 0) wdot[w] = mydot;
  __syncthreads();
  __shared__ bool am_last;
  if (threadIdx.x == 0) {
    double t0 = 0;
    for (int k = 0; k < NTT / 32; ++k) t0 += wdot[k];
    partials[blockIdx.x] = t0;
    __threadfence();
    am_last = atomicAdd(&st->cnt[0], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double sacc = 0;
  for (int k = threadIdx.x; k < (int)gridDim.x; k += NTT) sacc += __ldcg(partials + k);
  sacc = warp_sum(sacc);
  if (lane == 0) red[w] = sacc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double pq = 0;
    for (int k = 0; k < NTT / 32; ++k) pq += red[k];
    st->cnt[0] = 0;
    st->pq = pq;
    if (!(pq > 0) || !isfinite(pq)) { st->done = 1; st->status = DGAS_E_BREAKDOWN; }
    else { st->alpha = st->gamma / pq; alpha_hist[it] = st->alpha; }
  }
}

// p.q of the PCG SpMV: per-CTA partial, the last CTA to arrive sums the partials in CTA order
// (deterministic) and sets alpha = gamma / p.q (breakdown if p.q <= 0); same protocol as above
template <int NTT>
__device__ __forceinline__ void spmv_pq_epilogue(double mydot, double* wdot, double* red, PcgState* st, double* partials,
                                                 double* alpha_hist, int it) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  mydot = warp_sum(mydot);
  if (lane == 0) wdot[w] = mydot;
  __syncthreads();
  __shared__ bool am_last;
  if (threadIdx.x == 0) {
    double t0 = 0;
    for (int k = 0; k < NTT / 32; ++k) t0 += wdot[k];
    partials[blockIdx.x] = t0;
    __threadfence();
    am_last = atomicAdd(&st->cnt[0], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double sacc = 0;
  for (int k = threadIdx.x; k < (int)gridDim.x; k += NTT) sacc += __ldcg(partials + k);
  sacc = warp_sum(sacc);
  if (lane == 0) red[w] = sacc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double pq = 0;
    for (int k = 0; k < NTT / 32; ++k) pq += red[k];
    st->cnt[0] = 0;
    st->pq = pq;
    if (!(pq > 0) || !isfinite(pq)) { st->done = 1; st->status = DGAS_E_BREAKDOWN; }
    else { st->alpha = st->gamma / pq; alpha_hist[it] = st->alpha; }
  }
}

// ------------------------------------------------------------------------------------------------
// k_spmv_cls — q = A p (+ the same PCG fusion) over de-duplicated A, cells grouped by their distinct
// row-block ("class"; config 3: 262,144 cells, 1,225 classes). A work item is a run of cells of one
// class; its warp loads the class row-block ONCE into registers (lane (a, h) holds A[a][h + LPR t])
// and then only gathers neighbour values per cell (one cell ahead) and multiplies: no per-cell
// re-read of the 4-8 KB row-block through L1/L2 (k_spmv_dd: ~200 instructions and ~5 us of latency
// per cell on config 3). Same product order as k_spmv_dd within a slice h (t ascending), slices
// summed by shuffles in h order. Items are dealt round-robin to the grid's warps.
template <int NP>
struct ClsCfg {
  static constexpr int LPR = 32 / NP > 0 ? 32 / NP : 1;
  static constexpr int LANES = NP * LPR;
  static constexpr int MAXC = (CLS_MAXDEG * NP + LPR - 1) / LPR;  // register columns per lane
  static constexpr int E = (CLS_MAXDEG * NP + 31) / 32;           // gathered entries per lane
  static constexpr int XS = (32 * E > LPR * MAXC ? 32 * E : LPR * MAXC);
};

// MINB = resident CTAs per SM the register allocation is capped for (1: uncapped, 168 registers at n_p = 10;
// 2: <= 128 registers, twice the warps per SM to hide the gather latency)
template <int NP, int MINB>
__global__ void __launch_bounds__(SR_NW * 32, MINB) k_spmv_cls(
    int mode, int nitems, const int4* __restrict__ items, const int64_t* __restrict__ cls_off,
    const int* __restrict__ cells, const int* __restrict__ cls_nb, const double* __restrict__ A, const double* x,
    double* y, const double* z, double* const* pbuf, PcgState* st, double* partials, double* alpha_hist) {
  using C = ClsCfg<NP>;
  constexpr int LPR = C::LPR, E = C::E, XS = C::XS, MAXC = C::MAXC;
  constexpr int NTT = SR_NW * 32;
  __shared__ double red[NTT / 32];
  __shared__ double wdot[NTT / 32];
  __shared__ double xs_all[SR_NW * CLS_DEPTH * XS];  // per warp: the gathered values of D cells
  int it = 0;
  double beta = 0;
  const double* pold = nullptr;
  double* pnew = nullptr;
  const bool pcg = mode == 1 || mode == 3;
  if (pcg) {
    if (st->done) return;
    it = st->it;
    beta = it > 0 ? st->beta : 0.0;
    pold = pbuf[it & 1];
    pnew = pbuf[(it + 1) & 1];
    if (mode == 3) x = pnew;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* xs = xs_all + w * (CLS_DEPTH * XS);
  for (int t = lane; t < CLS_DEPTH * XS; t += 32) xs[t] = 0.0;
  auto colval = [&](int64_t id) -> double {
    return mode == 1 ? (it > 0 ? z[id] + beta * pold[id] : z[id]) : x[id];
  };
  const int a = lane % NP, h = lane / NP;
  const bool rl = h < LPR && lane < C::LANES;
  double mydot = 0;
  const int gw = blockIdx.x * SR_NW + w, nw = gridDim.x * SR_NW;
  constexpr int D = CLS_DEPTH;
  for (int wi = gw; wi < nitems; wi += nw) {
    const int4 itm = items[wi];  // (class, first cell in `cells`, count, W = deg NP)
    const int W = itm.w, n = itm.z;
    const int* cl = cells + itm.y;
    const int* cnb = cls_nb + (size_t)itm.y * CLS_MAXDEG;  // neighbour cells of each cell, nbr order
    double Ar[MAXC];
    {
      const double* Ab = A + cls_off[itm.x] + a;
#pragma unroll
      for (int t = 0; t < MAXC; ++t) {
        const int col = h + LPR * t;
        Ar[t] = (rl && col < W) ? __ldg(Ab + col * NP) : 0.0;
      }
    }
    // software pipeline over the item's cells (slot d = i mod D): neighbour ids 2D cells ahead, gathered
    // values D cells ahead; lane j < deg holds neighbour j's id, the gather lanes take it by shuffle
    const int deg = W / NP;
    auto ids = [&](int i) -> int { return (i < n && lane < deg) ? __ldg(cnb + (size_t)i * CLS_MAXDEG + lane) : 0; };
    auto cid = [&](int i) -> int { return i < n ? __ldg(cl + i) : 0; };
    auto gather = [&](int idr, bool on, double* v) {
#pragma unroll
      for (int t = 0; t < E; ++t) {
        const int e = lane + 32 * t;
        const int nb = __shfl_sync(0xffffffffu, idr, (e / NP) & 31);
        v[t] = (on && e < W) ? colval((int64_t)nb * NP + e % NP) : 0.0;
      }
    };
    double v[D][E];
    int idr[D], cA[D], cB[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      cA[d] = cid(d);
      gather(ids(d), d < n, v[d]);
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      idr[d] = ids(d + D);
      cB[d] = cid(d + D);
    }
    // D cells per trip: their gathered values go to D shared-memory buffers behind ONE pair of warp barriers,
    // the gathers of the next D cells are issued, then the D products run as independent chains (the kernel is
    // latency-bound: ncu 0.32 issue slots per cycle with one cell at a time)
    for (int i0 = 0; i0 < n; i0 += D) {
      int cc[D];
      __syncwarp();  // the previous trip's reads of xs are done
#pragma unroll
      for (int d = 0; d < D; ++d) {
        cc[d] = cA[d];
        if (i0 + d < n) {
#pragma unroll
          for (int t = 0; t < E; ++t) xs[d * XS + lane + 32 * t] = v[d][t];
        }
      }
      __syncwarp();
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int i = i0 + d;
        gather(idr[d], i + D < n, v[d]);  // cell i + D
        cA[d] = cB[d];
        idr[d] = ids(i + 2 * D);
        cB[d] = cid(i + 2 * D);
      }
      double pn[D], tot[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        pn[d] = 0;
        if (pcg && h == 0 && lane < NP && i0 + d < n) {
          const size_t id = (size_t)cc[d] * NP + a;
          pn[d] = mode == 3 ? x[id] : it > 0 ? z[id] + beta * pold[id] : z[id];
        }
      }
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const double* xd = xs + d * XS;
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
#pragma unroll
        for (int t = 0; t + 3 < MAXC; t += 4) {
          s0 += Ar[t] * xd[h + LPR * t];
          s1 += Ar[t + 1] * xd[h + LPR * (t + 1)];
          s2 += Ar[t + 2] * xd[h + LPR * (t + 2)];
          s3 += Ar[t + 3] * xd[h + LPR * (t + 3)];
        }
#pragma unroll
        for (int t = MAXC / 4 * 4; t < MAXC; ++t) s0 += Ar[t] * xd[h + LPR * t];
        tot[d] = (s0 + s1) + (s2 + s3);
      }
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const double vv = tot[d];
        double tsum = vv;
#pragma unroll
        for (int h2 = 1; h2 < LPR; ++h2) tsum += __shfl_sync(0xffffffffu, vv, (a + NP * h2) & 31);
        if (h == 0 && lane < NP && i0 + d < n) {
          const size_t id = (size_t)cc[d] * NP + a;
          y[id] = tsum;
          if (pcg) {
            if (mode == 1) pnew[id] = pn[d];
            mydot += pn[d] * tsum;
          }
        }
      }
    }
  }
  if (!pcg) return;
  spmv_pq_epilogue<NTT>(mydot, wdot, red, st, partials, alpha_hist, it);
}

// ------------------------------------------------------------------------------------------------
// k_spmv_cls_t — the class-sorted SpMV on the FP64 tensor cores (mma.sync m8n8k4 f64). For a run of cells of
// one class the product is a dense contraction, Y (NP x 8 cells) = A_class (NP x W) X (W x 8 cells): the A
// fragments (2 m-tiles x W / 4 k-steps) are loaded ONCE per item into registers; per tile of 8 cells every
// lane gathers its own B-fragment entries (entry 4 s + l % 4 of the gathered vector of cell l / 4) straight
// from global memory, all W / 4 gathers in flight before the first DMMA, and stores its C-fragment entries
// of y. No shared-memory staging, no warp barrier on the loop, ~8x fewer instructions per cell than
// k_spmv_cls (ncu there: latency-bound on the gathers, 0.32 issue slots per cycle).
__device__ __forceinline__ void dmma884s(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int NP>
__global__ void __launch_bounds__(SR_NW * 32, 2) k_spmv_cls_t(
    int mode, int nitems, const int4* __restrict__ items, const int64_t* __restrict__ cls_off,
    const int* __restrict__ cells, const int* __restrict__ cls_nb, const double* __restrict__ A, const double* x,
    double* y, const double* z, double* const* pbuf, PcgState* st, double* partials, double* alpha_hist) {
  constexpr int NTT = SR_NW * 32;
  constexpr int MT = (NP + 7) / 8;                   // m-tiles of the NP rows
  constexpr int KSM = (CLS_MAXDEG * NP + 3) / 4;     // k-steps of the widest row-block
  __shared__ double red[NTT / 32];
  __shared__ double wdot[NTT / 32];
  int it = 0;
  double beta = 0;
  const double* pold = nullptr;
  double* pnew = nullptr;
  const bool pcg = mode == 1 || mode == 3;
  if (pcg) {
    if (st->done) return;
    it = st->it;
    beta = it > 0 ? st->beta : 0.0;
    pold = pbuf[it & 1];
    pnew = pbuf[(it + 1) & 1];
    if (mode == 3) x = pnew;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int lr = lane >> 2, lk = lane & 3;
  auto colval = [&](int64_t id) -> double {
    return mode == 1 ? (it > 0 ? z[id] + beta * pold[id] : z[id]) : x[id];
  };
  double mydot = 0;
  const int gw = blockIdx.x * SR_NW + w, nw = gridDim.x * SR_NW;
  for (int wi = gw; wi < nitems; wi += nw) {
    const int4 itm = items[wi];  // (class, first cell in `cells`, count, W = deg NP)
    const int W = itm.w, n = itm.z;
    const int* cl = cells + itm.y;
    const int* cnb = cls_nb + (size_t)itm.y * CLS_MAXDEG;
    // A fragments of the class row-block (column-major NP x W): a[t][s] = A[8 t + lr][4 s + lk]
    double af[MT][KSM];
    {
      const double* Ab = A + cls_off[itm.x];
#pragma unroll
      for (int s = 0; s < KSM; ++s) {
        const int col = 4 * s + lk;
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          const int row = 8 * t + lr;
          const bool ok = col < W && row < NP;
          af[t][s] = ok ? __ldg(Ab + (ok ? col * NP + row : 0)) : 0.0;
        }
      }
    }
    for (int i0 = 0; i0 < n; i0 += 8) {
      // this lane's B column is cell i0 + lr: its neighbour ids (nbr order, padded with the cell itself)
      const int ic = min(i0 + lr, n - 1);
      int ids[CLS_MAXDEG];
#pragma unroll
      for (int j = 0; j < CLS_MAXDEG; ++j) ids[j] = __ldg(cnb + (size_t)ic * CLS_MAXDEG + j);
      const int mycell = __ldg(cl + ic);
      double bf[KSM];
#pragma unroll
      for (int s = 0; s < KSM; ++s) {
        // entry 4 s + lk of the gathered vector: neighbour j = col / NP (one of two compile-time candidates)
        constexpr int dummy = 0;
        (void)dummy;
        const int col = 4 * s + lk;
        const int j0 = (4 * s) / NP;
        const bool hi = col >= NP * (j0 + 1);
        const int nb = hi ? ids[j0 + 1 < CLS_MAXDEG ? j0 + 1 : j0] : ids[j0];
        const int comp = col - NP * (hi ? j0 + 1 : j0);
        const bool ok = col < W;
        bf[s] = 0.0;
        if (4 * s < W) bf[s] = ok ? colval((int64_t)nb * NP + comp) : 0.0;  // (warp-uniform: k-steps beyond W skipped)
      }
      // own values of p_new for the dot product p.q (and the p write of mode 1): C-fragment positions
      const int ca = __shfl_sync(0xffffffffu, mycell, 8 * lk), cb = __shfl_sync(0xffffffffu, mycell, 8 * lk + 4);
      const bool va = i0 + 2 * lk < n, vb = i0 + 2 * lk + 1 < n;
      double pa[MT], pb[MT];
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        const int row = 8 * t + lr;
        pa[t] = 0.0;
        pb[t] = 0.0;
        if (pcg && row < NP) {
          if (va) pa[t] = colval((int64_t)ca * NP + row);
          if (vb) pb[t] = colval((int64_t)cb * NP + row);
        }
      }
      double c0[MT], c1[MT];
#pragma unroll
      for (int t = 0; t < MT; ++t) { c0[t] = 0.0; c1[t] = 0.0; }
#pragma unroll
      for (int s = 0; s < KSM; ++s)
        if (4 * s < W) {
#pragma unroll
          for (int t = 0; t < MT; ++t) dmma884s(c0[t], c1[t], af[t][s], bf[s]);
        }
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        const int row = 8 * t + lr;
        if (row < NP) {
          if (va) {
            const size_t id = (size_t)ca * NP + row;
            y[id] = c0[t];
            if (pcg) { if (mode == 1) pnew[id] = pa[t]; mydot += pa[t] * c0[t]; }
          }
          if (vb) {
            const size_t id = (size_t)cb * NP + row;
            y[id] = c1[t];
            if (pcg) { if (mode == 1) pnew[id] = pb[t]; mydot += pb[t] * c1[t]; }
          }
        }
      }
    }
  }
  if (!pcg) return;
  spmv_pq_epilogue<NTT>(mydot, wdot, red, st, partials, alpha_hist, it);
}

#define DISPATCH_P15S(P, ...)                               \
  switch (P) {                                              \
    case 1: { constexpr int NP_ = 3; __VA_ARGS__; } break;  \
    case 2: { constexpr int NP_ = 6; __VA_ARGS__; } break;  \
    case 3: { constexpr int NP_ = 10; __VA_ARGS__; } break; \
    case 4: { constexpr int NP_ = 15; __VA_ARGS__; } break; \
  }

#define DISPATCH_PSR(P, ...)                                \
  switch (P) {                                              \
    case 1: { constexpr int NP_ = 3; __VA_ARGS__; } break;  \
    case 2: { constexpr int NP_ = 6; __VA_ARGS__; } break;  \
    case 3: { constexpr int NP_ = 10; __VA_ARGS__; } break; \
    case 4: { constexpr int NP_ = 15; __VA_ARGS__; } break; \
    case 5: { constexpr int NP_ = 21; __VA_ARGS__; } break; \
    case 6: { constexpr int NP_ = 28; __VA_ARGS__; } break; \
  }

static size_t sr_base_bytes(dgas_ctx ctx, int chunk) {
  int xs = 0;
  DISPATCH_PSR(ctx->p, (xs = SrCfg<NP_>::XS));
  return SrLayout(chunk, xs).off_ring;
}

static int sr_chunk(dgas_ctx ctx) { return (ctx->nc + ctx->sr_grid - 1) / ctx->sr_grid; }

size_t spmv_ring_smem(dgas_ctx ctx) { return sr_base_bytes(ctx, sr_chunk(ctx)) + ctx->sr_ring_bytes; }

// degree limit of the gather (16 neighbours incl. self) and a ring that holds the largest block
int spmv_ring_configure(dgas_ctx ctx, int nsm) {
  tma_set_backoff(0);  // producer-lane back-off of this unit's streaming kernels (DGAS_PRODUCER_NS)
  if (ctx->max_deg > 16) return 1;
  int dev = 0, optin = 232448, smem_sm = 233472;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  // 2 CTAs/SM; 1 (one ~220 KB ring) when row-blocks are large (n_p = 28: 44 KB per cell, so a 110 KB
  // ring holds only two; measured config 5 p = q = 6: SpMV 0.159 -> 0.118 ms)
  const double avg_blk = (double)ctx->a_off_h[ctx->nc] * 8.0 / ctx->nc;
  int cps = avg_blk > 18432.0 ? 1 : 2;  // p = 5 (~23 KB): 0.086 -> 0.071 ms
  if (const char* e = std::getenv("DGAS_SR_CPS")) cps = std::max(1, std::atoi(e));
  size_t per = (size_t)smem_sm / cps - 2048;
  per = std::min(per, (size_t)optin - 2048);
  ctx->sr_grid = std::min(ctx->nc, cps * nsm);
  const size_t base = sr_base_bytes(ctx, sr_chunk(ctx));
  int64_t maxblk = 0;
  for (int c = 0; c < ctx->nc; ++c) maxblk = std::max(maxblk, ctx->a_off_h[c + 1] - ctx->a_off_h[c]);
  size_t rb = per > base ? (per - base) / 128 * 128 : 0;
  if (const char* e = std::getenv("DGAS_SR_RING_KB")) rb = std::min(rb, (size_t)std::atoi(e) * 1024);
  // cells per bulk copy: ~16 KB per copy (small row-blocks, e.g. 4 KB on config 3, cap the TMA rate)
  const double avg = avg_blk;
  int G = std::max(1, std::min(8, (int)std::lround(16384.0 / avg)));
  if (const char* e = std::getenv("DGAS_SR_G")) G = std::max(1, std::min(SR_NW, std::atoi(e)));
  while (G > 1 && rb < (size_t)G * maxblk * 8 * 2) --G;  // groups start at chunk offsets: bound by G blocks
  if (rb < (size_t)G * maxblk * 8 * 2) return 1;
  ctx->sr_G = G;
  ctx->sr_ring_bytes = (uint32_t)rb;
  // per-function attribute shared by every context: raise it to the opt-in maximum (see panel_set_smem)
  cudaError_t e = cudaSuccess;
  DISPATCH_PSR(ctx->p, ({
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, k_spmv_ring<NP_>);
    if (e == cudaSuccess && (size_t)optin < spmv_ring_smem(ctx) + fa.sharedSizeBytes) e = cudaErrorInvalidValue;
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_spmv_ring<NP_>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
  }));
  if (e != cudaSuccess) { ctx->detail = std::string("spmv ring smem: ") + cudaGetErrorString(e); return -1; }
  return 0;
}

// p_new = z + beta p_old (PCG direction update as its own streaming pass, DGAS_SPMV_PSPLIT=1): the
// SpMV then gathers one freshly written vector instead of two
__global__ void __launch_bounds__(256) k_pupdate(int64_t n, const double* z, double* const* pbuf, const PcgState* st) {
  if (st->done) return;
  const int it = st->it;
  const double beta = it > 0 ? st->beta : 0.0;
  const double* pold = pbuf[it & 1];
  double* pnew = pbuf[(it + 1) & 1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    pnew[i] = it > 0 ? z[i] + beta * pold[i] : z[i];
}

void launch_spmv_ring(dgas_ctx ctx, int mode, const double* x, double* y, PcgState* st, cudaStream_t s) {
  if (mode == 1 && ctx->spmv_psplit) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    k_pupdate<<<nsm * 8, 256, 0, s>>>(ctx->N, ctx->d_z, ctx->d_pbuf, st);
    mode = 3;
  }
  if (ctx->d_cls_items) {
    if (ctx->cls_tc) {
      DISPATCH_P15S(ctx->p, (k_spmv_cls_t<NP_><<<ctx->cls_grid, SR_NW * 32, 0, s>>>(
                                mode, ctx->cls_nitems, ctx->d_cls_items, ctx->d_cls_off, ctx->d_cls_cells, ctx->d_cls_nb,
                                ctx->d_A, x, y, ctx->d_z, ctx->d_pbuf, st, ctx->d_partials, ctx->d_alpha)));
    } else if (ctx->cls_minb == 2) {
      DISPATCH_P15S(ctx->p, (k_spmv_cls<NP_, 2><<<ctx->cls_grid, SR_NW * 32, 0, s>>>(
                                mode, ctx->cls_nitems, ctx->d_cls_items, ctx->d_cls_off, ctx->d_cls_cells, ctx->d_cls_nb,
                                ctx->d_A, x, y, ctx->d_z, ctx->d_pbuf, st, ctx->d_partials, ctx->d_alpha)));
    } else {
      DISPATCH_P15S(ctx->p, (k_spmv_cls<NP_, 1><<<ctx->cls_grid, SR_NW * 32, 0, s>>>(
                                mode, ctx->cls_nitems, ctx->d_cls_items, ctx->d_cls_off, ctx->d_cls_cells, ctx->d_cls_nb,
                                ctx->d_A, x, y, ctx->d_z, ctx->d_pbuf, st, ctx->d_partials, ctx->d_alpha)));
    }
    return;
  }
  if (ctx->d_a_dd) {
    const int grid = ctx->dd_grid, chunk = (ctx->nc + grid - 1) / grid;
    DISPATCH_PSR(ctx->p, (k_spmv_dd<NP_><<<grid, SR_NW * 32, 0, s>>>(mode, ctx->nc, chunk, ctx->d_nbr_ptr, ctx->d_nbr,
                                                                     ctx->d_a_dd, ctx->d_A, x, y, ctx->d_z, ctx->d_pbuf,
                                                                     st, ctx->d_partials, ctx->d_alpha)));
    return;
  }
  const int grid = ctx->sr_grid, chunk = sr_chunk(ctx);
  const size_t smem = spmv_ring_smem(ctx);
  DISPATCH_PSR(ctx->p, (k_spmv_ring<NP_><<<grid, (SR_NW + 1) * 32, smem, s>>>(
                           mode, ctx->nc, chunk, ctx->d_nbr_ptr, ctx->d_nbr, ctx->d_a_off, ctx->d_A, x, y, ctx->d_z,
                           ctx->d_pbuf, st, ctx->d_partials, ctx->d_alpha, ctx->sr_ring_bytes, ctx->sr_G, ctx->d_a_dd)));
}

// y = A x on the rows of cells [cb, ce) only (sharded solve, shard.cu; mode 0): the kernel addresses its
// cell range relative to its nbr_ptr / a_off / y pointers, and gathers x through absolute cell ids
void launch_spmv_range(dgas_ctx ctx, int cb, int ce, const double* x, double* y, cudaStream_t s) {
  const int n = ce - cb;
  if (n <= 0) return;
  if (ctx->d_a_dd) {
    const int grid = std::min(ctx->dd_grid, n), chunk = (n + grid - 1) / grid;
    DISPATCH_PSR(ctx->p, (k_spmv_dd<NP_><<<grid, SR_NW * 32, 0, s>>>(0, n, chunk, ctx->d_nbr_ptr + cb, ctx->d_nbr,
                                                                     ctx->d_a_dd + cb, ctx->d_A, x, y + (size_t)cb * NP_,
                                                                     ctx->d_z, ctx->d_pbuf, nullptr, ctx->d_partials,
                                                                     ctx->d_alpha)));
    return;
  }
  const int grid = std::min(ctx->sr_grid, n), chunk = (n + grid - 1) / grid;
  const size_t smem = spmv_ring_smem(ctx);  // sized for the full problem's (larger) chunk
  DISPATCH_PSR(ctx->p, (k_spmv_ring<NP_><<<grid, (SR_NW + 1) * 32, smem, s>>>(
                           0, n, chunk, ctx->d_nbr_ptr + cb, ctx->d_nbr, ctx->d_a_off + cb, ctx->d_A, x,
                           y + (size_t)cb * NP_, ctx->d_z, ctx->d_pbuf, nullptr, ctx->d_partials, ctx->d_alpha,
                           ctx->sr_ring_bytes, ctx->sr_G, ctx->d_a_dd ? ctx->d_a_dd + cb : nullptr)));
}

// Host: class-sorted work items for k_spmv_cls (dd[c] = compact offset of cell c's row-block). Cells of a
// class in ascending order, cut into runs of about nc / (5 x grid warps) cells. Off for p > 4 (register
// row-blocks) or cells with more than CLS_MAXDEG neighbours; DGAS_SPMV_CLS=0 disables it.
int spmv_cls_setup(dgas_ctx ctx, const std::vector<int64_t>& dd) {
  int on = 1;
  if (const char* e = std::getenv("DGAS_SPMV_CLS")) on = std::atoi(e) != 0;
  if (!on || ctx->p < 1 || ctx->p > 4 || ctx->max_deg > CLS_MAXDEG) return 0;
  const int nc = ctx->nc;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // two CTAs per SM where the 128-register cap does not spill (n_p <= 10): config 3 SpMV 134 -> 104 us
  int minb = ctx->np <= 10 ? 2 : 1;
  if (const char* e = std::getenv("DGAS_CLS_MINB")) minb = std::atoi(e) == 2 ? 2 : 1;
  ctx->cls_minb = minb;
  int tc = 1;  // tensor-core variant (k_spmv_cls_t; config 3: 0.077 -> 0.057 ms, 2989 -> 3097 PCG it/s): DGAS_CLS_TC=0 disables
  if (const char* e = std::getenv("DGAS_CLS_TC")) tc = std::atoi(e) != 0;
  if (ctx->np > 10) tc = 0;  // n_p = 15: the A fragments (46 doubles per lane) spill at the 128-register cap
  ctx->cls_tc = tc;
  int cps = 1;  // resident CTAs per SM (register-bound: the row-block lives in registers)
  if (tc) {
    DISPATCH_P15S(ctx->p, (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cps, k_spmv_cls_t<NP_>, SR_NW * 32, 0)));
  } else if (minb == 2) {
    DISPATCH_P15S(ctx->p, (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cps, k_spmv_cls<NP_, 2>, SR_NW * 32, 0)));
  } else {
    DISPATCH_P15S(ctx->p, (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cps, k_spmv_cls<NP_, 1>, SR_NW * 32, 0)));
  }
  cps = std::max(1, cps);
  if (const char* e = std::getenv("DGAS_CLS_CPS")) cps = std::max(1, std::atoi(e));
  const int grid = std::min(cps * nsm, std::max(1, nc / SR_NW));
  std::map<int64_t, std::vector<int>> cls;
  for (int c = 0; c < nc; ++c) cls[dd[c]].push_back(c);
  // runs of about nc / (5 x grid warps) cells, a multiple of the D cells a trip processes (config 3: 24 cells,
  // 0.077 ms; 12: 0.084, 18: 0.087, 36: 0.083)
  int run = (int)(nc / (5LL * grid * SR_NW));
  run = std::max(CLS_DEPTH, (run + CLS_DEPTH - 1) / CLS_DEPTH * CLS_DEPTH);
  if (const char* e = std::getenv("DGAS_CLS_RUN")) run = std::max(1, std::atoi(e));
  std::vector<int4> items;
  std::vector<int64_t> off;
  std::vector<int> cells;
  cells.reserve(nc);
  for (auto& kv : cls) {
    const int ci = (int)off.size();
    off.push_back(kv.first);
    const int c0 = kv.second[0];
    const int W = (ctx->nbr_ptr_h[c0 + 1] - ctx->nbr_ptr_h[c0]) * ctx->np;
    const int n = (int)kv.second.size(), nrun = (n + run - 1) / run;
    for (int t = 0; t < nrun; ++t) {
      const int b0 = (int)((int64_t)n * t / nrun), b1 = (int)((int64_t)n * (t + 1) / nrun);
      items.push_back(make_int4(ci, (int)cells.size() + b0, b1 - b0, W));
    }
    cells.insert(cells.end(), kv.second.begin(), kv.second.end());
  }
  // longest runs first so the round-robin deal ends evenly
  std::stable_sort(items.begin(), items.end(), [](const int4& u, const int4& v) { return u.z > v.z; });
  std::vector<int> nb((size_t)nc * CLS_MAXDEG);
  for (int i = 0; i < nc; ++i) {
    const int c = cells[i], lo = ctx->nbr_ptr_h[c], d = ctx->nbr_ptr_h[c + 1] - lo;
    for (int j = 0; j < CLS_MAXDEG; ++j) nb[(size_t)i * CLS_MAXDEG + j] = j < d ? ctx->nbr_h[lo + j] : c;
  }
  int st;
  if ((st = dev_upload(ctx, &ctx->d_cls_items, items)) || (st = dev_upload(ctx, &ctx->d_cls_off, off)) ||
      (st = dev_upload(ctx, &ctx->d_cls_cells, cells)) || (st = dev_upload(ctx, &ctx->d_cls_nb, nb)))
    return st;
  ctx->cls_nitems = (int)items.size();
  ctx->cls_grid = grid;
  if (std::getenv("DGAS_VERBOSE"))
    fprintf(stderr, "dgas: class SpMV: %zu row-block classes, %d items (runs <= %d cells), %d CTAs\n", cls.size(),
            ctx->cls_nitems, run, grid);
  return 0;
}
