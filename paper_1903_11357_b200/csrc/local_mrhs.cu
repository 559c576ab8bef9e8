// local_mrhs.cu — the local solves z_i = A_i^-1 r_i (the exact local solvers of the
// additive Schwarz operator) for subdomains that SHARE their factor, as one
// multiple-right-hand-side triangular solve per batch of subdomains.
//
// After exact de-duplication (dedup.cu) the 4,096 subdomains of config 3 use 64 distinct factors (one
// class of 3,844 interior subdomains). The per-subdomain kernels (k_local_warp, k_local_panel) run one
// dependent 2 x 64-step chain per subdomain: ~1 us per step, latency-bound (ncu: 21% occupancy, issue
// 0.51, L2 hit 96%). Here a CTA solves a batch of B subdomains of one class at once: every chain step
// is a small dense product with B columns instead of one,
//   forward  L y = r   : Y_k = P_k [R_k ; Y_{f_k..k-1}]          (NP x (NP + WU)) x (.. x B)
//   backward L^T z = y : V = P_k^T U_k, Z_k = V[0..NP), Y_{f_k..k-1} += V[NP..)    (U_k = Y_k)
// with P_k = [D_k | -U_k] the merged panel of cell k (local_panel.cu layout), so the chain runs 2m
// steps per BATCH instead of per subdomain and every factor element loaded is used B times.
//   * Y (m NP rows x B columns, fp64) lives in shared memory, row stride BS odd (conflict-free column
//     access); r is loaded into it, y overwrites r in place, z goes straight to global memory.
//   * One panel per step streamed by cp.async.bulk into an S-slot ring (thread 0 issues, S steps ahead;
//     the CTA barrier that ends a step releases its slot). The factors are L2-resident (20.5 MB on
//     config 3) and stay so (evict-last).
//   * Forward step: lanes = (column b of the batch, half), warps x halves = 16 column slices of the
//     step's panel; each thread accumulates all NP rows for its b over its slice, halves combine by a
//     shuffle, the 8 warps' partials by a shared-memory sum in fixed order (deterministic).
//   * Backward step: the same slices own panel columns; u_k (NP values per b) in registers.
// The batches (class, members) and the batch size are chosen on the host (mrhs_setup) so that all
// batches run in one wave; DGAS_MRHS=0 disables the kernel, DGAS_MR_B / DGAS_MR_S force B / slots.
#include <algorithm>
#include <map>

#include "internal.h"
#include "tma.cuh"

#define MR_T 256
#define MR_NW (MR_T / 32)

// panel layout helpers (same definitions as local_panel.cu)
template <int NP> __host__ __device__ constexpr int mr_dpk() { return (NP * (NP + 1) / 2 + 1) / 2 * 2; }
__host__ __device__ constexpr int mr_dcol(int np, int c) { return c * np - c * (c - 1) / 2; }

// dynamic smem: full[16] | fk[mc] | fm[mc] | slt[mc] | po[mc] | mb[32] | red[NW][NP][BMAX] | W[WC NP][BS] | ring
// W is a WINDOW of WC cells (row = (cell mod WC) NP + component, column b): the forward step k needs
// cells f_k..k, the backward step k cells fm_k..k (fm_k = min_{j >= k} f_j), both at most maxbw + 1 cells;
// r_{k+PD} / the y rows entering the backward window are prefetched PD steps ahead by cp.async into the
// slots of cells that are done, so WC = maxbw + PD + 1. y goes to global memory (the z array serves as
// the temporary: y_k is stored at z_k's place and read back by the backward sweep before z_k overwrites
// it), so shared memory no longer grows with the subdomain size and B = 32 fits several CTAs per SM.
#define MR_PD 6
struct MrLayout {
  size_t off_fk, off_fm, off_slt, off_po, off_mb, off_red, off_W, off_ring, total;
  __host__ __device__ MrLayout(int mc, int np, int bmax, int bs, int wc, int S, uint32_t slot) {
    off_fk = 128;
    off_fm = off_fk + (((size_t)mc * 4 + 15) & ~(size_t)15);
    off_slt = off_fm + (((size_t)mc * 4 + 15) & ~(size_t)15);
    off_po = off_slt + (((size_t)mc * 4 + 15) & ~(size_t)15);
    off_mb = off_po + (size_t)mc * 8;
    off_red = off_mb + 32 * 8;
    off_W = off_red + (size_t)MR_NW * np * bmax * 8;
    off_ring = (off_W + (size_t)wc * np * bs * 8 + 127) & ~(size_t)127;
    total = off_ring + (size_t)S * slot;
  }
};

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int NP>
__global__ void __launch_bounds__(MR_T) k_local_mrhs(int mode, int nbatch, const int4* __restrict__ batches,
                                                     const int* __restrict__ members, const int* __restrict__ sub_ptr,
                                                     const int* __restrict__ first, const int64_t* __restrict__ p_off,
                                                     const double* __restrict__ P, const double* r_in,
                                                     double* const* rbuf, double* z, const PcgState* st, int S,
                                                     uint32_t slot_bytes, int bmax, int BS, int WC, int max_cells) {
  constexpr int DPK = mr_dpk<NP>();
  extern __shared__ __align__(128) unsigned char sm[];
  const double* r = r_in;
  if (mode >= 1) {
    if (st->done) return;
    r = mode == 1 ? rbuf[0] : rbuf[(st->it + 1) & 1];
  }
  const MrLayout L(max_cells, NP, bmax, BS, WC, S, slot_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  int* fk = reinterpret_cast<int*>(sm + L.off_fk);
  int* fm = reinterpret_cast<int*>(sm + L.off_fm);
  int* slt = reinterpret_cast<int*>(sm + L.off_slt);
  int64_t* po = reinterpret_cast<int64_t*>(sm + L.off_po);
  int64_t* mb = reinterpret_cast<int64_t*>(sm + L.off_mb);
  double* red = reinterpret_cast<double*>(sm + L.off_red);
  double* W = reinterpret_cast<double*>(sm + L.off_W);
  unsigned char* ring = sm + L.off_ring;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int WR = WC * NP;  // window rows
  if (tid == 0) {
    for (int t = 0; t < S; ++t) mbar_init(&full[t], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = l2_evict_last();  // every batch of a class re-reads its factor: keep it in L2
  const int SM1 = S - 1;
  uint32_t gt = 0;  // steps this CTA has consumed: slot (g & SM1), parity (g / S) & 1
  for (int bi = blockIdx.x; bi < nbatch; bi += gridDim.x) {
    const int4 bt = batches[bi];
    const int rep = bt.x, moff = bt.y, B = bt.z;
    const int s0 = sub_ptr[rep], m = sub_ptr[rep + 1] - s0, T2 = 2 * m;
    for (int k = tid; k < m; k += MR_T) {
      fk[k] = first[s0 + k];
      po[k] = p_off[s0 + k];
      slt[k] = k % WC;
    }
    if (tid < B) mb[tid] = (int64_t)sub_ptr[members[moff + tid]] * NP;
    __syncthreads();
    if (tid == 0) {  // fm_k = min_{j >= k} f_j (the backward window's low end, monotone)
      int mn = 1 << 30;
      for (int k = m - 1; k >= 0; --k) { mn = min(mn, fk[k]); fm[k] = mn; }
    }
    // step t: forward cell t (t < m), backward cell 2m-1-t
    auto issue = [&](int t) {
      const int k = t < m ? t : T2 - 1 - t;
      const int n = DPK + (k - fk[k]) * NP * NP;  // D triangle + (k - f_k) NP columns of NP rows
      const uint32_t g = gt + (uint32_t)t;
      bulk_load(ring + (size_t)(g & SM1) * slot_bytes, P + po[k], (uint32_t)(((n + 1) & ~1) * 8), &full[g & SM1], pol);
    };
    if (tid == 0)
      for (int t = 0; t < min(S, T2); ++t) issue(t);
    // cp.async of NP rows x B columns of cell c from global (src: r or the y temporaries in z) into its slot
    auto fetch = [&](const double* src, int c) {
      double* dst = W + (size_t)slt[c] * NP * BS;
      for (int e = tid; e < NP * B; e += MR_T) {
        const int bb = e / NP, i = e - bb * NP;
        cp_async8(dst + (size_t)i * BS + bb, src + mb[bb] + (int64_t)c * NP + i);
      }
    };
    __syncthreads();  // slt / mb visible to fetch
    for (int c = 0; c < MR_PD; ++c) {
      if (c < m) fetch(r, c);
      cp_async_commit();
    }
    cp_async_wait<MR_PD - 1>();
    __syncthreads();
    const int H = B <= 16 ? 2 : 1;  // halves of a warp on different panel columns when B <= 16
    const int b = H == 2 ? (lane & 15) : lane, half = H == 2 ? (lane >> 4) : 0;
    const int NSL = MR_NW * H, sl = w * H + half;
    const bool act = b < B;
    // ------------------------------------------------ forward sweep
    for (int k = 0; k < m; ++k) {
      const uint32_t g = gt + (uint32_t)k;
      mbar_wait(&full[g & SM1], (g / S) & 1);
      const double* Ps = reinterpret_cast<const double*>(ring + (size_t)(g & SM1) * slot_bytes);
      const int f = fk[k], K = NP + (k - f) * NP, rk = slt[k] * NP, rf = slt[f] * NP;
      double acc[NP];
#pragma unroll
      for (int i = 0; i < NP; ++i) acc[i] = 0.0;
      if (act) {
        for (int q = sl; q < K; q += NSL) {
          if (q < NP) {  // D column q (rows q..NP-1) times r_k[q]
            const double rv = W[(size_t)(rk + q) * BS + b];
            const double* col = Ps + mr_dcol(NP, q) - q;
#pragma unroll
            for (int i = 0; i < NP; ++i)
              if (i >= q) acc[i] += col[i] * rv;
          } else {  // -U column j times y_old[j] (window rows wrap at WR)
            const int j = q - NP;
            int row = rf + j;
            row -= row >= WR ? WR : 0;
            const double yv = W[(size_t)row * BS + b];
            const double* col = Ps + DPK + j * NP;
            if constexpr (NP % 2 == 0) {
              const double2* c2 = reinterpret_cast<const double2*>(col);
#pragma unroll
              for (int i = 0; i < NP / 2; ++i) {
                const double2 pv = c2[i];
                acc[2 * i] += pv.x * yv;
                acc[2 * i + 1] += pv.y * yv;
              }
            } else {
#pragma unroll
              for (int i = 0; i < NP; ++i) acc[i] += col[i] * yv;
            }
          }
        }
      }
      if (H == 2) {
#pragma unroll
        for (int i = 0; i < NP; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 16);
      }
      if (act) {
#pragma unroll
        for (int i = 0; i < NP; ++i)
          if (H == 1 || (half == 0) == (i < NP / 2)) red[(w * NP + i) * bmax + b] = acc[i];
      }
      __syncthreads();  // partials written; the step's ring slot is consumed
      if (tid == 0 && k + S < T2) issue(k + S);
      if (k + MR_PD < m) fetch(r, k + MR_PD);  // slot of cell k + PD - WC < f_k: free
      cp_async_commit();
      for (int o = tid; o < NP * B; o += MR_T) {
        const int bb = o / NP, i = o - bb * NP;
        double s = 0;
#pragma unroll
        for (int ww = 0; ww < MR_NW; ++ww) s += red[(ww * NP + i) * bmax + bb];
        W[(size_t)(rk + i) * BS + bb] = s;
        z[mb[bb] + (int64_t)k * NP + i] = s;  // y_k, read back by the backward sweep
      }
      cp_async_wait<MR_PD - 1>();  // r_{k+1} landed
      __syncthreads();
    }
    // ------------------------------------------------ backward sweep
    // the window holds y of cells max(0, m - WC) .. m-1; cells below are fetched PD steps ahead
    int lo = max(0, m - WC);
    for (int kk = m - 1; kk >= max(0, m - MR_PD); --kk) {
      if (fm[kk] < lo) {
        for (int c = fm[kk]; c < lo; ++c) fetch(z, c);
        lo = fm[kk];
      }
      cp_async_commit();
    }
    cp_async_wait<MR_PD - 1>();
    __syncthreads();
    for (int k = m - 1; k >= 0; --k) {
      const int t = T2 - 1 - k;
      const uint32_t g = gt + (uint32_t)t;
      mbar_wait(&full[g & SM1], (g / S) & 1);
      const double* Ps = reinterpret_cast<const double*>(ring + (size_t)(g & SM1) * slot_bytes);
      const int f = fk[k], K = NP + (k - f) * NP, rk = slt[k] * NP, rf = slt[f] * NP;
      if (act) {
        double uk[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) uk[i] = W[(size_t)(rk + i) * BS + b];
        for (int q = sl; q < K; q += NSL) {
          if (q < NP) {  // z_k[q] = (D_k^T u_k)[q]
            const double* col = Ps + mr_dcol(NP, q) - q;
            double v = 0;
#pragma unroll
            for (int i = 0; i < NP; ++i)
              if (i >= q) v += col[i] * uk[i];
            z[mb[b] + (int64_t)k * NP + q] = v;
          } else {  // y_old[j] += (-U_k^T u_k)[j]
            const int j = q - NP;
            int row = rf + j;
            row -= row >= WR ? WR : 0;
            const double* col = Ps + DPK + j * NP;
            double v0 = 0, v1 = 0;
            if constexpr (NP % 2 == 0) {
              const double2* c2 = reinterpret_cast<const double2*>(col);
#pragma unroll
              for (int i = 0; i < NP / 2; ++i) {
                const double2 pv = c2[i];
                v0 += pv.x * uk[2 * i];
                v1 += pv.y * uk[2 * i + 1];
              }
            } else {
#pragma unroll
              for (int i = 0; i + 1 < NP; i += 2) {
                v0 += col[i] * uk[i];
                v1 += col[i + 1] * uk[i + 1];
              }
              v0 += col[NP - 1] * uk[NP - 1];
            }
            W[(size_t)row * BS + b] += v0 + v1;
          }
        }
      }
      // y rows of the cells the step k - PD needs (slots of cells > k, done)
      const int k2 = k - MR_PD;
      if (k2 >= 0 && fm[k2] < lo) {
        for (int c = fm[k2]; c < lo; ++c) fetch(z, c);
        lo = fm[k2];
      }
      cp_async_commit();
      cp_async_wait<MR_PD - 1>();
      __syncthreads();
      if (tid == 0 && t + S < T2) issue(t + S);
    }
    gt += (uint32_t)T2;
  }
}

// ------------------------------------------------------------------------------------------------
// k_local_mrhs_w — the same multi-RHS solve with INDEPENDENT WARP CHAINS (DGAS_MR_KERNEL=2). ncu on k_local_mrhs
// (config 3): ~2.4 us per chain step; stalls: shared-memory scoreboard 25%, CTA barrier 20%, fixed-latency
// waits 24%; every step pays two CTA barriers and a cross-warp reduction through shared memory. Here the
// right-hand sides of a batch are dealt to the warps, G per warp, and a warp never synchronises with the
// others: lane (g, ks) works on RHS column g and the panel columns q = ks (mod KS), KS = 32 / G.
//   forward  : acc[0..NP) over the lane's columns, summed over ks by KS-1 xor-shuffles per row
//   backward : u_k in registers, each lane owns its (q, g) entries (no reduction at all)
// The panels of the class are streamed once per CTA by a producer warp into the S-slot ring (full / empty
// mbarriers; empty counts one arrival per active consumer warp), so the warps drift apart by up to S steps.
// Each warp keeps its own window W_w (WC cells x NP rows x G columns) and its own cp.async prefetch of
// r (forward) / y (backward, from the temporaries in z); only __syncwarp on the chain.
// Lanes whose column is beyond the batch (g >= its count) mirror the last valid column: they compute and
// store the same values to the same addresses (benign), so the chain has no predication.
template <int NP, int G>
struct MrwCfg {
  static constexpr int KS = 32 / G;
  static constexpr int BS = G | 1;  // odd row stride of the window
};

struct MrwLayout {
  size_t off_fk, off_fm, off_slt, off_po, off_W, off_sc, off_ring, total;
  // sc = doubles of q staging per warp ((PD + 1) cells x NP rows x BS: the fused residual update, mode 3)
  __host__ __device__ MrwLayout(int mc, int np, int nw, int bs, int wc, int S, uint32_t slot, int sc = 0) {
    off_fk = 256;  // full[16] | empty[16]
    off_fm = off_fk + (((size_t)mc * 4 + 15) & ~(size_t)15);
    off_slt = off_fm + (((size_t)mc * 4 + 15) & ~(size_t)15);
    off_po = off_slt + (((size_t)mc * 4 + 15) & ~(size_t)15);
    off_W = off_po + (size_t)mc * 8;
    off_sc = off_W + (size_t)nw * wc * np * bs * 8;
    off_ring = (off_sc + (size_t)nw * sc * 8 + 127) & ~(size_t)127;
    total = off_ring + (size_t)S * slot;
  }
};

template <int NP, int G>
__global__ void __launch_bounds__(32 * 9) k_local_mrhs_w(int mode, int nbatch, const int4* __restrict__ batches,
                                                         const int* __restrict__ members,
                                                         const int* __restrict__ sub_ptr, const int* __restrict__ first,
                                                         const int64_t* __restrict__ p_off, const double* __restrict__ P,
                                                         const double* r_in, double* const* rbuf, double* z,
                                                         const PcgState* st, int NW, int S, uint32_t slot_bytes, int WC,
                                                         int max_cells, const double* qvec) {
  constexpr int DPK = mr_dpk<NP>(), KS = MrwCfg<NP, G>::KS, BS = MrwCfg<NP, G>::BS, PD = MR_PD;
  constexpr int SCW = (PD + 1) * NP * BS;  // q staging per warp (doubles), mode 3
  extern __shared__ __align__(128) unsigned char sm[];
  // mode 3 (PCG iteration, residual update fused; needs qvec and the q staging in the layout): r = r_old -
  // alpha q formed here with k_restrict_chunk's expression, so the restriction can run beside this kernel.
  // Built and measured on config 3: no gain (2011 vs 1997 PCG it/s; the coarse chain behind the restriction
  // is then as long as the local solve, and the 13 KB of staging cost 15%), so the launcher passes no qvec.
  const double* r = r_in;
  double alpha = 0;
  const bool fuse = mode == 3;
  if (mode >= 1) {
    if (st->done) return;
    const int it = st->it;
    r = mode == 1 ? rbuf[0] : mode == 2 ? rbuf[(it + 1) & 1] : rbuf[it & 1];
    if (fuse) alpha = st->alpha;
  }
  const MrwLayout L(max_cells, NP, NW, BS, WC, S, slot_bytes, qvec ? SCW : 0);  // staging only when launched for mode 3
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 16;
  int* fk = reinterpret_cast<int*>(sm + L.off_fk);
  int* fm = reinterpret_cast<int*>(sm + L.off_fm);
  int* slt = reinterpret_cast<int*>(sm + L.off_slt);
  int64_t* po = reinterpret_cast<int64_t*>(sm + L.off_po);
  unsigned char* ring = sm + L.off_ring;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int4 bt = batches[blockIdx.x];
  const int rep = bt.x, moff = bt.y, B = bt.z;
  const int s0 = sub_ptr[rep], m = sub_ptr[rep + 1] - s0, T2 = 2 * m;
  const int nwact = (B + G - 1) / G;  // consumer warps with at least one right-hand side
  for (int k = tid; k < m; k += blockDim.x) {
    fk[k] = first[s0 + k];
    po[k] = p_off[s0 + k];
    slt[k] = k % WC;
  }
  if (tid == 0) {
    for (int t = 0; t < S; ++t) { mbar_init(&full[t], 1); mbar_init(&empty[t], nwact); }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {  // fm_k = min_{j >= k} f_j (the backward window's low end, monotone)
    int mn = 1 << 30;
    for (int k = m - 1; k >= 0; --k) { mn = min(mn, fk[k]); fm[k] = mn; }
  }
  __syncthreads();
  const int SM1 = S - 1;
  if (w == NW) {
    // ---------------- producer warp: step t = forward cell t (t < m), backward cell 2m-1-t
    if (lane != 0) return;
    const uint64_t pol = l2_evict_last();  // every batch of the class re-reads its factor: keep it in L2
    for (int t = 0; t < T2; ++t) {
      const int sl = t & SM1;
      if (t >= S) mbar_wait_backoff(&empty[sl], (uint32_t)(((t / S) - 1) & 1));
      const int k = t < m ? t : T2 - 1 - t;
      const int n = DPK + (k - fk[k]) * NP * NP;
      bulk_load(ring + (size_t)sl * slot_bytes, P + po[k], (uint32_t)(((n + 1) & ~1) * 8), &full[sl], pol);
    }
    return;
  }
  if (w >= nwact) return;
  // ---------------- consumer warp w: columns w G .. w G + G - 1 of the batch
  const int g = lane % G, ks = lane / G;
  const int cnt = min(G, B - w * G);           // valid columns of this warp (>= 1)
  const int ge = min(g, cnt - 1);              // mirrored column
  const int64_t mbase = (int64_t)sub_ptr[members[moff + w * G + ge]] * NP;
  double* Ww = reinterpret_cast<double*>(sm + L.off_W) + (size_t)w * WC * NP * BS;
  const int WR = WC * NP;
  // cp.async of NP rows x G columns of cell c (src: r, or the y temporaries in z) into its window slot
  double* Qw = reinterpret_cast<double*>(sm + L.off_sc) + (size_t)w * SCW;
  // cp.async of NP rows x G columns of cell c (src: r, or the y temporaries in z) into its window slot. The
  // element (column gb, row i) a lane copies in round t is fixed: its source offset and window offset are
  // computed once (no division or shuffle on the chain)
  constexpr int FR = (NP * G + 31) / 32;
  int64_t fsrc[FR];
  int fdst[FR];
#pragma unroll
  for (int t = 0; t < FR; ++t) {
    const int e = t * 32 + lane;
    const int gb = e / NP, i = e - gb * NP;
    const int64_t mbb = __shfl_sync(0xffffffffu, mbase, gb & 31);  // lane gb (ks = 0) holds column gb's base
    fsrc[t] = e < NP * G ? mbb + i : -1;
    fdst[t] = i * BS + gb;
  }
  auto fetch = [&](const double* src, int c, bool withq) {
    double* dst = Ww + slt[c] * (NP * BS);
    double* dq = Qw + (c % (PD + 1)) * (NP * BS);
#pragma unroll
    for (int t = 0; t < FR; ++t)
      if (fsrc[t] >= 0) {
        cp_async8(dst + fdst[t], src + fsrc[t] + c * NP);
        if (withq) cp_async8(dq + fdst[t], qvec + fsrc[t] + c * NP);
      }
  };
  // mode 3: r_c = r_old - alpha q on the entries this lane copied itself (landed: its own wait_group)
  auto combine = [&](int c) {
    double* dst = Ww + slt[c] * (NP * BS);
    const double* dq = Qw + (c % (PD + 1)) * (NP * BS);
#pragma unroll
    for (int t = 0; t < FR; ++t)
      if (fsrc[t] >= 0) dst[fdst[t]] = fma(-alpha, dq[fdst[t]], dst[fdst[t]]);
  };
  for (int c = 0; c < PD; ++c) {
    if (c < m) fetch(r, c, fuse);
    cp_async_commit();
  }
  cp_async_wait<PD - 1>();
  if (fuse) combine(0);
  __syncwarp();
  // ------------------------------------------------ forward sweep
  // U columns of the panel per loop trip, all their loads issued before the first product (the chain is
  // latency-bound: ncu 0.37 issue slots per cycle, stalls on fixed latencies and shared-memory loads); a
  // column beyond the panel is clamped to column 0 with a zero multiplier, so there is no remainder loop
  constexpr int U = NP <= 10 ? 4 : 2;
  constexpr int NPAD = (NP + KS - 1) / KS * KS, RPL = NPAD / KS;  // rows per lane after the reduce-scatter
  for (int k = 0; k < m; ++k) {
    const int sl = k & SM1;
    mbar_wait(&full[sl], (uint32_t)((k / S) & 1));
    const double* __restrict__ Ps = reinterpret_cast<const double*>(ring + (size_t)sl * slot_bytes);
    const int f = fk[k], KU = (k - f) * NP, rk = slt[k] * NP, rf = slt[f] * NP;
    double acc[NPAD];
#pragma unroll
    for (int i = 0; i < NPAD; ++i) acc[i] = 0.0;
    for (int q = ks; q < NP; q += KS) {  // D column q (rows q..NP-1) times r_k[q]
      const double rv = Ww[(rk + q) * BS + g];
      const double* col = Ps + mr_dcol(NP, q) - q;
#pragma unroll
      for (int i = 0; i < NP; ++i)
        if (i >= q) acc[i] += col[i] * rv;
    }
    for (int j0 = ks; j0 < KU; j0 += KS * U) {  // -U column j times y_old[j] (window rows wrap at WR)
      double yv[U];
      const double* col[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int jj = j0 + u * KS;
        const bool ok = jj < KU;
        const int j = ok ? jj : 0;
        int row = rf + j;
        row -= row >= WR ? WR : 0;
        const double wv = Ww[row * BS + g];
        yv[u] = ok ? wv : 0.0;
        col[u] = Ps + DPK + j * NP;
      }
      if constexpr (NP % 2 == 0) {
        double2 pv[U][NP / 2];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int i = 0; i < NP / 2; ++i) pv[u][i] = reinterpret_cast<const double2*>(col[u])[i];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int i = 0; i < NP / 2; ++i) {
            acc[2 * i] += pv[u][i].x * yv[u];
            acc[2 * i + 1] += pv[u][i].y * yv[u];
          }
      } else {
        double pv[U][NP];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int i = 0; i < NP; ++i) pv[u][i] = col[u][i];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int i = 0; i < NP; ++i) acc[i] += pv[u][i] * yv[u];
      }
    }
    // reduce-scatter over the KS slices: at each level a lane keeps one half of its rows and adds the
    // partner's sums of that half; lane ks ends with the rows RPL ks .. RPL ks + RPL - 1 (fixed order)
    {
      int n = NPAD;
#pragma unroll
      for (int o = 16; o >= G; o >>= 1) {
        const int h = n / 2;
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < NPAD / 2; ++i)
          if (i < h) {
            const double snd = up ? acc[i] : acc[h + i];
            const double kep = up ? acc[h + i] : acc[i];
            acc[i] = kep + __shfl_xor_sync(0xffffffffu, snd, o);
          }
        n = h;
      }
    }
    __syncwarp();  // every lane is done with the ring slot and with the window rows it read
    if (lane == 0) mbar_arrive(&empty[sl]);
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int row = ks * RPL + i;
      if (row < NP) {
        Ww[(rk + row) * BS + g] = acc[i];
        z[mbase + (int64_t)k * NP + row] = acc[i];  // y_k, read back by the backward sweep
      }
    }
    if (k + PD < m) fetch(r, k + PD, fuse);  // slot of cell k + PD - WC < f_k: free
    cp_async_commit();
    cp_async_wait<PD - 1>();  // r_{k+1} landed (this lane's copies)
    if (fuse && k + 1 < m) combine(k + 1);
    __syncwarp();             // ... and everybody's, and y_k is visible
  }
  // ------------------------------------------------ backward sweep
  // the window holds y of cells max(0, m - WC) .. m-1; cells below are fetched PD steps ahead
  int lo = max(0, m - WC);
  for (int kk = m - 1; kk >= max(0, m - PD); --kk) {
    if (fm[kk] < lo) {
      for (int c = fm[kk]; c < lo; ++c) fetch(z, c, false);
      lo = fm[kk];
    }
    cp_async_commit();
  }
  cp_async_wait<PD - 1>();
  __syncwarp();
  for (int k = m - 1; k >= 0; --k) {
    const int t = T2 - 1 - k, sl = t & SM1;
    mbar_wait(&full[sl], (uint32_t)((t / S) & 1));
    const double* __restrict__ Ps = reinterpret_cast<const double*>(ring + (size_t)sl * slot_bytes);
    const int f = fk[k], KU = (k - f) * NP, rk = slt[k] * NP, rf = slt[f] * NP;
    double uk[NP];
#pragma unroll
    for (int i = 0; i < NP; ++i) uk[i] = Ww[(rk + i) * BS + g];
    for (int q = ks; q < NP; q += KS) {  // z_k[q] = (D_k^T u_k)[q]
      const double* col = Ps + mr_dcol(NP, q) - q;
      double v = 0;
#pragma unroll
      for (int i = 0; i < NP; ++i)
        if (i >= q) v += col[i] * uk[i];
      z[mbase + (int64_t)k * NP + q] = v;
    }
    for (int j0 = ks; j0 < KU; j0 += KS * U) {  // y_old[j] += (-U_k^T u_k)[j]: U independent columns per trip
      double* wp[U];
      double wv[U], v0[U], v1[U];
      const double* col[U];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int jj = j0 + u * KS;
        ok[u] = jj < KU;
        const int j = ok[u] ? jj : 0;
        int row = rf + j;
        row -= row >= WR ? WR : 0;
        wp[u] = Ww + row * BS + g;
        wv[u] = *wp[u];
        col[u] = Ps + DPK + j * NP;
        v0[u] = 0;
        v1[u] = 0;
      }
      if constexpr (NP % 2 == 0) {
        double2 pv[U][NP / 2];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int i = 0; i < NP / 2; ++i) pv[u][i] = reinterpret_cast<const double2*>(col[u])[i];
#pragma unroll
        for (int i = 0; i < NP / 2; ++i)
#pragma unroll
          for (int u = 0; u < U; ++u) {
            v0[u] += pv[u][i].x * uk[2 * i];
            v1[u] += pv[u][i].y * uk[2 * i + 1];
          }
      } else {
        double pv[U][NP];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int i = 0; i < NP; ++i) pv[u][i] = col[u][i];
#pragma unroll
        for (int i = 0; i + 1 < NP; i += 2)
#pragma unroll
          for (int u = 0; u < U; ++u) {
            v0[u] += pv[u][i] * uk[i];
            v1[u] += pv[u][i + 1] * uk[i + 1];
          }
#pragma unroll
        for (int u = 0; u < U; ++u) v0[u] += pv[u][NP - 1] * uk[NP - 1];
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (ok[u]) *wp[u] = wv[u] + (v0[u] + v1[u]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[sl]);
    // y rows of the cells the step k - PD needs (slots of cells > k, done)
    const int k2 = k - PD;
    if (k2 >= 0 && fm[k2] < lo) {
      for (int c = fm[k2]; c < lo; ++c) fetch(z, c, false);
      lo = fm[k2];
    }
    cp_async_commit();
    cp_async_wait<PD - 1>();
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------------------
// k_local_mrhs_r — warp chains with ROW lanes in the forward sweep (DGAS_MR_KERNEL=3). ncu on k_local_mrhs_w
// (config 3, 8 warps x 2 columns): ~470 warp instructions per chain step for 2 right-hand sides, 13% of
// them DFMA; a third is the cross-lane reduction of the K-sliced forward product (selects, shuffles) and
// its index arithmetic. Here a warp owns G = 32 / NP right-hand sides and lane (g, i) is
//   forward  : row i of y_k for column g: one sequential dot product over the panel's columns (4 independent
//              partial sums), the panel read column-major (lanes i consecutive), the window value of column g
//              broadcast to its NP lanes. No reduction, no shuffle.
//   backward : K-slice i (columns q = i mod NP) for column g, u_k in registers (as k_local_mrhs_w).
// The window is stored per column, W_w[g][row], so both sweeps read it conflict-free. Same ring / producer /
// prefetch protocol as k_local_mrhs_w; lanes beyond G NP idle.
struct MrrLayout {
  size_t off_fk, off_fm, off_slt, off_po, off_W, off_ring, total;
  int wrp;
  __host__ __device__ MrrLayout(int mc, int np, int nw, int g, int wc, int S, uint32_t slot) {
    wrp = (wc * np) | 1;  // odd column stride
    off_fk = 256;         // full[16] | empty[16]
    off_fm = off_fk + (((size_t)mc * 4 + 15) & ~(size_t)15);
    off_slt = off_fm + (((size_t)mc * 4 + 15) & ~(size_t)15);
    off_po = off_slt + (((size_t)mc * 4 + 15) & ~(size_t)15);
    off_W = off_po + (size_t)mc * 8;
    off_ring = (off_W + (size_t)nw * g * wrp * 8 + 127) & ~(size_t)127;
    total = off_ring + (size_t)S * slot;
  }
};

template <int NP>
__global__ void __launch_bounds__(32 * 9) k_local_mrhs_r(int mode, int nbatch, const int4* __restrict__ batches,
                                                         const int* __restrict__ members,
                                                         const int* __restrict__ sub_ptr, const int* __restrict__ first,
                                                         const int64_t* __restrict__ p_off, const double* __restrict__ P,
                                                         const double* r_in, double* const* rbuf, double* z,
                                                         const PcgState* st, int NW, int S, uint32_t slot_bytes, int WC,
                                                         int max_cells) {
  constexpr int DPK = mr_dpk<NP>(), G = 32 / NP, PD = MR_PD;
  extern __shared__ __align__(128) unsigned char sm[];
  const double* r = r_in;
  if (mode >= 1) {
    if (st->done) return;
    r = mode == 1 ? rbuf[0] : rbuf[(st->it + 1) & 1];
  }
  const MrrLayout L(max_cells, NP, NW, G, WC, S, slot_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 16;
  int* fk = reinterpret_cast<int*>(sm + L.off_fk);
  int* fm = reinterpret_cast<int*>(sm + L.off_fm);
  int* slt = reinterpret_cast<int*>(sm + L.off_slt);
  int64_t* po = reinterpret_cast<int64_t*>(sm + L.off_po);
  unsigned char* ring = sm + L.off_ring;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int4 bt = batches[blockIdx.x];
  const int rep = bt.x, moff = bt.y, B = bt.z;
  const int s0 = sub_ptr[rep], m = sub_ptr[rep + 1] - s0, T2 = 2 * m;
  const int nwact = (B + G - 1) / G;  // consumer warps with at least one right-hand side
  for (int k = tid; k < m; k += blockDim.x) {
    fk[k] = first[s0 + k];
    po[k] = p_off[s0 + k];
    slt[k] = (k % WC) * NP;  // first window row of cell k
  }
  if (tid == 0) {
    for (int t = 0; t < S; ++t) { mbar_init(&full[t], 1); mbar_init(&empty[t], nwact); }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {  // fm_k = min_{j >= k} f_j (the backward window's low end, monotone)
    int mn = 1 << 30;
    for (int k = m - 1; k >= 0; --k) { mn = min(mn, fk[k]); fm[k] = mn; }
  }
  __syncthreads();
  const int SM1 = S - 1;
  if (w == NW) {
    // ---------------- producer warp: step t = forward cell t (t < m), backward cell 2m-1-t
    if (lane != 0) return;
    const uint64_t pol = l2_evict_last();  // every batch of the class re-reads its factor: keep it in L2
    for (int t = 0; t < T2; ++t) {
      const int sl = t & SM1;
      if (t >= S) mbar_wait_backoff(&empty[sl], (uint32_t)(((t / S) - 1) & 1));
      const int k = t < m ? t : T2 - 1 - t;
      const int n = DPK + (k - fk[k]) * NP * NP;
      bulk_load(ring + (size_t)sl * slot_bytes, P + po[k], (uint32_t)(((n + 1) & ~1) * 8), &full[sl], pol);
    }
    return;
  }
  if (w >= nwact) return;
  // ---------------- consumer warp w: columns w G .. w G + G - 1 of the batch
  const int cnt = min(G, B - w * G);  // valid columns of this warp (>= 1)
  const int g = min(lane / NP, G - 1), i = lane - g * NP;
  const bool act = lane < G * NP && g < cnt;
  const int WRP = L.wrp, WR = WC * NP;
  const int64_t mbase = (int64_t)sub_ptr[members[moff + w * G + min(g, cnt - 1)]] * NP;
  double* Wg = reinterpret_cast<double*>(sm + L.off_W) + ((size_t)w * G + g) * WRP;  // this lane's column
  // cp.async of cell c (src: r, or the y temporaries in z): lane (g, i) copies entry i of its column
  auto fetch = [&](const double* src, int c) {
    if (act) cp_async8(Wg + slt[c] + i, src + mbase + (int64_t)c * NP + i);
  };
  for (int c = 0; c < PD; ++c) {
    if (c < m) fetch(r, c);
    cp_async_commit();
  }
  cp_async_wait<PD - 1>();
  __syncwarp();
  // ------------------------------------------------ forward sweep: y_k[i] = sum_q P_k[i][q] [r_k ; y_old][q]
  for (int k = 0; k < m; ++k) {
    const int sl = k & SM1;
    mbar_wait(&full[sl], (uint32_t)((k / S) & 1));
    const double* __restrict__ Ps = reinterpret_cast<const double*>(ring + (size_t)sl * slot_bytes);
    const int f = fk[k], KU = (k - f) * NP, rk = slt[k], rf = slt[f];
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    if (act) {
      // D_k r_k: column c holds rows c..NP-1 at dcol(c); row i takes columns c <= i
      const double* wr = Wg + rk;
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        const double dv = Ps[mr_dcol(NP, c) + (i >= c ? i - c : 0)];
        const double t = i >= c ? dv : 0.0;
        if (c & 1) a1 += t * wr[c];
        else a0 += t * wr[c];
      }
      // -U_k y_old, one cell (NP columns) per trip: its NP panel values and NP window values are all loaded
      // before the first product (no remainder: the column count is a multiple of NP; the window wraps at a
      // cell boundary)
      const double* pc = Ps + DPK + i;  // column j at pc[j NP]
      int slot = rf;
#pragma unroll 2
      for (int c = f; c < k; ++c) {
        const double* wv = Wg + slot;
        double pv[NP], wq[NP];
#pragma unroll
        for (int t = 0; t < NP; ++t) { pv[t] = pc[t * NP]; wq[t] = wv[t]; }
#pragma unroll
        for (int t = 0; t < NP; ++t) {
          if ((t & 3) == 0) a0 += pv[t] * wq[t];
          else if ((t & 3) == 1) a1 += pv[t] * wq[t];
          else if ((t & 3) == 2) a2 += pv[t] * wq[t];
          else a3 += pv[t] * wq[t];
        }
        pc += NP * NP;
        slot += NP;
        slot -= slot >= WR ? WR : 0;
      }
    }
    const double yk = (a0 + a1) + (a2 + a3);
    __syncwarp();  // every lane is done with the ring slot and with the window rows it read
    if (lane == 0) mbar_arrive(&empty[sl]);
    if (act) {
      Wg[rk + i] = yk;
      z[mbase + (int64_t)k * NP + i] = yk;  // y_k, read back by the backward sweep
    }
    if (k + PD < m) fetch(r, k + PD);  // slot of cell k + PD - WC < f_k: free
    cp_async_commit();
    cp_async_wait<PD - 1>();  // r_{k+1} landed (this lane's copies)
    __syncwarp();             // ... and everybody's, and y_k is visible
  }
  // ------------------------------------------------ backward sweep
  // the window holds y of cells max(0, m - WC) .. m-1; cells below are fetched PD steps ahead
  int lo = max(0, m - WC);
  for (int kk = m - 1; kk >= max(0, m - PD); --kk) {
    if (fm[kk] < lo) {
      for (int c = fm[kk]; c < lo; ++c) fetch(z, c);
      lo = fm[kk];
    }
    cp_async_commit();
  }
  cp_async_wait<PD - 1>();
  __syncwarp();
  constexpr int U = NP <= 10 ? 3 : 2;  // independent panel columns per loop trip
  for (int k = m - 1; k >= 0; --k) {
    const int t = T2 - 1 - k, sl = t & SM1;
    mbar_wait(&full[sl], (uint32_t)((t / S) & 1));
    const double* __restrict__ Ps = reinterpret_cast<const double*>(ring + (size_t)sl * slot_bytes);
    const int f = fk[k], KU = (k - f) * NP, rk = slt[k], rf = slt[f];
    if (act) {
      double uk[NP];
#pragma unroll
      for (int a = 0; a < NP; ++a) uk[a] = Wg[rk + a];
      {  // z_k[i] = (D_k^T u_k)[i]: column i of D_k holds rows i..NP-1
        const double* col = Ps + mr_dcol(NP, i) - i;
        double v = 0;
#pragma unroll
        for (int a = 0; a < NP; ++a)
          if (a >= i) v += col[a] * uk[a];
        z[mbase + (int64_t)k * NP + i] = v;
      }
      for (int j0 = i; j0 < KU; j0 += NP * U) {  // y_old[j] += (-U_k^T u_k)[j], U independent columns per trip
        double* wp[U];
        double wv[U], v0[U], v1[U];
        const double* col[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int jj = j0 + u * NP;
          ok[u] = jj < KU;
          const int j = ok[u] ? jj : 0;
          int row = rf + j;
          row -= row >= WR ? WR : 0;
          wp[u] = Wg + row;
          wv[u] = *wp[u];
          col[u] = Ps + DPK + j * NP;
          v0[u] = 0;
          v1[u] = 0;
        }
        if constexpr (NP % 2 == 0) {
          double2 pv[U][NP / 2];
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int a = 0; a < NP / 2; ++a) pv[u][a] = reinterpret_cast<const double2*>(col[u])[a];
#pragma unroll
          for (int a = 0; a < NP / 2; ++a)
#pragma unroll
            for (int u = 0; u < U; ++u) {
              v0[u] += pv[u][a].x * uk[2 * a];
              v1[u] += pv[u][a].y * uk[2 * a + 1];
            }
        } else {
          double pv[U][NP];
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int a = 0; a < NP; ++a) pv[u][a] = col[u][a];
#pragma unroll
          for (int a = 0; a + 1 < NP; a += 2)
#pragma unroll
            for (int u = 0; u < U; ++u) {
              v0[u] += pv[u][a] * uk[a];
              v1[u] += pv[u][a + 1] * uk[a + 1];
            }
#pragma unroll
          for (int u = 0; u < U; ++u) v0[u] += pv[u][NP - 1] * uk[NP - 1];
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (ok[u]) *wp[u] = wv[u] + (v0[u] + v1[u]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[sl]);
    // y rows of the cells the step k - PD needs (slots of cells > k, done)
    const int k2 = k - PD;
    if (k2 >= 0 && fm[k2] < lo) {
      for (int c = fm[k2]; c < lo; ++c) fetch(z, c);
      lo = fm[k2];
    }
    cp_async_commit();
    cp_async_wait<PD - 1>();
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------------------
// k_local_mrhs_t — the multi-RHS warp chains on the FP64 TENSOR CORES (mma.sync m8n8k4 f64; the default).
// With many right-hand sides per factor the chain step IS a dense contraction: Y_k (NP x 8) = P_k (NP x K) .
// W (K x 8) forward, and [z_k ; y_old] (K x 8) += P_k^T (K x NP) . U_k (NP x 8) backward, for the 8 columns a
// warp owns. One DMMA does 8 x 8 x 4 = 256 FMAs and sums over k inside the instruction: no K-slicing across
// lanes, no shuffle reduction, ~5x fewer instructions per right-hand side than k_local_mrhs_w (ncu there:
// instruction-bound, 13% DFMA). Fragments (PTX ISA, m8n8k4 f64): lane l holds A[l / 4][l % 4], B[l % 4][l / 4],
// C[l / 4][2 (l % 4) .. + 1]. The window is W_w[row][8] (8 columns, no padding): a B fragment reads 32
// consecutive doubles, a C fragment is one 16-byte access per lane, both conflict-free.
//   forward  : C(2 m-tiles of 8 rows x 8 columns) = sum over k-steps of 4 panel columns; the D triangle first
//              (masked to its lower part), columns beyond the panel masked to zero in A and B.
//   backward : B = u_k (NP x 8) loaded once (3 k-steps); z_k = D_k^T u_k (2 m-tiles), then per tile of 8 rows
//              of y_old: C = y_old (16-byte loads), C += (-U_k^T) u_k, stored back.
// Ring, producer warp, windows, cp.async prefetch and the y temporaries in z as in k_local_mrhs_w.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int NP>
__global__ void __launch_bounds__(32 * 9) k_local_mrhs_t(int mode, int nbatch, const int4* __restrict__ batches,
                                                         const int* __restrict__ members,
                                                         const int* __restrict__ sub_ptr, const int* __restrict__ first,
                                                         const int64_t* __restrict__ p_off, const double* __restrict__ P,
                                                         const double* r_in, double* const* rbuf, double* z,
                                                         const PcgState* st, int NW, int S, uint32_t slot_bytes, int WC,
                                                         int max_cells) {
  constexpr int DPK = mr_dpk<NP>(), G = 8, BS = 8, PD = MR_PD;
  constexpr int MT = (NP + 7) / 8;  // m-tiles of the NP rows
  constexpr int KT = (NP + 3) / 4;  // k-steps over NP
  extern __shared__ __align__(128) unsigned char sm[];
  const double* r = r_in;
  if (mode >= 1) {
    if (st->done) return;
    r = mode == 1 ? rbuf[0] : rbuf[(st->it + 1) & 1];
  }
  const MrwLayout L(max_cells, NP, NW, BS, WC, S, slot_bytes, 0);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 16;
  int* fk = reinterpret_cast<int*>(sm + L.off_fk);
  int* fm = reinterpret_cast<int*>(sm + L.off_fm);
  int* slt = reinterpret_cast<int*>(sm + L.off_slt);
  int64_t* po = reinterpret_cast<int64_t*>(sm + L.off_po);
  unsigned char* ring = sm + L.off_ring;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int4 bt = batches[blockIdx.x];
  const int rep = bt.x, moff = bt.y, B = bt.z;
  const int s0 = sub_ptr[rep], m = sub_ptr[rep + 1] - s0, T2 = 2 * m;
  const int nwact = (B + G - 1) / G;
  for (int k = tid; k < m; k += blockDim.x) {
    fk[k] = first[s0 + k];
    po[k] = p_off[s0 + k];
    slt[k] = (k % WC) * NP;  // first window row of cell k
  }
  if (tid == 0) {
    for (int t = 0; t < S; ++t) { mbar_init(&full[t], 1); mbar_init(&empty[t], nwact); }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    int mn = 1 << 30;
    for (int k = m - 1; k >= 0; --k) { mn = min(mn, fk[k]); fm[k] = mn; }
  }
  // the ring is read up to 6 doubles past a panel (rows 10..15 of a fragment) and the window holds padding
  // rows: start from finite data
  for (int e = tid; e < (int)((size_t)S * slot_bytes / 8); e += blockDim.x) reinterpret_cast<double*>(ring)[e] = 0.0;
  __syncthreads();
  const int SM1 = S - 1;
  if (w == NW) {
    if (lane != 0) return;
    fence_proxy_async();  // the zero fill (generic proxy) before the bulk copies (async proxy) into the ring
    const uint64_t pol = l2_evict_last();
    for (int t = 0; t < T2; ++t) {
      const int sl = t & SM1;
      if (t >= S) mbar_wait_backoff(&empty[sl], (uint32_t)(((t / S) - 1) & 1));
      const int k = t < m ? t : T2 - 1 - t;
      const int n = DPK + (k - fk[k]) * NP * NP;
      bulk_load(ring + (size_t)sl * slot_bytes, P + po[k], (uint32_t)(((n + 1) & ~1) * 8), &full[sl], pol);
    }
    return;
  }
  if (w >= nwact) return;
  // ---------------- consumer warp w: columns 8 w .. 8 w + 7 of the batch
  const int cnt = min(G, B - w * G);
  const int lr = lane >> 2, lk = lane & 3;  // fragment row / k index of this lane
  bool rowok[MT], kok[KT];                  // lane-constant masks: fragment row 8 t + lr / k index 4 kt + lk < NP
#pragma unroll
  for (int t = 0; t < MT; ++t) rowok[t] = 8 * t + lr < NP;
#pragma unroll
  for (int kt = 0; kt < KT; ++kt) kok[kt] = 4 * kt + lk < NP;
  const int gcol = lane & 7;                // lanes 0..7 (and their mirrors) hold column gcol's base
  const int64_t mbase = (int64_t)sub_ptr[members[moff + w * G + min(gcol, cnt - 1)]] * NP;
  const int64_t mb0 = __shfl_sync(0xffffffffu, mbase, 2 * lk), mb1 = __shfl_sync(0xffffffffu, mbase, 2 * lk + 1);
  double* Ww = reinterpret_cast<double*>(sm + L.off_W) + (size_t)w * WC * NP * BS;
  const int WR = WC * NP;
  for (int e = lane; e < WR * BS; e += 32) Ww[e] = 0.0;
  constexpr int FR = (NP * G + 31) / 32;
  int64_t fsrc[FR];
  int fdst[FR];
#pragma unroll
  for (int t = 0; t < FR; ++t) {
    const int e = t * 32 + lane;
    const int gb = e / NP, i = e - gb * NP;
    const int64_t mbb = __shfl_sync(0xffffffffu, mbase, gb & 7);
    fsrc[t] = e < NP * G ? mbb + i : -1;
    fdst[t] = i * BS + gb;
  }
  auto fetch = [&](const double* src, int c) {
    double* dst = Ww + slt[c] * BS;
#pragma unroll
    for (int t = 0; t < FR; ++t)
      if (fsrc[t] >= 0) cp_async8(dst + fdst[t], src + fsrc[t] + c * NP);
  };
  __syncwarp();
  for (int c = 0; c < PD; ++c) {
    if (c < m) fetch(r, c);
    cp_async_commit();
  }
  cp_async_wait<PD - 1>();
  __syncwarp();
  // ------------------------------------------------ forward sweep
  for (int k = 0; k < m; ++k) {
    const int sl = k & SM1;
    mbar_wait(&full[sl], (uint32_t)((k / S) & 1));
    const double* __restrict__ Ps = reinterpret_cast<const double*>(ring + (size_t)sl * slot_bytes);
    const int f = fk[k], KU = (k - f) * NP, rk = slt[k], rf = slt[f];
    double c0[MT], c1[MT];
#pragma unroll
    for (int t = 0; t < MT; ++t) { c0[t] = 0.0; c1[t] = 0.0; }
    // D_k r_k: k-steps over the NP columns of the packed lower triangle
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      const int c = 4 * kt + lk;
      const bool cv = c < NP;
      const int cc = cv ? c : 0;
      const double bv = cv ? Ww[(rk + cc) * BS + lr] : 0.0;
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        const int row = 8 * t + lr;
        const bool av = cv && row < NP && row >= c;
        const double a = av ? Ps[mr_dcol(NP, cc) + (av ? row - cc : 0)] : 0.0;
        dmma884(c0[t], c1[t], a, bv);
      }
    }
    // -U_k y_old: k-steps of 4 panel columns (window rows wrap at WR), UK k-steps per trip with all fragment
    // loads first and one accumulator set per k-step of the trip (independent DMMA chains: with ~1 warp per
    // scheduler the chain latency is what the step costs)
    constexpr int UK = 4;
    double ca[UK][MT][2];
#pragma unroll
    for (int u = 0; u < UK; ++u)
#pragma unroll
      for (int t = 0; t < MT; ++t) { ca[u][t][0] = 0.0; ca[u][t][1] = 0.0; }
    {
      // full trips (16 columns, no column masks): lane-constant fragment pointers advanced per trip
      const double* pA = Ps + DPK + lk * NP + lr;  // A[row lr (+ 8 t)][column lk] of the trip's first k-step
      int wrow = rf + lk;                          // window row of that column, kept in [0, WR)
      wrow -= wrow >= WR ? WR : 0;
      int j0 = 0;
      for (; j0 + 4 * UK <= KU; j0 += 4 * UK) {
        double av[UK][MT], bv[UK];
#pragma unroll
        for (int u = 0; u < UK; ++u) {
          int row = wrow + 4 * u;
          row -= row >= WR ? WR : 0;
          bv[u] = Ww[row * BS + lr];
#pragma unroll
          for (int t = 0; t < MT; ++t) {
            const double pv = pA[4 * u * NP + 8 * t];  // rows beyond NP: masked below (reads stay inside the ring + its 128-byte pad)
            if (8 * t + 7 < NP) av[u][t] = pv;  // every row of this m-tile exists (compile time)
            else av[u][t] = rowok[t] ? pv : 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < UK; ++u)
#pragma unroll
          for (int t = 0; t < MT; ++t) dmma884(ca[u][t][0], ca[u][t][1], av[u][t], bv[u]);
        pA += 4 * UK * NP;
        wrow += 4 * UK;
        wrow -= wrow >= WR ? WR : 0;
      }
      if (j0 < KU) {  // last, partial trip: columns beyond the panel masked to zero in A and B
        double av[UK][MT], bv[UK];
#pragma unroll
        for (int u = 0; u < UK; ++u) {
          const bool jv = j0 + 4 * u + lk < KU;
          int row = wrow + 4 * u;
          row -= row >= WR ? WR : 0;
          const double wv = Ww[(jv ? row : 0) * BS + lr];
          bv[u] = jv ? wv : 0.0;
#pragma unroll
          for (int t = 0; t < MT; ++t) {
            const bool ok = jv && rowok[t];
            const double pv = pA[ok ? 4 * u * NP + 8 * t : 0];
            av[u][t] = ok ? pv : 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < UK; ++u)
#pragma unroll
          for (int t = 0; t < MT; ++t) dmma884(ca[u][t][0], ca[u][t][1], av[u][t], bv[u]);
      }
    }
#pragma unroll
    for (int t = 0; t < MT; ++t) {
      c0[t] += (ca[0][t][0] + ca[1][t][0]) + (ca[2][t][0] + ca[3][t][0]);
      c1[t] += (ca[0][t][1] + ca[1][t][1]) + (ca[2][t][1] + ca[3][t][1]);
    }
    __syncwarp();  // every lane is done with the ring slot and with the window rows it read
    if (lane == 0) mbar_arrive(&empty[sl]);
#pragma unroll
    for (int t = 0; t < MT; ++t) {
      const int row = 8 * t + lr;
      if (row < NP) {
        *reinterpret_cast<double2*>(Ww + (rk + row) * BS + 2 * lk) = make_double2(c0[t], c1[t]);
        z[mb0 + (int64_t)k * NP + row] = c0[t];  // y_k, read back by the backward sweep
        z[mb1 + (int64_t)k * NP + row] = c1[t];
      }
    }
    if (k + PD < m) fetch(r, k + PD);
    cp_async_commit();
    cp_async_wait<PD - 1>();
    __syncwarp();
  }
  // ------------------------------------------------ backward sweep
  int lo = max(0, m - WC);
  for (int kk = m - 1; kk >= max(0, m - PD); --kk) {
    if (fm[kk] < lo) {
      for (int c = fm[kk]; c < lo; ++c) fetch(z, c);
      lo = fm[kk];
    }
    cp_async_commit();
  }
  cp_async_wait<PD - 1>();
  __syncwarp();
  for (int k = m - 1; k >= 0; --k) {
    const int t2 = T2 - 1 - k, sl = t2 & SM1;
    mbar_wait(&full[sl], (uint32_t)((t2 / S) & 1));
    const double* __restrict__ Ps = reinterpret_cast<const double*>(ring + (size_t)sl * slot_bytes);
    const int f = fk[k], KU = (k - f) * NP, rk = slt[k], rf = slt[f];
    double bu[KT];  // B fragments of u_k (NP x 8)
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      const int i = 4 * kt + lk;
      const double wv = Ww[(rk + (i < NP ? i : 0)) * BS + lr];
      bu[kt] = i < NP ? wv : 0.0;
    }
    // z_k = D_k^T u_k: row q, k-dimension i >= q (column q of D_k holds rows q..NP-1)
#pragma unroll
    for (int t = 0; t < MT; ++t) {
      const int q = 8 * t + lr;
      double z0 = 0.0, z1 = 0.0;
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        const int i = 4 * kt + lk;
        const bool av = q < NP && i < NP && i >= q;
        const double a = av ? Ps[mr_dcol(NP, av ? q : 0) + (av ? i - q : 0)] : 0.0;
        dmma884(z0, z1, a, bu[kt]);
      }
      if (q < NP) {
        z[mb0 + (int64_t)k * NP + q] = z0;
        z[mb1 + (int64_t)k * NP + q] = z1;
      }
    }
    // y_old += (-U_k^T) u_k, tiles of 8 rows of y_old, UT independent tiles per trip (loads first)
    constexpr int UT = 3;
    {
      const double* pB = Ps + DPK + lr * NP + lk;  // A[row j = lr (+ 8 u)][i = lk (+ 4 kt)] = (-U_k)[i][j]
      int wrow = rf + lr;                          // window row of y_old row lr, kept in [0, WR)
      wrow -= wrow >= WR ? WR : 0;
      int jt = 0;
      for (; jt + 8 * UT <= KU; jt += 8 * UT) {  // full trips: no row masks
        double2* wp[UT];
        double2 cv[UT];
        double av[UT][KT];
#pragma unroll
        for (int u = 0; u < UT; ++u) {
          int row = wrow + 8 * u;
          row -= row >= WR ? WR : 0;
          wp[u] = reinterpret_cast<double2*>(Ww + row * BS + 2 * lk);
          cv[u] = *wp[u];
#pragma unroll
          for (int kt = 0; kt < KT; ++kt) {
            if (4 * kt + 3 < NP) {  // every k index of this k-step exists (compile time)
              av[u][kt] = pB[8 * u * NP + 4 * kt];
            } else {
              const double pv = pB[8 * u * NP + (kok[kt] ? 4 * kt : 0)];
              av[u][kt] = kok[kt] ? pv : 0.0;
            }
          }
        }
#pragma unroll
        for (int kt = 0; kt < KT; ++kt)
#pragma unroll
          for (int u = 0; u < UT; ++u) dmma884(cv[u].x, cv[u].y, av[u][kt], bu[kt]);
#pragma unroll
        for (int u = 0; u < UT; ++u) *wp[u] = cv[u];
        pB += 8 * UT * NP;
        wrow += 8 * UT;
        wrow -= wrow >= WR ? WR : 0;
        wrow -= wrow >= WR ? WR : 0;
      }
      if (jt < KU) {  // last, partial trip
        double2* wp[UT];
        double2 cv[UT];
        double av[UT][KT];
        bool jv[UT];
#pragma unroll
        for (int u = 0; u < UT; ++u) {
          jv[u] = jt + 8 * u + lr < KU;
          int row = wrow + 8 * u;
          row -= row >= WR ? WR : 0;
          wp[u] = reinterpret_cast<double2*>(Ww + (jv[u] ? row : 0) * BS + 2 * lk);
          cv[u] = *wp[u];
#pragma unroll
          for (int kt = 0; kt < KT; ++kt) {
            const bool ok = jv[u] && kok[kt];
            const double pv = pB[ok ? 8 * u * NP + 4 * kt : 0];
            av[u][kt] = ok ? pv : 0.0;
          }
        }
#pragma unroll
        for (int kt = 0; kt < KT; ++kt)
#pragma unroll
          for (int u = 0; u < UT; ++u) dmma884(cv[u].x, cv[u].y, av[u][kt], bu[kt]);
#pragma unroll
        for (int u = 0; u < UT; ++u)
          if (jv[u]) *wp[u] = cv[u];
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[sl]);
    const int k2 = k - PD;
    if (k2 >= 0 && fm[k2] < lo) {
      for (int c = fm[k2]; c < lo; ++c) fetch(z, c);
      lo = fm[k2];
    }
    cp_async_commit();
    cp_async_wait<PD - 1>();
    __syncwarp();
  }
}

#define DISPATCH_MR(P, ...)                                 \
  switch (P) {                                              \
    case 1: { constexpr int NP_ = 3; __VA_ARGS__; } break;  \
    case 2: { constexpr int NP_ = 6; __VA_ARGS__; } break;  \
    case 3: { constexpr int NP_ = 10; __VA_ARGS__; } break; \
    case 4: { constexpr int NP_ = 15; __VA_ARGS__; } break; \
  }

#define DISPATCH_MRG(G, ...)                          \
  switch (G) {                                        \
    case 2: { constexpr int G_ = 2; __VA_ARGS__; } break;   \
    case 4: { constexpr int G_ = 4; __VA_ARGS__; } break;   \
    case 8: { constexpr int G_ = 8; __VA_ARGS__; } break;   \
    case 16: { constexpr int G_ = 16; __VA_ARGS__; } break; \
    case 32: { constexpr int G_ = 32; __VA_ARGS__; } break; \
  }

// Host: classes of subdomains sharing a factor (rep_of from dedup.cu), batch size and geometry.
// Cost model: the chain is 2m steps per batch whatever B, a step's shared-memory traffic grows with B,
// so take the B that runs every batch in the fewest waves, then the smallest such B.
int mrhs_setup(dgas_ctx ctx, const std::vector<int>& rep_of) {
  int on = 1;
  if (const char* e = std::getenv("DGAS_MRHS")) on = std::atoi(e) != 0;
  if (!on || ctx->p < 1 || ctx->p > 4 || ctx->max_sub_cells <= 1) return 0;
  const int nsub = ctx->nsub, np = ctx->np, mc = ctx->max_sub_cells;
  std::map<int, std::vector<int>> cls;
  for (int s2 = 0; s2 < nsub; ++s2) cls[rep_of[s2]].push_back(s2);
  // worth it only when subdomains really share factors (on average several per class)
  double minavg = 4.0;
  if (const char* e = std::getenv("DGAS_MR_MINAVG")) minavg = std::atof(e);  // tests: small meshes
  if ((double)nsub / (double)cls.size() < minavg) return 0;
  int dev = 0, nsm = 148, smem_sm = 233472, optin = 232448;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // widest panel of the representatives (bytes, 128-aligned slot)
  const int dpk = (np * (np + 1) / 2 + 1) / 2 * 2;
  int maxn = 0;
  for (auto& kv : cls) {
    const int rep = kv.first;
    for (int c = ctx->sub_ptr_h[rep]; c < ctx->sub_ptr_h[rep + 1]; ++c) {
      const int k = c - ctx->sub_ptr_h[rep];
      maxn = std::max(maxn, dpk + (k - ctx->first_h[c]) * np * np);
    }
  }
  const uint32_t slot = (uint32_t)((((maxn + 1) & ~1) * 8 + 127) / 128 * 128);
  // window: the widest backward reach k - min_{j >= k} f_j (>= the forward reach k - f_k) + prefetch distance
  int maxbw = 0;
  for (auto& kv : cls) {
    const int rep = kv.first, c0 = ctx->sub_ptr_h[rep], m = ctx->sub_ptr_h[rep + 1] - c0;
    int mn = 1 << 30;
    for (int k = m - 1; k >= 0; --k) {
      mn = std::min(mn, ctx->first_h[c0 + k]);
      maxbw = std::max(maxbw, k - mn);
    }
  }
  const int WC = std::min(mc, maxbw + MR_PD + 1);
  int S = 4;
  if (const char* e = std::getenv("DGAS_MR_S")) S = std::max(2, std::atoi(e));
  while (S & (S - 1)) ++S;  // power of two
  // room for one coarse-solve CTA per SM beside the local solves (the coarse chain runs concurrently)
  size_t reserve = 8 * 1024;
  if (ctx->coarse_mode == 2) reserve += (size_t)std::max(ctx->nd.maxN, ctx->nd.maxF + ctx->nd.maxU) * 8 + 1024;
  // 3: warp chains with row lanes forward (k_local_mrhs_r), 2: warp chains with K-slice lanes
  // (k_local_mrhs_w), 1: CTA-wide steps (k_local_mrhs)
  // config 3 (PCG it/s with everything else equal): kernel 4 (FP64 tensor cores, 2 warps x 8 columns) local
  // 0.160 ms / 2989; kernel 2 0.187 ms / 2750; kernel 3 0.210 ms (fewer instructions than 2, but its
  // sequential forward dot product is latency-bound)
  int kern = 4;
  if (const char* e = std::getenv("DGAS_MR_KERNEL")) kern = std::max(1, std::min(4, std::atoi(e)));
  if (kern >= 2) {
    // config 3 sweep (PCG it/s): 8 warps x 2 columns 2028, 4 x 4 1751, 4 x 8 1758, 8 x 4 1756, 4 x 2 1750
    int G = 2, NW = 8;
    if (!std::getenv("DGAS_MR_S")) S = 8;
    if (const char* e = std::getenv("DGAS_MR_G")) G = std::atoi(e);
    if (const char* e = std::getenv("DGAS_MR_NW")) NW = std::max(1, std::min(8, std::atoi(e)));
    if (G != 2 && G != 4 && G != 8 && G != 16 && G != 32) G = 2;
    if (kern == 3) G = 32 / np;  // one lane per (column, row)
    if (kern == 4) {             // tensor-core chains: 8 columns per warp (the n of m8n8k4)
      G = 8;
      if (!std::getenv("DGAS_MR_NW")) NW = 2;  // config 3: 2 warps 2989, 4 warps 2870, 8 warps 2915 PCG it/s
    }
    if (S > 16) S = 16;
    const int B = G * NW, BSw = kern == 4 ? 8 : (G | 1);
    const size_t need = kern == 4 ? MrwLayout(mc, np, NW, BSw, WC, S, slot, 0).total + 128 :
                        kern == 3 ? MrrLayout(mc, np, NW, G, WC, S, slot).total
                                  : MrwLayout(mc, np, NW, BSw, WC, S, slot, 0).total;
    if (need > (size_t)optin) kern = 1;
    else {
      std::vector<int4> bat;
      std::vector<int> mem;
      for (auto& kv : cls) {
        const int n = (int)kv.second.size(), nbat = (n + B - 1) / B;
        int off = 0;
        for (int t = 0; t < nbat; ++t) {
          const int cnt = n / nbat + (t < n % nbat ? 1 : 0);
          bat.push_back(make_int4(kv.first, (int)mem.size(), cnt, 0));
          for (int u = 0; u < cnt; ++u) mem.push_back(kv.second[off + u]);
          off += cnt;
        }
      }
      std::stable_sort(bat.begin(), bat.end(), [](const int4& a, const int4& b2) { return a.z > b2.z; });
      int st;
      if ((st = dev_upload(ctx, &ctx->d_mr_batches, bat)) || (st = dev_upload(ctx, &ctx->d_mr_members, mem))) return st;
      ctx->mr_nbatch = (int)bat.size();
      ctx->mr_B = B;
      ctx->mr_BS = BSw;
      ctx->mr_S = S;
      ctx->mr_slot = slot;
      ctx->mr_WC = WC;
      ctx->mr_G = G;
      ctx->mr_NW = NW;
      ctx->mr_smem = need;
      ctx->mr_grid = ctx->mr_nbatch;
      ctx->mr_classes = (int)cls.size();
      cudaError_t e = cudaSuccess;
      if (kern == 4) {
        DISPATCH_MR(ctx->p, ({
          cudaFuncAttributes fa;
          e = cudaFuncGetAttributes(&fa, k_local_mrhs_t<NP_>);
          if (e == cudaSuccess && (size_t)optin < ctx->mr_smem + fa.sharedSizeBytes) e = cudaErrorInvalidValue;
          if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_local_mrhs_t<NP_>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     optin - (int)fa.sharedSizeBytes);
        }));
      } else if (kern == 3) {
        DISPATCH_MR(ctx->p, ({
          cudaFuncAttributes fa;
          e = cudaFuncGetAttributes(&fa, k_local_mrhs_r<NP_>);
          if (e == cudaSuccess && (size_t)optin < ctx->mr_smem + fa.sharedSizeBytes) e = cudaErrorInvalidValue;
          if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_local_mrhs_r<NP_>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     optin - (int)fa.sharedSizeBytes);
        }));
      } else {
        DISPATCH_MR(ctx->p, DISPATCH_MRG(G, ({
          cudaFuncAttributes fa;
          e = cudaFuncGetAttributes(&fa, k_local_mrhs_w<NP_, G_>);
          if (e == cudaSuccess && (size_t)optin < ctx->mr_smem + fa.sharedSizeBytes) e = cudaErrorInvalidValue;
          if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_local_mrhs_w<NP_, G_>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     optin - (int)fa.sharedSizeBytes);
        })));
      }
      if (e != cudaSuccess) { ctx->detail = std::string("mrhs local smem: ") + cudaGetErrorString(e); return DGAS_E_CUDA; }
      if (std::getenv("DGAS_VERBOSE")) {
        size_t big = 0;
        for (auto& kv : cls) big = std::max(big, kv.second.size());
        fprintf(stderr, kern == 3 ? "dgas: multi-RHS local solve (warp chains, row lanes): %d classes (largest %zu), %d batches "
                "of <= %d (%d warps x %d columns, %d), window %d cells, ring %d x %u B, smem/CTA %zu\n" :
                "dgas: multi-RHS local solve (warp chains): %d classes (largest %zu), %d batches of <= %d "
                "(%d warps x %d columns, %d K-slices), window %d cells, ring %d x %u B, smem/CTA %zu\n", ctx->mr_classes,
                big, ctx->mr_nbatch, B, NW, G, 32 / G, WC, S, slot, ctx->mr_smem);
      }
      ctx->mr_kernel = kern;
      ctx->local_kernel = 5;
      return 0;
    }
  }
  ctx->mr_kernel = 1;
  int bforce = 0;
  if (const char* e = std::getenv("DGAS_MR_B")) bforce = std::max(1, std::min(32, std::atoi(e)));
  // fewest waves, then fewest batches (a step's instruction count per warp hardly depends on B <= 32)
  int bestB = 0, bestW = 1 << 30, bestCps = 0;
  int64_t bestNb = 1LL << 40;
  for (int B = 1; B <= 32; ++B) {
    if (bforce && B != bforce) continue;
    const int BS = B | 1;
    const size_t need = MrLayout(mc, np, B, BS, WC, S, slot).total;
    if (need > (size_t)optin) continue;
    const int cps = std::min<int>(2048 / MR_T, (int)(((size_t)smem_sm - std::min((size_t)smem_sm / 2, reserve)) / (need + 1024)));
    if (cps < 1) continue;
    int64_t nb = 0;
    for (auto& kv : cls) nb += ((int64_t)kv.second.size() + B - 1) / B;
    const int waves = (int)((nb + (int64_t)cps * nsm - 1) / ((int64_t)cps * nsm));
    if (waves < bestW || (waves == bestW && nb < bestNb)) { bestW = waves; bestB = B; bestCps = cps; bestNb = nb; }
  }
  if (!bestB) return 0;
  const int B = bestB, BS = B | 1;
  // batches: each class split into ceil(n/B) batches of near-equal size, largest first
  std::vector<int4> bat;
  std::vector<int> mem;
  for (auto& kv : cls) {
    const int n = (int)kv.second.size(), nbat = (n + B - 1) / B;
    int off = 0;
    for (int t = 0; t < nbat; ++t) {
      const int cnt = n / nbat + (t < n % nbat ? 1 : 0);
      bat.push_back(make_int4(kv.first, (int)mem.size(), cnt, 0));
      for (int u = 0; u < cnt; ++u) mem.push_back(kv.second[off + u]);
      off += cnt;
    }
  }
  std::stable_sort(bat.begin(), bat.end(), [](const int4& a, const int4& b2) { return a.z > b2.z; });
  int st;
  if ((st = dev_upload(ctx, &ctx->d_mr_batches, bat)) || (st = dev_upload(ctx, &ctx->d_mr_members, mem))) return st;
  ctx->mr_nbatch = (int)bat.size();
  ctx->mr_B = B;
  ctx->mr_BS = BS;
  ctx->mr_S = S;
  ctx->mr_slot = slot;
  ctx->mr_WC = WC;
  ctx->mr_smem = MrLayout(mc, np, B, BS, WC, S, slot).total;
  ctx->mr_grid = std::min(ctx->mr_nbatch, bestCps * nsm);
  ctx->mr_classes = (int)cls.size();
  cudaError_t e = cudaSuccess;
  DISPATCH_MR(ctx->p, ({
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, k_local_mrhs<NP_>);
    if (e == cudaSuccess && (size_t)optin < ctx->mr_smem + fa.sharedSizeBytes) e = cudaErrorInvalidValue;
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_local_mrhs<NP_>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
  }));
  if (e != cudaSuccess) { ctx->detail = std::string("mrhs local smem: ") + cudaGetErrorString(e); return DGAS_E_CUDA; }
  if (std::getenv("DGAS_VERBOSE")) {
    size_t big = 0;
    for (auto& kv : cls) big = std::max(big, kv.second.size());
    fprintf(stderr, "dgas: multi-RHS local solve: %d classes (largest %zu), %d batches of <= %d, %d CTAs (%d/SM, %d wave(s)), "
            "window %d cells, ring %d x %u B, smem/CTA %zu\n", ctx->mr_classes, big, ctx->mr_nbatch, B, ctx->mr_grid,
            bestCps, bestW, WC, S, slot, ctx->mr_smem);
  }
  ctx->local_kernel = 5;
  return 0;
}

void launch_local_mrhs(dgas_ctx ctx, int mode, const PcgState* st, const double* r, double* z, cudaStream_t s) {
  if (ctx->mr_kernel == 4) {
    DISPATCH_MR(ctx->p, (k_local_mrhs_t<NP_><<<ctx->mr_grid, (ctx->mr_NW + 1) * 32, ctx->mr_smem, s>>>(
                            mode, ctx->mr_nbatch, ctx->d_mr_batches, ctx->d_mr_members, ctx->d_sub_ptr, ctx->d_first,
                            ctx->d_p_off, reinterpret_cast<const double*>(ctx->d_P), r, ctx->d_rbuf, z, st, ctx->mr_NW,
                            ctx->mr_S, ctx->mr_slot, ctx->mr_WC, ctx->max_sub_cells)));
    return;
  }
  if (ctx->mr_kernel == 3) {
    DISPATCH_MR(ctx->p, (k_local_mrhs_r<NP_><<<ctx->mr_grid, (ctx->mr_NW + 1) * 32, ctx->mr_smem, s>>>(
                            mode, ctx->mr_nbatch, ctx->d_mr_batches, ctx->d_mr_members, ctx->d_sub_ptr, ctx->d_first,
                            ctx->d_p_off, reinterpret_cast<const double*>(ctx->d_P), r, ctx->d_rbuf, z, st, ctx->mr_NW,
                            ctx->mr_S, ctx->mr_slot, ctx->mr_WC, ctx->max_sub_cells)));
    return;
  }
  if (ctx->mr_kernel == 2) {
    DISPATCH_MR(ctx->p, DISPATCH_MRG(ctx->mr_G, (k_local_mrhs_w<NP_, G_><<<ctx->mr_grid, (ctx->mr_NW + 1) * 32, ctx->mr_smem, s>>>(
                            mode, ctx->mr_nbatch, ctx->d_mr_batches, ctx->d_mr_members, ctx->d_sub_ptr, ctx->d_first,
                            ctx->d_p_off, reinterpret_cast<const double*>(ctx->d_P), r, ctx->d_rbuf, z, st, ctx->mr_NW,
                            ctx->mr_S, ctx->mr_slot, ctx->mr_WC, ctx->max_sub_cells, (const double*)nullptr))));
    return;
  }
  DISPATCH_MR(ctx->p, (k_local_mrhs<NP_><<<ctx->mr_grid, MR_T, ctx->mr_smem, s>>>(
                          mode, ctx->mr_nbatch, ctx->d_mr_batches, ctx->d_mr_members, ctx->d_sub_ptr, ctx->d_first,
                          ctx->d_p_off, reinterpret_cast<const double*>(ctx->d_P), r, ctx->d_rbuf, z, st, ctx->mr_S,
                          ctx->mr_slot, ctx->mr_B, ctx->mr_BS, ctx->mr_WC, ctx->max_sub_cells)));
}
