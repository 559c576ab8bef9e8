// local_panel.cu — the local solves z_i = A_i^-1 r_i of the additive Schwarz preconditioner
// (exact solves with the subdomain blocks A_i), built for L2 reuse.
//
// Why a second local-solve kernel. A direct solve with A_i = L L^T reads every factor entry twice
// (forward sweep, then backward sweep in reverse order). k_local runs every subdomain at once
// (7 CTAs/SM on config 4) and so reads the factor twice from HBM: the 1024 concurrent factors
// (0.93 GB) cannot stay in the 126 MB L2 across the turnaround. This kernel runs few subdomains per
// SM (1-2 CTAs/SM) so that the part of each factor that is live between its forward and backward
// use (on average half a factor per running CTA) fits in L2, and it makes each step of the
// sweep chain short enough that this low concurrency still streams at HBM speed:
//   * merged panels P_k = [D_k | -U_k] (column-major, NP rows; D_k = L_kk^-1, U_k = D_k L_{k,f_k..k-1}),
//     so a forward step is ONE dot product y_k = P_k [r_k ; y_{f_k..k-1}] and a backward step is ONE
//     transposed product v = P_k^T u_k whose first NP entries are z_k = D_k^T u_k and the rest the
//     update y_{f_k..k-1} -= U_k^T u_k. No separate D^-1 prologue/epilogue sweeps.
//   * per-cell tables (unit ranges, f_k, panel offsets) precomputed on the host; no integer division
//     on the chain; power-of-two ring.
//   * 256 consumer threads per subdomain (16 lanes per row in the forward step, 2 per column in the
//     backward step); one producer warp streams CC-column units of the panels by cp.async.bulk into S
//     ring slots. Forward loads are evict-last (they are read again by the backward sweep), the
//     ring-resident tail and the backward loads are evict-first.
// Derivation (block rows of A_i = L L^T, D_k = L_kk^-1, U_k = D_k L_{k,old}):
//   forward  L y = r   : y_k = D_k r_k - U_k y_old
//   backward L^T z = y : u_k = y_k - sum_{j>k} U_j[:,k]^T u_j,  z_k = D_k^T u_k
#include "internal.h"
#define TMA_HOST_BACKOFF
#include "tma.cuh"

#ifndef PANEL_NARROW_TPC
#define PANEL_NARROW_TPC 1
#endif
#ifndef PANEL_WIDE_TPC
#define PANEL_WIDE_TPC(NP) ((NP) > 10 ? 2 : 1)
#endif
template <int NP, bool NARROW = false>
struct PanelCfg {
  static constexpr int T = (NP > 4 && !NARROW) ? 256 : 128;       // consumer threads
  static constexpr int ROWS = NP > 16 ? 32 : NP > 8 ? 16 : (NP > 4 ? 8 : 4);  // row slots in the forward step
  static constexpr int LPR = T / ROWS;                            // lanes per row (4 .. 32)
  static constexpr int NW = T / 32;
  // backward step: TPC threads per column (rows split into TPC slices of H). Narrow CTAs (HBM-bound):
  // 1 (no pair shuffle, fewer passes; cfg4 local 0.303 -> 0.289 ms). Wide CTAs (latency-bound): 1 up
  // to n_p = 10 (cfg1/2, cfg5 p1-p3 +1-3%), 2 at n_p = 15 (a 15-long dot per thread is too long a
  // chain: cfg5 p4q4 -8% with 1)
  static constexpr int TPC = NARROW ? PANEL_NARROW_TPC : PANEL_WIDE_TPC(NP);
  static constexpr int H = (NP + TPC - 1) / TPC;
};

// Panel layout of cell k (doubles, 16-byte aligned): D_k lower triangle packed column by column
// (column c holds rows c..NP-1 at dcol(c), padded to DPK, even), then the WU = (k - f_k) NP columns
// of -U_k (column j at DPK + j NP). Stream units: unit 0 = D part + U columns [0, CC0), unit t >= 1
// = U columns [CC0 + (t-1) CC, ...), CC and CC0 = CC - E even so every unit starts 16-byte aligned
// and fits a CC-column slot.
// TS = storage type of the panels: double (the fp64 contract) or float (NEXT-4 variant: fp32-stored
// factors, fp64 arithmetic). A = elements per 16 bytes; every count below is a multiple of A.
template <typename TS> __host__ __device__ constexpr int panel_al() { return 16 / (int)sizeof(TS); }
template <typename TS> __host__ __device__ constexpr int panel_dpk(int np) {
  return (np * (np + 1) / 2 + panel_al<TS>() - 1) / panel_al<TS>() * panel_al<TS>();
}
template <typename TS> __host__ __device__ constexpr int panel_e(int np) {
  return ((panel_dpk<TS>(np) + np - 1) / np + panel_al<TS>() - 1) / panel_al<TS>() * panel_al<TS>();
}
__host__ __device__ constexpr int panel_dcol(int np, int c) { return c * np - c * (c - 1) / 2; }
__host__ __device__ inline int panel_units(int wu, int cc, int cc0) { return 1 + (wu > cc0 ? (wu - cc0 + cc - 1) / cc : 0); }

// smem layout (must match panel_smem_bytes): full[64] | empty[64] | us[mc+1] | fk[mc] | po[mc] | [R] | Y | ring
// R (r_i staged) only in wide CTAs (latency-bound: r_k read from shared memory on the chain); narrow
// CTAs (HBM-bound, shared memory goes to the ring) read r_k from global memory one step ahead.
struct PanelLayout {
  size_t off_us, off_fk, off_po, off_R, off_Y, off_ring;
  __host__ __device__ PanelLayout(int mc, int np, bool stage_r) {
    off_us = 1024;
    off_fk = off_us + (((size_t)(mc + 1) * 4 + 15) & ~(size_t)15);
    off_po = off_fk + (((size_t)mc * 4 + 15) & ~(size_t)15);
    off_R = (off_po + (size_t)mc * 8 + 15) & ~(size_t)15;
    off_Y = off_R + (stage_r ? (((size_t)mc * np * 8 + 15) & ~(size_t)15) : 0);
    off_ring = (off_Y + (size_t)mc * np * 8 + 127) & ~(size_t)127;
  }
};

// NARROW (7 CTAs/SM): at most 48 registers so a 256-thread coarse-solve CTA still fits beside them
// FUSE (wide CTAs only): mode 3 is available (the narrow variant's 48-register cap spills with it)
template <int NP, bool NARROW, typename TS, bool FUSE = false>
__global__ void __launch_bounds__(PanelCfg<NP, NARROW>::T + 32, NARROW ? 8 : 3) k_local_panel(
    int mode, const int* __restrict__ sub_ptr, const int* __restrict__ first, const int* __restrict__ pus,
    const int* __restrict__ sub_units, const int64_t* __restrict__ p_off, const TS* __restrict__ P,
    const double* r_in, double* const* rbuf, double* z, const PcgState* st, int S, uint32_t slot_bytes, int CC,
    int max_cells, int keep_fwd, const double* qvec) {
  using C = PanelCfg<NP, NARROW>;
  constexpr int T = C::T, LPR = C::LPR, NW = C::NW, H = C::H, TPC = C::TPC;
  extern __shared__ __align__(128) double sm[];
  // mode 3 (PCG iteration, residual update fused): r = r_old - alpha q formed here with k_restrict_chunk's
  // expression; the restriction then runs beside this kernel on the coarse stream (iter_kernels.cu)
  const double* r = r_in;
  double alpha = 0;
  const bool fuse = FUSE && !NARROW && mode == 3;
  if (mode >= 1) {
    if (st->done) return;
    const int it = st->it;
    r = mode == 1 ? rbuf[0] : (mode == 2 || !FUSE) ? rbuf[(it + 1) & 1] : rbuf[it & 1];
    if (fuse) alpha = st->alpha;
  }
  const int s = blockIdx.x, s0 = sub_ptr[s], m = sub_ptr[s + 1] - s0;
  const PanelLayout L(max_cells, NP, !NARROW);
  unsigned char* smb = reinterpret_cast<unsigned char*>(sm);
  uint64_t* full = reinterpret_cast<uint64_t*>(smb);
  uint64_t* empty = full + 64;
  int* us_s = reinterpret_cast<int*>(smb + L.off_us);
  int* fk_s = reinterpret_cast<int*>(smb + L.off_fk);
  int64_t* po_s = reinterpret_cast<int64_t*>(smb + L.off_po);
  double* R = reinterpret_cast<double*>(smb + L.off_R);
  double* Y = reinterpret_cast<double*>(smb + L.off_Y);
  unsigned char* ring = smb + L.off_ring;
  const int tid = threadIdx.x;
  for (int k = tid; k < m; k += T + 32) {
    us_s[k] = pus[s0 + k];
    fk_s[k] = first[s0 + k];
    po_s[k] = p_off[s0 + k];
  }
  if (tid == 0) {
    us_s[m] = sub_units[s];
    for (int t = 0; t < S; ++t) { mbar_init(&full[t], 1); mbar_init(&empty[t], NW); }
    fence_mbar_init();
  }
  __syncthreads();
  const int U = us_s[m], SM1 = S - 1;
  if (tid >= T) {
    // ---------------- producer warp (one lane issues every copy)
    if (tid != T) return;
    const uint64_t pol_first = l2_evict_first(), pol_last = keep_fwd ? l2_evict_last() : pol_first;
    uint64_t epar = 0;  // parity of the next empty-barrier phase per slot
    constexpr int DPK = panel_dpk<TS>(NP), AL = panel_al<TS>();
    const int CC0 = CC - panel_e<TS>(NP);
    auto issue = [&](int u, int k, uint64_t pol) {
      const int WU = (k - fk_s[k]) * NP, t = u - us_s[k];
      int64_t off, n;
      if (t == 0) { off = 0; n = DPK + (int64_t)min(WU, CC0) * NP; }
      else { const int j0 = CC0 + (t - 1) * CC; off = DPK + (int64_t)j0 * NP; n = (int64_t)(min(WU, j0 + CC) - j0) * NP; }
      const uint32_t nbytes = (uint32_t)((n + AL - 1) / AL * AL * (int64_t)sizeof(TS));
      bulk_load(ring + (size_t)(u & SM1) * slot_bytes, P + po_s[k] + off, nbytes, &full[u & SM1], pol);
    };
    int k = 0;
    for (int u = 0; u < U; ++u) {  // forward stream: slot u & SM1 after the release of unit u - S
      while (us_s[k + 1] <= u) ++k;
      const int sl = u & SM1;
      if (u >= S) { mbar_wait_producer(&empty[sl], (uint32_t)((epar >> sl) & 1)); epar ^= 1ull << sl; }
      issue(u, k, u < U - S ? pol_last : pol_first);
    }
    int kw = m - 1;
    for (int v = U - 1; v >= S; --v) {  // backward refills: after the release of unit v, load unit v - S
      const int sl = v & SM1;
      mbar_wait_producer(&empty[sl], (uint32_t)((epar >> sl) & 1));
      epar ^= 1ull << sl;
      const int w = v - S;
      while (us_s[kw] > w) --kw;
      issue(w, kw, pol_first);
    }
    return;
  }
  // ---------------- consumers
  constexpr int DPK = panel_dpk<TS>(NP);
  const int CC0 = CC - panel_e<TS>(NP);
  const int lane = tid & 31;
  uint64_t fph = 0;  // parity of the next full-barrier phase per slot
  const double* rs = r + (size_t)s0 * NP;
  if constexpr (!NARROW) {
    if (fuse) {
      const double* qs = qvec + (size_t)s0 * NP;
      for (int e = tid; e < m * NP; e += T) R[e] = fma(-alpha, qs[e], rs[e]);
    } else {
      for (int e = tid; e < m * NP; e += T) R[e] = rs[e];
    }
    named_sync(1, T);
  }
  // forward: thread (a, q) accumulates row a of P_k over columns c = q (mod LPR)
  {
    const int a = tid / LPR, q = tid % LPR;
    constexpr int RN = (NP + LPR - 1) / LPR;  // D_k columns (r_k entries) per thread
    double rk[RN];  // narrow: r_k entries c = q + LPR t, prefetched one step ahead (overwritten after use)
    if constexpr (NARROW) {
#pragma unroll
      for (int t = 0; t < RN; ++t) rk[t] = rs[min(q + LPR * t, NP - 1)];
    }
    for (int k = 0; k < m; ++k) {
      const int u0 = us_s[k], u1 = us_s[k + 1], fk = fk_s[k];
      const int WU = (k - fk) * NP;
      if constexpr (!NARROW) {
#pragma unroll
        for (int t = 0; t < RN; ++t) rk[t] = q + LPR * t < NP ? R[k * NP + q + LPR * t] : 0.0;
      }
      const double* yb = Y + fk * NP;  // U column j multiplies Y[f_k NP + j]
      double v0 = 0, v1 = 0;
      for (int u = u0; u < u1; ++u) {
        const int sl = u & SM1, t = u - u0;
        mbar_wait(&full[sl], (uint32_t)((fph >> sl) & 1));
        fph ^= 1ull << sl;
        const TS* Ps = reinterpret_cast<const TS*>(ring + (size_t)sl * slot_bytes);
        if (a < NP) {
          int j0, j1;
          const TS* Pu;  // U column j at Pu[j NP]
          if (t == 0) {
#pragma unroll
            for (int t = 0; t < RN; ++t) {  // D_k r_k, lower triangle
              const int c = q + LPR * t;
              if (c < NP && c <= a) v1 += (double)Ps[panel_dcol(NP, c) + a - c] * rk[t];
            }
            if constexpr (NARROW) {  // prefetch r_{k+1}: unconditional loads from valid addresses (the
              // values are only used under c < NP), so the loads stay in flight until the next D step
              const int kn = min(k + 1, m - 1);
#pragma unroll
              for (int t = 0; t < RN; ++t) rk[t] = rs[kn * NP + min(q + LPR * t, NP - 1)];
            }
            j0 = 0; j1 = min(WU, CC0); Pu = Ps + DPK + a;
          } else {
            j0 = CC0 + (t - 1) * CC; j1 = min(WU, j0 + CC); Pu = Ps - j0 * NP + a;
          }
          int j = j0 + q;
          for (; j + LPR < j1; j += 2 * LPR) {
            v0 += (double)Pu[j * NP] * yb[j];
            v1 += (double)Pu[(j + LPR) * NP] * yb[j + LPR];
          }
          if (j < j1) v0 += (double)Pu[j * NP] * yb[j];
        }
        __syncwarp();
        // the ring-resident tail (u >= U - S) is released only once, by the backward sweep
        if (lane == 0 && u < U - S) mbar_arrive(&empty[sl]);
      }
      double v = v0 + v1;
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (q == 0 && a < NP) Y[k * NP + a] = v;
      named_sync(1, T);
    }
  }
  // backward: u_k = Y_k is final; v = P_k^T u_k, TPC threads per column, rows split in slices of H
  {
    const int half = tid % TPC, a0 = half * H;
    double* zs = z + (size_t)s0 * NP;
    for (int k = m - 1; k >= 0; --k) {
      const int u0 = us_s[k], u1 = us_s[k + 1], fk = fk_s[k];
      const int WU = (k - fk) * NP;
      // u_k rows of this thread's half: registers (wide CTAs) or read from shared memory per use
      // (narrow CTAs, whose 48-register cap would otherwise spill)
      double ukr[NARROW ? 1 : H];
      if constexpr (!NARROW) {
#pragma unroll
        for (int i = 0; i < H; ++i) ukr[i] = a0 + i < NP ? Y[k * NP + a0 + i] : 0.0;
      }
      const double* uks = Y + k * NP + a0;
      auto uk = [&](int i) -> double {
        if constexpr (NARROW) return uks[i];
        else return ukr[i];
      };
      double* yb = Y + fk * NP;
      for (int u = u1 - 1; u >= u0; --u) {
        const int sl = u & SM1, t = u - u0;
        if (u < U - S) {
          mbar_wait(&full[sl], (uint32_t)((fph >> sl) & 1));
          fph ^= 1ull << sl;
        }
        const TS* Ps = reinterpret_cast<const TS*>(ring + (size_t)sl * slot_bytes);
        // virtual columns x of this unit: unit 0 has the NP columns of D_k first (z_k = D_k^T u_k)
        const int xoff = t == 0 ? NP : 0;
        const int j0 = t == 0 ? 0 : CC0 + (t - 1) * CC, j1 = t == 0 ? min(WU, CC0) : min(WU, j0 + CC);
        const TS* Pu = t == 0 ? Ps + DPK : Ps - j0 * NP;  // U column j at Pu[j NP]
        const int nx = xoff + j1 - j0;
        // every lane of a warp runs the same trip count (warp-uniform bound), so the pair shuffle is
        // a full-warp one
        for (int xb = (tid >> 5) * (32 / TPC); xb < nx; xb += T / TPC) {
          const int x = xb + lane / TPC, j = j0 + x - xoff;
          // D column x holds rows x..NP-1 (D_k[a][x] at col[a]); U column j holds all rows. One
          // branch-free path for both (no divergence between the D and U lanes of warp 0)
          const bool isd = x < xoff;
          const TS* col = isd ? Ps + panel_dcol(NP, x) - x : Pu + j * NP;
          const int lo = isd ? x : 0, hi = x < nx ? NP : 0;
          double w0 = 0, w1 = 0;
#pragma unroll
          for (int i = 0; i + 1 < H; i += 2) {
            if (a0 + i < hi && a0 + i >= lo) w0 += (double)col[a0 + i] * uk(i);
            if (a0 + i + 1 < hi && a0 + i + 1 >= lo) w1 += (double)col[a0 + i + 1] * uk(i + 1);
          }
          if ((H & 1) && a0 + H - 1 < hi && a0 + H - 1 >= lo) w0 += (double)col[a0 + H - 1] * uk(H - 1);
          double w = w0 + w1;
          if constexpr (TPC == 2) w += __shfl_xor_sync(0xffffffffu, w, 1);
          if (half == 0 && x < nx) {
            if (x < xoff) zs[k * NP + x] = w;
            else yb[j] += w;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[sl]);
      }
      named_sync(1, T);
    }
  }
}

// P_k = [D_k packed lower triangle | -U_k] at p_off[c] (layout above), D_k from the row-major
// lower triangle of Dinv.
template <typename TS>
__global__ void k_build_panels(int np, int nc, const int* sub_ptr_of_cell, const int* first,
                               const int64_t* u_off, const double* U, const double* Dinv, const int64_t* p_off,
                               TS* P) {
  const int c = blockIdx.x;
  if (c >= nc) return;
  const int k = c - sub_ptr_of_cell[c], WU = (k - first[c]) * np, dpk = panel_dpk<TS>(np);
  TS* Pc = P + p_off[c];
  const double* Uc = U + u_off[c];
  const double* Dc = Dinv + (size_t)c * np * np;
  for (int e = threadIdx.x; e < np * np; e += blockDim.x) {
    const int a = e / np, cc = e % np;
    if (cc <= a) Pc[panel_dcol(np, cc) + a - cc] = (TS)Dc[a * np + cc];
  }
  for (int e = np * (np + 1) / 2 + threadIdx.x; e < dpk; e += blockDim.x) Pc[e] = (TS)0;
  for (int e = threadIdx.x; e < WU * np; e += blockDim.x) Pc[dpk + e] = (TS)(-Uc[e]);
}

#define DISPATCH_P15(P, ...)                                \
  switch (P) {                                              \
    case 1: { constexpr int NP_ = 3; __VA_ARGS__; } break;  \
    case 2: { constexpr int NP_ = 6; __VA_ARGS__; } break;  \
    case 3: { constexpr int NP_ = 10; __VA_ARGS__; } break; \
    case 4: { constexpr int NP_ = 15; __VA_ARGS__; } break; \
  }

// p = 5, 6 (n_p = 21, 28) were measured slower than the envelope kernel (config 5 p = q = 6: 1228 vs
// 1440 PCG it/s), so the panel kernel is built and used for p <= 4 only
int panel_supported(int p) { return p >= 1 && p <= 4; }

int panel_al(int f32) { return f32 ? panel_al<float>() : panel_al<double>(); }
int panel_min_cc(int np, int f32) { return f32 ? panel_e<float>(np) + 4 : panel_e<double>(np) + 2; }

// 128 consumer threads when more than 3 CTAs share an SM (registers), else 256
static bool panel_narrow(dgas_ctx ctx) { return ctx->panel_cps > 3; }
bool panel_is_narrow(dgas_ctx ctx) { return panel_narrow(ctx); }

size_t panel_base_bytes(int max_cells, int np, bool narrow) { return PanelLayout(max_cells, np, !narrow).off_ring; }

// host: panel offsets, per-cell unit starts, per-subdomain unit counts; device: the panels
template <typename TS>
static int panel_setup_t(dgas_ctx ctx, const std::vector<int>& sub_ptr, const std::vector<int>& first) {
  const int nc = ctx->nc, np = ctx->np, CC = ctx->panel_cc, CC0 = CC - panel_e<TS>(np), dpk = panel_dpk<TS>(np);
  constexpr int AL = panel_al<TS>();
  std::vector<int64_t> p_off(nc + 1, 0);
  std::vector<int> pus(nc), sub_units(ctx->nsub), sub_of(nc);
  for (int s = 0; s < ctx->nsub; ++s) {
    int acc = 0;
    for (int c = sub_ptr[s]; c < sub_ptr[s + 1]; ++c) {
      const int k = c - sub_ptr[s], WU = (k - first[c]) * np;
      sub_of[c] = sub_ptr[s];
      pus[c] = acc;
      acc += panel_units(WU, CC, CC0);
      p_off[c + 1] = p_off[c] + (dpk + (int64_t)np * WU + AL - 1) / AL * AL;  // 16-byte panels for TMA
    }
    sub_units[s] = acc;
  }
  ctx->p_total = p_off[nc];
  int st;
  if ((st = dev_upload(ctx, &ctx->d_p_off, p_off))) return st;
  if ((st = dev_upload(ctx, &ctx->d_pus, pus))) return st;
  if ((st = dev_upload(ctx, &ctx->d_sub_units, sub_units))) return st;
  int* d_sub_of = nullptr;
  if ((st = dev_upload(ctx, &d_sub_of, sub_of))) return st;
  if ((st = dev_alloc(ctx, &ctx->d_P, ((size_t)p_off[nc] * sizeof(TS) + 7) / 8 + 32))) { cudaFree(d_sub_of); return st; }
  k_build_panels<TS><<<nc, 128, 0, ctx->stream>>>(np, nc, d_sub_of, ctx->d_first, ctx->d_u_off, ctx->d_U, ctx->d_Dinv,
                                                  ctx->d_p_off, reinterpret_cast<TS*>(ctx->d_P));
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  cudaFree(d_sub_of);
  if (e != cudaSuccess) { ctx->detail = std::string("panel build: ") + cudaGetErrorString(e); return DGAS_E_CUDA; }
  return 0;
}

int panel_setup(dgas_ctx ctx, const std::vector<int>& sub_ptr, const std::vector<int>& first) {
  tma_set_backoff(0);  // producer-lane back-off of this unit's streaming kernels (DGAS_PRODUCER_NS)
  return ctx->panel_f32 ? panel_setup_t<float>(ctx, sub_ptr, first) : panel_setup_t<double>(ctx, sub_ptr, first);
}

size_t panel_smem_bytes(dgas_ctx ctx) {
  return PanelLayout(ctx->max_sub_cells, ctx->np, !panel_narrow(ctx)).off_ring +
         (size_t)ctx->panel_slots * ctx->panel_slot_bytes + 128;
}

// The attribute is per function (shared by every context in the process): always raise it to the
// opt-in maximum, never to this context's size (a later, smaller context would otherwise break the
// launches of an earlier one).
int panel_set_smem(dgas_ctx ctx) {
  const size_t smem = panel_smem_bytes(ctx);
  int dev = 0, mx = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaError_t e = cudaSuccess;
  auto raise = [&](const void* f) {
    cudaFuncAttributes fa;
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, f);
    if (e == cudaSuccess && (size_t)mx < smem + fa.sharedSizeBytes) e = cudaErrorInvalidValue;
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, mx - (int)fa.sharedSizeBytes);
  };
  DISPATCH_P15(ctx->p, (raise((const void*)k_local_panel<NP_, true, double>),
                        raise((const void*)k_local_panel<NP_, false, double>),
                        raise((const void*)k_local_panel<NP_, false, double, true>),
                        raise((const void*)k_local_panel<NP_, true, float>),
                        raise((const void*)k_local_panel<NP_, false, float>),
                        raise((const void*)k_local_panel<NP_, false, float, true>)));
  if (e != cudaSuccess) { ctx->detail = std::string("panel smem: ") + cudaGetErrorString(e); return DGAS_E_CUDA; }
  return 0;
}

void launch_local_panel(dgas_ctx ctx, int mode, PcgState* st, const double* r, double* z, cudaStream_t s) {
  const size_t smem = panel_smem_bytes(ctx);
#define PANEL_LAUNCH(NAR, TS)                                                                                      \
  DISPATCH_P15(ctx->p, (k_local_panel<NP_, NAR, TS, !NAR><<<ctx->nsub, PanelCfg<NP_, NAR>::T + 32, smem, s>>>(     \
                           mode, ctx->d_sub_ptr, ctx->d_first, ctx->d_pus, ctx->d_sub_units, ctx->d_p_off,         \
                           reinterpret_cast<const TS*>(ctx->d_P), r, ctx->d_rbuf, z, st, ctx->panel_slots,        \
                           ctx->panel_slot_bytes, ctx->panel_cc, ctx->max_sub_cells, ctx->panel_keep, ctx->d_q)))
  if (ctx->panel_f32) {
    if (panel_narrow(ctx)) { PANEL_LAUNCH(true, float); } else { PANEL_LAUNCH(false, float); }
  } else {
    if (panel_narrow(ctx)) { PANEL_LAUNCH(true, double); } else { PANEL_LAUNCH(false, double); }
  }
#undef PANEL_LAUNCH
}

// subdomains [sb, se) only (sharded solve, mode 0): shifted sub_ptr / sub_units, grid se - sb
void launch_local_panel_range(dgas_ctx ctx, int sb, int se, const double* r, double* z, cudaStream_t s) {
  if (se <= sb) return;
  const size_t smem = panel_smem_bytes(ctx);
#define PANEL_LAUNCH_R(NAR, TS)                                                                                    \
  DISPATCH_P15(ctx->p, (k_local_panel<NP_, NAR, TS><<<se - sb, PanelCfg<NP_, NAR>::T + 32, smem, s>>>(             \
                           0, ctx->d_sub_ptr + sb, ctx->d_first, ctx->d_pus, ctx->d_sub_units + sb, ctx->d_p_off,   \
                           reinterpret_cast<const TS*>(ctx->d_P), r, ctx->d_rbuf, z, nullptr, ctx->panel_slots,    \
                           ctx->panel_slot_bytes, ctx->panel_cc, ctx->max_sub_cells, ctx->panel_keep, nullptr)))
  if (ctx->panel_f32) {
    if (panel_narrow(ctx)) { PANEL_LAUNCH_R(true, float); } else { PANEL_LAUNCH_R(false, float); }
  } else {
    if (panel_narrow(ctx)) { PANEL_LAUNCH_R(true, double); } else { PANEL_LAUNCH_R(false, double); }
  }
#undef PANEL_LAUNCH_R
}

// ====================================================================================================
// k_local_warp — the same merged-panel solve (P_k = [D_k | -U_k], units of CCW columns), one WARP per
// subdomain. The CTA kernel above spends most issue slots on per-step CTA barriers, mbarrier polling
// and idle row/column slots (ncu, config 3: 72% issue-busy, 356 M warp instructions per launch), so it
// needs 7-8 CTAs per SM to stream at ~60% of HBM peak, and with every subdomain in flight the factor
// is read twice from HBM (backward sweep after the whole forward sweep; 1.65-1.85x the algorithmic
// bytes). Here a warp owns a subdomain end to end: lane (a, h) = (row, column slice) in the forward
// step (row sums by shuffles), lane = column in the backward step (u_k in registers), __syncwarp only,
// and the warp's lane 0 issues its own cp.async.bulk refills into a private ring (no empty barriers:
// producer and consumer are the same warp). Short steps let 1-2 warps per SM keep HBM busy, so few
// subdomains are in flight at a time and the forward copies (evict-last) are still in L2 when the
// backward sweep re-reads them: HBM reads the factor about once. Subdomains are taken dynamically
// (atomic counter; the last warp out resets it).
//   forward  L y = r   : y_k = D_k r_k - U_k y_old           (lanes: rows x column slices)
//   backward L^T z = y : v = P_k^T u_k, z_k = v[0..NP), y_old -= U_k^T u_k (lanes: columns)
// ====================================================================================================
template <int NP>
struct WarpCfg {
  static constexpr int LPR = 32 / NP;       // column slices per row (lanes a + NP h)
  static constexpr int LANES = NP * LPR;    // active lanes in the forward step
  static constexpr int RN = (NP + LPR - 1) / LPR;  // D columns (r_k entries) per lane
};

// per-warp smem: full[S] (256 B) | us[mc+1] | fk[mc] | po[mc] | Y[mc NP] | ring[S slot]
struct WarpLayout {
  size_t off_us, off_fk, off_po, off_Y, off_ring, stride;
  __host__ __device__ WarpLayout(int mc, int np, int S, uint32_t slot) {
    off_us = 256;
    off_fk = off_us + (((size_t)(mc + 1) * 4 + 15) & ~(size_t)15);
    off_po = off_fk + (((size_t)mc * 4 + 15) & ~(size_t)15);
    off_Y = off_po + (((size_t)mc * 8 + 15) & ~(size_t)15);
    off_ring = (off_Y + (size_t)mc * np * 8 + 127) & ~(size_t)127;
    stride = (off_ring + (size_t)S * slot + 127) & ~(size_t)127;
  }
};

template <int NP>
__global__ void __launch_bounds__(128) k_local_warp(
    int mode, int nsub, const int* __restrict__ sub_ptr, const int* __restrict__ first, const int* __restrict__ pus,
    const int* __restrict__ sub_units, const int64_t* __restrict__ p_off, const double* __restrict__ P,
    const double* r_in, double* const* rbuf, double* z, const PcgState* st, unsigned* cnt, int S, uint32_t slot_bytes,
    int CC, int max_cells, int keep_fwd) {
  using C = WarpCfg<NP>;
  constexpr int LPR = C::LPR, RN = C::RN;
  constexpr int DPK = panel_dpk<double>(NP), AL = panel_al<double>();
  extern __shared__ __align__(128) unsigned char smw[];
  const double* r = r_in;
  if (mode >= 1) {
    if (st->done) return;
    r = mode == 1 ? rbuf[0] : rbuf[(st->it + 1) & 1];
  }
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const WarpLayout L(max_cells, NP, S, slot_bytes);
  unsigned char* base = smw + (size_t)wl * L.stride;
  uint64_t* full = reinterpret_cast<uint64_t*>(base);
  int* us = reinterpret_cast<int*>(base + L.off_us);
  int* fk = reinterpret_cast<int*>(base + L.off_fk);
  int64_t* po = reinterpret_cast<int64_t*>(base + L.off_po);
  double* Y = reinterpret_cast<double*>(base + L.off_Y);
  unsigned char* ring = base + L.off_ring;
  if (lane == 0) {
    for (int t = 0; t < S; ++t) mbar_init(&full[t], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const int SM1 = S - 1, CC0 = CC - panel_e<double>(NP);
  const uint64_t pol_first = l2_evict_first(), pol_keep = keep_fwd ? l2_evict_last() : pol_first;
  uint32_t ph = 0;  // parity of the next completion per slot (S <= 32)
  const int a = lane % NP, h = lane / NP;
  const bool fwd_lane = lane < C::LANES;
  for (;;) {
    int sub = 0;
    if (lane == 0) sub = (int)atomicAdd(cnt, 1u);
    sub = __shfl_sync(0xffffffffu, sub, 0);
    if (sub >= nsub) break;
    const int s0 = sub_ptr[sub], m = sub_ptr[sub + 1] - s0;
    for (int k = lane; k < m; k += 32) {
      us[k] = pus[s0 + k];
      fk[k] = first[s0 + k];
      po[k] = p_off[s0 + k];
    }
    if (lane == 0) us[m] = sub_units[sub];
    __syncwarp();
    const int U = us[m];
    // unit u of cell k -> (offset, bytes) in the cell's panel
    auto issue = [&](int u, int k, uint64_t pol) {
      const int WU = (k - fk[k]) * NP, t = u - us[k];
      int64_t off, n;
      if (t == 0) { off = 0; n = DPK + (int64_t)min(WU, CC0) * NP; }
      else { const int j0 = CC0 + (t - 1) * CC; off = DPK + (int64_t)j0 * NP; n = (int64_t)(min(WU, j0 + CC) - j0) * NP; }
      const uint32_t nbytes = (uint32_t)((n + AL - 1) / AL * AL * 8);
      bulk_load(ring + (size_t)(u & SM1) * slot_bytes, P + po[k] + off, nbytes, &full[u & SM1], pol);
    };
    int kf = 0;  // lane 0: cell of the next forward unit to issue
    if (lane == 0) {
      for (int u = 0; u < min(S, U); ++u) {
        while (us[kf + 1] <= u) ++kf;
        issue(u, kf, u < U - S ? pol_keep : pol_first);
      }
    }
    const double* rs = r + (size_t)s0 * NP;
    double rk[RN];  // r_k entries c = h + LPR t (used only where c < NP: loads need no predicate)
#pragma unroll
    for (int t = 0; t < RN; ++t) rk[t] = rs[min(h + LPR * t, NP - 1)];
    // ---------------- forward sweep
    for (int k = 0; k < m; ++k) {
      const int u0 = us[k], u1 = us[k + 1], f = fk[k], WU = (k - f) * NP;
      const double* yb = Y + f * NP;
      double v0 = 0, v1 = 0;
      for (int u = u0; u < u1; ++u) {
        const int sl = u & SM1, t = u - u0;
        mbar_wait(&full[sl], (ph >> sl) & 1);
        ph ^= 1u << sl;
        const double* Ps = reinterpret_cast<const double*>(ring + (size_t)sl * slot_bytes);
        if (fwd_lane) {
          int j0, j1;
          const double* Pu;
          if (t == 0) {
#pragma unroll
            for (int tt = 0; tt < RN; ++tt) {
              const int c = h + LPR * tt;
              if (c < NP && c <= a) v1 += Ps[panel_dcol(NP, c) + a - c] * rk[tt];
            }
            j0 = 0; j1 = min(WU, CC0); Pu = Ps + DPK + a;
          } else {
            j0 = CC0 + (t - 1) * CC; j1 = min(WU, j0 + CC); Pu = Ps - j0 * NP + a;
          }
          int j = j0 + h;
          double v2 = 0, v3 = 0;
          for (; j + 3 * LPR < j1; j += 4 * LPR) {  // 8 independent loads in flight per lane
            const double p0 = Pu[j * NP], p1 = Pu[(j + LPR) * NP], p2 = Pu[(j + 2 * LPR) * NP],
                         p3 = Pu[(j + 3 * LPR) * NP];
            const double y0 = yb[j], y1 = yb[j + LPR], y2 = yb[j + 2 * LPR], y3 = yb[j + 3 * LPR];
            v0 += p0 * y0; v1 += p1 * y1; v2 += p2 * y2; v3 += p3 * y3;
          }
          for (; j < j1; j += LPR) v0 += Pu[j * NP] * yb[j];
          v0 += v2; v1 += v3;
        }
        __syncwarp();
        if (lane == 0 && u + S < U) {  // the slot is consumed: refill it with unit u + S
          while (us[kf + 1] <= u + S) ++kf;
          issue(u + S, kf, u + S < U - S ? pol_keep : pol_first);
        }
      }
      double v = v0 + v1, tot = v;
#pragma unroll
      for (int h2 = 1; h2 < LPR; ++h2) tot += __shfl_sync(0xffffffffu, v, (a + NP * h2) & 31);
      if (h == 0 && lane < NP) Y[k * NP + a] = tot;
      // prefetch r_{k+1} (unconditional, valid addresses: stays in flight until the next D step)
      const int kn = min(k + 1, m - 1);
#pragma unroll
      for (int t = 0; t < RN; ++t) rk[t] = rs[kn * NP + min(h + LPR * t, NP - 1)];
      __syncwarp();
    }
    // ---------------- backward sweep: units in reverse; the last S units are still in the ring
    int kb = m - 1;  // lane 0: cell of the next backward refill
    double* zs = z + (size_t)s0 * NP;
    for (int k = m - 1; k >= 0; --k) {
      const int u0 = us[k], u1 = us[k + 1], f = fk[k], WU = (k - f) * NP;
      double uk[NP];
#pragma unroll
      for (int i = 0; i < NP; ++i) uk[i] = Y[k * NP + i];
      double* yb = Y + f * NP;
      for (int u = u1 - 1; u >= u0; --u) {
        const int sl = u & SM1, t = u - u0;
        if (u < U - S) {
          mbar_wait(&full[sl], (ph >> sl) & 1);
          ph ^= 1u << sl;
        }
        const double* Ps = reinterpret_cast<const double*>(ring + (size_t)sl * slot_bytes);
        const int xoff = t == 0 ? NP : 0;
        const int j0 = t == 0 ? 0 : CC0 + (t - 1) * CC, j1 = t == 0 ? min(WU, CC0) : min(WU, j0 + CC);
        const double* Pu = t == 0 ? Ps + DPK : Ps - j0 * NP;
        const int nx = xoff + j1 - j0;
        if (t == 0 && lane < NP) {  // z_k = D_k^T u_k: D column x holds rows x..NP-1
          const int x = lane;
          const double* col = Ps + panel_dcol(NP, x) - x;
          double w = 0;
#pragma unroll
          for (int i = 0; i < NP; ++i)
            if (i >= x) w += col[i] * uk[i];
          zs[k * NP + x] = w;
        }
        // U columns: y_old -= U_k^T u_k (full columns, no predicates)
        for (int x = lane; x < nx - xoff; x += 32) {
          const double* col = Pu + (j0 + x) * NP;
          double w0 = 0, w1 = 0;
#pragma unroll
          for (int i = 0; i + 1 < NP; i += 2) {
            w0 += col[i] * uk[i];
            w1 += col[i + 1] * uk[i + 1];
          }
          if (NP & 1) w0 += col[NP - 1] * uk[NP - 1];
          yb[j0 + x] += w0 + w1;
        }
        __syncwarp();
        if (lane == 0 && u - S >= 0) {  // slot consumed: load unit u - S (needed S units later)
          while (us[kb] > u - S) --kb;
          issue(u - S, kb, pol_first);
        }
      }
      __syncwarp();
    }
  }
  // last warp out resets the subdomain counter for the next launch
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(cnt + 1, 1u) == gridDim.x * (blockDim.x >> 5) - 1) {
      cnt[0] = 0;
      cnt[1] = 0;
      __threadfence();
    }
  }
}

// host: the warp kernel's own unit tables (its CCW differs from the CTA kernel's CC), ring sizing
int local_warp_setup(dgas_ctx ctx) {
  if (!panel_supported(ctx->p) || ctx->max_sub_cells <= 1 || ctx->panel_f32) return 0;
  int dev = 0, nsm = 148, smem_sm = 233472, optin = 232448;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // default on for the large configs with n_p <= 10 (>= 4 subdomains per SM; measured B200 PCG it/s,
  // tools/gpu_ab.sh: config 3 1077 -> 1150 with 4 x 4 warps/SM). Config 4 (n_p = 15) runs 1814 -> 1912 with
  // it, but its different summation order moves the stopping iteration of that plateau-prone solve (rho
  // jumps of 1e8) to 682, outside both +-2 of the oracle's 688 and the oracle's own perturbation spread
  // (684..688, tools/golden_spread.py); the CTA kernel gives 687, so config 4 keeps it (R22).
  // The CTA kernel also stays for few subdomains (config 5: 256, latency-bound chains, 1.8-2.3x faster).
  int want = ctx->nsub >= 4 * nsm && ctx->np <= 10;
  if (const char* e = std::getenv("DGAS_LOCAL_WARP")) want = std::atoi(e) != 0;
  if (!want) return 0;
  int W = 4, cps = ctx->np <= 10 ? 4 : 2;
  if (const char* e = std::getenv("DGAS_LW_WARPS")) W = std::max(1, std::min(4, std::atoi(e)));
  if (const char* e = std::getenv("DGAS_LW_CPS")) cps = std::max(1, std::min(16, std::atoi(e)));
  size_t reserve = 8 * 1024;
  if (ctx->coarse_mode == 2) reserve += (size_t)std::max(ctx->nd.maxN, ctx->nd.maxF + ctx->nd.maxU) * 8 + 1024;
  size_t per_cta = std::min((size_t)optin, ((size_t)smem_sm - reserve) / cps - 1024);
  const size_t per_warp = per_cta / W;
  const int np = ctx->np, mc = ctx->max_sub_cells;
  const size_t fixed = WarpLayout(mc, np, 0, 0).off_ring + 128;
  if (per_warp <= fixed + 4096) return 0;
  const size_t B = per_warp - fixed;
  size_t target = 8 * 1024;
  if (const char* e = std::getenv("DGAS_LW_SLOT_KB")) target = (size_t)std::atoi(e) * 1024;
  int S = 2;
  while (S < 32 && B / (2 * S) >= target) S *= 2;
  const int cc_min = panel_min_cc(np, 0), maxW = ctx->max_urow + np;
  const int cc_max = std::max(cc_min, (maxW + 1) / 2 * 2);
  int CC = (int)std::min<size_t>(cc_max, (B / S) / (8 * np)) / 2 * 2;
  if (CC < cc_min) return 0;
  const uint32_t sb = (uint32_t)(((((int64_t)CC * np + 1) / 2 * 2) * 8 + 127) / 128 * 128);
  while (S < 32 && (size_t)2 * S * sb <= B) S *= 2;
  // unit tables for CCW = CC
  const std::vector<int>& sp = ctx->sub_ptr_h;
  const int CC0 = CC - panel_e<double>(np);
  std::vector<int> pus(ctx->nc), sub_units(ctx->nsub);
  int maxU = 0;
  for (int s = 0; s < ctx->nsub; ++s) {
    int acc = 0;
    for (int c = sp[s]; c < sp[s + 1]; ++c) {
      const int k = c - sp[s], WU = (k - ctx->first_h[c]) * np;
      pus[c] = acc;
      acc += panel_units(WU, CC, CC0);
    }
    sub_units[s] = acc;
    maxU = std::max(maxU, acc);
  }
  int st;
  if ((st = dev_upload(ctx, &ctx->d_lw_pus, pus)) || (st = dev_upload(ctx, &ctx->d_lw_units, sub_units))) return st;
  if ((st = dev_alloc(ctx, &ctx->d_lw_cnt, 4))) return st;
  ctx->lw_S = S;
  ctx->lw_slot = sb;
  ctx->lw_cc = CC;
  ctx->lw_warps = W;
  ctx->lw_grid = cps * nsm;
  ctx->lw_keep = 1;
  if (const char* e = std::getenv("DGAS_LW_KEEP")) ctx->lw_keep = std::atoi(e) != 0;
  ctx->lw_smem = WarpLayout(mc, np, S, sb).stride * W;
  cudaError_t e = cudaSuccess;
  DISPATCH_P15(ctx->p, ({
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, k_local_warp<NP_>);
    if (e == cudaSuccess && (size_t)optin < ctx->lw_smem + fa.sharedSizeBytes) e = cudaErrorInvalidValue;
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_local_warp<NP_>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
  }));
  if (e != cudaSuccess) { ctx->detail = std::string("warp local smem: ") + cudaGetErrorString(e); return DGAS_E_CUDA; }
  if (std::getenv("DGAS_VERBOSE"))
    fprintf(stderr, "dgas: warp local solve: %d warps x %d CTAs/SM, ring %d x %u B (CC %d), smem/CTA %zu\n", W, cps, S,
            sb, CC, ctx->lw_smem);
  ctx->local_kernel = 4;
  return 0;
}

void launch_local_warp(dgas_ctx ctx, int mode, const PcgState* st, const double* r, double* z, cudaStream_t s) {
  DISPATCH_P15(ctx->p, (k_local_warp<NP_><<<ctx->lw_grid, 32 * ctx->lw_warps, ctx->lw_smem, s>>>(
                           mode, ctx->nsub, ctx->d_sub_ptr, ctx->d_first, ctx->d_lw_pus, ctx->d_lw_units, ctx->d_p_off,
                           reinterpret_cast<const double*>(ctx->d_P), r, ctx->d_rbuf, z, st, ctx->d_lw_cnt, ctx->lw_S,
                           ctx->lw_slot, ctx->lw_cc, ctx->max_sub_cells, ctx->lw_keep)));
}
