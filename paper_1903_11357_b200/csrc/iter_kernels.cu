// iter_kernels.cu — per-iteration kernels of ASPCG with the additive Schwarz
// preconditioner P^-1 = Q A0^-1 Q^T + sum_i E_i A_i^-1 E_i^T (R8).
//
// One PCG iteration (captured in a CUDA graph WHILE node, abi.cu):
//   k_spmv_ring (spmv_ring.cu)  p = z + beta p_old (fused), q = A p, p.q -> alpha      (I1, I7)
//                               [k_spmv3 here: the slot-ring variant, DGAS_SPMV_KERNEL=3]
//   k_restrict_chunk            x += alpha p, r -= alpha q, r.r -> stop test; r0 = Q^T r  (I2, I3)
//   k_coarse | k_nd_fwd/bwd     z0 = A0^-1 r0 on a forked stream                        (I4)
//   k_local_panel | k_local     z_i = A_i^-1 r_i for all subdomains                     (I5)
//   k_prolong                   z += Q z0, r.z -> beta, bookkeeping, graph condition    (I6)
// Reductions are deterministic: per-CTA partials, the last CTA to arrive sums them in a fixed order.
#include <cfloat>

#include "internal.h"
#define TMA_HOST_BACKOFF
#include "tma.cuh"
#include <cstdlib>

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

// restriction / prolongation: n_p lanes per piece (cell), 32 / n_p pieces per warp (lanes beyond
// idle): 94% of the lanes busy at n_p = 10, 15 (62% / 94% with power-of-two groups)
template <int NP>
struct PackCfg {
  static constexpr int PPW = 32 / NP > 0 ? 32 / NP : 1;
};
int pack_ppw(int np) { return 32 / np > 0 ? 32 / np : 1; }
int restrict_chunk_threads() { return 256; }  // RC_T

// lanes per cell row in the block-Jacobi kernel (shuffles within power-of-two lane groups), cells per warp
template <int NP>
struct ProlongCfg {
  static constexpr int L = NP <= 4 ? 4 : NP <= 8 ? 8 : NP <= 16 ? 16 : 32;  // lanes per cell
  static constexpr int CPW = 32 / L;                                         // cells per warp
};

// ------------------------------------------------------------------ SpMV: persistent, batched, TMA ring
// Each CTA owns a contiguous range of cell rows, processed in batches of G cells whose (contiguous,
// column-major, 16-byte padded) row-blocks arrive by ONE cp.async.bulk per batch into a ring of S
// shared-memory slots. Thread (g, a, q) of a batch computes the partial dot product of row a of cell
// g over the columns col = q (mod SPTR); SPTR adjacent lanes finish it with shuffles. The input
// columns of the next batch are gathered two batches ahead in a register pipeline (neighbour index,
// then value), so no global load sits on the per-batch critical path.
// mode 0: y = A x.  mode 1 (PCG): p_new = z + beta p_old (fused), q = A p_new, p.q -> alpha.
#define SP_T 256
template <int NP>
struct SpmvCfg {
  static constexpr int TR = NP >= 21 ? 8 : 4;             // threads per row (adjacent lanes)
  static constexpr int E = NP >= 21 ? 3 : 2;              // gathered columns per thread per batch
  static constexpr int G = (SP_T / (NP * TR)) > 0 ? SP_T / (NP * TR) : 1;  // cells per batch
};
// NG independent consumer groups (SP_T / NG threads each, own named barrier, every NG-th batch): the
// per-batch barrier then spans half the threads and no group waits for the other's cells
template <int NP, int NG>
struct SpmvGrp {
  static constexpr int GT = SP_T / NG;
  // two groups: 4 lanes per row from n_p = 15 up (n_p = 28: 112 threads per cell), 2 below (n_p = 10:
  // 20 threads per cell, 6 cells = ~24 KB per batch)
  static constexpr int TR = NG == 1 ? SpmvCfg<NP>::TR : (NP >= 15 ? 4 : 2);
  static constexpr int E = NG == 1 ? SpmvCfg<NP>::E : 3;
  static constexpr int G = (GT / (NP * TR)) > 0 ? GT / (NP * TR) : 1;
  static constexpr bool ok = NP * TR <= GT;
};

template <int NP, int NG>
__global__ void __launch_bounds__(SP_T + 32) k_spmv3(int mode, int nc, int chunk, const int* __restrict__ nbr_ptr,
                                                const int* __restrict__ nbr, const int64_t* __restrict__ a_off,
                                                const double* __restrict__ A, const double* x, double* y,
                                                const double* z, double* const* pbuf, PcgState* st,
                                                double* partials, double* alpha_hist, int S, uint32_t slot_bytes,
                                                int maxW, int G) {
  constexpr int GMAX = SpmvGrp<NP, NG>::G, SPTR = SpmvGrp<NP, NG>::TR, SP_MAXE = SpmvGrp<NP, NG>::E;
  constexpr int GT = SpmvGrp<NP, NG>::GT;  // threads of one consumer group
  extern __shared__ __align__(128) double sm[];
  constexpr int NTT = SP_T + 32;  // consumers + producer warp
  __shared__ double red[NTT / 32];
  __shared__ double wdot[NTT / 32];
  __shared__ double own_all[NG][2][GMAX * NP];
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
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c0 = min(nc, blockIdx.x * chunk), c1 = min(nc, c0 + chunk), ncell = c1 - c0;
  const int nb = (ncell + G - 1) / G;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);          // full[16]
  uint64_t* empt = bars + 16;                                 // empty[16]
  int64_t* ao_s = reinterpret_cast<int64_t*>(bars + 32);                  // a_off[c0 .. c1]
  int* np_s = reinterpret_cast<int*>(ao_s + chunk + 2);                    // nbr_ptr[c0 .. c1]
  const int xstride = G * ((maxW + 1) & ~1);
  double* xs_all = reinterpret_cast<double*>(np_s + ((chunk + 2 + 3) & ~3));   // [NG][2][G][maxW]
  unsigned char* ring = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(xs_all + NG * 2 * xstride) + 127) & ~(uintptr_t)127);
  for (int k = threadIdx.x; k <= ncell; k += SP_T + 32) { np_s[k] = nbr_ptr[c0 + k]; ao_s[k] = a_off[c0 + k]; }
  if (threadIdx.x == 0) {
    for (int t = 0; t < S; ++t) { mbar_init(&bars[t], 1); mbar_init(&empt[t], GT / 32); }
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x >= SP_T) {
    // producer warp: batch bi goes to slot bi % S as soon as the consumers released batch bi - S
    if (threadIdx.x == SP_T)
      for (int bi = 0; bi < nb; ++bi) {
        if (bi >= S) mbar_wait(&empt[bi % S], (uint32_t)(((bi - S) / S) & 1));
        const int k0 = bi * G, k1 = min(ncell, k0 + G);
        bulk_load(ring + (size_t)(bi % S) * slot_bytes, A + ao_s[k0], (uint32_t)((ao_s[k1] - ao_s[k0]) * 8),
                  &bars[bi % S]);
      }
  }
  double mydot = 0;
  if (threadIdx.x < SP_T) {  // ---------------- consumers (group gid takes batches gid, gid + NG, ...)
  const int gid = threadIdx.x / GT, tl = threadIdx.x % GT;
  double* xs = xs_all + gid * 2 * xstride;
  double (*own)[GMAX * NP] = own_all[gid];
  auto colval = [&](int64_t id) -> double {
    return mode == 1 ? (it > 0 ? z[id] + beta * pold[id] : z[id]) : x[id];
  };
  // gather stage A: entry e of batch bi -> (cell g, column col) -> global index (-1 if none)
  int idxA[SP_MAXE], slotA[SP_MAXE];
  auto stage_idx = [&](int bi, int* idx, int* slot) {
    const int k0 = bi * G, k1 = min(ncell, k0 + G);
#pragma unroll
    for (int t = 0; t < SP_MAXE; ++t) {
      idx[t] = -1;
      slot[t] = 0;
      int e = tl + GT * t;  // flat entry of the batch
      for (int k = k0; k < k1; ++k) {
        const int W = (np_s[k + 1] - np_s[k]) * NP;
        if (e < W) {
          idx[t] = __ldg(nbr + np_s[k] + e / NP) * NP + e % NP;
          slot[t] = (k - k0) * ((maxW + 1) & ~1) + e;
          break;
        }
        e -= W;
      }
    }
  };
  int idxB[SP_MAXE], slotB[SP_MAXE], idxC[SP_MAXE], slotC[SP_MAXE];
  double vB[SP_MAXE], vC[SP_MAXE];
  auto publish = [&](int bi, const int* idx, const int* slot, const double* v) {  // values of batch bi -> xs
    double* xn = xs + ((bi / NG) & 1) * xstride;
    const int nk0 = bi * G;
    for (int t = 0; t < SP_MAXE; ++t)
      if (idx[t] >= 0) {
        xn[slot[t]] = v[t];
        const int gg = slot[t] / ((maxW + 1) & ~1);
        if (idx[t] / NP == c0 + nk0 + gg) own[(bi / NG) & 1][gg * NP + idx[t] % NP] = v[t];
      }
  };
  // prologue: the group's batch 0 published, batch 1 values in registers (vB), batch 2 indices (idxC)
  stage_idx(gid, idxA, slotA);
  for (int t = 0; t < SP_MAXE; ++t) vC[t] = idxA[t] >= 0 ? colval(idxA[t]) : 0.0;
  publish(gid, idxA, slotA, vC);
  stage_idx(gid + NG, idxB, slotB);
  for (int t = 0; t < SP_MAXE; ++t) vB[t] = idxB[t] >= 0 ? colval(idxB[t]) : 0.0;
  stage_idx(gid + 2 * NG, idxC, slotC);
  named_sync(1 + gid, GT);
  const int g = tl / (NP * SPTR), a = (tl / SPTR) % NP, q = tl % SPTR;
  for (int bi = gid; bi < nb; bi += NG) {
    const int cur = (bi / NG) & 1;
    // values of the group's next-but-one batch (in flight for two batch computes), indices of the one after
    for (int t = 0; t < SP_MAXE; ++t) vC[t] = idxC[t] >= 0 ? colval(idxC[t]) : 0.0;
    stage_idx(bi + 3 * NG, idxA, slotA);
    const int k0 = bi * G, kg = k0 + g;
    mbar_wait(&bars[bi % S], (uint32_t)((bi / S) & 1));
    if (g < G && kg < ncell) {
      const int W = (np_s[kg + 1] - np_s[kg]) * NP;
      const double* Ak = reinterpret_cast<const double*>(ring + (size_t)(bi % S) * slot_bytes) + (ao_s[kg] - ao_s[k0]) + a;
      const double* xk = xs + cur * xstride + g * ((maxW + 1) & ~1);
      double v0 = 0, v1 = 0;
      int col = q;
      for (; col + SPTR < W; col += 2 * SPTR) {
        v0 += Ak[(size_t)col * NP] * xk[col];
        v1 += Ak[(size_t)(col + SPTR) * NP] * xk[col + SPTR];
      }
      if (col < W) v0 += Ak[(size_t)col * NP] * xk[col];
      double v = v0 + v1;
#pragma unroll
      for (int o = 1; o < SPTR; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (q == 0) {
        const size_t id = (size_t)(c0 + kg) * NP + a;
        y[id] = v;
        if (mode == 1) {
          const double pn = own[cur][g * NP + a];
          pnew[id] = pn;
          mydot += pn * v;
        }
      }
    } else {
      double v = 0;
#pragma unroll
      for (int o = 1; o < SPTR; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empt[bi % S]);  // this warp is done with the ring slot of batch bi
    publish(bi + NG, idxB, slotB, vB);  // xs[cur^1] is not read during batch bi
    for (int t = 0; t < SP_MAXE; ++t) {
      idxB[t] = idxC[t]; slotB[t] = slotC[t]; vB[t] = vC[t];
      idxC[t] = idxA[t]; slotC[t] = slotA[t];
    }
    named_sync(1 + gid, GT);  // the group's next batch published
  }
  }  // consumers
  if (mode != 1) return;
  mydot = warp_sum(mydot);
  if (lane == 0) wdot[w] = mydot;
  __syncthreads();
  double tot[1] = {0};
  if (threadIdx.x == 0)
    for (int k = 0; k < NTT / 32; ++k) tot[0] += wdot[k];
  double res[1];
  if (last_block<NTT, 1>(tot, partials, &st->cnt[0], res, red)) {
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
// Pieces of J are spread over wpj warps of a CTA and, when J has many pieces (e.g. 16 coarse elements
// over 16384 cells), over cpj CTAs whose partial sums the last-arriving CTA of J adds in split order
// (deterministic). L lanes per piece (ProlongCfg), 32/L pieces per warp step; per-lane accumulation,
// one warp reduction per coarse dof at the end.
#define RT 256
#ifndef RESTRICT_MINB
#define RESTRICT_MINB 1  // 6 (40 registers, spills): cfg3 +1%, cfg4 -2% (measured)
#endif
template <int NP, int NQ>
__global__ void __launch_bounds__(RT, RESTRICT_MINB) k_restrict(int mode, int ncoarse, int wpj, int cpj, const int* __restrict__ cov_ptr,
                                                 const int2* __restrict__ rrec,
                                                 const double* __restrict__ G, const double* r_in, double* const* rbuf,
                                                 const double* q, double* const* pbuf, double* x, const double* b,
                                                 double* r0, double* rpart, unsigned* jcnt, PcgState* st,
                                                 double* partials) {
  constexpr int L = NP, PPW = PackCfg<NP>::PPW;
  __shared__ double red[RT / 32];
  __shared__ double part[RT / 32][NQ];
  __shared__ double wsum[RT / 32][2];
  __shared__ bool j_last;
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
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, a = lane % L;
  const int jpc = cpj > 1 ? 1 : (RT / 32) / wpj;
  const int J = cpj > 1 ? blockIdx.x / cpj : blockIdx.x * jpc + w / wpj;
  const int split = cpj > 1 ? blockIdx.x % cpj : 0;
  const int wj = w % wpj, TW = wpj * cpj, gw = split * wpj + wj;
  double accq[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) accq[k] = 0;
  double rr = 0, bb = 0;
  if (J < ncoarse) {
    // packed records (cell, piece | owner << 31): one load per piece, the next one prefetched
    const int ke = cov_ptr[J + 1], kstep = TW * PPW;
    const bool act = lane / L < PPW;
    int k = act ? cov_ptr[J] + gw * PPW + lane / L : ke;
    int2 rec = k < ke ? rrec[k] : make_int2(0, 0);
    for (; k < ke; k += kstep) {
      const int2 nrec = k + kstep < ke ? rrec[k + kstep] : rec;
      if (a < NP) {
        const int cell = rec.x, o = rec.y & 0x7fffffff;
        const bool owner = rec.y < 0;
        const size_t id = (size_t)cell * NP + a;
        const double* Go = G + ((size_t)o * NP + a) * NQ;
        double gv[NQ];
        if constexpr (NQ % 2 == 0) {
#pragma unroll
          for (int c = 0; c < NQ; c += 2) {
            const double2 g2 = __ldg(reinterpret_cast<const double2*>(Go + c));
            gv[c] = g2.x; gv[c + 1] = g2.y;
          }
        } else {
#pragma unroll
          for (int c = 0; c < NQ; ++c) gv[c] = __ldg(Go + c);
        }
        double rv;
        if (mode == 0) rv = rold[id];
        else if (mode == 1) rv = fma(-alpha, q[id], rold[id]);  // one rounding; the fused local solves form the same r
        else rv = b[id] - q[id];
        if (owner && mode >= 1) {
          rnew[id] = rv;
          rr += rv * rv;
          if (mode == 1) x[id] += alpha * pnew[id];
          else bb += b[id] * b[id];
        }
#pragma unroll
        for (int c = 0; c < NQ; ++c) accq[c] += gv[c] * rv;
      }
      rec = nrec;
    }
  }
#pragma unroll
  for (int c = 0; c < NQ; ++c) {
    const double v = warp_sum(accq[c]);
    if (lane == 0) part[w][c] = v;
  }
  rr = warp_sum(rr); bb = warp_sum(bb);
  if (lane == 0) { wsum[w][0] = rr; wsum[w][1] = bb; }
  __syncthreads();
  if (cpj == 1) {
    for (int e = threadIdx.x; e < jpc * NQ; e += RT) {
      const int jl = e / NQ, c = e % NQ, JJ = blockIdx.x * jpc + jl;
      if (JJ >= ncoarse) continue;
      double v = 0;
      for (int k = 0; k < wpj; ++k) v += part[jl * wpj + k][c];
      r0[(size_t)JJ * NQ + c] = v;
    }
  } else {
    if (threadIdx.x < NQ) {
      double v = 0;
      for (int k = 0; k < wpj; ++k) v += part[k][threadIdx.x];
      rpart[((size_t)J * cpj + split) * NQ + threadIdx.x] = v;
      __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) j_last = atomicAdd(&jcnt[J], 1u) == (unsigned)cpj - 1;
    __syncthreads();
    if (j_last) {
      __threadfence();
      if (threadIdx.x < NQ) {
        double v = 0;
        for (int sp = 0; sp < cpj; ++sp) v += __ldcg(rpart + ((size_t)J * cpj + sp) * NQ + threadIdx.x);
        r0[(size_t)J * NQ + threadIdx.x] = v;
      }
      if (threadIdx.x == 0) jcnt[J] = 0;
    }
  }
  if (mode == 0) return;
  double mine[2] = {0, 0};
  if (threadIdx.x == 0)
    for (int k = 0; k < RT / 32; ++k) { mine[0] += wsum[k][0]; mine[1] += wsum[k][1]; }
  double tot[2];
  if (last_block<RT, 2>(mine, partials, &st->cnt[1], tot, red)) {
    if (threadIdx.x == 0) {
      st->rr = tot[0];
      if (mode == 2) { st->bb = tot[1]; st->rtol2_bb *= tot[1]; }
      if (!isfinite(tot[0])) { st->done = 1; st->status = DGAS_E_BREAKDOWN; }
      else if (tot[0] <= st->rtol2_bb) { st->done = 1; st->status = DGAS_OK; if (mode == 1) st->it = it + 1; }
    }
  }
}

// ------------------------------------------------------------------ restriction, chunked (default)
// Same arithmetic as k_restrict, organised for latency: the pieces of every coarse element J are cut
// into chunks of at most PPW * RC_STEPS pieces (host table: J, first, last piece); persistent warps
// take chunks round-robin and work independently (no CTA barrier until the end). A warp writes its
// chunk's n_q partial sums; the last warp to finish a chunk of J (per-J counter) adds J's chunk
// partials in chunk order (deterministic) into r0[J]. r.r (and b.b) go through the usual
// deterministic last-CTA sum.
#define RC_T 256
template <int NP, int NQ>
__global__ void __launch_bounds__(RC_T) k_restrict_chunk(int mode, int nchunk, const int4* __restrict__ chunks,
                                                         const int* __restrict__ jchunk_ptr,
                                                         const int2* __restrict__ rrec, const double* __restrict__ G,
                                                         const double* r_in, double* const* rbuf, const double* q,
                                                         double* const* pbuf, double* x, const double* b, double* r0,
                                                         double* cpart, unsigned* jcnt, PcgState* st,
                                                         double* partials) {
  constexpr int L = NP, PPW = PackCfg<NP>::PPW;
  __shared__ double red[RC_T / 32];
  __shared__ double wsum[RC_T / 32][2];
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
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, a = lane % L;
  const bool act = lane / L < PPW;
  double rr = 0, bb = 0;
  const int wstep = gridDim.x * (RC_T / 32);
  for (int ch = blockIdx.x * (RC_T / 32) + w; ch < nchunk; ch += wstep) {
    const int4 cd = chunks[ch];  // (J, first piece, end piece, chunk index within J)
    double accq[NQ];
#pragma unroll
    for (int c = 0; c < NQ; ++c) accq[c] = 0;
    const int ke = cd.z;
    int k = act ? cd.y + lane / L : ke;
    int2 rec = k < ke ? rrec[k] : make_int2(0, 0);
    if constexpr (NQ <= 3) {
      // two warp steps per trip with the loads of both issued first (latency-bound: one dependent round of
      // loads per step); the sums keep the piece order (step A, then step B)
      int2 recB = k + PPW < ke ? rrec[k + PPW] : rec;
      for (; k < ke; k += 2 * PPW) {
        const int2 recA2 = k + 2 * PPW < ke ? rrec[k + 2 * PPW] : rec;
        const int2 recB2 = k + 3 * PPW < ke ? rrec[k + 3 * PPW] : rec;
        const bool okB = k + PPW < ke;
        const int2 rB = okB ? recB : rec;
        const int cellA = rec.x, oA = rec.y & 0x7fffffff, cellB = rB.x, oB = rB.y & 0x7fffffff;
        const bool ownA = rec.y < 0 && mode >= 1, ownB = okB && rB.y < 0 && mode >= 1;
        const size_t idA = (size_t)cellA * NP + a, idB = (size_t)cellB * NP + a;
        double gA[NQ], gB[NQ];
        const double* GoA = G + ((size_t)oA * NP + a) * NQ;
        const double* GoB = G + ((size_t)oB * NP + a) * NQ;
#pragma unroll
        for (int c = 0; c < NQ; ++c) { gA[c] = __ldg(GoA + c); gB[c] = __ldg(GoB + c); }
        double r1A = 0, r2A = 0, r1B = 0, r2B = 0, xA = 0, pA = 0, xB = 0, pB = 0;
        if (mode == 0) { r1A = rold[idA]; r1B = rold[idB]; }
        else if (mode == 1) { r1A = rold[idA]; r2A = q[idA]; r1B = rold[idB]; r2B = q[idB]; }
        else { r1A = b[idA]; r2A = q[idA]; r1B = b[idB]; r2B = q[idB]; }
        if (mode == 1) {
          if (ownA) { xA = x[idA]; pA = pnew[idA]; }
          if (ownB) { xB = x[idB]; pB = pnew[idB]; }
        }
        const double rvA = mode == 0 ? r1A : mode == 1 ? fma(-alpha, r2A, r1A) : r1A - r2A;
        const double rvB = mode == 0 ? r1B : mode == 1 ? fma(-alpha, r2B, r1B) : r1B - r2B;
        if (ownA) {
          rnew[idA] = rvA;
          rr += rvA * rvA;
          if (mode == 1) x[idA] = xA + alpha * pA;
          else bb += r1A * r1A;
        }
#pragma unroll
        for (int c = 0; c < NQ; ++c) accq[c] += gA[c] * rvA;
        if (okB) {
          if (ownB) {
            rnew[idB] = rvB;
            rr += rvB * rvB;
            if (mode == 1) x[idB] = xB + alpha * pB;
            else bb += r1B * r1B;
          }
#pragma unroll
          for (int c = 0; c < NQ; ++c) accq[c] += gB[c] * rvB;
        }
        rec = recA2;
        recB = recB2;
      }
    } else {
    for (; k < ke; k += PPW) {
      const int2 nrec = k + PPW < ke ? rrec[k + PPW] : rec;
      const int cell = rec.x, o = rec.y & 0x7fffffff;
      const bool owner = rec.y < 0;
      const size_t id = (size_t)cell * NP + a;
      const double* Go = G + ((size_t)o * NP + a) * NQ;
      double gv[NQ];
      if constexpr (NQ % 2 == 0) {
#pragma unroll
        for (int c = 0; c < NQ; c += 2) {
          const double2 g2 = __ldg(reinterpret_cast<const double2*>(Go + c));
          gv[c] = g2.x; gv[c + 1] = g2.y;
        }
      } else {
#pragma unroll
        for (int c = 0; c < NQ; ++c) gv[c] = __ldg(Go + c);
      }
      double rv;
      if (mode == 0) rv = rold[id];
      else if (mode == 1) rv = fma(-alpha, q[id], rold[id]);  // one rounding; the fused local solves form the same r
      else rv = b[id] - q[id];
      if (owner && mode >= 1) {
        rnew[id] = rv;
        rr += rv * rv;
        if (mode == 1) x[id] += alpha * pnew[id];
        else bb += b[id] * b[id];
      }
#pragma unroll
      for (int c = 0; c < NQ; ++c) accq[c] += gv[c] * rv;
      rec = nrec;
    }
    }
    double mine[NQ];
#pragma unroll
    for (int c = 0; c < NQ; ++c) mine[c] = warp_sum(accq[c]);
    const int J = cd.x, nch = jchunk_ptr[J + 1] - jchunk_ptr[J];
    if (nch == 1) {
      if (lane < NQ) {
        double v = 0;
#pragma unroll
        for (int c = 0; c < NQ; ++c) if (c == lane) v = mine[c];
        r0[(size_t)J * NQ + lane] = v;
      }
    } else {
      if (lane < NQ) {
        double v = 0;
#pragma unroll
        for (int c = 0; c < NQ; ++c) if (c == lane) v = mine[c];
        cpart[(size_t)ch * NQ + lane] = v;
      }
      __threadfence();
      __syncwarp();
      unsigned last = 0;
      if (lane == 0) last = atomicAdd(&jcnt[J], 1u) == (unsigned)nch - 1;
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        __threadfence();
        if (lane < NQ) {
          double v = 0;
          for (int c2 = jchunk_ptr[J]; c2 < jchunk_ptr[J + 1]; ++c2) v += __ldcg(cpart + (size_t)c2 * NQ + lane);
          r0[(size_t)J * NQ + lane] = v;
        }
        if (lane == 0) jcnt[J] = 0;
      }
    }
  }
  if (mode == 0) return;
  rr = warp_sum(rr); bb = warp_sum(bb);
  if (lane == 0) { wsum[w][0] = rr; wsum[w][1] = bb; }
  __syncthreads();
  double mine2[2] = {0, 0};
  if (threadIdx.x == 0)
    for (int k2 = 0; k2 < RC_T / 32; ++k2) { mine2[0] += wsum[k2][0]; mine2[1] += wsum[k2][1]; }
  double tot[2];
  if (last_block<RC_T, 2>(mine2, partials, &st->cnt[1], tot, red)) {
    if (threadIdx.x == 0) {
      st->rr = tot[0];
      if (mode == 2) { st->bb = tot[1]; st->rtol2_bb *= tot[1]; }
      if (!isfinite(tot[0])) { st->done = 1; st->status = DGAS_E_BREAKDOWN; }
      else if (tot[0] <= st->rtol2_bb) { st->done = 1; st->status = DGAS_OK; if (mode == 1) st->it = it + 1; }
    }
  }
}

// ------------------------------------------------------------------ coarse solve z0 = A0^-1 r0
// dense: z0 = X r0 with the explicit inverse (warp per row, 4 x 16-byte streaming loads in flight per
// lane); banded: one CTA runs the forward / backward tile sweeps of the band Cholesky factor.
// Launched on a forked stream so it runs concurrently with the local solves (the paths join at I6).
#define CO_T 256
__global__ void __launch_bounds__(CO_T) k_coarse(int mode, int dense, int64_t N0, int64_t ldX, int nT, int bt,
                                                 const double* __restrict__ X, const double* __restrict__ A0t,
                                                 const double* __restrict__ Dinv0, const double* r0, double* z0,
                                                 const PcgState* st) {
  __shared__ double acc[CT];
  if (mode >= 1 && st->done) return;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (dense) {
    const int64_t rows_per = (N0 + gridDim.x - 1) / gridDim.x;
    const int64_t r_lo = blockIdx.x * rows_per, r_hi = min(N0, r_lo + rows_per);
    for (int64_t row = r_lo + w; row < r_hi; row += CO_T / 32) {
      const double* xr = X + row * ldX;
      double v0 = 0, v1 = 0, v2 = 0, v3 = 0;
      int64_t c = 2 * lane;
      for (; c + 192 < N0; c += 256) {
        const double2 a0 = __ldcs(reinterpret_cast<const double2*>(xr + c));
        const double2 a1 = __ldcs(reinterpret_cast<const double2*>(xr + c + 64));
        const double2 a2 = __ldcs(reinterpret_cast<const double2*>(xr + c + 128));
        const double2 a3 = __ldcs(reinterpret_cast<const double2*>(xr + c + 192));
        v0 += a0.x * __ldg(r0 + c) + a0.y * __ldg(r0 + c + 1);
        v1 += a1.x * __ldg(r0 + c + 64) + a1.y * __ldg(r0 + c + 65);
        v2 += a2.x * __ldg(r0 + c + 128) + a2.y * __ldg(r0 + c + 129);
        v3 += a3.x * __ldg(r0 + c + 192) + a3.y * __ldg(r0 + c + 193);
      }
      for (; c < N0; c += 64) {
        v0 += xr[c] * __ldg(r0 + c);
        if (c + 1 < N0) v1 += xr[c + 1] * __ldg(r0 + c + 1);
      }
      const double v = warp_sum((v0 + v1) + (v2 + v3));
      if (lane == 0) z0[row] = v;
    }
    return;
  }
  if (blockIdx.x != 0) return;
  for (int64_t i = threadIdx.x; i < (int64_t)nT * CT; i += CO_T) z0[i] = i < N0 ? r0[i] : 0.0;
  __syncthreads();
  for (int I = 0; I < nT; ++I) {
    for (int a = w; a < CT; a += CO_T / 32) {
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
      const int a = threadIdx.x;
      double v = 0;
      for (int c = a; c < CT; ++c) v += Dinv0[(size_t)I * CT * CT + c * CT + a] * z0[(size_t)I * CT + c];
      acc[a] = v;
    }
    __syncthreads();
    if (threadIdx.x < CT) z0[(size_t)I * CT + threadIdx.x] = acc[threadIdx.x];
    __syncthreads();
    const int K0 = max(0, I - bt);
    for (int e = threadIdx.x; e < (I - K0) * CT; e += CO_T) {
      int K = K0 + e / CT, col = e % CT;
      const double* t = A0t + ((size_t)I * (bt + 1) + (K - I + bt)) * CT * CT + col;
      double v = 0;
      for (int a = 0; a < CT; ++a) v += t[a * CT] * acc[a];
      z0[(size_t)K * CT + col] -= v;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ local solves z_i = A_i^-1 r_i
// One CTA per subdomain: s = D^-1 r, U y = s (forward), U^T u = y (backward), z = D^-T u, with
// A_i = L L^T and U = D_b^-1-scaled block-envelope rows (setup_kernels.cu). Warp-specialised:
//   * a producer warp streams the column-major row-blocks U_k through S shared-memory slots with
//     cp.async.bulk, in units of CC columns (unit u in slot u % S). Forward order u = 0..U-1; the
//     last S units stay resident for the backward sweep, which consumes u = U-1..0 and refills the
//     slot of unit v with unit v - S. A slot is refilled as soon as every consumer warp has released
//     it (per-slot "empty" mbarrier), so prefetch depth does not depend on row-block sizes;
//   * consumer warps run the two sweeps; the only CTA-level dependency per row-block (y_k complete
//     before step k+1) is a named barrier among the consumers.
template <int NP>
struct LocalCfg {
  static constexpr int T = NP <= 15 ? 128 : 256;   // consumer threads
  static constexpr int W = T / 32;                 // consumer warps
};

__device__ __forceinline__ int nd_slot_events(int U, int S, int s) { return s < U ? (U - 1 - s) / S + 1 : 0; }

template <int NP>
__global__ void __launch_bounds__(LocalCfg<NP>::T + 32) k_local(int mode, const int* __restrict__ sub_ptr,
                                                                const int* __restrict__ first,
                                                                const int64_t* __restrict__ u_off,
                                                                const double* __restrict__ U,
                                                                const double* __restrict__ Dinv, const double* r_in,
                                                                double* const* rbuf, double* z, const PcgState* st,
                                                                int S, uint32_t slot_bytes, int ymax_cells, int CC,
                                                                int reuse, const double* qvec) {
  constexpr int T = LocalCfg<NP>::T, NW = LocalCfg<NP>::W;
  extern __shared__ __align__(128) double sm[];
  // mode 3: residual update fused (r = r_old - alpha q formed here, see apply_fuses_restrict)
  const double* r = r_in;
  double alpha = 0;
  const bool fuse = mode == 3;
  if (mode >= 1) {
    if (st->done) return;
    const int it = st->it;
    r = mode == 1 ? rbuf[0] : mode == 2 ? rbuf[(it + 1) & 1] : rbuf[it & 1];
    if (fuse) alpha = st->alpha;
  }
  const int s = blockIdx.x;
  const int s0 = sub_ptr[s], m = sub_ptr[s + 1] - s0;
  // layout (must match apply_smem_bytes): full[64] | empty[64] | fk | us | uo | y | ring
  const size_t off_fk = 1024;
  const size_t off_us = off_fk + (((size_t)(ymax_cells + 1) * 4 + 7) & ~(size_t)7);
  const size_t off_uo = off_us + (((size_t)(ymax_cells + 2) * 4 + 7) & ~(size_t)7);
  const size_t off_y = (off_uo + (size_t)ymax_cells * 8 + 127) & ~(size_t)127;
  unsigned char* smb = reinterpret_cast<unsigned char*>(sm);
  uint64_t* full = reinterpret_cast<uint64_t*>(smb);
  uint64_t* empty = full + 64;
  int* fk_s = reinterpret_cast<int*>(smb + off_fk);
  int* us_s = reinterpret_cast<int*>(smb + off_us);
  int64_t* uo_s = reinterpret_cast<int64_t*>(smb + off_uo);
  double* y = reinterpret_cast<double*>(smb + off_y);
  unsigned char* ring = reinterpret_cast<unsigned char*>(y) + (((size_t)ymax_cells * NP * 8 + 127) & ~(size_t)127);
  for (int k = threadIdx.x; k < m; k += T + 32) { fk_s[k] = first[s0 + k]; uo_s[k] = u_off[s0 + k]; }
  if (threadIdx.x == 0) {
    for (int t = 0; t < S; ++t) { mbar_init(&full[t], 1); mbar_init(&empty[t], NW); }
    fence_mbar_init();
    int acc = 0;
    for (int k = 0; k < m; ++k) {
      us_s[k] = acc;
      acc += k == 0 ? 0 : ((k - first[s0 + k]) * NP + CC - 1) / CC;
    }
    us_s[m] = acc;
  }
  __syncthreads();
  const int nunits = us_s[m];
  auto unit_cols = [&](int u, int k, int& cA, int& cB) {
    cA = (u - us_s[k]) * CC;
    cB = min((k - fk_s[k]) * NP, cA + CC);
  };
  if (threadIdx.x >= T) {
    // ---------------- producer warp (lane 0 issues every copy)
    if (threadIdx.x != T) return;
    // the `reuse` units the backward sweep re-reads first (just below the ring-resident tail) are
    // streamed evict-last in the forward sweep, everything else evict-first
    const uint64_t pol_first = l2_evict_first(), pol_last = l2_evict_last();
    const int keep_lo = nunits - S - reuse, keep_hi = nunits - S;
    auto issue = [&](int u, int k, bool fwd) {
      int cA, cB;
      unit_cols(u, k, cA, cB);
      const uint32_t nbytes = (uint32_t)((((int64_t)(cB - cA) * NP + 1) & ~1LL) * 8);
      const bool keep = fwd && u >= keep_lo && u < keep_hi;
      bulk_load(ring + (size_t)(u % S) * slot_bytes, U + uo_s[k] + (int64_t)cA * NP, nbytes, &full[u % S],
                keep ? pol_last : pol_first);
    };
    int k = 1;
    for (int u = 0; u < nunits; ++u) {  // forward stream
      while (us_s[k + 1] <= u) ++k;
      if (u >= S) {  // wait for the forward release of unit u - S (event (u - S) / S of its slot)
        mbar_wait_producer(&empty[u % S], (uint32_t)(((u - S) / S) & 1));
      }
      issue(u, k, true);
    }
    int kv = m - 1, kw = m - 1;
    for (int v = nunits - 1; v >= S; --v) {  // backward refills: after releasing v, load v - S
      const int sl = v % S;
      const int vmax = sl + S * (nd_slot_events(nunits, S, sl) - 1);  // largest unit of the slot
      const int Fs = nd_slot_events(nunits - S, S, sl);               // forward releases of the slot
      const int ev = Fs + (vmax - v) / S;  // index of v's backward release event in its slot
      mbar_wait_producer(&empty[sl], (uint32_t)(ev & 1));
      const int w = v - S;
      while (us_s[kw] > w) --kw;
      (void)kv;
      issue(w, kw, false);
    }
    return;
  }
  // ---------------- consumers
  const int lane = threadIdx.x & 31;
  uint64_t ph = 0;
  const double* rs = r + (size_t)s0 * NP;
  if (fuse) {
    const double* qs = qvec + (size_t)s0 * NP;
    for (int e = threadIdx.x; e < m * NP; e += T) {
      const int k = e / NP, a = e % NP;
      const double* D = Dinv + ((size_t)(s0 + k) * NP + a) * NP;
      double v = 0;
      for (int c = 0; c <= a; ++c) v += __ldg(D + c) * fma(-alpha, qs[k * NP + c], rs[k * NP + c]);
      y[e] = v;
    }
  } else {
    for (int e = threadIdx.x; e < m * NP; e += T) {
      const int k = e / NP, a = e % NP;
      const double* D = Dinv + ((size_t)(s0 + k) * NP + a) * NP;
      double v = 0;
      for (int c = 0; c <= a; ++c) v += __ldg(D + c) * rs[k * NP + c];
      y[e] = v;
    }
  }
  named_sync(1, T);
  // forward: thread (a, q) accumulates row a over columns col = q (mod 8) of every unit of U_k
  const int fa = threadIdx.x >> 3, fq = threadIdx.x & 7;
  for (int k = 1; k < m; ++k) {
    const int u0 = us_s[k], u1 = us_s[k + 1];
    if (u1 > u0) {
      const double* yw = y + fk_s[k] * NP;
      double v = 0;
      for (int u = u0; u < u1; ++u) {
        const int sl = u % S;
        mbar_wait(&full[sl], (uint32_t)((ph >> sl) & 1u));
        ph ^= 1ull << sl;
        int cA, cB;
        unit_cols(u, k, cA, cB);
        const double* Uc = reinterpret_cast<const double*>(ring + (size_t)sl * slot_bytes);
        if (fa < NP) {
          double v1 = 0;
          int col = cA + fq;
          for (; col + 8 < cB; col += 16) {
            v += Uc[(col - cA) * NP + fa] * yw[col];
            v1 += Uc[(col + 8 - cA) * NP + fa] * yw[col + 8];
          }
          if (col < cB) v += Uc[(col - cA) * NP + fa] * yw[col];
          v += v1;
        }
        __syncwarp();
        // resident units (u >= U - S) are released only once, in the backward sweep: every slot's
        // release events then alternate with producer refills (no mbarrier phase aliasing)
        if (lane == 0 && u < nunits - S) mbar_arrive(&empty[sl]);
      }
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      if (fa < NP && fq == 0) y[k * NP + fa] -= v;
    }
    named_sync(1, T);
  }
  // backward: u_k is final; y[f_k .. k) -= U_k^T u_k (thread per column)
  for (int k = m - 1; k > 0; --k) {
    const int u0 = us_s[k], u1 = us_s[k + 1];
    if (u1 > u0) {
      const double* uk = y + k * NP;
      double* yw = y + fk_s[k] * NP;
      for (int u = u1 - 1; u >= u0; --u) {
        const int sl = u % S;
        if (u < nunits - S) {
          mbar_wait(&full[sl], (uint32_t)((ph >> sl) & 1u));
          ph ^= 1ull << sl;
        }
        int cA, cB;
        unit_cols(u, k, cA, cB);
        const double* Uc = reinterpret_cast<const double*>(ring + (size_t)sl * slot_bytes);
        for (int col = cA + threadIdx.x; col < cB; col += T) {
          const double* uc = Uc + (size_t)(col - cA) * NP;
          double v0 = 0, v1 = 0;
#pragma unroll
          for (int a = 0; a + 1 < NP; a += 2) { v0 += uc[a] * uk[a]; v1 += uc[a + 1] * uk[a + 1]; }
          if (NP & 1) v0 += uc[NP - 1] * uk[NP - 1];
          yw[col] -= v0 + v1;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[sl]);
      }
    }
    named_sync(1, T);
  }
  double* zs = z + (size_t)s0 * NP;
  for (int e = threadIdx.x; e < m * NP; e += T) {
    const int k = e / NP, a = e % NP;
    const double* D = Dinv + (size_t)(s0 + k) * NP * NP;
    double v = 0;
    for (int c = a; c < NP; ++c) v += __ldg(D + c * NP + a) * y[k * NP + c];
    zs[e] = v;
  }
}

// ------------------------------------------------------------------ prolongation + r.z
// z_kappa += sum_{pieces o of kappa} G_o z0_J(o).  mode 0: apply only.  mode 1: PCG init (gamma_0).
// mode 2: PCG iteration (beta = gamma_new / gamma, history, it++, maxit, graph condition).
#define PW 8
template <int NP, int NQ>
__global__ void __launch_bounds__(PW * 32) k_prolong(int mode, int nc, const int4* __restrict__ crec,
                                                     const int2* __restrict__ prec,
                                                     const double* __restrict__ G, const double* z0, double* z,
                                                     double* const* rbuf, PcgState* st, double* partials,
                                                     double* beta_hist, cudaGraphConditionalHandle h, int use_h) {
  constexpr int L = NP, CPW = PackCfg<NP>::PPW;
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
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, a = lane % L;
  const bool act = lane / L < CPW;
  double d = 0;
  // persistent grid-stride over groups of CPW cells per warp (few CTAs: few last-block atomics);
  // the next group's cell record is loaded before the current group is processed
  const int ngroups = (nc + CPW - 1) / CPW, gstep = gridDim.x * PW;
  int g = blockIdx.x * PW + w;
  int c = g * CPW + lane / L;
  int4 rc = act && c < nc ? crec[c] : make_int4(0, 0, 0, 0);
  // further pieces (non-nested cells) from prec, in piece order
  auto extra = [&](const int4& q4, double v) -> double {
    for (int t = 1; t < q4.z; ++t) {
      const int2 pr = prec[q4.w + t];
      const double* Go = G + ((size_t)pr.x * NP + a) * NQ;
      const double* zj = z0 + (size_t)pr.y * NQ;
      if constexpr (NQ % 2 == 0) {
#pragma unroll
        for (int b = 0; b < NQ; b += 2) {
          const double2 g2 = __ldg(reinterpret_cast<const double2*>(Go + b));
          v += g2.x * zj[b] + g2.y * zj[b + 1];
        }
      } else {
#pragma unroll
        for (int b = 0; b < NQ; ++b) v += __ldg(Go + b) * zj[b];
      }
    }
    return v;
  };
  if constexpr (NQ <= 3) {  // (NQ = 6: 128 registers, measured slower on config 4: 30 -> 40 us)
    // two groups per trip, all first-piece loads of both issued before the first use (the kernel is
    // latency-bound: one dependent round of loads per group), records two groups ahead
    int cB = (g + gstep) * CPW + lane / L;
    int4 rcB = act && g + gstep < ngroups && cB < nc ? crec[cB] : rc;
    for (; g < ngroups; g += 2 * gstep) {
      const int gA2 = g + 2 * gstep, gB2 = g + 3 * gstep;
      const int cA2 = gA2 * CPW + lane / L, cB2 = gB2 * CPW + lane / L;
      const int4 rcA2 = act && gA2 < ngroups && cA2 < nc ? crec[cA2] : rc;
      const int4 rcB2 = act && gB2 < ngroups && cB2 < nc ? crec[cB2] : rc;
      const bool okA = act && c < nc, okB = act && g + gstep < ngroups && cB < nc;
      const size_t idA = (size_t)(okA ? c : 0) * NP + a, idB = (size_t)(okB ? cB : 0) * NP + a;
      double vA = 0, vB = 0, rA = 0, rB = 0, gA[NQ], gB[NQ], zA[NQ], zB[NQ];
      if (okA) {
        vA = z[idA];
        if (mode >= 1) rA = r[idA];
        const double* Go = G + ((size_t)rc.x * NP + a) * NQ;
        const double* zj = z0 + (size_t)rc.y * NQ;
#pragma unroll
        for (int b = 0; b < NQ; ++b) { gA[b] = __ldg(Go + b); zA[b] = zj[b]; }
      }
      if (okB) {
        vB = z[idB];
        if (mode >= 1) rB = r[idB];
        const double* Go = G + ((size_t)rcB.x * NP + a) * NQ;
        const double* zj = z0 + (size_t)rcB.y * NQ;
#pragma unroll
        for (int b = 0; b < NQ; ++b) { gB[b] = __ldg(Go + b); zB[b] = zj[b]; }
      }
      if (okA) {
        if (rc.z > 0) {
          if constexpr (NQ % 2 == 0) {
#pragma unroll
            for (int b = 0; b < NQ; b += 2) vA += gA[b] * zA[b] + gA[b + 1] * zA[b + 1];
          } else {
#pragma unroll
            for (int b = 0; b < NQ; ++b) vA += gA[b] * zA[b];
          }
        }
        if (rc.z > 1) vA = extra(rc, vA);
        z[idA] = vA;
        d += rA * vA;
      }
      if (okB) {
        if (rcB.z > 0) {
          if constexpr (NQ % 2 == 0) {
#pragma unroll
            for (int b = 0; b < NQ; b += 2) vB += gB[b] * zB[b] + gB[b + 1] * zB[b + 1];
          } else {
#pragma unroll
            for (int b = 0; b < NQ; ++b) vB += gB[b] * zB[b];
          }
        }
        if (rcB.z > 1) vB = extra(rcB, vB);
        z[idB] = vB;
        d += rB * vB;
      }
      rc = rcA2; c = cA2;
      rcB = rcB2; cB = cB2;
    }
  } else {
  for (; g < ngroups; g += gstep) {
    const int gn = g + gstep, cn = gn * CPW + lane / L;
    const int4 rcn = act && gn < ngroups && cn < nc ? crec[cn] : rc;
    if (act && c < nc) {
      const size_t id = (size_t)c * NP + a;
      double v = z[id];
      const double rv = mode >= 1 ? r[id] : 0.0;
      // first piece from the cell record (o, J, n, k), further pieces (non-nested) from prec
      if (rc.z > 0) {
        const double* Go = G + ((size_t)rc.x * NP + a) * NQ;
        const double* zj = z0 + (size_t)rc.y * NQ;
        if constexpr (NQ % 2 == 0) {
#pragma unroll
          for (int b = 0; b < NQ; b += 2) {
            const double2 g2 = __ldg(reinterpret_cast<const double2*>(Go + b));
            v += g2.x * zj[b] + g2.y * zj[b + 1];
          }
        } else {
#pragma unroll
          for (int b = 0; b < NQ; ++b) v += __ldg(Go + b) * zj[b];
        }
      }
      if (rc.z > 1) v = extra(rc, v);
      z[id] = v;
      d += rv * v;
    }
    rc = rcn;
    c = cn;
  }
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

static int SpmvCfgMax(int p, int ng) {
  int G = 1;
  if (ng == 2) {
    DISPATCH_P(p, (G = SpmvGrp<NP_, 2>::G));
  } else {
    DISPATCH_P(p, (G = SpmvGrp<NP_, 1>::G));
  }
  return G;
}

int spmv_groups_ok(int p) {
  bool ok = false;
  DISPATCH_P(p, (ok = SpmvGrp<NP_, 2>::ok));
  return ok ? 2 : 1;
}

int spmv_gather_cap(int p, int ng) {
  int e = 2;
  if (ng == 2) {
    DISPATCH_P(p, (e = SpmvGrp<NP_, 2>::E));
  } else {
    DISPATCH_P(p, (e = SpmvGrp<NP_, 1>::E));
  }
  return e * (SP_T / ng);
}

int spmv_batch_cells(int p, int ng) {
  int G = SpmvCfgMax(p, ng);
  if (const char* e = std::getenv("DGAS_SPMV_G")) G = std::max(1, std::min(SpmvCfgMax(p, ng), std::atoi(e)));
  return G;
}

size_t spmv_smem_bytes(dgas_ctx ctx) {
  const int chunk = (ctx->nc + ctx->spmv_grid - 1) / std::max(1, ctx->spmv_grid);
  const int maxW = ctx->max_deg * ctx->np, G = ctx->spmv_G;
  size_t b = 32 * 8 + (size_t)(chunk + 2) * 8 + (size_t)((chunk + 2 + 3) & ~3) * 4 +
             (size_t)ctx->spmv_groups * 2 * (size_t)G * ((maxW + 1) & ~1) * 8;
  return ((b + 127) & ~(size_t)127) + (size_t)ctx->spmv_slots * ctx->spmv_slot_bytes + 128;
}

void launch_spmv(dgas_ctx ctx, int mode, const double* x, double* y, PcgState* st, cudaStream_t s) {
  if (ctx->spmv_kernel == 4) {
    launch_spmv_ring(ctx, mode, x, y, st, s);
    return;
  }
  const int grid = ctx->spmv_grid, chunk = (ctx->nc + grid - 1) / grid;
  const size_t smem = spmv_smem_bytes(ctx);
#define SPMV_LAUNCH(NG_)                                                                                       \
  DISPATCH_P(ctx->p, (k_spmv3<NP_, NG_><<<grid, SP_T + 32, smem, s>>>(                                          \
                         mode, ctx->nc, chunk, ctx->d_nbr_ptr, ctx->d_nbr, ctx->d_a_off, ctx->d_A, x, y, ctx->d_z, \
                         ctx->d_pbuf, st, ctx->d_partials, ctx->d_alpha, ctx->spmv_slots, ctx->spmv_slot_bytes,   \
                         ctx->max_deg * ctx->np, ctx->spmv_G)))
  if (ctx->spmv_groups == 2) {
    SPMV_LAUNCH(2);
  } else {
    SPMV_LAUNCH(1);
  }
#undef SPMV_LAUNCH
}

int spmv_set_smem(dgas_ctx ctx, size_t smem) {
  cudaError_t e = cudaSuccess;
  int dev = 0, mx = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if ((int)smem > mx) { ctx->detail = "SpMV kernel needs more shared memory than available"; return DGAS_E_INVALID_ARG; }
#define SPMV_ATTR(NG_)                                                                                        \
  DISPATCH_P(ctx->p, ({                                                                                        \
    cudaFuncAttributes fa;                                                                                     \
    e = cudaFuncGetAttributes(&fa, k_spmv3<NP_, NG_>);                                                         \
    if (e == cudaSuccess && (size_t)mx < smem + fa.sharedSizeBytes) e = cudaErrorInvalidValue;                 \
    if (e == cudaSuccess)                                                                                      \
      e = cudaFuncSetAttribute(k_spmv3<NP_, NG_>, cudaFuncAttributeMaxDynamicSharedMemorySize,                 \
                               mx - (int)fa.sharedSizeBytes);                                                  \
  }))
  if (ctx->spmv_groups == 2) {
    SPMV_ATTR(2);
  } else {
    SPMV_ATTR(1);
  }
#undef SPMV_ATTR
  if (e != cudaSuccess) { ctx->detail = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e); return DGAS_E_CUDA; }
  return 0;
}

void launch_restrict(dgas_ctx ctx, int mode, PcgState* st, const double* r, cudaStream_t s) {
  if (ctx->d_chunks) {
    DISPATCH_P(ctx->p, DISPATCH_Q(ctx->q, (k_restrict_chunk<NP_, NQ_><<<ctx->rc_grid, RC_T, 0, s>>>(
                                              mode, ctx->nchunk, ctx->d_chunks, ctx->d_jchunk_ptr,
                                              ctx->d_rrec_it ? ctx->d_rrec_it : ctx->d_rrec, ctx->d_G_it ? ctx->d_G_it : ctx->d_G,
                                              r, ctx->d_rbuf, ctx->d_q, ctx->d_pbuf, ctx->d_x, ctx->d_b, ctx->d_r0,
                                              ctx->d_cpart, ctx->d_jcnt2, st, ctx->d_partials))));
    return;
  }
  const int wpj = ctx->restrict_wpj, cpj = ctx->restrict_cpj;
  const int grid = cpj > 1 ? ctx->ncoarse * cpj : (ctx->ncoarse + (RT / 32 / wpj) - 1) / (RT / 32 / wpj);
  DISPATCH_P(ctx->p, DISPATCH_Q(ctx->q, (k_restrict<NP_, NQ_><<<grid, RT, 0, s>>>(
                                            mode, ctx->ncoarse, wpj, cpj, ctx->d_cov_ptr,
                                            ctx->d_rrec_it ? ctx->d_rrec_it : ctx->d_rrec,
                                            ctx->d_G_it ? ctx->d_G_it : ctx->d_G, r, ctx->d_rbuf, ctx->d_q, ctx->d_pbuf,
                                            ctx->d_x, ctx->d_b, ctx->d_r0, ctx->d_rpart, ctx->d_jcnt, st,
                                            ctx->d_partials))));
}

size_t apply_smem_bytes(dgas_ctx ctx) {
  const size_t mc = ctx->max_sub_cells, n = ctx->np;
  const size_t off_us = 1024 + ((mc + 1) * 4 + 7) / 8 * 8;
  const size_t off_uo = off_us + ((mc + 2) * 4 + 7) / 8 * 8;
  const size_t off_y = (off_uo + mc * 8 + 127) / 128 * 128;
  const size_t ybytes = (mc * n * 8 + 127) / 128 * 128;
  return off_y + ybytes + (size_t)ctx->ring_slots * ctx->slot_bytes + 128;
}

int local_threads(int p) {
  int t = 128;
  DISPATCH_P(p, (t = LocalCfg<NP_>::T));
  return t;
}

// z = P^-1 r minus the prolongation: coarse solve on the side stream || local solves on s
// preconditioner variants without local solves (dgas_set_precond): z = r (NONE) or z = 0 (COARSE); the
// coarse part is added by k_prolong as for the two-level operator
__global__ void k_zfill(int mode, int copy, int64_t n, const double* r_in, double* const* rbuf, double* z,
                        const PcgState* st) {
  const double* r = r_in;
  if (mode >= 1) {
    if (st->done) return;
    r = mode == 1 ? rbuf[0] : rbuf[(st->it + 1) & 1];
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z[i] = copy ? r[i] : 0.0;
}

// dense / band coarse solve z0 = A0^-1 r0, plus the calibrated refinement steps of the dense path
// (R30: z0 += X (r0 - A0 z0), residual from the A0 pair blocks)
void launch_coarse_dense(dgas_ctx ctx, int mode, const PcgState* st, const double* r0, double* z0, cudaStream_t s) {
  k_coarse<<<ctx->n_coarse_ctas, CO_T, 0, s>>>(mode, ctx->coarse_dense, ctx->N0, ctx->ldX, ctx->nT, ctx->bt, ctx->d_X,
                                                ctx->d_A0t, ctx->d_Dinv0, r0, z0, st);
  if (!ctx->coarse_dense) return;
  for (int it = 0; it < ctx->dense_refine; ++it) {
    launch_a0_resid(ctx, ctx->d_prow, r0, z0, ctx->d_rb0, st, mode, s);
    k_coarse<<<ctx->n_coarse_ctas, CO_T, 0, s>>>(mode, 1, ctx->N0, ctx->ldX, ctx->nT, ctx->bt, ctx->d_X, ctx->d_A0t,
                                                  ctx->d_Dinv0, ctx->d_rb0, ctx->d_zb0, st);
    launch_axpy_add(ctx->N0, ctx->d_zb0, z0, st, mode, s);
  }
}

static void launch_coarse_part(dgas_ctx ctx, int mode, PcgState* st, cudaStream_t s) {
  if (ctx->coarse_mode == 2) nd_solve_launch(ctx, mode, st, s);
  else launch_coarse_dense(ctx, mode, st, ctx->d_r0, ctx->d_z0, s);
}

// T_HH = T_h (the paper's regime): every subdomain is one cell, A_i^-1 = D^T D with
// D = L_kk^-1 (row-major lower triangle), so the local solve is two tiny triangular GEMVs per cell.
// L lanes per cell (ProlongCfg), the cell's r and y exchanged by shuffles.
template <int NP>
__global__ void __launch_bounds__(256) k_bjacobi(int mode, int nc, const double* __restrict__ Dinv, const double* r_in,
                                                 double* const* rbuf, double* z, const PcgState* st) {
  constexpr int L = ProlongCfg<NP>::L, CPW = ProlongCfg<NP>::CPW;
  const double* r = r_in;
  if (mode >= 1) {
    if (st->done) return;
    r = mode == 1 ? rbuf[0] : rbuf[(st->it + 1) & 1];
  }
  const int lane = threadIdx.x & 31, a = lane % L, base = lane - a;
  const int c = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * CPW + lane / L;
  const bool on = c < nc && a < NP;
  const double rv = on ? r[(size_t)c * NP + a] : 0.0;
  const double* D = Dinv + (size_t)(c < nc ? c : 0) * NP * NP;
  double y = 0;
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const double rk = __shfl_sync(0xffffffffu, rv, base + k);
    if (on && k <= a) y += __ldg(D + a * NP + k) * rk;
  }
  double v = 0;
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const double yk = __shfl_sync(0xffffffffu, y, base + k);
    if (on && k >= a) v += __ldg(D + k * NP + a) * yk;
  }
  if (on) z[(size_t)c * NP + a] = v;
}

// all local solves z_i = A_i^-1 r_i
static void launch_local(dgas_ctx ctx, int mode, PcgState* st, const double* r, double* z, cudaStream_t s) {
  if (ctx->max_sub_cells == 1) {
    unsigned grid = 1;
    DISPATCH_P(ctx->p, (grid = (ctx->nc + 8 * ProlongCfg<NP_>::CPW - 1) / (8 * ProlongCfg<NP_>::CPW)));
    DISPATCH_P(ctx->p, (k_bjacobi<NP_><<<grid, 256, 0, s>>>(mode, ctx->nc, ctx->d_Dinv, r, ctx->d_rbuf, z, st)));
    return;
  }
  if (ctx->local_kernel == 2) {
    launch_local_panel(ctx, mode, st, r, z, s);
    return;
  }
  if (ctx->local_kernel == 3) {
    launch_local_inv(ctx, mode, st, r, z, s);
    return;
  }
  if (ctx->local_kernel == 4) {
    launch_local_warp(ctx, mode, st, r, z, s);
    return;
  }
  if (ctx->local_kernel == 5) {
    launch_local_mrhs(ctx, mode, st, r, z, s);
    return;
  }
  const size_t smem = apply_smem_bytes(ctx);
  DISPATCH_P(ctx->p, (k_local<NP_><<<ctx->nsub, LocalCfg<NP_>::T + 32, smem, s>>>(
                         mode, ctx->d_sub_ptr, ctx->d_first, ctx->d_u_off, ctx->d_U, ctx->d_Dinv, r, ctx->d_rbuf, z,
                         st, ctx->ring_slots, ctx->slot_bytes, ctx->max_sub_cells, ctx->ring_rows, ctx->local_reuse,
                         ctx->d_q)));
}

// local solves of subdomains [sb, se) only (sharded solve, shard.cu; mode 0): the single-GPU kernels
// index subdomains through sub_ptr[blockIdx] (absolute cell numbers), so a shifted sub_ptr and a grid
// of se - sb CTAs run exactly the solves of that range
void launch_local_range(dgas_ctx ctx, int sb, int se, const double* r, double* z, cudaStream_t s) {
  if (se <= sb) return;
  if (ctx->max_sub_cells == 1) {
    const int c0 = ctx->sub_ptr_h[sb], n = ctx->sub_ptr_h[se] - c0;
    unsigned grid = 1;
    DISPATCH_P(ctx->p, (grid = (n + 8 * ProlongCfg<NP_>::CPW - 1) / (8 * ProlongCfg<NP_>::CPW)));
    DISPATCH_P(ctx->p, (k_bjacobi<NP_><<<grid, 256, 0, s>>>(0, n, ctx->d_Dinv + (size_t)c0 * NP_ * NP_,
                                                            r + (size_t)c0 * NP_, ctx->d_rbuf, z + (size_t)c0 * NP_,
                                                            nullptr)));
    return;
  }
  if (ctx->local_kernel == 2) { launch_local_panel_range(ctx, sb, se, r, z, s); return; }
  if (ctx->local_kernel == 3) { launch_local_inv_range(ctx, sb, se, r, z, s); return; }
  const size_t smem = apply_smem_bytes(ctx);
  DISPATCH_P(ctx->p, (k_local<NP_><<<se - sb, LocalCfg<NP_>::T + 32, smem, s>>>(
                         0, ctx->d_sub_ptr + sb, ctx->d_first, ctx->d_u_off, ctx->d_U, ctx->d_Dinv, r, ctx->d_rbuf, z,
                         nullptr, ctx->ring_slots, ctx->slot_bytes, ctx->max_sub_cells, ctx->ring_rows, ctx->local_reuse,
                         nullptr)));
}

// Residual update fused into the local solve (PCG iterations): the wide panel kernel, the envelope kernel and
// the explicit-inverse kernel (latency-bound configs: one wave of CTAs, idle SMs) form r = r_old - alpha q itself (mode 3), so k_restrict_chunk (x,
// r, r.r, stop test, r0 = Q^T r) leaves the critical path: it runs on the coarse stream in front of the coarse
// solve, beside the local solves, and both join before the prolongation. The caller then skips its own
// launch_restrict. Config 5 p3q3: 7380 -> 7922 PCG it/s. On the HBM- or issue-bound configs 3 and 4 it was
// measured neutral (the GPU is full: what the restriction takes, the local solve loses), so the narrow panel
// kernel and the multi-RHS kernels keep the serial order. DGAS_FUSE_R=0 keeps the serial order everywhere.
bool apply_fuses_restrict(dgas_ctx ctx) {
  static const bool no_fork = std::getenv("DGAS_NO_FORK") != nullptr;
  if (ctx->fuse_r < 0) {  // read once per context (the PCG graph is built with one choice)
    const char* e = std::getenv("DGAS_FUSE_R");
    ctx->fuse_r = e ? (std::atoi(e) != 0) : 1;
  }
  if (!ctx->fuse_r || no_fork || ctx->precond != 0 || ctx->max_sub_cells == 1) return false;
  return (ctx->local_kernel == 2 && !panel_is_narrow(ctx)) || ctx->local_kernel == 1 || ctx->local_kernel == 3;
}

void launch_apply(dgas_ctx ctx, int mode, PcgState* st, const double* r, double* z, cudaStream_t s) {
  static const bool no_fork = std::getenv("DGAS_NO_FORK") != nullptr;
  if (ctx->precond != 0) {
    // variants (z0 is zeroed by dgas_set_precond when the coarse part is off)
    if (ctx->precond == 2) launch_coarse_part(ctx, mode, st, s);
    if (ctx->precond == 1) launch_local(ctx, mode, st, r, z, s);
    else k_zfill<<<2 * 148, 256, 0, s>>>(mode, ctx->precond == 3, ctx->N, r, ctx->d_rbuf, z, st);
    return;
  }
  if (no_fork) {
    launch_coarse_part(ctx, mode, st, s);
    launch_local(ctx, mode, st, r, z, s);
    return;
  }
  cudaStream_t side = ctx->side[ctx->side_sel];
  cudaEvent_t ef = ctx->ev_fork[ctx->side_sel], ej = ctx->ev_join[ctx->side_sel];
  cudaEventRecord(ef, s);
  cudaStreamWaitEvent(side, ef, 0);
  if (mode == 2 && apply_fuses_restrict(ctx)) {
    launch_restrict(ctx, 1, st, nullptr, side);
    launch_coarse_part(ctx, mode, st, side);
    launch_local(ctx, 3, st, r, z, s);
  } else {
    launch_coarse_part(ctx, mode, st, side);
    launch_local(ctx, mode, st, r, z, s);
  }
  cudaEventRecord(ej, side);
  cudaStreamWaitEvent(s, ej, 0);
}

void launch_local_only(dgas_ctx ctx, const double* r, double* z, cudaStream_t s) {
  launch_local(ctx, 0, nullptr, r, z, s);
}

void launch_coarse_only(dgas_ctx ctx, cudaStream_t s) {
  if (ctx->coarse_mode == 2) { nd_solve_launch(ctx, 0, nullptr, s); return; }
  launch_coarse_dense(ctx, 0, nullptr, ctx->d_r0, ctx->d_z0, s);
}

void launch_prolong(dgas_ctx ctx, int mode, PcgState* st, const double* r, double* z, cudaStream_t s,
                    cudaGraphConditionalHandle h, int use_handle) {
  (void)r;
  unsigned grid = 1;
  DISPATCH_P(ctx->p, (grid = (ctx->nc + PW * PackCfg<NP_>::PPW - 1) / (PW * PackCfg<NP_>::PPW)));
  grid = std::min<unsigned>(grid, (unsigned)ctx->prolong_grid);
  DISPATCH_P(ctx->p, DISPATCH_Q(ctx->q, (k_prolong<NP_, NQ_><<<grid, PW * 32, 0, s>>>(
                                            mode, ctx->nc, ctx->d_crec_it ? ctx->d_crec_it : ctx->d_crec,
                                            ctx->d_prec_it ? ctx->d_prec_it : ctx->d_prec,
                                            ctx->d_G_it ? ctx->d_G_it : ctx->d_G,
                                            ctx->d_z0, z, ctx->d_rbuf, st, ctx->d_partials, ctx->d_beta, h,
                                            use_handle))));
}

// resident CTAs per SM of the persistent restriction / prolongation kernels (their grids are sized to one wave)
int restrict_ctas_per_sm(dgas_ctx ctx) {
  int n = 1;
  DISPATCH_P(ctx->p, DISPATCH_Q(ctx->q, (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_restrict_chunk<NP_, NQ_>, RC_T, 0))));
  return std::max(1, n);
}
int prolong_ctas_per_sm(dgas_ctx ctx) {
  int n = 1;
  DISPATCH_P(ctx->p, DISPATCH_Q(ctx->q, (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_prolong<NP_, NQ_>, PW * 32, 0))));
  return std::max(1, n);
}

void launch_init_state(dgas_ctx ctx, PcgState* st, int maxit, double rtol, cudaStream_t s) {
  (void)ctx;
  k_init_state<<<1, 1, 0, s>>>(st, maxit, rtol);
}

void launch_lanczos(dgas_ctx ctx, cudaStream_t s) {
  k_lanczos<<<1, 256, 0, s>>>(ctx->d_state, ctx->d_alpha, ctx->d_beta, ctx->d_lanczos);
}

// The attribute is per function (shared by all contexts): always raise it to the opt-in maximum.
int apply_set_smem(dgas_ctx ctx, size_t smem) {
  tma_set_backoff(0);  // producer-lane back-off of this unit's streaming kernels (DGAS_PRODUCER_NS)
  cudaError_t e = cudaSuccess;
  int dev = 0, mx = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if ((int)smem > mx) { ctx->detail = "fused apply kernel needs more shared memory than available"; return DGAS_E_INVALID_ARG; }
  DISPATCH_P(ctx->p, ({
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, k_local<NP_>);
    if (e == cudaSuccess && (size_t)mx < smem + fa.sharedSizeBytes) e = cudaErrorInvalidValue;
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_local<NP_>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx - (int)fa.sharedSizeBytes);
  }));
  if (e != cudaSuccess) { ctx->detail = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e); return DGAS_E_CUDA; }
  return 0;
}
