// dedup.cu — exact de-duplication of the per-iteration operator data (SURVEY.md §8(f) NEXT-4,
// "Cartesian de-duplication of identical interior A_i and element blocks").
//
// On a uniform Cartesian mesh with constant rho (config 3) every interior cell sees the same geometry,
// and the GPU assembly produces BITWISE-identical row-blocks (config 3: 1225 distinct row-blocks for
// 262,144 cells) and bitwise-identical local factors (64 distinct for 4,096 subdomains). Storing each
// distinct block once changes no arithmetic at all (same bits, same order of operations); it only moves
// the SpMV's 1.05 GB of A and the local solve's 1.6 GB of factors into a few MB that stay in L2:
//   * A: k_spmv_dd reads cell c's row-block from a_dd[c] in the compact store through the L2 (the byte
//     ring with one bulk copy per cell was measured slower: 0.40 ms vs 0.18 ms on config 3);
//   * local factors: the panel kernels address the factor of cell c through p_off[c], so every cell of
//     a subdomain is pointed at the same relative position in the representative subdomain's panels.
// Detection hashes and then memcmp-verifies the data at setup (host copy once). Off on meshes without
// repetition (Voronoi: every block distinct) and with DGAS_DEDUP=0.
#include <cstring>
#include <unordered_map>

#include "internal.h"

static uint64_t fnv_bytes(const void* p, size_t n, uint64_t h = 1469598103934665603ULL) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) { h ^= b[i]; h *= 1099511628211ULL; }
  return h;
}

int dedup_setup(dgas_ctx ctx) {
  int on = 1;
  if (const char* e = std::getenv("DGAS_DEDUP")) on = std::atoi(e) != 0;
  if (!on || ctx->spmv_kernel != 4) return 0;
  const int nc = ctx->nc;
  cudaStream_t s = ctx->stream;
  double maxfrac = 0.25;  // stored / total above which de-duplication is not worth it (tests: small meshes)
  if (const char* e = std::getenv("DGAS_DEDUP_MAXFRAC")) maxfrac = std::atof(e);
  DGAS_CUDA(cudaStreamSynchronize(s));
  // ---------------- A row-blocks
  {
    const std::vector<int64_t>& ao = ctx->a_off_h;
    std::vector<double> A((size_t)ao[nc]);
    DGAS_CUDA(cudaMemcpy(A.data(), ctx->d_A, A.size() * 8, cudaMemcpyDeviceToHost));
    std::unordered_map<uint64_t, std::vector<int>> rep;  // hash -> representative cells
    std::vector<int64_t> dd(nc);
    std::vector<int> reps;
    int64_t stored = 0;
    for (int c = 0; c < nc; ++c) {
      const int64_t n = ao[c + 1] - ao[c];
      const uint64_t h = fnv_bytes(A.data() + ao[c], (size_t)n * 8) ^ (uint64_t)n;
      auto& lst = rep[h];
      int found = -1;
      for (int r : lst)
        if (ao[r + 1] - ao[r] == n && std::memcmp(A.data() + ao[r], A.data() + ao[c], (size_t)n * 8) == 0) { found = r; break; }
      if (found < 0) {
        lst.push_back(c);
        reps.push_back(c);
        dd[c] = stored;
        stored += n;
      } else {
        dd[c] = dd[found];
      }
    }
    // worth it only with real repetition (the compact store then fits L2 and the copies are L2 hits)
    if ((double)stored < maxfrac * (double)ao[nc]) {
      std::vector<double> Ac((size_t)stored);
      for (int r : reps) std::memcpy(Ac.data() + dd[r], A.data() + ao[r], (size_t)(ao[r + 1] - ao[r]) * 8);
      double* dA = nullptr;
      int st;
      if ((st = dev_upload(ctx, &dA, Ac)) || (st = dev_upload(ctx, &ctx->d_a_dd, dd))) return st;
      cudaFree(ctx->d_A);
      ctx->d_A = dA;
      ctx->a_dd_h = dd;
      ctx->a_unique = (int64_t)reps.size();
      ctx->a_bytes_stored = stored * 8;
      int dev = 0, nsm = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      ctx->dd_grid = std::min(nc, 8 * nsm);  // k_spmv_dd: 8 x 256-thread CTAs per SM
      if (const char* e = std::getenv("DGAS_DD_CPS")) ctx->dd_grid = std::min(nc, std::max(1, std::atoi(e)) * nsm);
      if ((st = spmv_cls_setup(ctx, dd))) return st;  // class-sorted SpMV (row-block in registers)
    }
  }
  // ---------------- local factors (merged panels), whole subdomains at a time
  if ((ctx->local_kernel == 2 || ctx->local_kernel == 4) && !ctx->panel_f32) {
    const int nsub = ctx->nsub;
    const std::vector<int>& sp = ctx->sub_ptr_h;
    std::vector<int64_t> po(nc + 1);
    DGAS_CUDA(cudaMemcpy(po.data(), ctx->d_p_off, (nc + 1) * 8, cudaMemcpyDeviceToHost));
    std::vector<double> Pp((size_t)ctx->p_total);
    DGAS_CUDA(cudaMemcpy(Pp.data(), ctx->d_P, Pp.size() * 8, cudaMemcpyDeviceToHost));
    std::unordered_map<uint64_t, std::vector<int>> rep;
    std::vector<int> rep_of(nsub);
    std::vector<int> reps;
    auto same_shape = [&](int a, int b) {
      const int m = sp[a + 1] - sp[a];
      if (sp[b + 1] - sp[b] != m) return false;
      for (int k = 0; k <= m; ++k)
        if (po[sp[a] + k] - po[sp[a]] != po[sp[b] + k] - po[sp[b]]) return false;
      for (int k = 0; k < m; ++k)
        if (ctx->first_h[sp[a] + k] != ctx->first_h[sp[b] + k]) return false;
      return true;
    };
    for (int s2 = 0; s2 < nsub; ++s2) {
      const int64_t a0 = po[sp[s2]], a1 = po[sp[s2 + 1]];
      uint64_t h = fnv_bytes(Pp.data() + a0, (size_t)(a1 - a0) * 8);
      h = fnv_bytes(ctx->first_h.data() + sp[s2], (size_t)(sp[s2 + 1] - sp[s2]) * 4, h);
      auto& lst = rep[h];
      int found = -1;
      for (int r : lst)
        if (same_shape(r, s2) && std::memcmp(Pp.data() + po[sp[r]], Pp.data() + a0, (size_t)(a1 - a0) * 8) == 0) { found = r; break; }
      if (found < 0) { lst.push_back(s2); reps.push_back(s2); rep_of[s2] = s2; }
      else rep_of[s2] = found;
    }
    int64_t stored = 0;
    std::vector<int64_t> base(nsub, -1);
    for (int r : reps) { base[r] = stored; stored += po[sp[r + 1]] - po[sp[r]]; }
    if ((double)stored < maxfrac * (double)ctx->p_total) {
      std::vector<double> Pc((size_t)stored + 32);
      for (int r : reps) std::memcpy(Pc.data() + base[r], Pp.data() + po[sp[r]], (size_t)(po[sp[r + 1]] - po[sp[r]]) * 8);
      std::vector<int64_t> pn(nc + 1);
      for (int s2 = 0; s2 < nsub; ++s2) {
        const int r = rep_of[s2];
        for (int c = sp[s2]; c < sp[s2 + 1]; ++c) pn[c] = base[r] + (po[sp[r] + (c - sp[s2])] - po[sp[r]]);
      }
      pn[nc] = stored;
      double* dP = nullptr;
      int64_t* dpo = nullptr;
      int st;
      if ((st = dev_upload(ctx, &dP, Pc)) || (st = dev_upload(ctx, &dpo, pn))) return st;
      cudaFree(ctx->d_P);
      cudaFree(ctx->d_p_off);
      ctx->d_P = dP;
      ctx->d_p_off = dpo;
      ctx->p_unique = (int)reps.size();
      ctx->p_bytes_stored = stored * 8;
      if ((st = mrhs_setup(ctx, rep_of))) return st;  // batched solves over the shared factors
    }
  }
  // ---------------- restriction / prolongation blocks G (one np x nq block per overlap piece): nested
  // Cartesian tilings repeat them. The iteration kernels get a compact store and copies of the piece
  // records that index its distinct blocks (same bits, same order of operations); the originals stay
  // for the sharded solve, which addresses G by piece.
  {
    int gon = 1;
    if (const char* e = std::getenv("DGAS_DEDUP_G")) gon = std::atoi(e) != 0;
    const int nov = ctx->nov;
    const size_t blk = (size_t)ctx->np * ctx->nq;
    if (gon && nov > 0) {
      std::vector<double> G((size_t)nov * blk);
      DGAS_CUDA(cudaMemcpy(G.data(), ctx->d_G, G.size() * 8, cudaMemcpyDeviceToHost));
      std::unordered_map<uint64_t, std::vector<int>> rep;
      std::vector<int> uidx(nov), reps;
      for (int o = 0; o < nov; ++o) {
        const uint64_t h = fnv_bytes(G.data() + (size_t)o * blk, blk * 8);
        auto& lst = rep[h];
        int found = -1;
        for (int r : lst)
          if (std::memcmp(G.data() + (size_t)r * blk, G.data() + (size_t)o * blk, blk * 8) == 0) { found = r; break; }
        if (found < 0) { lst.push_back(o); uidx[o] = (int)reps.size(); reps.push_back(o); }
        else uidx[o] = uidx[found];
      }
      if ((double)reps.size() < maxfrac * (double)nov) {
        std::vector<double> Gc(reps.size() * blk);
        for (size_t u = 0; u < reps.size(); ++u) std::memcpy(Gc.data() + u * blk, G.data() + (size_t)reps[u] * blk, blk * 8);
        std::vector<int2> rrec(nov), prec(nov);
        std::vector<int4> crec(nc);
        DGAS_CUDA(cudaMemcpy(rrec.data(), ctx->d_rrec, (size_t)nov * sizeof(int2), cudaMemcpyDeviceToHost));
        DGAS_CUDA(cudaMemcpy(prec.data(), ctx->d_prec, (size_t)nov * sizeof(int2), cudaMemcpyDeviceToHost));
        DGAS_CUDA(cudaMemcpy(crec.data(), ctx->d_crec, (size_t)nc * sizeof(int4), cudaMemcpyDeviceToHost));
        for (int k = 0; k < nov; ++k) {
          const int o = rrec[k].y & 0x7fffffff;
          rrec[k].y = (rrec[k].y & (int)0x80000000u) | uidx[o];
          prec[k].x = uidx[prec[k].x];
        }
        for (int c = 0; c < nc; ++c) crec[c].x = uidx[crec[c].x];
        int st;
        if ((st = dev_upload(ctx, &ctx->d_G_it, Gc)) || (st = dev_upload(ctx, &ctx->d_rrec_it, rrec)) ||
            (st = dev_upload(ctx, &ctx->d_prec_it, prec)) || (st = dev_upload(ctx, &ctx->d_crec_it, crec)))
          return st;
        ctx->g_unique = (int64_t)reps.size();
      }
    }
  }
  if (std::getenv("DGAS_VERBOSE") && ctx->g_unique)
    fprintf(stderr, "dgas: dedup: G %lld distinct blocks for %d pieces (%.2f MB stored)\n", (long long)ctx->g_unique,
            ctx->nov, ctx->g_unique * ctx->np * ctx->nq * 8 / 1e6);
  if (std::getenv("DGAS_VERBOSE"))
    fprintf(stderr, "dgas: dedup: A %lld distinct row-blocks (%.1f MB stored), local factors %d distinct (%.1f MB)\n",
            (long long)ctx->a_unique, ctx->a_bytes_stored / 1e6, ctx->p_unique, ctx->p_bytes_stored / 1e6);
  return 0;
}
