// nd_host.cu — symbolic nested dissection of the coarse problem (integer plumbing on the host).
//
// The coarse operator A0 = Q^T A Q (eq:A0) is block-sparse over coarse elements.
// For large N0 it is factorised by a multifrontal nested-dissection Cholesky (DESIGN.md "Coarse
// solve"): recursive coordinate bisection of the coarse-element centroids gives a binary tree of
// fronts; front F eliminates its own elements after its descendants, U_F are the later elements it
// couples to. Per front the GPU stores X_F = S_FF^-1 and M_F = S_UF S_FF^-1 (S = front matrix after
// the children's Schur updates), so each tree level of the solve is a single GEMV-only launch:
//   forward (leaves -> root):  u_F = t_U - M_F t_F,            t = b + children's u (extend-add)
//   backward (root -> leaves): x_F = X_F t_F - M_F^T x_U.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <numeric>
#include <vector>

#include "internal.h"

namespace {
struct Front {
  std::vector<int> F, U;      // coarse elements (U in elimination order)
  std::vector<int> child;
  int parent = -1, depth = 0;
};
}  // namespace

int nd_build(dgas_ctx ctx, const std::vector<int>& pair_h, const std::vector<double>& centroid, int leaf) {
  const int NC = ctx->ncoarse, nq = ctx->nq;
  // adjacency of coarse elements (from the coupled pairs of A0)
  std::vector<std::vector<int>> adj(NC);
  for (size_t k = 0; k < pair_h.size() / 2; ++k) {
    int a = pair_h[2 * k], b = pair_h[2 * k + 1];
    if (a != b) adj[a].push_back(b);
  }
  for (auto& l : adj) { std::sort(l.begin(), l.end()); l.erase(std::unique(l.begin(), l.end()), l.end()); }
  // recursive bisection -> fronts (children before parents after the final postorder sort)
  std::vector<Front> fr;
  struct Task { std::vector<int> nodes; int parent, depth; };
  std::vector<Task> stack;
  std::vector<int> all(NC);
  std::iota(all.begin(), all.end(), 0);
  stack.push_back({all, -1, 0});
  std::vector<int> side(NC, 0);
  while (!stack.empty()) {
    Task t = std::move(stack.back());
    stack.pop_back();
    const int id = (int)fr.size();
    fr.push_back(Front());
    fr[id].parent = t.parent;
    fr[id].depth = t.depth;
    if (t.parent >= 0) fr[t.parent].child.push_back(id);
    if ((int)t.nodes.size() <= leaf) { fr[id].F = t.nodes; continue; }
    double x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300;
    for (int v : t.nodes) {
      x0 = std::min(x0, centroid[2 * v]); x1 = std::max(x1, centroid[2 * v]);
      y0 = std::min(y0, centroid[2 * v + 1]); y1 = std::max(y1, centroid[2 * v + 1]);
    }
    const int ax = (x1 - x0) >= (y1 - y0) ? 0 : 1;
    std::vector<int> nodes = t.nodes;
    std::sort(nodes.begin(), nodes.end(), [&](int a, int b) {
      double ca = centroid[2 * a + ax], cb = centroid[2 * b + ax];
      return ca < cb || (ca == cb && a < b);
    });
    const size_t half = nodes.size() / 2;
    for (size_t i = 0; i < nodes.size(); ++i) side[nodes[i]] = i < half ? 1 : 2;
    std::vector<int> L, R, S;
    for (size_t i = 0; i < nodes.size(); ++i) {
      int v = nodes[i];
      if (side[v] == 1) {
        bool sep = false;
        for (int w : adj[v]) if (side[w] == 2) { sep = true; break; }
        (sep ? S : L).push_back(v);
      } else R.push_back(v);
    }
    for (int v : nodes) side[v] = 0;
    fr[id].F = S;
    if (!L.empty()) stack.push_back({L, id, t.depth + 1});
    if (!R.empty()) stack.push_back({R, id, t.depth + 1});
    if (S.empty() && (L.empty() || R.empty())) {  // degenerate split: make it a leaf
      fr[id].F = t.nodes;
      for (int c : fr[id].child) (void)c;
      fr[id].child.clear();
      stack.resize(stack.size() - (!L.empty()) - (!R.empty()));
    }
  }
  // postorder: children before parents (process by decreasing depth, then id)
  const int nf = (int)fr.size();
  std::vector<int> order(nf);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return fr[a].depth > fr[b].depth; });
  std::vector<int> pos(nf);
  for (int i = 0; i < nf; ++i) pos[order[i]] = i;
  std::vector<int> rank(NC, -1);
  for (int i = 0; i < nf; ++i)
    for (int v : fr[order[i]].F) rank[v] = i;
  for (int v = 0; v < NC; ++v)
    if (rank[v] < 0) { ctx->detail = "nested dissection lost a coarse element"; return DGAS_E_MESH; }
  // symbolic: U_F = (adj(F) U children's U) restricted to later ranks, sorted by (rank, id)
  for (int i = 0; i < nf; ++i) {
    Front& f = fr[order[i]];
    std::vector<int> u;
    for (int v : f.F)
      for (int w : adj[v]) if (rank[w] > i) u.push_back(w);
    for (int c : f.child)
      for (int w : fr[c].U) if (rank[w] > i) u.push_back(w);
    std::sort(u.begin(), u.end(), [&](int a, int b) { return rank[a] < rank[b] || (rank[a] == rank[b] && a < b); });
    u.erase(std::unique(u.begin(), u.end()), u.end());
    f.U = u;
  }
  // ---- flatten (fronts in postorder), dof-level sizes, storage offsets, maps
  NdPlan& P = ctx->nd;
  P = NdPlan();
  P.nf = nf;
  int maxdepth = 0;
  for (auto& f : fr) maxdepth = std::max(maxdepth, f.depth);
  P.nlev = maxdepth + 1;
  std::vector<int> nF(nf), nU(nf);
  std::vector<int64_t> offX(nf + 1, 0), offM(nf + 1, 0), offUpd(nf + 1, 0), offS(nf + 1, 0);
  std::vector<int> offT(nf + 1, 0), offu(nf + 1, 0), offFe(nf + 1, 0), offUe(nf + 1, 0);
  std::vector<int> Fe, Ue;  // coarse elements of F and U, flattened
  std::vector<int> childptr(nf + 1, 0), childs, cmap_ptr(1, 0), cmap;  // child -> parent local index
  std::vector<int> lev_of(nf);
  for (int i = 0; i < nf; ++i) {
    const Front& f = fr[order[i]];
    nF[i] = (int)f.F.size() * nq;
    nU[i] = (int)f.U.size() * nq;
    offX[i + 1] = offX[i] + (int64_t)nF[i] * nF[i];
    offM[i + 1] = offM[i] + (int64_t)nU[i] * nF[i];
    offUpd[i + 1] = offUpd[i] + (int64_t)nU[i] * nU[i];
    offS[i + 1] = offS[i] + (int64_t)(nF[i] + nU[i]) * (nF[i] + nU[i]);
    offT[i + 1] = offT[i] + nF[i];
    offu[i + 1] = offu[i] + nU[i];
    Fe.insert(Fe.end(), f.F.begin(), f.F.end());
    Ue.insert(Ue.end(), f.U.begin(), f.U.end());
    offFe[i + 1] = (int)Fe.size();
    offUe[i + 1] = (int)Ue.size();
    lev_of[i] = f.depth;
    P.maxF = std::max(P.maxF, nF[i]);
    P.maxU = std::max(P.maxU, nU[i]);
    P.maxN = std::max(P.maxN, nF[i] + nU[i]);
  }
  for (int i = 0; i < nf; ++i) {
    const Front& f = fr[order[i]];
    // local index of every element of F u U
    std::vector<std::pair<int, int>> loc;
    for (size_t k = 0; k < f.F.size(); ++k) loc.push_back({f.F[k], (int)k});
    for (size_t k = 0; k < f.U.size(); ++k) loc.push_back({f.U[k], (int)(f.F.size() + k)});
    std::sort(loc.begin(), loc.end());
    auto local = [&](int e) {
      auto it = std::lower_bound(loc.begin(), loc.end(), std::make_pair(e, -1));
      return (it != loc.end() && it->first == e) ? it->second : -1;
    };
    for (int c : f.child) {
      const int ci = pos[c];
      childs.push_back(ci);
      // map of the child's U elements into this front's local element index
      for (int w : fr[c].U) {
        int l = local(w);
        if (l < 0) { ctx->detail = "nested dissection: child update not covered by parent"; return DGAS_E_MESH; }
        cmap.push_back(l);
      }
      cmap_ptr.push_back((int)cmap.size());
    }
    childptr[i + 1] = (int)childs.size();
  }
  // children's cmap offsets are stored per child (indexed by child position in `childs`)
  // assembly list: for every coupled pair (v, w), v in F, rank(w) >= rank(F): (pair, local v, local w)
  std::vector<int> asm_ptr(nf + 1, 0);
  std::vector<int4> asmv;
  {
    // pair index lookup
    std::vector<std::vector<std::pair<int, int>>> prs(NC);
    for (size_t k = 0; k < pair_h.size() / 2; ++k) prs[pair_h[2 * k]].push_back({pair_h[2 * k + 1], (int)k});
    for (int i = 0; i < nf; ++i) {
      const Front& f = fr[order[i]];
      std::vector<std::pair<int, int>> loc;
      for (size_t k = 0; k < f.F.size(); ++k) loc.push_back({f.F[k], (int)k});
      for (size_t k = 0; k < f.U.size(); ++k) loc.push_back({f.U[k], (int)(f.F.size() + k)});
      std::sort(loc.begin(), loc.end());
      for (size_t k = 0; k < f.F.size(); ++k) {
        int v = f.F[k];
        for (auto& pw : prs[v]) {
          int w = pw.first;
          if (rank[w] < i) continue;
          auto it = std::lower_bound(loc.begin(), loc.end(), std::make_pair(w, -1));
          if (it == loc.end() || it->first != w) { ctx->detail = "nested dissection: coupling outside front"; return DGAS_E_MESH; }
          asmv.push_back(make_int4(pw.second, (int)k, it->second, 0));
        }
      }
      asm_ptr[i + 1] = (int)asmv.size();
    }
  }
  // levels: fronts grouped by depth (forward: deepest first)
  std::vector<int> lev_ptr(P.nlev + 1, 0), lev_fronts;
  for (int d = P.nlev - 1, k = 0; d >= 0; --d, ++k) {
    for (int i = 0; i < nf; ++i) if (lev_of[i] == d) lev_fronts.push_back(i);
    lev_ptr[k + 1] = (int)lev_fronts.size();
  }
  P.h_lev_ptr = lev_ptr;
  P.h_lev_fronts = lev_fronts;
  P.h_nF = nF; P.h_nU = nU;
  P.h_offX = offX; P.h_offM = offM; P.h_offUpd = offUpd; P.h_offS = offS;
  P.h_offT = offT; P.h_offu = offu; P.h_offFe = offFe; P.h_offUe = offUe;
  P.h_Fe = Fe; P.h_Ue = Ue; P.h_childptr = childptr; P.h_childs = childs; P.h_cmap_ptr = cmap_ptr; P.h_cmap = cmap;
  P.h_asm_ptr = asm_ptr; P.h_asm = asmv;
  P.h_prow.assign(NC + 1, 0);
  for (size_t k = 0; k < pair_h.size() / 2; ++k) P.h_prow[pair_h[2 * k] + 1]++;
  for (int J = 0; J < NC; ++J) P.h_prow[J + 1] += P.h_prow[J];
  if (const char* e = std::getenv("DGAS_ND_REFINE")) P.refine = P.refine_env = std::max(0, std::atoi(e));
  return 0;
}
