// dgas_gen/gen.cpp — seeded synthetic INPUT generator (meshes, partitions, coarse agglomerates).
//
// This module is input generation only. It is shared by the oracle (oracle/) and the CUDA path
// (paper_1903_11357_b200/) and holds none of the method's arithmetic: no quadrature, no basis,
// no assembly, no solver. It produces
//   * the fine polygonal mesh T_h ("tessellation of Omega consisting of disjoint
//     polytopic elements"),
//   * the subdomain partition T_HH ("each subdomain Omega_i is the union of some
//     elements"),
//   * the coarse partition T_H either as a parent map (nested) or, for the
//     non-nested "edge coarsening" reading (reading R17), as coarse polygons
//     plus the intersection pieces kappa ∩ D_J (pure geometry),
//   * the piecewise-constant diffusion coefficient rho (BASELINE calls it kappa).
//
// Recipe: SplitMix64-seeded xoshiro256**, uniform seeds in [0,1]^2,
// clipped Voronoi by half-plane clipping, 5 Lloyd iterations, vertex welding, RCB partitions
// (split the longer centroid-bbox extent at the count median, ties by cell id), lexicographic
// tiles for Cartesian grids, merged-edge (chord) coarse polygons for config 4.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <numeric>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

namespace {

// ------------------------------------------------------------------ RNG
struct Rng {
  uint64_t s[4];
  static uint64_t splitmix(uint64_t& x) {
    uint64_t z = (x += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  explicit Rng(uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) s[i] = splitmix(x);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
    return r;
  }
  double uniform() { return double(next() >> 11) * (1.0 / 9007199254740992.0); }
};

struct P2 { double x, y; };
using Poly = std::vector<P2>;

double poly_area(const Poly& p) {
  double a = 0;
  for (size_t i = 0, n = p.size(); i < n; ++i) {
    const P2 &u = p[i], &v = p[(i + 1) % n];
    a += u.x * v.y - v.x * u.y;
  }
  return 0.5 * a;
}
P2 poly_centroid(const Poly& p) {
  double a = 0, cx = 0, cy = 0;
  for (size_t i = 0, n = p.size(); i < n; ++i) {
    const P2 &u = p[i], &v = p[(i + 1) % n];
    double c = u.x * v.y - v.x * u.y;
    a += c; cx += (u.x + v.x) * c; cy += (u.y + v.y) * c;
  }
  a *= 0.5;
  return {cx / (6 * a), cy / (6 * a)};
}

// keep {x : (x - m) . d <= 0}
Poly clip_halfplane(const Poly& in, P2 m, P2 d) {
  Poly out;
  size_t n = in.size();
  if (!n) return out;
  out.reserve(n + 2);
  for (size_t i = 0; i < n; ++i) {
    const P2 &a = in[i], &b = in[(i + 1) % n];
    double fa = (a.x - m.x) * d.x + (a.y - m.y) * d.y;
    double fb = (b.x - m.x) * d.x + (b.y - m.y) * d.y;
    bool ia = fa <= 0, ib = fb <= 0;
    if (ia) out.push_back(a);
    if (ia != ib) {
      double t = fa / (fa - fb);
      out.push_back({a.x + t * (b.x - a.x), a.y + t * (b.y - a.y)});
    }
  }
  return out;
}

// ------------------------------------------------------------------ Voronoi (clipped to unit square)
void voronoi(const std::vector<P2>& seeds, std::vector<Poly>& cells) {
  const int N = (int)seeds.size();
  int G = std::max(1, (int)std::ceil(std::sqrt(N / 2.0)));
  double bs = 1.0 / G;
  std::vector<std::vector<int>> bucket(G * G);
  auto bidx = [&](double v) { return std::min(G - 1, std::max(0, (int)(v * G))); };
  for (int i = 0; i < N; ++i) bucket[bidx(seeds[i].y) * G + bidx(seeds[i].x)].push_back(i);
  cells.assign(N, {});
  for (int i = 0; i < N; ++i) {
    const P2 s = seeds[i];
    Poly c = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
    int bx = bidx(s.x), by = bidx(s.y);
    for (int r = 0; r <= G; ++r) {
      double rmax2 = 0;
      for (auto& v : c) rmax2 = std::max(rmax2, (v.x - s.x) * (v.x - s.x) + (v.y - s.y) * (v.y - s.y));
      double lb = (r - 1) * bs;
      if (r >= 2 && 4 * rmax2 <= lb * lb) break;
      for (int yy = by - r; yy <= by + r; ++yy)
        for (int xx = bx - r; xx <= bx + r; ++xx) {
          if (std::max(std::abs(yy - by), std::abs(xx - bx)) != r) continue;
          if (xx < 0 || yy < 0 || xx >= G || yy >= G) continue;
          for (int j : bucket[yy * G + xx]) {
            if (j == i) continue;
            P2 t = seeds[j];
            P2 m = {0.5 * (s.x + t.x), 0.5 * (s.y + t.y)}, d = {t.x - s.x, t.y - s.y};
            c = clip_halfplane(c, m, d);
          }
        }
    }
    cells[i] = c;
  }
}

struct Mesh {
  std::vector<double> xy;
  std::vector<int> cptr, cvtx;
  int ncells() const { return (int)cptr.size() - 1; }
  P2 v(int i) const { return {xy[2 * i], xy[2 * i + 1]}; }
  Poly poly(int c) const {
    Poly p;
    for (int k = cptr[c]; k < cptr[c + 1]; ++k) p.push_back(v(cvtx[k]));
    return p;
  }
};

// weld vertices of independently clipped cells into one shared vertex table
bool weld(const std::vector<Poly>& cells, Mesh& m, std::string& err) {
  const double q = 1e-9, tol = 1e-11;
  std::unordered_map<uint64_t, std::vector<int>> grid;
  auto key = [](int64_t ix, int64_t iy) { return (uint64_t)(ix + (1LL << 31)) << 32 | (uint64_t)(iy + (1LL << 31)); };
  m.xy.clear(); m.cptr.assign(1, 0); m.cvtx.clear();
  for (const Poly& c : cells) {
    std::vector<int> ids;
    for (const P2& p : c) {
      // snap exact boundary coordinates
      P2 v = p;
      if (std::fabs(v.x) < 1e-13) v.x = 0;
      if (std::fabs(v.y) < 1e-13) v.y = 0;
      if (std::fabs(v.x - 1) < 1e-13) v.x = 1;
      if (std::fabs(v.y - 1) < 1e-13) v.y = 1;
      int64_t ix = (int64_t)std::floor(v.x / q), iy = (int64_t)std::floor(v.y / q);
      int found = -1;
      for (int dy = -1; dy <= 1 && found < 0; ++dy)
        for (int dx = -1; dx <= 1 && found < 0; ++dx) {
          auto it = grid.find(key(ix + dx, iy + dy));
          if (it == grid.end()) continue;
          for (int id : it->second) {
            double ex = m.xy[2 * id] - v.x, ey = m.xy[2 * id + 1] - v.y;
            if (ex * ex + ey * ey <= tol * tol) { found = id; break; }
          }
        }
      if (found < 0) {
        found = (int)m.xy.size() / 2;
        m.xy.push_back(v.x); m.xy.push_back(v.y);
        grid[key(ix, iy)].push_back(found);
      }
      if (ids.empty() || ids.back() != found) ids.push_back(found);
    }
    while (ids.size() > 1 && ids.front() == ids.back()) ids.pop_back();
    if (ids.size() < 3) { err = "degenerate cell after welding"; return false; }
    for (int id : ids) m.cvtx.push_back(id);
    m.cptr.push_back((int)m.cvtx.size());
  }
  return true;
}

bool make_voronoi(int N, uint64_t seed, int lloyd, Mesh& m, std::string& err) {
  Rng rng(seed);
  std::vector<P2> seeds;
  seeds.reserve(N);
  // uniform seeds in [0,1]^2, drawn (x_i, y_i) in order; near-duplicates redrawn
  {
    int G = std::max(1, (int)std::ceil(std::sqrt((double)N)));
    std::vector<std::vector<int>> b(G * G);
    while ((int)seeds.size() < N) {
      P2 s = {rng.uniform(), rng.uniform()};
      int bx = std::min(G - 1, (int)(s.x * G)), by = std::min(G - 1, (int)(s.y * G));
      bool dup = false;
      for (int yy = std::max(0, by - 1); yy <= std::min(G - 1, by + 1) && !dup; ++yy)
        for (int xx = std::max(0, bx - 1); xx <= std::min(G - 1, bx + 1) && !dup; ++xx)
          for (int j : b[yy * G + xx])
            if (std::hypot(seeds[j].x - s.x, seeds[j].y - s.y) < 1e-12) { dup = true; break; }
      if (dup) continue;
      b[by * G + bx].push_back((int)seeds.size());
      seeds.push_back(s);
    }
  }
  std::vector<Poly> cells;
  for (int it = 0; it < lloyd; ++it) {
    voronoi(seeds, cells);
    for (int i = 0; i < N; ++i) seeds[i] = poly_centroid(cells[i]);
  }
  voronoi(seeds, cells);
  return weld(cells, m, err);
}

void make_cartesian(int n, Mesh& m) {
  m.xy.clear(); m.cptr.assign(1, 0); m.cvtx.clear();
  for (int j = 0; j <= n; ++j)
    for (int i = 0; i <= n; ++i) { m.xy.push_back((double)i / n); m.xy.push_back((double)j / n); }
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      int v0 = j * (n + 1) + i;
      m.cvtx.push_back(v0); m.cvtx.push_back(v0 + 1); m.cvtx.push_back(v0 + n + 2); m.cvtx.push_back(v0 + n + 1);
      m.cptr.push_back((int)m.cvtx.size());
    }
}

// ------------------------------------------------------------------ L-shaped domain (paper Ex.1)
// L = [0,1]^2 minus the quadrant (1/2,1] x [0,1/2) (re-entrant corner at (1/2,1/2); the paper's
// (-1,1)^2-type L scaled by 1/2, which leaves K unchanged). A Voronoi cell of the unit square is cut to
// the L as A = cell ∩ {x <= 1/2} and B = cell ∩ {x >= 1/2, y >= 1/2}; when both are non-empty the cell is
// split into the two convex polygons A and B unless cell ∩ L is already a single half-plane clip
// (only cells around the corner split, which can add one or two cells to the requested count).
const double LC = 0.5;
bool in_L(P2 s) { return !(s.x > LC && s.y < LC); }

void clip_L(const Poly& c, std::vector<Poly>& out) {
  Poly a = clip_halfplane(c, {LC, 0}, {1, 0});                         // x <= 1/2
  Poly b = clip_halfplane(clip_halfplane(c, {LC, 0}, {-1, 0}), {0, LC}, {0, -1});  // x >= 1/2, y >= 1/2
  double ac = std::fabs(poly_area(c)), tol = 1e-12 * ac;
  double aa = a.size() >= 3 ? std::fabs(poly_area(a)) : 0, ab = b.size() >= 3 ? std::fabs(poly_area(b)) : 0;
  if (std::fabs(aa + ab - ac) <= tol) { out.push_back(c); return; }   // cell inside L
  // cell ∩ L is convex when it is a single half-plane clip of the cell; only otherwise split into A, B
  Poly up = clip_halfplane(c, {0, LC}, {0, -1});                      // y >= 1/2
  double au = up.size() >= 3 ? std::fabs(poly_area(up)) : 0;
  if (std::fabs(au - (aa + ab)) <= tol) { out.push_back(up); return; }
  if (std::fabs(aa - (aa + ab)) <= tol) { out.push_back(a); return; }
  if (aa > tol) out.push_back(a);
  if (ab > tol) out.push_back(b);
}

// insert every mesh vertex that lies strictly inside another cell's edge into that cell's loop, so that
// faces are conforming vertex pairs (the split above creates such hanging vertices)
void insert_hanging(Mesh& m) {
  const int NV = (int)m.xy.size() / 2;
  const int G = std::max(1, (int)std::sqrt((double)NV));
  std::vector<std::vector<int>> bk(G * G);
  auto bi = [&](double v) { return std::min(G - 1, std::max(0, (int)(v * G))); };
  for (int i = 0; i < NV; ++i) bk[bi(m.xy[2 * i + 1]) * G + bi(m.xy[2 * i])].push_back(i);
  std::vector<int> nptr(1, 0), nv;
  for (int c = 0; c < m.ncells(); ++c) {
    const int n = m.cptr[c + 1] - m.cptr[c];
    for (int k = 0; k < n; ++k) {
      int ia = m.cvtx[m.cptr[c] + k], ib = m.cvtx[m.cptr[c] + (k + 1) % n];
      nv.push_back(ia);
      P2 a = m.v(ia), b = m.v(ib);
      double L2 = (b.x - a.x) * (b.x - a.x) + (b.y - a.y) * (b.y - a.y);
      std::vector<std::pair<double, int>> hits;
      for (int yy = bi(std::min(a.y, b.y)); yy <= bi(std::max(a.y, b.y)); ++yy)
        for (int xx = bi(std::min(a.x, b.x)); xx <= bi(std::max(a.x, b.x)); ++xx)
          for (int j : bk[yy * G + xx]) {
            if (j == ia || j == ib) continue;
            P2 v = m.v(j);
            double t = ((v.x - a.x) * (b.x - a.x) + (v.y - a.y) * (b.y - a.y)) / L2;
            if (t <= 1e-9 || t >= 1 - 1e-9) continue;
            double cr = (b.x - a.x) * (v.y - a.y) - (b.y - a.y) * (v.x - a.x);
            if (cr * cr <= 1e-22 * L2 * L2) hits.push_back({t, j});
          }
      std::sort(hits.begin(), hits.end());
      for (auto& h : hits) nv.push_back(h.second);
    }
    nptr.push_back((int)nv.size());
  }
  m.cptr = nptr; m.cvtx = nv;
}

bool make_voronoi_L(int N, uint64_t seed, int lloyd, Mesh& m, std::string& err) {
  Rng rng(seed);
  std::vector<P2> seeds;
  while ((int)seeds.size() < N) {                                       // uniform in L by rejection
    P2 s = {rng.uniform(), rng.uniform()};
    if (in_L(s)) seeds.push_back(s);
  }
  std::vector<Poly> cells, parts;
  for (int it = 0; it < lloyd; ++it) {                                  // Lloyd on cell ∩ L
    voronoi(seeds, cells);
    for (int i = 0; i < N; ++i) {
      parts.clear();
      clip_L(cells[i], parts);
      double A = 0, cx = 0, cy = 0;
      for (auto& q : parts) { double a = poly_area(q); P2 c = poly_centroid(q); A += a; cx += a * c.x; cy += a * c.y; }
      if (A > 0) seeds[i] = {cx / A, cy / A};
    }
  }
  voronoi(seeds, cells);
  std::vector<Poly> out;
  for (auto& c : cells) clip_L(c, out);
  if (!weld(out, m, err)) return false;
  insert_hanging(m);
  return true;
}

// one level of centroid-midpoint refinement ("successive refinement of elements"): an
// n-gon v_0..v_{n-1} with centroid c becomes the n quadrilaterals (c, m_{i-1,i}, v_i, m_{i,i+1});
// shared edges are split at the same midpoint on both sides, so the result is conforming.
// parent[c'] = the cell c' came from; children of one cell are consecutive.
void refine_once(const Mesh& m, Mesh& out, std::vector<int>& parent, std::string& err) {
  std::vector<Poly> cells;
  parent.clear();
  for (int c = 0; c < m.ncells(); ++c) {
    Poly p = m.poly(c);
    P2 g = poly_centroid(p);
    const int n = (int)p.size();
    for (int i = 0; i < n; ++i) {
      P2 vp = p[(i + n - 1) % n], v = p[i], vn = p[(i + 1) % n];
      cells.push_back({g, {0.5 * (vp.x + v.x), 0.5 * (vp.y + v.y)}, v, {0.5 * (v.x + vn.x), 0.5 * (v.y + vn.y)}});
      parent.push_back(c);
    }
  }
  weld(cells, out, err);
}

// ------------------------------------------------------------------ partitions
std::vector<P2> centroids(const Mesh& m) {
  std::vector<P2> c(m.ncells());
  for (int i = 0; i < m.ncells(); ++i) c[i] = poly_centroid(m.poly(i));
  return c;
}

// recursive coordinate bisection; part ids = leaf index in depth-first (low, high) order
void rcb_rec(const std::vector<P2>& cen, std::vector<int>& ids, int lo, int hi, int k, int first, std::vector<int>& part) {
  if (k == 1) { for (int i = lo; i < hi; ++i) part[ids[i]] = first; return; }
  double x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300;
  for (int i = lo; i < hi; ++i) {
    const P2& c = cen[ids[i]];
    x0 = std::min(x0, c.x); x1 = std::max(x1, c.x); y0 = std::min(y0, c.y); y1 = std::max(y1, c.y);
  }
  bool byx = (x1 - x0) >= (y1 - y0);
  std::sort(ids.begin() + lo, ids.begin() + hi, [&](int a, int b) {
    double ca = byx ? cen[a].x : cen[a].y, cb = byx ? cen[b].x : cen[b].y;
    return ca < cb || (ca == cb && a < b);
  });
  int kl = k / 2;
  int n = hi - lo;
  int nl = (int)((long long)n * kl / k);
  rcb_rec(cen, ids, lo, lo + nl, kl, first, part);
  rcb_rec(cen, ids, lo + nl, hi, k - kl, first + kl, part);
}

std::vector<int> rcb(const Mesh& m, int k) {
  auto cen = centroids(m);
  std::vector<int> ids(m.ncells()), part(m.ncells());
  std::iota(ids.begin(), ids.end(), 0);
  rcb_rec(cen, ids, 0, m.ncells(), k, 0, part);
  return part;
}

// face adjacency: for every cell edge (a,b) the neighbouring cell (or -1)
struct EdgeAdj {
  std::vector<int> nb;  // per cvtx slot k (edge cvtx[k] -> cvtx[next]) : neighbour cell or -1
};
EdgeAdj edge_adjacency(const Mesh& m) {
  EdgeAdj e;
  e.nb.assign(m.cvtx.size(), -1);
  std::unordered_map<uint64_t, std::pair<int, int>> mp;  // key -> (cell, slot)
  mp.reserve(m.cvtx.size() * 2);
  for (int c = 0; c < m.ncells(); ++c)
    for (int k = m.cptr[c]; k < m.cptr[c + 1]; ++k) {
      int a = m.cvtx[k], b = m.cvtx[k + 1 < m.cptr[c + 1] ? k + 1 : m.cptr[c]];
      uint64_t key = (uint64_t)std::min(a, b) << 32 | (uint64_t)std::max(a, b);
      auto it = mp.find(key);
      if (it == mp.end()) mp[key] = {c, k};
      else { e.nb[k] = it->second.first; e.nb[it->second.second] = c; }
    }
  return e;
}

// reassign non-largest connected components of each part to the adjacent part sharing most faces
void fix_connectivity(const Mesh& m, std::vector<int>& part, int nparts) {
  EdgeAdj ea = edge_adjacency(m);
  for (int pass = 0; pass < 4; ++pass) {
    std::vector<int> comp(m.ncells(), -1);
    std::vector<std::vector<int>> comps;
    for (int c = 0; c < m.ncells(); ++c) {
      if (comp[c] >= 0) continue;
      int id = (int)comps.size();
      comps.push_back({});
      std::vector<int> st = {c};
      comp[c] = id;
      while (!st.empty()) {
        int u = st.back(); st.pop_back();
        comps[id].push_back(u);
        for (int k = m.cptr[u]; k < m.cptr[u + 1]; ++k) {
          int v = ea.nb[k];
          if (v >= 0 && comp[v] < 0 && part[v] == part[u]) { comp[v] = id; st.push_back(v); }
        }
      }
    }
    std::vector<int> best(nparts, -1);
    for (int id = 0; id < (int)comps.size(); ++id) {
      int p = part[comps[id][0]];
      if (best[p] < 0 || comps[id].size() > comps[best[p]].size()) best[p] = id;
    }
    bool changed = false;
    for (int id = 0; id < (int)comps.size(); ++id) {
      int p = part[comps[id][0]];
      if (best[p] == id) continue;
      std::map<int, int> cnt;
      for (int u : comps[id])
        for (int k = m.cptr[u]; k < m.cptr[u + 1]; ++k) {
          int v = ea.nb[k];
          if (v >= 0 && part[v] != p) cnt[part[v]]++;
        }
      if (cnt.empty()) continue;
      int tgt = -1, bc = -1;
      for (auto& kv : cnt) if (kv.second > bc) { bc = kv.second; tgt = kv.first; }
      for (int u : comps[id]) part[u] = tgt;
      changed = true;
    }
    if (!changed) break;
  }
}

// ------------------------------------------------------------------ merged-edge coarse polygons
bool seg_intersect_proper(P2 a, P2 b, P2 c, P2 d) {
  auto orient = [](P2 p, P2 q, P2 r) { return (q.x - p.x) * (r.y - p.y) - (q.y - p.y) * (r.x - p.x); };
  double o1 = orient(a, b, c), o2 = orient(a, b, d), o3 = orient(c, d, a), o4 = orient(c, d, b);
  const double eps = 1e-15;
  return ((o1 > eps && o2 < -eps) || (o1 < -eps && o2 > eps)) && ((o3 > eps && o4 < -eps) || (o3 < -eps && o4 > eps));
}
bool poly_simple(const Poly& p) {
  int n = (int)p.size();
  if (n < 3) return false;
  for (int i = 0; i < n; ++i)
    for (int j = i + 2; j < n; ++j) {
      if (i == 0 && j == n - 1) continue;
      if (seg_intersect_proper(p[i], p[(i + 1) % n], p[j], p[(j + 1) % n])) return false;
    }
  // repeated vertices are also non-simple
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      if (p[i].x == p[j].x && p[i].y == p[j].y) return false;
  return poly_area(p) > 0;
}

struct CoarseOut {
  std::vector<Poly> polys;
};

// Sutherland–Hodgman: subject (possibly non-convex, CCW) clipped by convex CCW window.
Poly clip_convex(const Poly& subject, const Poly& win) {
  Poly out = subject;
  int n = (int)win.size();
  for (int i = 0; i < n && !out.empty(); ++i) {
    P2 a = win[i], b = win[(i + 1) % n];
    // inside = left of a->b : cross(b-a, x-a) >= 0  <=>  (x - a) . d <= 0 with d = outward normal (dy, -dx)
    P2 d = {b.y - a.y, -(b.x - a.x)};
    out = clip_halfplane(out, a, d);
  }
  return out;
}

struct Overlaps {
  std::vector<int> fine, coarse, ptr;
  std::vector<double> xy;
};

// overlap pieces kappa ∩ D_J for every fine cell; returns false with bad cells listed if coverage fails
bool compute_overlaps(const Mesh& m, const std::vector<Poly>& cp, Overlaps& ov, std::vector<int>& bad_coarse) {
  int NC = (int)cp.size();
  std::vector<double> bb(4 * NC);
  const int G = std::max(1, (int)std::sqrt((double)NC));
  std::vector<std::vector<int>> grid(G * G);
  auto gi = [&](double v) { return std::min(G - 1, std::max(0, (int)(v * G))); };
  for (int J = 0; J < NC; ++J) {
    double x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300;
    for (auto& v : cp[J]) { x0 = std::min(x0, v.x); x1 = std::max(x1, v.x); y0 = std::min(y0, v.y); y1 = std::max(y1, v.y); }
    bb[4 * J] = x0; bb[4 * J + 1] = x1; bb[4 * J + 2] = y0; bb[4 * J + 3] = y1;
    for (int yy = gi(y0); yy <= gi(y1); ++yy)
      for (int xx = gi(x0); xx <= gi(x1); ++xx) grid[yy * G + xx].push_back(J);
  }
  ov.fine.clear(); ov.coarse.clear(); ov.ptr.assign(1, 0); ov.xy.clear();
  std::set<int> bad;
  for (int c = 0; c < m.ncells(); ++c) {
    Poly k = m.poly(c);
    double kx0 = 1e300, kx1 = -1e300, ky0 = 1e300, ky1 = -1e300;
    for (auto& v : k) { kx0 = std::min(kx0, v.x); kx1 = std::max(kx1, v.x); ky0 = std::min(ky0, v.y); ky1 = std::max(ky1, v.y); }
    std::set<int> cand;
    for (int yy = gi(ky0); yy <= gi(ky1); ++yy)
      for (int xx = gi(kx0); xx <= gi(kx1); ++xx)
        for (int J : grid[yy * G + xx])
          if (bb[4 * J] <= kx1 && bb[4 * J + 1] >= kx0 && bb[4 * J + 2] <= ky1 && bb[4 * J + 3] >= ky0) cand.insert(J);
    double ak = poly_area(k), sum = 0;
    std::vector<int> here;
    for (int J : cand) {
      Poly piece = clip_convex(cp[J], k);
      if (piece.size() < 3) continue;
      double a = poly_area(piece);
      if (a <= 1e-12 * ak) continue;
      sum += a;
      here.push_back(J);
      ov.fine.push_back(c); ov.coarse.push_back(J);
      for (auto& v : piece) { ov.xy.push_back(v.x); ov.xy.push_back(v.y); }
      ov.ptr.push_back((int)ov.xy.size() / 2);
    }
    if (std::fabs(sum - ak) > 1e-10 * ak) for (int J : cand) bad.insert(J);
  }
  bad_coarse.assign(bad.begin(), bad.end());
  return bad.empty();
}

// Build merged-edge ("coarsened edge") coarse polygons from an agglomeration (R17).
bool merged_edge_coarse(const Mesh& m, const std::vector<int>& part, int NC, std::vector<Poly>& out, Overlaps& ov,
                        std::string& err) {
  EdgeAdj ea = edge_adjacency(m);
  int NV = (int)m.xy.size() / 2;
  // parts incident to every vertex (-1 = outside)
  std::vector<std::set<int>> vparts(NV);
  for (int c = 0; c < m.ncells(); ++c)
    for (int k = m.cptr[c]; k < m.cptr[c + 1]; ++k) {
      int a = m.cvtx[k];
      vparts[a].insert(part[c]);
      if (ea.nb[k] < 0) {
        int b = m.cvtx[k + 1 < m.cptr[c + 1] ? k + 1 : m.cptr[c]];
        vparts[a].insert(-1); vparts[b].insert(-1);
      }
    }
  auto is_corner = [&](int v) {
    double x = m.xy[2 * v], y = m.xy[2 * v + 1];
    return (x == 0 || x == 1) && (y == 0 || y == 1);
  };
  // boundary loop of every part: directed edges a->b with the part on the left
  std::vector<std::vector<int>> loop(NC), loopnb(NC);
  {
    std::vector<std::unordered_map<int, std::pair<int, int>>> nxt(NC);  // a -> (b, neighbour part)
    for (int c = 0; c < m.ncells(); ++c)
      for (int k = m.cptr[c]; k < m.cptr[c + 1]; ++k) {
        int nbc = ea.nb[k];
        int pn = nbc < 0 ? -1 : part[nbc];
        if (pn == part[c]) continue;
        int a = m.cvtx[k], b = m.cvtx[k + 1 < m.cptr[c + 1] ? k + 1 : m.cptr[c]];
        if (nxt[part[c]].count(a)) { err = "pinched agglomerate boundary"; return false; }
        nxt[part[c]][a] = {b, pn};
      }
    for (int J = 0; J < NC; ++J) {
      if (nxt[J].empty()) { err = "empty agglomerate"; return false; }
      int start = nxt[J].begin()->first;
      // deterministic start: smallest vertex id
      for (auto& kv : nxt[J]) start = std::min(start, kv.first);
      int a = start;
      size_t guard = 0;
      do {
        auto it = nxt[J].find(a);
        if (it == nxt[J].end()) { err = "open agglomerate boundary"; return false; }
        loop[J].push_back(a); loopnb[J].push_back(it->second.second);
        a = it->second.first;
        if (++guard > nxt[J].size()) { err = "boundary walk failed"; return false; }
      } while (a != start);
      if (loop[J].size() != nxt[J].size()) { err = "agglomerate with several boundary loops"; return false; }
    }
  }
  // keep-vertex flags: junctions (>=3 parts incl. outside) and corners; plus DP refinements
  std::vector<char> keep(NV, 0);
  for (int v = 0; v < NV; ++v) if (vparts[v].size() >= 3 || is_corner(v)) keep[v] = 1;
  for (int iter = 0; iter < 64; ++iter) {
    out.assign(NC, {});
    std::vector<int> badJ;
    for (int J = 0; J < NC; ++J) {
      const auto& L = loop[J];
      int n = (int)L.size();
      int first = -1;
      for (int i = 0; i < n; ++i) if (keep[L[i]]) { first = i; break; }
      if (first < 0) {  // island interface: keep everything
        for (int i = 0; i < n; ++i) out[J].push_back(m.v(L[i]));
        continue;
      }
      for (int t = 0; t < n; ++t) {
        int v = L[(first + t) % n];
        if (keep[v]) out[J].push_back(m.v(v));
      }
      if (!poly_simple(out[J])) badJ.push_back(J);
    }
    if (badJ.empty()) {
      std::vector<int> badc;
      if (compute_overlaps(m, out, ov, badc)) return true;
      badJ = badc;
    }
    // Douglas–Peucker step on every interface of the bad polygons: keep the farthest vertex
    bool changed = false;
    for (int J : badJ) {
      const auto& L = loop[J];
      int n = (int)L.size();
      std::vector<int> ks;
      for (int i = 0; i < n; ++i) if (keep[L[i]]) ks.push_back(i);
      if (ks.empty()) continue;
      for (size_t s = 0; s < ks.size(); ++s) {
        int i0 = ks[s], i1 = ks[(s + 1) % ks.size()];
        if (ks.size() == 1) i1 = i0 + n;
        if (i1 <= i0) i1 += n;
        if (i1 - i0 < 2) continue;
        P2 a = m.v(L[i0 % n]), b = m.v(L[i1 % n]);
        double best = -1; int bi = -1;
        for (int i = i0 + 1; i < i1; ++i) {
          P2 p = m.v(L[i % n]);
          double dx = b.x - a.x, dy = b.y - a.y, ll = std::hypot(dx, dy);
          double d = ll > 0 ? std::fabs((p.x - a.x) * dy - (p.y - a.y) * dx) / ll : std::hypot(p.x - a.x, p.y - a.y);
          if (d > best) { best = d; bi = i; }
        }
        if (bi >= 0 && !keep[L[bi % n]]) { keep[L[bi % n]] = 1; changed = true; }
      }
    }
    if (!changed) { err = "merged-edge coarsening could not be repaired"; return false; }
  }
  err = "merged-edge coarsening did not converge";
  return false;
}

struct Problem {
  Mesh mesh;
  std::vector<int> part;
  int nsub = 0, ncoarse = 0, nested = 1;
  std::vector<int> parent;
  Overlaps ov;
  std::vector<int> cpoly_ptr;
  std::vector<double> cpoly_xy;
  std::vector<double> kappa;
  std::string err;
};

std::vector<int> cart_tiles(int n, int t) {
  std::vector<int> p(n * n);
  int nt = n / t;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) p[j * n + i] = (j / t) * nt + (i / t);
  return p;
}

}  // namespace

extern "C" {

// kind: 0 = Cartesian n x n, 1 = Voronoi with n cells, 2 = L-shape Voronoi of n_coarse cells refined n
//       times, 3 = L-shape Voronoi with n cells
// sub_mode: 0 = Cartesian tiles of sub_tile^2 cells, 1 = RCB into n_sub parts, 2 = one cell per subdomain
// coarse_mode: 0 = coarse = subdomains (nested), 1 = RCB into n_coarse (nested), 2 = Cartesian tiles
//              of coarse_tile^2 (nested), 3 = RCB into n_coarse + merged edges (non-nested),
//              4 = independent Voronoi mesh of n_coarse cells (non-nested, paper Ex.4),
//              5 = the refinement parent of kind 2 (nested)
// kappa_mode: 0 = 1 everywhere, 1 = 10^U(-4,4) per subdomain (stream seeded with seed ^ 0x6b617070)
void* dgas_gen_problem(int kind, int n, uint64_t seed, int lloyd, int sub_mode, int sub_tile, int n_sub,
                       int coarse_mode, int coarse_tile, int n_coarse, int kappa_mode) {
  Problem* P = new Problem();
  Mesh& m = P->mesh;
  std::vector<int> refine_parent;
  if (kind == 0) make_cartesian(n, m);
  else if (kind == 1) { if (!make_voronoi(n, seed, lloyd, m, P->err)) return P; }
  else if (kind == 2) {
    // L-shape: Voronoi mesh of n_coarse cells refined n times (Ex.1, first variant); parent = refinement
    Mesh cur;
    if (!make_voronoi_L(n_coarse, seed, lloyd, cur, P->err)) return P;
    refine_parent.resize(cur.ncells());
    std::iota(refine_parent.begin(), refine_parent.end(), 0);
    P->ncoarse = cur.ncells();
    for (int l = 0; l < n; ++l) {
      Mesh nx;
      std::vector<int> par;
      refine_once(cur, nx, par, P->err);
      if (!P->err.empty()) return P;
      for (int& v : par) v = refine_parent[v];
      refine_parent = par;
      cur = nx;
    }
    m = cur;
  } else if (kind == 3) { if (!make_voronoi_L(n, seed, lloyd, m, P->err)) return P; }
  else { P->err = "unknown mesh kind"; return P; }
  int NC = m.ncells();
  if (sub_mode == 0) { P->part = cart_tiles(n, sub_tile); P->nsub = (n / sub_tile) * (n / sub_tile); }
  else if (sub_mode == 2) { P->part.resize(NC); std::iota(P->part.begin(), P->part.end(), 0); P->nsub = NC; }
  else { P->part = rcb(m, n_sub); P->nsub = n_sub; }
  P->nested = 1;
  if (coarse_mode == 0) { P->parent = P->part; P->ncoarse = P->nsub; }
  else if (coarse_mode == 1) { P->parent = rcb(m, n_coarse); P->ncoarse = n_coarse; }
  else if (coarse_mode == 5) {
    if (kind != 2) { P->err = "coarse_mode 5 needs kind 2 (refinement hierarchy)"; return P; }
    P->parent = refine_parent;
  }
  else if (coarse_mode == 2) { P->parent = cart_tiles(n, coarse_tile); P->ncoarse = (n / coarse_tile) * (n / coarse_tile); }
  else if (coarse_mode == 4) {
    // independent Voronoi coarse mesh (Ex.4 "independently generated"): seeds from the
    // stream seed ^ 0x636f61727365, same Lloyd count; pieces kappa ∩ D_J by convex clipping
    Mesh cm;
    if (!make_voronoi(n_coarse, seed ^ 0x636f61727365ULL, lloyd, cm, P->err)) return P;
    std::vector<Poly> cp(cm.ncells());
    for (int J = 0; J < cm.ncells(); ++J) cp[J] = cm.poly(J);
    std::vector<int> bad;
    if (!compute_overlaps(m, cp, P->ov, bad)) { P->err = "independent coarse mesh: overlap coverage failed"; return P; }
    P->nested = 0; P->ncoarse = cm.ncells();
    P->cpoly_ptr.assign(1, 0);
    for (auto& poly : cp) {
      for (auto& v : poly) { P->cpoly_xy.push_back(v.x); P->cpoly_xy.push_back(v.y); }
      P->cpoly_ptr.push_back((int)P->cpoly_xy.size() / 2);
    }
  } else {
    std::vector<int> agg = rcb(m, n_coarse);
    fix_connectivity(m, agg, n_coarse);
    std::vector<Poly> cp;
    if (!merged_edge_coarse(m, agg, n_coarse, cp, P->ov, P->err)) return P;
    P->nested = 0; P->ncoarse = n_coarse;
    P->cpoly_ptr.assign(1, 0);
    for (auto& poly : cp) {
      for (auto& v : poly) { P->cpoly_xy.push_back(v.x); P->cpoly_xy.push_back(v.y); }
      P->cpoly_ptr.push_back((int)P->cpoly_xy.size() / 2);
    }
  }
  P->kappa.assign(NC, 1.0);
  if (kappa_mode == 1) {
    Rng r2(seed ^ 0x6b617070ULL);
    std::vector<double> ks(P->nsub);
    for (int i = 0; i < P->nsub; ++i) ks[i] = std::pow(10.0, 8.0 * r2.uniform() - 4.0);
    for (int c = 0; c < NC; ++c) P->kappa[c] = ks[P->part[c]];
  }
  return P;
}

const char* dgas_gen_error(void* h) { return ((Problem*)h)->err.empty() ? nullptr : ((Problem*)h)->err.c_str(); }

// sizes: [n_vertices, n_cells, n_cell_vtx, n_sub, n_coarse, nested, n_ov, n_ov_xy_points, n_cpoly_points]
void dgas_gen_sizes(void* h, int64_t* s) {
  Problem* P = (Problem*)h;
  s[0] = (int64_t)P->mesh.xy.size() / 2; s[1] = P->mesh.ncells(); s[2] = (int64_t)P->mesh.cvtx.size();
  s[3] = P->nsub; s[4] = P->ncoarse; s[5] = P->nested; s[6] = (int64_t)P->ov.fine.size();
  s[7] = (int64_t)P->ov.xy.size() / 2; s[8] = (int64_t)P->cpoly_xy.size() / 2;
}

void dgas_gen_copy(void* h, double* xy, int* cptr, int* cvtx, int* part, int* parent, double* kappa, int* ov_fine,
                   int* ov_coarse, int* ov_ptr, double* ov_xy, int* cpoly_ptr, double* cpoly_xy) {
  Problem* P = (Problem*)h;
  std::memcpy(xy, P->mesh.xy.data(), P->mesh.xy.size() * 8);
  std::memcpy(cptr, P->mesh.cptr.data(), P->mesh.cptr.size() * 4);
  std::memcpy(cvtx, P->mesh.cvtx.data(), P->mesh.cvtx.size() * 4);
  std::memcpy(part, P->part.data(), P->part.size() * 4);
  std::memcpy(kappa, P->kappa.data(), P->kappa.size() * 8);
  if (P->nested) std::memcpy(parent, P->parent.data(), P->parent.size() * 4);
  else {
    std::memcpy(ov_fine, P->ov.fine.data(), P->ov.fine.size() * 4);
    std::memcpy(ov_coarse, P->ov.coarse.data(), P->ov.coarse.size() * 4);
    std::memcpy(ov_ptr, P->ov.ptr.data(), P->ov.ptr.size() * 4);
    std::memcpy(ov_xy, P->ov.xy.data(), P->ov.xy.size() * 8);
    std::memcpy(cpoly_ptr, P->cpoly_ptr.data(), P->cpoly_ptr.size() * 4);
    std::memcpy(cpoly_xy, P->cpoly_xy.data(), P->cpoly_xy.size() * 8);
  }
}

void dgas_gen_free(void* h) { delete (Problem*)h; }

// Uniform N(0,1)-ish test vectors: counter-based (SplitMix64 of (seed, i)), Box–Muller. Shared by
// both sides for parity inputs; holds no method arithmetic.
void dgas_gen_normal(uint64_t seed, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    uint64_t x = seed * 0x632be59bd9b4e019ULL + (uint64_t)i * 2;
    uint64_t a = Rng::splitmix(x), b = Rng::splitmix(x);
    double u1 = (double(a >> 11) + 0.5) * (1.0 / 9007199254740992.0), u2 = double(b >> 11) * (1.0 / 9007199254740992.0);
    out[i] = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
}

}  // extern "C"
