// oracle/oracle.cpp — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow CPU implementation of what the hot path computes, written from
// arXiv 1903.11357 in fp64 (plus a long-double variant of the preconditioner for the
// sensitivity check of DESIGN.md reading R30). It shares NO code with the CUDA path
// (paper_1903_11357_b200/): its own topology, quadrature (Golub–Welsch Gauss–Legendre), basis,
// assembly, Cholesky, PCG and Lanczos. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it. The product path never calls it.
// Threads: everything is sequential except the loops over independent subdomains (local Cholesky
// factors, local solves), which OpenMP may spread over or_set_threads(n) threads; each subdomain's
// arithmetic is the same plain loop whatever the thread count, so results are bitwise identical.
//
// Citations: P:n = /root/reference/PAPER.md line n (the reference is not present at run time).
//   SIPDG form            P:83-98  (eq:Ah, eq:lifting_R_2, eq:Sigma), harmonic average P:53-59,
//                         jumps/averages P:61-69, assembled in face form P:467-469 (Lemma 5.8 proof).
//   DG space              P:74-77  (eq:Vh), physical-frame P_p(kappa).
//   local solvers         P:129-137 (A_i = A_h(R_i^T u, R_i^T v), R_i^T = extension by zero).
//   coarse space / R0^T   P:140-151 (eq:R0T L2 prolongation, eq:A0 Galerkin).
//   additive operator     P:160-165 (P_ad = sum_i P_i).
//   ASPCG protocol        P:741 (Euclidean relative residual < 1e-8, x0 = 0, Lanczos estimate).
//   DG energy norm        P:240-241 (eq:DGnorm_2).
// Readings where the paper is silent are listed in DESIGN.md (R1..R30).
//
// Parity pins: see tests/test_oracle_*.py (closed forms, worked examples, invariants). Every
// function below is pinned by at least one of them; none is "parity unpinned".
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <type_traits>
#include <utility>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace orc {

// -------------------------------------------------------------- Gauss–Legendre (Golub–Welsch)
// Nodes = eigenvalues of the Jacobi matrix of the Legendre recurrence, weights = 2 v_0^2.
// Eigen-decomposition by cyclic Jacobi rotations (plain, m <= 16).
void gauss_legendre(int m, std::vector<double>& x, std::vector<double>& w) {
  std::vector<double> J(m * m, 0.0), V(m * m, 0.0);
  for (int i = 0; i < m; ++i) V[i * m + i] = 1.0;
  for (int k = 1; k < m; ++k) {
    double b = k / std::sqrt(4.0 * k * k - 1.0);
    J[(k - 1) * m + k] = J[k * m + (k - 1)] = b;
  }
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0;
    for (int i = 0; i < m; ++i)
      for (int j = i + 1; j < m; ++j) off += J[i * m + j] * J[i * m + j];
    if (off < 1e-32) break;
    for (int p = 0; p < m; ++p)
      for (int q = p + 1; q < m; ++q) {
        double apq = J[p * m + q];
        if (std::fabs(apq) < 1e-300) continue;
        double theta = (J[q * m + q] - J[p * m + p]) / (2 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1));
        double c = 1 / std::sqrt(t * t + 1), s = t * c;
        for (int k = 0; k < m; ++k) {
          double akp = J[k * m + p], akq = J[k * m + q];
          J[k * m + p] = c * akp - s * akq;
          J[k * m + q] = s * akp + c * akq;
        }
        for (int k = 0; k < m; ++k) {
          double apk = J[p * m + k], aqk = J[q * m + k];
          J[p * m + k] = c * apk - s * aqk;
          J[q * m + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < m; ++k) {
          double vkp = V[k * m + p], vkq = V[k * m + q];
          V[k * m + p] = c * vkp - s * vkq;
          V[k * m + q] = s * vkp + c * vkq;
        }
      }
  }
  std::vector<std::pair<double, double>> nw(m);
  for (int i = 0; i < m; ++i) nw[i] = {J[i * m + i], 2.0 * V[0 * m + i] * V[0 * m + i]};
  std::sort(nw.begin(), nw.end());
  x.resize(m); w.resize(m);
  for (int i = 0; i < m; ++i) { x[i] = nw[i].first; w[i] = nw[i].second; }
}

struct QP { double x, y, w; };

// Collapsed (Duffy) Gauss–Legendre rule on the reference triangle {u,v >= 0, u+v <= 1}:
// u = (1+s)/2, v = (1-u)(1+t)/2, Jacobian (1-u)/4; exact for total degree <= 2m-2.
void ref_triangle_rule(int m, std::vector<QP>& r) {
  std::vector<double> x, w;
  gauss_legendre(m, x, w);
  r.clear();
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      double u = 0.5 * (1 + x[i]);
      double v = (1 - u) * 0.5 * (1 + x[j]);
      r.push_back({u, v, w[i] * w[j] * (1 - u) * 0.25});
    }
}

// physical rule on triangle (a, b, c) with SIGNED Jacobian 2*area (signed fans are exact)
void triangle_rule(const double* a, const double* b, const double* c, const std::vector<QP>& ref, std::vector<QP>& out) {
  double jx1 = b[0] - a[0], jy1 = b[1] - a[1], jx2 = c[0] - a[0], jy2 = c[1] - a[1];
  double det = jx1 * jy2 - jx2 * jy1;
  for (const QP& q : ref) out.push_back({a[0] + q.x * jx1 + q.y * jx2, a[1] + q.x * jy1 + q.y * jy2, q.w * det});
}

// -------------------------------------------------------------- polygons
struct Polygon { std::vector<double> v; int n() const { return (int)v.size() / 2; } };

double area(const Polygon& P) {
  double a = 0;
  for (int i = 0; i < P.n(); ++i) {
    int j = (i + 1) % P.n();
    a += P.v[2 * i] * P.v[2 * j + 1] - P.v[2 * j] * P.v[2 * i + 1];
  }
  return 0.5 * a;
}

// centroid-fan rule (cells: convex, "each cell sub-triangulated from its centroid", B:8)
void cell_rule(const Polygon& P, int m, std::vector<QP>& out) {
  std::vector<QP> ref;
  ref_triangle_rule(m, ref);
  double cx = 0, cy = 0;
  for (int i = 0; i < P.n(); ++i) { cx += P.v[2 * i]; cy += P.v[2 * i + 1]; }
  double c[2] = {cx / P.n(), cy / P.n()};
  out.clear();
  for (int i = 0; i < P.n(); ++i) {
    int j = (i + 1) % P.n();
    triangle_rule(c, &P.v[2 * i], &P.v[2 * j], ref, out);
  }
}

// signed fan from vertex 0 (overlap pieces kappa ∩ D_J, possibly non-convex)
void piece_rule(const Polygon& P, int m, std::vector<QP>& out) {
  std::vector<QP> ref;
  ref_triangle_rule(m, ref);
  out.clear();
  for (int i = 1; i + 1 < P.n(); ++i) triangle_rule(&P.v[0], &P.v[2 * i], &P.v[2 * i + 2], ref, out);
}

// -------------------------------------------------------------- basis (R6)
// Legendre polynomials and derivatives by the three-term recurrences.
void legendre(int p, double t, double* L, double* dL) {
  L[0] = 1; dL[0] = 0;
  if (p >= 1) { L[1] = t; dL[1] = 1; }
  for (int n = 1; n < p; ++n) {
    L[n + 1] = ((2 * n + 1) * t * L[n] - n * L[n - 1]) / (n + 1);
    dL[n + 1] = dL[n - 1] + (2 * n + 1) * L[n];
  }
}

struct Basis {
  int p = 0, np = 0;
  double x0 = 0, x1 = 1, y0 = 0, y1 = 1;
  std::vector<double> C;  // np x np : phi_a = sum_b C[a][b] g_b
  // g_i = L_a(xi) L_b(eta), graded: degree d = 0..p, a = d..0, b = d - a
  void raw(double x, double y, double* g, double* gx, double* gy) const {
    double La[16], dLa[16], Lb[16], dLb[16];
    double sx = 2.0 / (x1 - x0), sy = 2.0 / (y1 - y0);
    legendre(p, (x - x0) * sx - 1, La, dLa);
    legendre(p, (y - y0) * sy - 1, Lb, dLb);
    int i = 0;
    for (int d = 0; d <= p; ++d)
      for (int a = d; a >= 0; --a, ++i) {
        int b = d - a;
        g[i] = La[a] * Lb[b];
        if (gx) { gx[i] = dLa[a] * sx * Lb[b]; gy[i] = La[a] * dLb[b] * sy; }
      }
  }
  void eval(double x, double y, double* phi, double* px, double* py) const {
    double g[64], gx[64], gy[64];
    raw(x, y, g, px ? gx : nullptr, py ? gy : nullptr);
    for (int a = 0; a < np; ++a) {
      double s = 0, sx = 0, sy = 0;
      for (int b = 0; b < np; ++b) {
        s += C[a * np + b] * g[b];
        if (px) { sx += C[a * np + b] * gx[b]; sy += C[a * np + b] * gy[b]; }
      }
      phi[a] = s;
      if (px) { px[a] = sx; py[a] = sy; }
    }
  }
};

// plain Cholesky M = L L^T (row-major, lower), returns false if a pivot <= 0
template <typename T>
bool cholesky(int n, std::vector<T>& M) {
  for (int j = 0; j < n; ++j) {
    T s = M[j * n + j];
    for (int k = 0; k < j; ++k) s -= M[j * n + k] * M[j * n + k];
    if (!(s > 0)) return false;
    T d = std::sqrt(s);
    M[j * n + j] = d;
    for (int i = j + 1; i < n; ++i) {
      T t = M[i * n + j];
      for (int k = 0; k < j; ++k) t -= M[i * n + k] * M[j * n + k];
      M[i * n + j] = t / d;
    }
    for (int k = j + 1; k < n; ++k) M[j * n + k] = 0;
  }
  return true;
}
// inverse of lower-triangular L (row-major)
std::vector<double> tri_inverse(int n, const std::vector<double>& L) {
  std::vector<double> X(n * n, 0.0);
  for (int c = 0; c < n; ++c)
    for (int i = c; i < n; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = c; k < i; ++k) s -= L[i * n + k] * X[k * n + c];
      X[i * n + c] = s / L[i * n + i];
    }
  return X;
}

// orthonormalise the raw basis over a region given by its quadrature rule: CholQR applied twice
bool orthonormalise(Basis& B, const std::vector<QP>& rule) {
  int n = B.np;
  B.C.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i) B.C[i * n + i] = 1.0;
  for (int pass = 0; pass < 2; ++pass) {
    std::vector<double> M(n * n, 0.0), phi(n);
    for (const QP& q : rule) {
      B.eval(q.x, q.y, phi.data(), nullptr, nullptr);
      for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) M[a * n + b] += q.w * phi[a] * phi[b];
    }
    if (!cholesky(n, M)) return false;
    std::vector<double> Li = tri_inverse(n, M), C2(n * n, 0.0);
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b) {
        double s = 0;
        for (int k = 0; k < n; ++k) s += Li[a * n + k] * B.C[k * n + b];
        C2[a * n + b] = s;
      }
    B.C = C2;
  }
  return true;
}

// -------------------------------------------------------------- problem
struct Face { int kp, km; double ax, ay, bx, by, nx, ny, len; };  // km = -1 on the boundary

template <typename T>
struct Factors {
  std::vector<std::vector<T>> Lloc;  // per subdomain (dense lower Cholesky), empty if not factored
  std::vector<T> L0;                 // coarse: dense lower (N0 <= dense_max) or band storage
  int band = -1;                     // -1: dense; else half bandwidth
};

struct Ctx {
  int nc = 0, p = 1, q = 1, np = 3, nq = 3, nsub = 0, ncoarse = 0;
  double Cs = 10.0;
  std::vector<Polygon> cell;
  std::vector<double> kappa, hk;
  std::vector<int> part;
  std::vector<Face> faces;
  std::vector<Basis> basis;
  // A as per-row map: neighbour cell -> np x np block
  std::vector<std::map<int, std::vector<double>>> A;
  // subdomains
  std::vector<std::vector<int>> sub_cells;
  // coarse
  std::vector<Basis> cbasis;
  std::vector<int> ov_fine, ov_coarse;
  std::vector<Polygon> ov_poly;
  std::vector<std::vector<double>> G;             // per overlap np x nq
  std::vector<std::vector<int>> ov_of_cell;
  std::vector<double> A0;                          // dense (N0 small) — or empty
  std::vector<double> A0band;                      // band (lower) storage N0 x (band+1)
  int band = -1;
  Factors<double> F;
  Factors<long double> FL;
  bool use_coarse = true, use_local = true, have_schwarz = false;
  int refine = 0;  // iterative-refinement steps of the band coarse solve (R30)
  double perturb = 0;  // relative last-bit perturbation of G (sensitivity measurement, R30)
  uint64_t perturb_seed = 1;
  int status = 0;
  char msg[256] = {0};
};

static int fail(Ctx* c, int code, const char* m) {
  c->status = code;
  std::snprintf(c->msg, sizeof c->msg, "%s", m);
  return code;
}

// harmonic average <eta>
static double harm(double a, double b) { return 2 * a * b / (a + b); }


}  // namespace orc

using namespace orc;

extern "C" {

const char* or_message(void* h) { return ((Ctx*)h)->msg; }
int or_status(void* h) { return ((Ctx*)h)->status; }

// Build topology, geometry and the per-cell orthonormal basis; assemble A (face form) — P:83-98,467.
void* or_create(int nv, const double* xy, int nc, const int* cptr, const int* cvtx, const int* part, int nsub,
                const double* kappa, int p, double Cs) {
  Ctx* c = new Ctx();
  c->nc = nc; c->p = p; c->np = (p + 1) * (p + 2) / 2; c->Cs = Cs; c->nsub = nsub;
  c->cell.resize(nc); c->kappa.assign(kappa, kappa + nc); c->part.assign(part, part + nc);
  c->hk.resize(nc);
  for (int i = 0; i < nc; ++i) {
    for (int k = cptr[i]; k < cptr[i + 1]; ++k) { c->cell[i].v.push_back(xy[2 * cvtx[k]]); c->cell[i].v.push_back(xy[2 * cvtx[k] + 1]); }
    // h_kappa = diameter = max vertex-pair distance (R1)
    double h = 0;
    const Polygon& P = c->cell[i];
    for (int a = 0; a < P.n(); ++a)
      for (int b = a + 1; b < P.n(); ++b) h = std::max(h, std::hypot(P.v[2 * a] - P.v[2 * b], P.v[2 * a + 1] - P.v[2 * b + 1]));
    c->hk[i] = h;
    if (!(kappa[i] > 0) || !std::isfinite(kappa[i])) { fail(c, -1, "kappa must be positive and finite"); return c; }
    if (area(P) <= 0) { fail(c, -2, "non-CCW or zero-area cell"); return c; }
  }
  (void)nv;
  // faces
  std::map<std::pair<int, int>, std::vector<std::pair<int, int>>> edges;
  for (int i = 0; i < nc; ++i) {
    int n = cptr[i + 1] - cptr[i];
    for (int k = 0; k < n; ++k) {
      int a = cvtx[cptr[i] + k], b = cvtx[cptr[i] + (k + 1) % n];
      edges[{std::min(a, b), std::max(a, b)}].push_back({i, k});
    }
  }
  for (auto& e : edges) {
    if (e.second.size() > 2) { fail(c, -2, "non-manifold edge"); return c; }
    int kp = e.second[0].first, km = e.second.size() == 2 ? e.second[1].first : -1;
    int kl = e.second[0].second;
    if (km >= 0 && km < kp) { std::swap(kp, km); kl = e.second[1].second; }
    const Polygon& P = c->cell[kp];
    int n = P.n();
    double ax = P.v[2 * kl], ay = P.v[2 * kl + 1], bx = P.v[2 * ((kl + 1) % n)], by = P.v[2 * ((kl + 1) % n) + 1];
    double len = std::hypot(bx - ax, by - ay);
    // CCW loop: outward normal of the edge a->b is (dy, -dx)/len
    c->faces.push_back({kp, km, ax, ay, bx, by, (by - ay) / len, -(bx - ax) / len, len});
  }
  // basis (R6): bbox-scaled Legendre products, orthonormalised over the cell (CholQR2)
  c->basis.resize(nc);
  for (int i = 0; i < nc; ++i) {
    Basis& B = c->basis[i];
    const Polygon& P = c->cell[i];
    B.p = p; B.np = c->np;
    B.x0 = B.y0 = 1e300; B.x1 = B.y1 = -1e300;
    for (int k = 0; k < P.n(); ++k) {
      B.x0 = std::min(B.x0, P.v[2 * k]); B.x1 = std::max(B.x1, P.v[2 * k]);
      B.y0 = std::min(B.y0, P.v[2 * k + 1]); B.y1 = std::max(B.y1, P.v[2 * k + 1]);
    }
    std::vector<QP> rule;
    cell_rule(P, p + 1, rule);
    if (!orthonormalise(B, rule)) { fail(c, -2, "basis Gram not SPD"); return c; }
  }
  // assembly (face form of eq:Ah, P:83-98 with P:467-469)
  int np = c->np;
  c->A.assign(nc, {});
  auto blk = [&](int i, int j) -> std::vector<double>& {
    auto& m = c->A[i];
    auto it = m.find(j);
    if (it == m.end()) it = m.emplace(j, std::vector<double>(np * np, 0.0)).first;
    return it->second;
  };
  std::vector<double> phi(np), px(np), py(np), phi2(np), px2(np), py2(np);
  for (int i = 0; i < nc; ++i) {  // volume: int rho grad u . grad v
    std::vector<QP> rule;
    cell_rule(c->cell[i], p + 1, rule);
    auto& Ab = blk(i, i);
    for (const QP& qp : rule) {
      c->basis[i].eval(qp.x, qp.y, phi.data(), px.data(), py.data());
      for (int a = 0; a < np; ++a)
        for (int b = 0; b < np; ++b) Ab[a * np + b] += c->kappa[i] * qp.w * (px[a] * px[b] + py[a] * py[b]);
    }
  }
  std::vector<double> gx, gw;
  gauss_legendre(p + 1, gx, gw);
  double p2 = (double)p * p;
  for (const Face& F : c->faces) {
    if (F.km < 0) {
      // boundary: <rho> = rho_k, <h> = h_k, {tau}_w = tau_k, [v] = v n
      int k = F.kp;
      double sigma = Cs * c->kappa[k] * p2 / c->hk[k];  // eq:Sigma
      auto& Ab = blk(k, k);
      for (int g = 0; g < (int)gx.size(); ++g) {
        double t = 0.5 * (1 + gx[g]), w = 0.5 * gw[g] * F.len;
        double x = F.ax + t * (F.bx - F.ax), y = F.ay + t * (F.by - F.ay);
        c->basis[k].eval(x, y, phi.data(), px.data(), py.data());
        for (int a = 0; a < np; ++a)
          for (int b = 0; b < np; ++b) {
            double dna = px[a] * F.nx + py[a] * F.ny, dnb = px[b] * F.nx + py[b] * F.ny;
            Ab[a * np + b] += w * (sigma * phi[a] * phi[b] - c->kappa[k] * (dnb * phi[a] + dna * phi[b]));
          }
      }
    } else {
      int kp = F.kp, km = F.km;
      double rp = c->kappa[kp], rm = c->kappa[km];
      double rho_h = harm(rp, rm), h_h = harm(c->hk[kp], c->hk[km]);
      double sigma = Cs * rho_h * p2 / h_h;  // eq:Sigma
      // omega = rho-/(rho+ + rho-) => omega rho+ = (1-omega) rho- = <rho>/2
      double wp = rm / (rp + rm) * rp, wm = (1 - rm / (rp + rm)) * rm;
      int side[2] = {kp, km};
      double eps[2] = {1.0, -1.0}, wgt[2] = {wp, wm};
      for (int g = 0; g < (int)gx.size(); ++g) {
        double t = 0.5 * (1 + gx[g]), w = 0.5 * gw[g] * F.len;
        double x = F.ax + t * (F.bx - F.ax), y = F.ay + t * (F.by - F.ay);
        c->basis[kp].eval(x, y, phi.data(), px.data(), py.data());
        c->basis[km].eval(x, y, phi2.data(), px2.data(), py2.data());
        const double* V[2] = {phi.data(), phi2.data()};
        const double* GX[2] = {px.data(), px2.data()};
        const double* GY[2] = {py.data(), py2.data()};
        for (int s = 0; s < 2; ++s)        // test side
          for (int tt = 0; tt < 2; ++tt) { // trial side
            auto& Ab = blk(side[s], side[tt]);
            for (int a = 0; a < np; ++a)
              for (int b = 0; b < np; ++b) {
                double va = V[s][a], ub = V[tt][b];
                double dnu = GX[tt][b] * F.nx + GY[tt][b] * F.ny;  // n from + to -
                double dnv = GX[s][a] * F.nx + GY[s][a] * F.ny;
                // sigma [u].[v] - {rho grad u}_w . [v] - {rho grad v}_w . [u]
                Ab[a * np + b] += w * (sigma * eps[s] * eps[tt] * ub * va - wgt[tt] * dnu * eps[s] * va -
                                       wgt[s] * dnv * eps[tt] * ub);
              }
          }
      }
    }
  }
  // subdomain cell lists (cells in increasing caller order)
  c->sub_cells.assign(nsub, {});
  for (int i = 0; i < nc; ++i) {
    if (part[i] < 0 || part[i] >= nsub) { fail(c, -1, "partition out of range"); return c; }
    c->sub_cells[part[i]].push_back(i);
  }
  for (int s = 0; s < nsub; ++s)
    if (c->sub_cells[s].empty()) { fail(c, -1, "empty subdomain"); return c; }
  return c;
}

void or_free(void* h) { delete (Ctx*)h; }

int or_sizes(void* h, int64_t* out) {
  Ctx* c = (Ctx*)h;
  int64_t nnzb = 0;
  for (auto& m : c->A) nnzb += (int64_t)m.size();
  out[0] = c->nc; out[1] = c->np; out[2] = (int64_t)c->faces.size(); out[3] = nnzb; out[4] = c->nq; out[5] = c->ncoarse;
  return c->status;
}

// basis coefficients (np x np) of a cell and its bbox
void or_basis(void* h, int cell, double* C, double* bbox) {
  Ctx* c = (Ctx*)h;
  const Basis& B = c->basis[cell];
  std::memcpy(C, B.C.data(), sizeof(double) * B.np * B.np);
  bbox[0] = B.x0; bbox[1] = B.x1; bbox[2] = B.y0; bbox[3] = B.y1;
}

// evaluate basis of `cell` at points
void or_eval_basis(void* h, int cell, int npts, const double* pts, double* phi, double* px, double* py) {
  Ctx* c = (Ctx*)h;
  int np = c->np;
  for (int k = 0; k < npts; ++k) c->basis[cell].eval(pts[2 * k], pts[2 * k + 1], phi + k * np, px + k * np, py + k * np);
}

// the A block (i, j) (zeros if not coupled); returns 1 if the block exists
int or_block(void* h, int i, int j, double* out) {
  Ctx* c = (Ctx*)h;
  auto it = c->A[i].find(j);
  if (it == c->A[i].end()) { std::memset(out, 0, sizeof(double) * c->np * c->np); return 0; }
  std::memcpy(out, it->second.data(), sizeof(double) * c->np * c->np);
  return 1;
}

// dense A (only for small N)
void or_dense_A(void* h, double* out) {
  Ctx* c = (Ctx*)h;
  int np = c->np;
  int64_t N = (int64_t)c->nc * np;
  std::memset(out, 0, sizeof(double) * N * N);
  for (int i = 0; i < c->nc; ++i)
    for (auto& kv : c->A[i])
      for (int a = 0; a < np; ++a)
        for (int b = 0; b < np; ++b) out[((int64_t)i * np + a) * N + (int64_t)kv.first * np + b] = kv.second[a * np + b];
}

// y = A x  (caller order)
void or_spmv(void* h, const double* x, double* y) {
  Ctx* c = (Ctx*)h;
  int np = c->np;
  for (int i = 0; i < c->nc; ++i)
    for (int a = 0; a < np; ++a) {
      double s = 0;
      for (auto& kv : c->A[i])
        for (int b = 0; b < np; ++b) s += kv.second[a * np + b] * x[(int64_t)kv.first * np + b];
      y[(int64_t)i * np + a] = s;
    }
}

// y = |A| |x| (entrywise absolute values): the scale of the rounding error of any y = A x, used by the
// parity tests to bound the SpMV difference (|fl(Ax) - Ax| <= gamma_n |A||x|)
void or_spmv_abs(void* h, const double* x, double* y) {
  Ctx* c = (Ctx*)h;
  int np = c->np;
  for (int i = 0; i < c->nc; ++i)
    for (int a = 0; a < np; ++a) {
      double s = 0;
      for (auto& kv : c->A[i])
        for (int b = 0; b < np; ++b) s += std::fabs(kv.second[a * np + b] * x[(int64_t)kv.first * np + b]);
      y[(int64_t)i * np + a] = s;
    }
}

// right-hand side b_a = int_kappa f phi_a  (eq:dG); f_kind: 0 = 2pi^2 sin sin, 1 = 1, 2 = 2[x(1-x)+y(1-y)]
// fixed Duffy rule with m = p + 4 (R10)
void or_rhs(void* h, int f_kind, double* b) {
  Ctx* c = (Ctx*)h;
  int np = c->np;
  std::vector<double> phi(np);
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < c->nc; ++i) {
    std::vector<QP> rule;
    cell_rule(c->cell[i], c->p + 4, rule);
    for (int a = 0; a < np; ++a) b[(int64_t)i * np + a] = 0;
    for (const QP& qp : rule) {
      double f = f_kind == 0 ? 2 * pi * pi * std::sin(pi * qp.x) * std::sin(pi * qp.y)
                 : f_kind == 1 ? 1.0 : 2 * (qp.x * (1 - qp.x) + qp.y * (1 - qp.y));
      c->basis[i].eval(qp.x, qp.y, phi.data(), nullptr, nullptr);
      for (int a = 0; a < np; ++a) b[(int64_t)i * np + a] += qp.w * f * phi[a];
    }
  }
}

// L2 projection coefficients of u (u_kind: 0 = sin(pi x) sin(pi y), 1 = x(1-x)y(1-y)); orthonormal basis => c_a = int u phi_a
void or_project(void* h, int u_kind, double* out) {
  Ctx* c = (Ctx*)h;
  int np = c->np;
  std::vector<double> phi(np);
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < c->nc; ++i) {
    std::vector<QP> rule;
    cell_rule(c->cell[i], c->p + 4, rule);
    for (int a = 0; a < np; ++a) out[(int64_t)i * np + a] = 0;
    for (const QP& qp : rule) {
      double u = u_kind == 0 ? std::sin(pi * qp.x) * std::sin(pi * qp.y) : qp.x * (1 - qp.x) * qp.y * (1 - qp.y);
      c->basis[i].eval(qp.x, qp.y, phi.data(), nullptr, nullptr);
      for (int a = 0; a < np; ++a) out[(int64_t)i * np + a] += qp.w * u * phi[a];
    }
  }
}

// errors of a DG function x against u = sin(pi x) sin(pi y): [L2 error, DG-norm error] (eq:DGnorm_2)
// ||w||_DG^2 = sum_k int rho |grad w|^2 + sum_F int sigma |[w]|^2, with w = u_h - u (u continuous, zero on bdry)
void or_errors(void* h, const double* x, double* out) {
  Ctx* c = (Ctx*)h;
  int np = c->np, p = c->p;
  const double pi = 3.14159265358979323846;
  std::vector<double> phi(np), px(np), py(np);
  double l2 = 0, dg = 0;
  for (int i = 0; i < c->nc; ++i) {
    std::vector<QP> rule;
    cell_rule(c->cell[i], p + 4, rule);
    for (const QP& qp : rule) {
      c->basis[i].eval(qp.x, qp.y, phi.data(), px.data(), py.data());
      double uh = 0, ux = 0, uy = 0;
      for (int a = 0; a < np; ++a) { uh += x[(int64_t)i * np + a] * phi[a]; ux += x[(int64_t)i * np + a] * px[a]; uy += x[(int64_t)i * np + a] * py[a]; }
      double u = std::sin(pi * qp.x) * std::sin(pi * qp.y);
      double gx = pi * std::cos(pi * qp.x) * std::sin(pi * qp.y), gy = pi * std::sin(pi * qp.x) * std::cos(pi * qp.y);
      l2 += qp.w * (uh - u) * (uh - u);
      dg += qp.w * c->kappa[i] * ((ux - gx) * (ux - gx) + (uy - gy) * (uy - gy));
    }
  }
  std::vector<double> gxs, gws;
  gauss_legendre(p + 4, gxs, gws);
  double p2 = (double)p * p;
  std::vector<double> phi2(np);
  for (const Face& F : c->faces) {
    double sigma = F.km < 0 ? c->Cs * c->kappa[F.kp] * p2 / c->hk[F.kp]
                            : c->Cs * harm(c->kappa[F.kp], c->kappa[F.km]) * p2 / harm(c->hk[F.kp], c->hk[F.km]);
    for (int g = 0; g < (int)gxs.size(); ++g) {
      double t = 0.5 * (1 + gxs[g]), w = 0.5 * gws[g] * F.len;
      double X = F.ax + t * (F.bx - F.ax), Y = F.ay + t * (F.by - F.ay);
      c->basis[F.kp].eval(X, Y, phi.data(), nullptr, nullptr);
      double up = 0, um = 0;
      for (int a = 0; a < np; ++a) up += x[(int64_t)F.kp * np + a] * phi[a];
      if (F.km >= 0) {
        c->basis[F.km].eval(X, Y, phi2.data(), nullptr, nullptr);
        for (int a = 0; a < np; ++a) um += x[(int64_t)F.km * np + a] * phi2[a];
      }
      dg += w * sigma * (up - um) * (up - um);  // the exact u has no jump and vanishes on the boundary
    }
  }
  out[0] = std::sqrt(l2); out[1] = std::sqrt(dg);
}

// ---------------------------------------------------------------- Schwarz preconditioner
// coarse description: overlap pieces (fine cell, coarse element, polygon). For nested problems the
// pieces are the fine cells themselves (Remark 3.2).
// sample: if n_sample >= 0, only the listed subdomains get local factors (sampled full-size parity).
int or_setup_schwarz(void* h, int ncoarse, int q, int n_ov, const int* ov_fine, const int* ov_coarse,
                     const int* ov_ptr, const double* ov_xy, int use_coarse, int use_local, int n_sample,
                     const int* sample, int long_double_too, int dense_max) {
  Ctx* c = (Ctx*)h;
  if (c->status) return c->status;
  if (q < 1 || q > c->p) return fail(c, -1, "need 1 <= q <= p (P:140)");
  c->q = q; c->nq = (q + 1) * (q + 2) / 2; c->ncoarse = ncoarse;
  c->use_coarse = use_coarse; c->use_local = use_local;
  int np = c->np, nq = c->nq;
  // --- local Cholesky factors of A_i = principal submatrices
  c->F.Lloc.assign(c->nsub, {});
  c->FL.Lloc.assign(c->nsub, {});
  std::vector<char> want(c->nsub, n_sample < 0 ? 1 : 0);
  for (int k = 0; k < n_sample; ++k) want[sample[k]] = 1;
  // subdomains are independent: factored in parallel (OpenMP, one subdomain per thread; the
  // arithmetic of each factor is the same plain loop whatever the thread count)
  int bad_sub = -1, bad_ld = 0;
  if (use_local) {
#pragma omp parallel for schedule(dynamic)
    for (int s = 0; s < c->nsub; ++s) {
      if (!want[s]) continue;
      const auto& cells = c->sub_cells[s];
      int m = (int)cells.size(), n = m * np;
      std::map<int, int> loc;
      for (int k = 0; k < m; ++k) loc[cells[k]] = k;
      std::vector<double> M((size_t)n * n, 0.0);
      for (int k = 0; k < m; ++k)
        for (auto& kv : c->A[cells[k]]) {
          auto it = loc.find(kv.first);
          if (it == loc.end()) continue;
          for (int a = 0; a < np; ++a)
            for (int b = 0; b < np; ++b) M[(size_t)(k * np + a) * n + it->second * np + b] = kv.second[a * np + b];
        }
      if (long_double_too) {
        std::vector<long double> ML(M.begin(), M.end());
        if (!cholesky(n, ML)) {
#pragma omp critical
          { bad_ld = 1; bad_sub = s; }
        }
        c->FL.Lloc[s] = std::move(ML);
      }
      if (!cholesky(n, M)) {
#pragma omp critical
        { if (bad_sub < 0 || s < bad_sub) bad_sub = s; }
      }
      c->F.Lloc[s] = std::move(M);
    }
  }
  if (bad_sub >= 0) {
    if (bad_ld) return fail(c, -3, "local block not SPD (long double)");
    char b[64]; std::snprintf(b, 64, "local %d not SPD", bad_sub); return fail(c, -3, b);
  }
  if (!use_coarse) { c->have_schwarz = true; return 0; }
  // --- coarse basis psi_J: bbox-Legendre products of degree q orthonormalised over D_J (R8)
  c->ov_fine.assign(ov_fine, ov_fine + n_ov);
  c->ov_coarse.assign(ov_coarse, ov_coarse + n_ov);
  c->ov_poly.assign(n_ov, {});
  c->ov_of_cell.assign(c->nc, {});
  c->cbasis.assign(ncoarse, {});
  for (int J = 0; J < ncoarse; ++J) {
    Basis& B = c->cbasis[J];
    B.p = q; B.np = nq; B.x0 = B.y0 = 1e300; B.x1 = B.y1 = -1e300;
  }
  for (int o = 0; o < n_ov; ++o) {
    for (int k = ov_ptr[o]; k < ov_ptr[o + 1]; ++k) {
      c->ov_poly[o].v.push_back(ov_xy[2 * k]); c->ov_poly[o].v.push_back(ov_xy[2 * k + 1]);
      Basis& B = c->cbasis[ov_coarse[o]];
      B.x0 = std::min(B.x0, ov_xy[2 * k]); B.x1 = std::max(B.x1, ov_xy[2 * k]);
      B.y0 = std::min(B.y0, ov_xy[2 * k + 1]); B.y1 = std::max(B.y1, ov_xy[2 * k + 1]);
    }
    c->ov_of_cell[ov_fine[o]].push_back(o);
  }
  {
    std::vector<std::vector<QP>> rules(ncoarse);
    for (int o = 0; o < n_ov; ++o) {
      std::vector<QP> r;
      piece_rule(c->ov_poly[o], q + 1, r);
      auto& R = rules[ov_coarse[o]];
      R.insert(R.end(), r.begin(), r.end());
    }
    for (int J = 0; J < ncoarse; ++J)
      if (!orthonormalise(c->cbasis[J], rules[J])) return fail(c, -2, "coarse basis Gram not SPD");
  }
  // --- G = int_{kappa ∩ D_J} phi psi (eq:R0T); Q = M_h^{-1} G = G (orthonormal phi)
  c->G.assign(n_ov, std::vector<double>(np * nq, 0.0));
  {
    int m = (c->p + q + 1) / 2 + 1;
    std::vector<double> phi(np), psi(nq);
    for (int o = 0; o < n_ov; ++o) {
      std::vector<QP> r;
      piece_rule(c->ov_poly[o], m, r);
      for (const QP& qp : r) {
        c->basis[ov_fine[o]].eval(qp.x, qp.y, phi.data(), nullptr, nullptr);
        c->cbasis[ov_coarse[o]].eval(qp.x, qp.y, psi.data(), nullptr, nullptr);
        for (int a = 0; a < np; ++a)
          for (int b = 0; b < nq; ++b) c->G[o][a * nq + b] += qp.w * phi[a] * psi[b];
      }
    }
  }
  if (c->perturb != 0) {  // sensitivity probe: G *= (1 + perturb * u), u uniform in [-1, 1]
    uint64_t x = c->perturb_seed;
    for (auto& g : c->G)
      for (auto& v : g) {
        x = x * 6364136223846793005ULL + 1442695040888963407ULL;
        double u = (double)(x >> 11) * (1.0 / 9007199254740992.0) * 2 - 1;
        v *= 1 + c->perturb * u;
      }
  }
  // --- A0 = Q^T A Q (eq:A0)
  int64_t N0 = (int64_t)ncoarse * nq;
  int bw = 0;
  for (int i = 0; i < c->nc; ++i)
    for (auto& kv : c->A[i])
      for (int o1 : c->ov_of_cell[i])
        for (int o2 : c->ov_of_cell[kv.first]) {
          int d = std::abs(c->ov_coarse[o1] - c->ov_coarse[o2]);
          bw = std::max(bw, (d + 1) * nq - 1);
        }
  bool dense = N0 <= dense_max;
  c->band = dense ? -1 : bw;
  int64_t ld = dense ? N0 : (int64_t)bw + 1;
  std::vector<double> A0(N0 * ld, 0.0);
  // dense: A0[I][Jc]; band (lower): row I, column Jc <= I stored at A0[I*ld + (Jc - I + bw)]
  auto at = [&](int64_t I, int64_t Jc) -> double* {
    if (dense) return &A0[I * N0 + Jc];
    if (Jc > I || I - Jc > bw) return nullptr;
    return &A0[I * ld + (Jc - I + bw)];
  };
  std::vector<double> T(np * nq);
  for (int i = 0; i < c->nc; ++i)
    for (auto& kv : c->A[i]) {
      int j = kv.first;
      const auto& Ab = kv.second;
      for (int o2 : c->ov_of_cell[j]) {
        // T = A_ij G_o2  (np x nq)
        for (int a = 0; a < np; ++a)
          for (int b = 0; b < nq; ++b) {
            double s = 0;
            for (int k = 0; k < np; ++k) s += Ab[a * np + k] * c->G[o2][k * nq + b];
            T[a * nq + b] = s;
          }
        for (int o1 : c->ov_of_cell[i]) {
          int J1 = c->ov_coarse[o1], J2 = c->ov_coarse[o2];
          for (int a = 0; a < nq; ++a)
            for (int b = 0; b < nq; ++b) {
              double* d = at((int64_t)J1 * nq + a, (int64_t)J2 * nq + b);
              if (!d) continue;
              double s = 0;
              for (int k = 0; k < np; ++k) s += c->G[o1][k * nq + a] * T[k * nq + b];
              *d += s;
            }
        }
      }
    }
  if (dense) {
    c->A0 = A0;
    if (long_double_too) {
      std::vector<long double> L(A0.begin(), A0.end());
      if (!cholesky((int)N0, L)) return fail(c, -3, "coarse not SPD (long double)");
      c->FL.L0 = std::move(L);
    }
    if (!cholesky((int)N0, A0)) return fail(c, -3, "coarse not SPD");
    c->F.L0 = std::move(A0);
    c->F.band = -1;
  } else {
    // plain band Cholesky (lower band, half bandwidth bw)
    c->A0band = A0;
    for (int64_t j = 0; j < N0; ++j) {
      double s = A0[j * ld + bw];
      for (int64_t k = std::max<int64_t>(0, j - bw); k < j; ++k) { double v = A0[j * ld + (k - j + bw)]; s -= v * v; }
      if (!(s > 0)) return fail(c, -3, "coarse not SPD");
      double d = std::sqrt(s);
      A0[j * ld + bw] = d;
      for (int64_t i = j + 1; i <= std::min(N0 - 1, j + bw); ++i) {
        double t = A0[i * ld + (j - i + bw)];
        for (int64_t k = std::max<int64_t>(0, i - bw); k < j; ++k) t -= A0[i * ld + (k - i + bw)] * A0[j * ld + (k - j + bw)];
        A0[i * ld + (j - i + bw)] = t / d;
      }
    }
    c->F.L0 = std::move(A0);
    c->F.band = bw;
  }
  c->have_schwarz = true;
  return 0;
}

}  // extern "C"

namespace orc {
// solve L L^T x = b in place (dense lower)
template <typename T>
void chol_solve(int n, const std::vector<T>& L, std::vector<T>& x) {
  for (int i = 0; i < n; ++i) {
    T s = x[i];
    for (int k = 0; k < i; ++k) s -= L[(size_t)i * n + k] * x[k];
    x[i] = s / L[(size_t)i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    T s = x[i];
    for (int k = i + 1; k < n; ++k) s -= L[(size_t)k * n + i] * x[k];
    x[i] = s / L[(size_t)i * n + i];
  }
}
void band_solve(int64_t n, int bw, const std::vector<double>& L, std::vector<double>& x) {
  int64_t ld = bw + 1;
  for (int64_t i = 0; i < n; ++i) {
    double s = x[i];
    for (int64_t k = std::max<int64_t>(0, i - bw); k < i; ++k) s -= L[i * ld + (k - i + bw)] * x[k];
    x[i] = s / L[i * ld + bw];
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = x[i];
    for (int64_t k = i + 1; k <= std::min(n - 1, i + bw); ++k) s -= L[k * ld + (i - k + bw)] * x[k];
    x[i] = s / L[i * ld + bw];
  }
}

// z = Q A0^{-1} Q^T r + sum_i E_i A_i^{-1} E_i^T r  (P:160-165 in matrix form; R0 = Q^T, R8)
template <typename T>
int apply_t(Ctx* c, const Factors<T>& F, const double* r, double* z, const std::vector<char>* only) {
  int np = c->np, nq = c->nq;
  int64_t N = (int64_t)c->nc * np;
  std::vector<T> zz(N, T(0));
  if (c->use_local) {
    for (int s = 0; s < c->nsub; ++s)
      if (!(only && !(*only)[s]) && F.Lloc[s].empty()) return -1;
    // independent subdomain solves (disjoint cells): parallel over subdomains, same arithmetic
#pragma omp parallel for schedule(dynamic)
    for (int s = 0; s < c->nsub; ++s) {
      if (only && !(*only)[s]) continue;
      const auto& cells = c->sub_cells[s];
      int n = (int)cells.size() * np;
      std::vector<T> x(n);
      for (int k = 0; k < (int)cells.size(); ++k)
        for (int a = 0; a < np; ++a) x[k * np + a] = r[(int64_t)cells[k] * np + a];
      chol_solve(n, F.Lloc[s], x);
      for (int k = 0; k < (int)cells.size(); ++k)
        for (int a = 0; a < np; ++a) zz[(int64_t)cells[k] * np + a] += x[k * np + a];
    }
  }
  if (c->use_coarse) {
    int64_t N0 = (int64_t)c->ncoarse * nq;
    std::vector<T> r0(N0, T(0));
    for (size_t o = 0; o < c->G.size(); ++o)  // r0 = Q^T r
      for (int b = 0; b < nq; ++b) {
        T s = 0;
        for (int a = 0; a < np; ++a) s += (T)c->G[o][a * nq + b] * (T)r[(int64_t)c->ov_fine[o] * np + a];
        r0[(int64_t)c->ov_coarse[o] * nq + b] += s;
      }
    if (c->F.band < 0) chol_solve((int)N0, F.L0, r0);
    else {
      // band path (N0 > dense_max): the fp64 band factor, plus c->refine refinement steps with a
      // long-double residual (R30). The long-double apply (T = long double) uses the same
      // refined fp64 band solve for its coarse part (no long-double band factor is kept).
      const int bw = c->F.band;
      const int64_t ld = bw + 1;
      std::vector<double> b0(r0.begin(), r0.end()), x0(b0);
      band_solve(N0, bw, c->F.L0, x0);
      for (int it = 0; it < c->refine; ++it) {
        std::vector<double> res(N0);
        for (int64_t i = 0; i < N0; ++i) {
          long double s = b0[i];
          for (int64_t j = std::max<int64_t>(0, i - bw); j <= std::min<int64_t>(N0 - 1, i + bw); ++j) {
            double a = j <= i ? c->A0band[i * ld + (j - i + bw)] : c->A0band[j * ld + (i - j + bw)];
            s -= (long double)a * x0[j];
          }
          res[i] = (double)s;
        }
        band_solve(N0, bw, c->F.L0, res);
        for (int64_t i = 0; i < N0; ++i) x0[i] += res[i];
      }
      for (int64_t i = 0; i < N0; ++i) r0[i] = (T)x0[i];
    }
    for (size_t o = 0; o < c->G.size(); ++o) {  // z += Q z0
      int f = c->ov_fine[o];
      if (only && !(*only)[c->part[f]]) continue;
      for (int a = 0; a < np; ++a) {
        T s = 0;
        for (int b = 0; b < nq; ++b) s += (T)c->G[o][a * nq + b] * r0[(int64_t)c->ov_coarse[o] * nq + b];
        zz[(int64_t)f * np + a] += s;
      }
    }
  }
  for (int64_t i = 0; i < N; ++i) z[i] = (double)zz[i];
  return 0;
}
}  // namespace orc

extern "C" {

int or_apply(void* h, const double* r, double* z) { return apply_t(((Ctx*)h), ((Ctx*)h)->F, r, z, nullptr); }
int or_apply_ld(void* h, const double* r, double* z) { return apply_t(((Ctx*)h), ((Ctx*)h)->FL, r, z, nullptr); }
// apply restricted to the dofs of the listed subdomains (others left 0): sampled full-size parity
void or_set_refine(void* h, int steps) { ((Ctx*)h)->refine = steps; }
void or_set_perturb(void* h, double eps, uint64_t seed) { ((Ctx*)h)->perturb = eps; ((Ctx*)h)->perturb_seed = seed; }
// Sensitivity probe (R22/R30): A <- A (1 + eps u), u uniform in [-1, 1] from a hash of the unordered entry,
// so A stays symmetric. Models two correct assemblies of A that differ by ~kappa(Gram) eps (the basis is a
// CholQR2 of a Gram matrix). Call before setup_schwarz; the SpMV and every factor then use the result.
void or_perturb_A(void* h, double eps, uint64_t seed) {
  Ctx* c = (Ctx*)h;
  const int np = c->np;
  for (int i = 0; i < c->nc; ++i)
    for (auto& kv : c->A[i]) {
      const int j = kv.first;
      for (int a = 0; a < np; ++a)
        for (int b = 0; b < np; ++b) {
          uint64_t k0 = (uint64_t)std::min(i, j), k1 = (uint64_t)std::max(i, j);
          int aa = i < j ? a : i > j ? b : std::min(a, b), bb = i < j ? b : i > j ? a : std::max(a, b);
          uint64_t z = seed * 0x9e3779b97f4a7c15ULL ^ (k0 * 1000003ULL + k1) * 0xbf58476d1ce4e5b9ULL ^
                       (uint64_t)(aa * 64 + bb) * 0x94d049bb133111ebULL;
          z ^= z >> 31; z *= 0xbf58476d1ce4e5b9ULL; z ^= z >> 27; z *= 0x94d049bb133111ebULL; z ^= z >> 31;
          const double u = (double)(z >> 11) * (1.0 / 9007199254740992.0) * 2 - 1;
          kv.second[a * np + b] *= 1 + eps * u;
        }
    }
}
int or_apply_sampled(void* h, int n_sample, const int* sample, const double* r, double* z) {
  Ctx* c = (Ctx*)h;
  std::vector<char> only(c->nsub, 0);
  for (int k = 0; k < n_sample; ++k) only[sample[k]] = 1;
  return apply_t(c, c->F, r, z, &only);
}
// the same in long double (setup_schwarz with long_double_too; Z30 / DESIGN.md R30 reference)
int or_apply_sampled_ld(void* h, int n_sample, const int* sample, const double* r, double* z) {
  Ctx* c = (Ctx*)h;
  std::vector<char> only(c->nsub, 0);
  for (int k = 0; k < n_sample; ++k) only[sample[k]] = 1;
  return apply_t(c, c->FL, r, z, &only);
}

// G blocks (n_ov x np x nq) and dense A0 (N0 x N0, only if dense) for diagnostics
void or_get_G(void* h, double* out) {
  Ctx* c = (Ctx*)h;
  for (size_t o = 0; o < c->G.size(); ++o) std::memcpy(out + o * c->np * c->nq, c->G[o].data(), sizeof(double) * c->np * c->nq);
}
int or_get_A0(void* h, double* out) {
  Ctx* c = (Ctx*)h;
  if (c->A0.empty()) return -1;
  std::memcpy(out, c->A0.data(), sizeof(double) * c->A0.size());
  return 0;
}
void or_coarse_basis(void* h, int J, double* C, double* bbox) {
  Ctx* c = (Ctx*)h;
  const Basis& B = c->cbasis[J];
  std::memcpy(C, B.C.data(), sizeof(double) * B.np * B.np);
  bbox[0] = B.x0; bbox[1] = B.x1; bbox[2] = B.y0; bbox[3] = B.y1;
}

// ---------------------------------------------------------------- PCG (R11, R12)
// Hestenes–Stiefel PCG from x0 (normally 0): stop when ||r_k||_2 <= rtol ||b||_2 (checked after the
// x/r update, before the preconditioner). alpha/beta recorded for the Lanczos estimate.
// returns 0 converged, 1 not converged, -4 breakdown. precond: 1 = Schwarz, 0 = identity.
// or_pcg_ext: the same iteration, plus (for stored reference outputs) the iterate x restricted to the
// dofs idx[0..n_idx) after every iteration j, kept in a ring hist[(j % n_hist) * n_idx + t], and
// `extra` further iterations after the stop test fires (stop test skipped, *iters = the stopping
// iteration, *iters_run = iterations actually performed). or_pcg = or_pcg_ext with no history.
int or_pcg_ext(void* h, const double* b, double* x, double rtol, int maxit, int precond, int* iters, double* alphas,
               double* betas, double* resid, int n_idx, const int64_t* idx, int n_hist, double* hist, int extra,
               int* iters_run);
int or_pcg(void* h, const double* b, double* x, double rtol, int maxit, int precond, int* iters, double* alphas,
           double* betas, double* resid) {
  int run = 0;
  return or_pcg_ext(h, b, x, rtol, maxit, precond, iters, alphas, betas, resid, 0, nullptr, 0, nullptr, 0, &run);
}
int or_pcg_ext(void* h, const double* b, double* x, double rtol, int maxit, int precond, int* iters, double* alphas,
               double* betas, double* resid, int n_idx, const int64_t* idx, int n_hist, double* hist, int extra,
               int* iters_run) {
  Ctx* c = (Ctx*)h;
  *iters_run = 0;
  auto record = [&](int j) {
    if (n_hist > 0)
      for (int t = 0; t < n_idx; ++t) hist[(int64_t)(j % n_hist) * n_idx + t] = x[idx[t]];
  };
  int64_t N = (int64_t)c->nc * c->np;
  std::vector<double> r(N), z(N), p(N), q(N);
  or_spmv(h, x, q.data());
  double bb = 0;
  for (int64_t i = 0; i < N; ++i) { r[i] = b[i] - q[i]; bb += b[i] * b[i]; }
  double bnorm = std::sqrt(bb);
  *iters = 0;
  double rr0 = 0;
  for (int64_t i = 0; i < N; ++i) rr0 += r[i] * r[i];
  if (std::sqrt(rr0) <= rtol * bnorm) return 0;
  auto prec = [&](const std::vector<double>& in, std::vector<double>& out) {
    if (precond) return or_apply(h, in.data(), out.data());
    out = in;
    return 0;
  };
  if (prec(r, z)) return -1;
  double gamma = 0;
  for (int64_t i = 0; i < N; ++i) { p[i] = z[i]; gamma += r[i] * z[i]; }
  if (!(gamma > 0) || !std::isfinite(gamma)) return -4;
  int stop = -1;  // iteration at which the stop test fired (history mode continues `extra` more)
  for (int k = 0; k < maxit + extra; ++k) {
    if (stop < 0 && k >= maxit) break;
    if (stop >= 0 && k >= stop + extra) break;
    or_spmv(h, p.data(), q.data());
    double pq = 0;
    for (int64_t i = 0; i < N; ++i) pq += p[i] * q[i];
    if (!(pq > 0) || !std::isfinite(pq)) return -4;
    double alpha = gamma / pq;
    alphas[k] = alpha;
    double rr = 0;
    for (int64_t i = 0; i < N; ++i) { x[i] += alpha * p[i]; r[i] -= alpha * q[i]; rr += r[i] * r[i]; }
    if (resid) resid[k] = std::sqrt(rr) / bnorm;
    *iters_run = k + 1;
    record(k + 1);
    if (stop < 0) *iters = k + 1;
    if (stop < 0 && std::sqrt(rr) <= rtol * bnorm) {
      stop = k + 1;
      if (extra == 0) return 0;
    }
    if (prec(r, z)) return -1;
    double gnew = 0;
    for (int64_t i = 0; i < N; ++i) gnew += r[i] * z[i];
    if (!(gnew > 0) || !std::isfinite(gnew)) return -4;
    double beta = gnew / gamma;
    betas[k] = beta;
    gamma = gnew;
    for (int64_t i = 0; i < N; ++i) p[i] = z[i] + beta * p[i];
  }
  return stop >= 0 ? 0 : 1;
}

void or_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n);
#else
  (void)n;
#endif
}
int or_get_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

// Lanczos tridiagonal from the CG coefficients (R12):
// T_00 = 1/a_0, T_jj = 1/a_j + b_{j-1}/a_{j-1}, T_{j,j+1} = sqrt(b_j)/a_j ; extreme eigenvalues by
// Sturm-sequence bisection (Gershgorin bracket).
static int sturm_count(int m, const std::vector<double>& d, const std::vector<double>& e, double x) {
  int cnt = 0;
  double qv = d[0] - x;
  if (qv < 0) cnt++;
  for (int i = 1; i < m; ++i) {
    if (qv == 0) qv = 1e-300;
    qv = d[i] - x - e[i - 1] * e[i - 1] / qv;
    if (qv < 0) cnt++;
  }
  return cnt;
}
void or_lanczos(int m, const double* a, const double* b, double* out) {
  std::vector<double> d(m), e(m > 1 ? m - 1 : 1);
  for (int j = 0; j < m; ++j) d[j] = 1.0 / a[j] + (j > 0 ? b[j - 1] / a[j - 1] : 0.0);
  for (int j = 0; j + 1 < m; ++j) e[j] = std::sqrt(b[j]) / a[j];
  double lo = 1e300, hi = -1e300;
  for (int j = 0; j < m; ++j) {
    double r = (j > 0 ? std::fabs(e[j - 1]) : 0) + (j + 1 < m ? std::fabs(e[j]) : 0);
    lo = std::min(lo, d[j] - r); hi = std::max(hi, d[j] + r);
  }
  auto kth = [&](int k) {  // k-th smallest eigenvalue (0-based)
    double l = lo, u = hi;
    for (int it = 0; it < 200 && u - l > 1e-15 * std::max(std::fabs(l), std::fabs(u)); ++it) {
      double mid = 0.5 * (l + u);
      if (sturm_count(m, d, e, mid) > k) u = mid; else l = mid;
    }
    return 0.5 * (l + u);
  };
  out[0] = kth(0); out[1] = kth(m - 1); out[2] = out[1] / out[0];
}

// Triangle quadrature export (for the quadrature pins)
int or_triangle_rule(int m, double* out) {
  std::vector<QP> r;
  ref_triangle_rule(m, r);
  for (size_t i = 0; i < r.size(); ++i) { out[3 * i] = r[i].x; out[3 * i + 1] = r[i].y; out[3 * i + 2] = r[i].w; }
  return (int)r.size();
}
void or_gauss_legendre(int m, double* x, double* w) {
  std::vector<double> xs, ws;
  gauss_legendre(m, xs, ws);
  for (int i = 0; i < m; ++i) { x[i] = xs[i]; w[i] = ws[i]; }
}
// integrate x^a y^b over a polygon with the centroid-fan (convex) or signed vertex-0 fan rule
double or_poly_monomial(int n, const double* xy, int a, int b, int m, int fan) {
  Polygon P;
  P.v.assign(xy, xy + 2 * n);
  std::vector<QP> r;
  if (fan == 0) cell_rule(P, m, r); else piece_rule(P, m, r);
  double s = 0;
  for (auto& qp : r) s += qp.w * std::pow(qp.x, a) * std::pow(qp.y, b);
  return s;
}

}  // extern "C"
