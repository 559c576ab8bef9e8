// internal.h — context layout and device helpers of libdgas (B200 / sm_100a).
//
// Internal numbering: cells are renumbered subdomain-major (so R_i is a contiguous range,
// PAPER.md:129-137) and, inside a subdomain, in the face-graph ordering with the smallest block
// envelope among reverse Cuthill–McKee and several Sloan orderings (setup_host.cu), so the local
// Cholesky factors stay inside a narrow block envelope (DESIGN.md §5 "Local factors").
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/dgas.h"

#define DGAS_MAXP 6
#define DGAS_MAXNP 28
#define CT 32            // coarse tile size (tiled dense / banded Cholesky of A0)

// ---------------------------------------------------------------- PCG device state
struct PcgState {
  int it;          // completed iterations
  int done;        // 1 = stop (converged, breakdown or maxit)
  int status;      // DGAS_OK / DGAS_NOT_CONVERGED / DGAS_E_BREAKDOWN
  int maxit;
  double rtol2_bb; // rtol^2 ||b||^2
  double bb;       // ||b||^2
  double gamma;    // r.z of the current iterate
  double pq, alpha, beta, rr;
  unsigned int cnt[4];  // last-block counters of the reductions
};

// One deterministic two-stage reduction: per-CTA partials, the last CTA to arrive sums them in order.
struct Reduce {
  double* partials;   // [max CTAs]
  int cap;
};

// Nested-dissection plan of the coarse solve (nd_host.cu / nd_kernels.cu)
struct NdPlan {
  int nf = 0, nlev = 0, maxF = 0, maxU = 0, maxN = 0;
  int64_t bytes = 0;
  std::vector<int> h_lev_ptr, h_lev_fronts, h_nF, h_nU, h_offT, h_offu, h_offFe, h_offUe, h_Fe, h_Ue, h_childptr,
      h_childs, h_cmap_ptr, h_cmap, h_asm_ptr, h_wf_ptr, h_wb_ptr;
  std::vector<int64_t> h_offX, h_offM, h_offUpd, h_offS;
  std::vector<int4> h_asm;
  int *d_nF = nullptr, *d_nU = nullptr, *d_offT = nullptr, *d_offu = nullptr, *d_offFe = nullptr, *d_offUe = nullptr;
  int *d_Fe = nullptr, *d_Ue = nullptr, *d_childptr = nullptr, *d_childs = nullptr, *d_cmap_ptr = nullptr, *d_cmap = nullptr;
  int *d_asm_ptr = nullptr, *d_lev_fronts = nullptr;
  int4* d_asm = nullptr;
  int2 *d_wf = nullptr, *d_wb = nullptr;
  int64_t *d_offX = nullptr, *d_offM = nullptr, *d_offUpd = nullptr, *d_offS = nullptr;
  double *d_X = nullptr, *d_M = nullptr, *d_MT = nullptr, *d_T = nullptr, *d_u = nullptr;
  int refine = 0;                      // iterative-refinement steps of the coarse solve (R30; nd_calibrate)
  int refine_env = -1;                 // DGAS_ND_REFINE override (-1: calibrate)
  double calib_err = 0;                // measured relative error of one coarse solve (nd_calibrate)
  double calib_err0 = 0;               // the same without refinement
  std::vector<int> h_prow;             // coarse pair rows (pairs sorted by (J1, J2))
  int* d_prow = nullptr;
  double *d_rb = nullptr, *d_zb = nullptr;
  double* d_dsc = nullptr;             // diag(A0)^-1/2 (symmetric scaling of the fronts)
  // solve v2 (k_nd_fwd2 / k_nd_bwd2): one descriptor per work item, flat gather / child-source tables
  void *d_wf2 = nullptr, *d_wb2 = nullptr;  // NdItem[] per direction
  int *d_gF = nullptr, *d_gU = nullptr;
  int2* d_tsrc = nullptr;
  int v2 = 0, pdl = 0;
};

// Subdomain-sharded multi-GPU solve (shard.cu): this rank's view of the replicated context
struct ShardPlan {
  int active = 0, rank = 0, nranks = 1, cap = 1, nsend_own = 0, send_off = 0;
  std::vector<int> s_begin, c_begin;  // [nranks+1] subdomain / cell ranges (internal numbering)
  int *d_send_ptr = nullptr, *d_send = nullptr;  // border cells of every rank (CSR by rank)
  double* d_partials = nullptr;
  void* d_state = nullptr;
};

struct dgas_ctx_s {
  // sizes
  int p = 0, q = 0, np = 0, nq = 0, nc = 0, nsub = 0, ncoarse = 0, nface = 0, nov = 0;
  int64_t N = 0, N0 = 0;
  double penalty = 10;
  int coarse_dense = 1, coarse_bw = 0, nT = 0, bt = 0;  // coarse tiles
  int spmv_groups = 1;       // independent consumer groups in k_spmv3 (DGAS_SPMV_GROUPS)
  int restrict_cpj = 1;      // CTAs per coarse element in k_restrict (partials in d_rpart, counters d_jcnt)
  double* d_rpart = nullptr;
  unsigned* d_jcnt = nullptr;
  int local_reuse = 0;       // units per subdomain kept in L2 (evict-last) for the backward sweep
  int unroll = 4;            // PCG iterations per WHILE-body execution (DGAS_UNROLL)
  int precond = 0;           // DGAS_PRECOND_*: 0 two-level, 1 one-level, 2 coarse only, 3 none
  int coarse_mode = 0;       // 0 dense explicit inverse, 1 band Cholesky (tile sweeps), 2 nested dissection
  int nd_grid = 1 << 30;     // max CTAs per ND solve level (grid-stride over work items; DGAS_ND_GRID)
  int nd_l2 = 1;             // ND solve operator loads evict-last in L2 (DGAS_ND_L2)
  double nd_tol = 3e-11;     // coarse-solve relative error above which refinement steps are added (Z30; DGAS_ND_TOL)
  // dense coarse path: symmetric diagonal scaling and calibrated refinement (as the ND path, R30)
  int* d_prow = nullptr;     // coarse pair rows (pairs sorted by (J1, J2)), every coarse mode
  double* d_dsc0 = nullptr;  // diag(A0)^-1/2
  double *d_rb0 = nullptr, *d_zb0 = nullptr;  // refinement residual / correction (N0)
  int dense_refine = 0;
  double dense_err = 0, dense_err0 = 0;
  // explicit local inverses Z_i = A_i^-1 (local_inv.cu, local_kernel 3)
  double* d_inv_Z = nullptr;
  int64_t* d_inv_zoff = nullptr;
  int2* d_inv_items = nullptr;
  int inv_nitems = 0, inv_maxn = 0, inv_grid = 0;
  int64_t inv_bytes = 0;
  double inv_err = 0;
  std::vector<int> inv_item_ptr;  // [nsub+1] first work item of each subdomain
  // warp-per-subdomain local solve (local_panel.cu k_local_warp, local_kernel 4)
  int *d_lw_pus = nullptr, *d_lw_units = nullptr;
  unsigned* d_lw_cnt = nullptr;
  int lw_S = 0, lw_cc = 0, lw_warps = 2, lw_grid = 0, lw_keep = 1;
  uint32_t lw_slot = 0;
  size_t lw_smem = 0;
  ShardPlan sh;
  // exact de-duplication of bitwise-identical operator data (dedup.cu; NEXT-4 Cartesian de-duplication)
  int64_t* d_a_dd = nullptr;          // [nc] compact-store offset of each cell's row-block (nullptr: off)
  int dd_grid = 0;                     // persistent CTAs of k_spmv_dd
  int4* d_cls_items = nullptr;         // k_spmv_cls work items (class, first cell, count, W)
  int64_t* d_cls_off = nullptr;        // compact-store offset per row-block class
  int* d_cls_cells = nullptr;          // cells grouped by class
  int* d_cls_nb = nullptr;             // [nc][CLS_MAXDEG] neighbour cells of d_cls_cells[i]
  int cls_nitems = 0, cls_grid = 0, cls_minb = 1, cls_tc = 0;
  int fuse_r = -1;  // residual update fused into the local solve (apply_fuses_restrict), -1 = not decided yet
  std::vector<int64_t> a_dd_h;
  int64_t a_unique = 0, a_bytes_stored = 0;  // distinct row-blocks, bytes of the compact A
  int p_unique = 0;                   // distinct subdomain factors (panel store)
  // multiple-right-hand-side local solve over subdomains sharing a factor (local_mrhs.cu, local_kernel 5)
  int4* d_mr_batches = nullptr;       // (representative subdomain, first member, count, 0) per batch
  int* d_mr_members = nullptr;        // member subdomains, grouped by batch
  int mr_nbatch = 0, mr_B = 0, mr_BS = 1, mr_S = 4, mr_WC = 1, mr_grid = 0, mr_classes = 0;
  int mr_kernel = 1, mr_G = 8, mr_NW = 4, mr_sred = 0;  // 2: k_local_mrhs_w (warp chains: NW warps x G columns)
  uint32_t mr_slot = 0;
  size_t mr_smem = 0;
  int64_t p_bytes_stored = 0;
  NdPlan nd;
  double* d_A0b = nullptr;   // A0 blocks per coarse pair (n_pairs x nq x nq)
  int max_sub_cells = 0, max_urow = 0, max_deg = 0;
  int64_t nnzb = 0, u_total = 0;
  std::string detail;
  cudaStream_t stream = 0;
  // host mirrors needed later
  std::vector<int> perm, iperm;       // perm[new] = old cell, iperm[old] = new
  std::vector<int> nbr_ptr_h, nbr_h;  // internal neighbour lists (sorted, incl. self)
  std::vector<int64_t> a_off_h;       // row-block offsets of A (doubles, 16-byte padded)
  // ---- device: geometry (internal order)
  double* d_xy = nullptr;     // cell vertex coordinates, concatenated [cptr] x 2
  int* d_cptr = nullptr;      // [nc+1]
  double* d_kappa = nullptr;  // [nc]
  double* d_hk = nullptr;     // [nc] diameters
  double* d_C = nullptr;      // [nc][np*np] basis coefficients
  double* d_bbox = nullptr;   // [nc][4]
  double* d_glx = nullptr;    // Gauss–Legendre table, m = 1..16 at offset m(m-1)/2
  double* d_glw = nullptr;
  // faces
  int* d_face_cells = nullptr;    // [nface][2] internal (km = -1 on the boundary)
  double* d_face_xy = nullptr;    // [nface][4] a.x a.y b.x b.y (CCW for kp)
  int* d_cf_ptr = nullptr;        // cell -> faces CSR
  int* d_cf = nullptr;            // face id * 2 + side (0 = +, 1 = -)
  double* d_vol = nullptr;        // [nc][np*np] scratch (volume blocks)
  double* d_fblk = nullptr;       // [nface][4][np*np] scratch (face blocks)
  // A: per-cell row blocks np x (deg*np), row-major
  int* d_nbr_ptr = nullptr;
  int* d_nbr = nullptr;
  int64_t* d_a_off = nullptr;
  double* d_A = nullptr;
  // local envelope factors
  int* d_sub_ptr = nullptr;   // [nsub+1] cell ranges
  int* d_first = nullptr;     // [nc] first coupled local cell f_k (local index)
  int64_t* d_u_off = nullptr; // [nc] row-block offsets (doubles)
  double* d_U = nullptr;      // unit block-lower factor rows U_kj = L_kk^-1 L_kj
  double* d_Dinv = nullptr;   // [nc][np*np] L_kk^-1 (lower)
  // coarse
  int* d_ov_cell = nullptr;       // [nov] internal fine cell of each piece
  int* d_ov_coarse = nullptr;     // [nov]
  int* d_ov_pptr = nullptr;       // [nov+1] piece polygon points
  double* d_ov_xy = nullptr;      // points
  int* d_cov_ptr = nullptr;       // coarse J -> pieces CSR
  int* d_cov = nullptr;
  int* d_fov_ptr = nullptr;       // fine cell -> pieces CSR (first = owner)
  int* d_fov = nullptr;
  int2* d_rrec = nullptr;         // [nov] restriction order (cov): (cell, piece | owner << 31)
  int2* d_prec = nullptr;         // [nov] prolongation order (fov): (piece, coarse element)
  int4* d_crec = nullptr;         // [nc] per cell: (first piece, its coarse element, #pieces, fov index)
  int prolong_grid = 1 << 30;     // persistent CTAs of k_prolong
  // chunked restriction (k_restrict_chunk; DGAS_RESTRICT=1 selects k_restrict)
  int4* d_chunks = nullptr;       // [nchunk] (J, first piece, end piece, chunk index within J)
  int* d_jchunk_ptr = nullptr;    // [ncoarse+1] chunks of J
  double* d_cpart = nullptr;      // [nchunk][nq] chunk partial sums
  unsigned* d_jcnt2 = nullptr;    // [ncoarse] chunk arrival counters
  int nchunk = 0, rc_grid = 0;
  int* d_ctri_ptr = nullptr;      // coarse J -> fan triangles (piece, t)
  int* d_ctri = nullptr;
  double* d_Cc = nullptr;         // [ncoarse][nq*nq]
  double* d_cbbox = nullptr;      // [ncoarse][4]
  double* d_G = nullptr;          // [nov][np*nq]
  // iteration views of G and the piece records (launch_restrict / launch_prolong): the originals, or after
  // exact de-duplication of G (dedup.cu) a compact store with records that index its distinct blocks
  double* d_G_it = nullptr;
  int2* d_rrec_it = nullptr;
  int2* d_prec_it = nullptr;
  int4* d_crec_it = nullptr;
  int64_t g_unique = 0;
  double* d_A0t = nullptr;        // tile storage of A0 / its Cholesky factor
  double* d_Dinv0 = nullptr;      // [nT][CT*CT] inverse diagonal tiles
  double* d_W = nullptr;          // tile storage of L^-1 (dense only, scratch)
  double* d_X = nullptr;          // dense A0^-1, N0 x ldX row-major (dense only)
  int64_t ldX = 0;
  int64_t n_pairs = 0;
  int* d_pair = nullptr;          // coarse pairs (J1, J2)
  int* d_contrib_ptr = nullptr;   // pair -> contributions
  int4* d_contrib = nullptr;      // (cell, slot, o1, o2)
  // vectors (internal order)
  double *d_x = nullptr, *d_r = nullptr, *d_z = nullptr, *d_q = nullptr, *d_b = nullptr;
  double* d_p[2] = {nullptr, nullptr};
  double* d_r2 = nullptr;                    // second residual buffer (ping-pong with d_r)
  double** d_pbuf = nullptr;                 // device array {d_p[0], d_p[1]}
  double** d_rbuf = nullptr;                 // device array {d_r, d_r2}
  int* d_perm_dev = nullptr;                 // perm[new] = old (device)
  cudaStream_t cap_stream = nullptr, cap_stream2 = nullptr;
  cudaStream_t side[3] = {nullptr, nullptr, nullptr};      // fork streams of the coarse solve
  cudaEvent_t ev_fork[3] = {nullptr, nullptr, nullptr}, ev_join[3] = {nullptr, nullptr, nullptr};
  int side_sel = 0;                                        // 0: direct calls, 1: init capture, 2: body capture
  double *d_r0 = nullptr, *d_z0 = nullptr;
  double *d_t1 = nullptr, *d_t2 = nullptr;   // apply/spmv scratch (internal order)
  double* d_partials = nullptr;              // reduction partials
  int partial_cap = 0;
  PcgState* d_state = nullptr;               // PCG state
  PcgState* d_astate = nullptr;              // state used by standalone dgas_apply / dgas_spmv
  double *d_alpha = nullptr, *d_beta = nullptr;
  int hist_cap = 0;
  double* d_lanczos = nullptr;               // [3] lmin lmax cond
  int* d_err = nullptr;                      // [4] setup error flags
  PcgState* h_state = nullptr;               // pinned
  double* h_scal = nullptr;                  // pinned [8]
  // graph
  cudaGraphExec_t graph_exec = nullptr;
  cudaGraph_t graph = nullptr;
  int graph_maxit = 0;
  // last results
  int last_iters = 0, last_status = 0;
  double last_cond = 0, last_lmin = 0, last_lmax = 0, last_relres = 0;
  // launch geometry
  int n_coarse_ctas = 0;   // coarse CTAs in the fused apply kernel
  int ring_slots = 2;      // TMA ring slots of the local-solve CTAs
  uint32_t slot_bytes = 0; // bytes per slot (R rows of the widest U row-block, 128-aligned)
  int ring_rows = 1;       // CC: columns of a row-block per stream unit
  int spmv_slots = 2;
  uint32_t spmv_slot_bytes = 0;
  int spmv_grid = 0;
  int spmv_G = 1;
  int restrict_wpj = 8;     // warps per coarse element in k_restrict
  // local-solve kernel: 1 = k_local (envelope U + D, all subdomains resident), 2 = k_local_panel
  // (merged panels [D_k | -U_k], few CTAs per SM for L2 reuse across the forward/backward turnaround)
  int local_kernel = 1;
  std::vector<int> first_h, sub_ptr_h;   // host copies: f_k (local index), subdomain cell ranges
  double* d_P = nullptr;                 // panels [D_k | -U_k], column-major, 16-byte aligned
  int64_t* d_p_off = nullptr;            // [nc+1] panel offsets (doubles)
  int* d_pus = nullptr;                  // [nc] first stream unit of cell k within its subdomain
  int* d_sub_units = nullptr;            // [nsub] stream units per subdomain
  int64_t p_total = 0;
  int panel_cc = 2, panel_slots = 2, panel_keep = 1, panel_cps = 1;
  int panel_f32 = 0;   // NEXT-4 variant (DGAS_PANEL_F32=1): fp32-stored panels, fp64 arithmetic
  // SpMV kernel: 3 = k_spmv3 (fixed slots, consumer groups), 4 = k_spmv_ring (byte ring, warp per cell)
  int spmv_kernel = 3;
  uint32_t sr_ring_bytes = 0;
  int sr_grid = 0, sr_G = 1;  // persistent CTAs; cells per bulk copy
  int spmv_psplit = 0;        // PCG direction update as a separate pass before the SpMV (DGAS_SPMV_PSPLIT)
  uint32_t panel_slot_bytes = 0;
};

// ---------------------------------------------------------------- helpers
#define DGAS_CUDA(call)                                                        \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      ctx->detail = std::string(#call) + ": " + cudaGetErrorString(e_);        \
      return e_ == cudaErrorMemoryAllocation ? DGAS_E_NOMEM : DGAS_E_CUDA;     \
    }                                                                          \
  } while (0)

__host__ __device__ inline int np_of(int p) { return (p + 1) * (p + 2) / 2; }
__host__ __device__ inline int gl_off(int m) { return m * (m - 1) / 2; }

// Legendre L_0..L_p and derivatives at t (three-term recurrences)
__device__ inline void dev_legendre(int p, double t, double* L, double* dL) {
  L[0] = 1.0; dL[0] = 0.0;
  if (p >= 1) { L[1] = t; dL[1] = 1.0; }
  for (int n = 1; n < p; ++n) {
    L[n + 1] = ((2 * n + 1) * t * L[n] - n * L[n - 1]) / (n + 1);
    dL[n + 1] = dL[n - 1] + (2 * n + 1) * L[n];
  }
}

// raw graded bbox-Legendre products g_i and their gradients (R6)
__device__ inline void dev_raw(int p, const double* bb, double x, double y, double* g, double* gx, double* gy) {
  double La[DGAS_MAXP + 1], dLa[DGAS_MAXP + 1], Lb[DGAS_MAXP + 1], dLb[DGAS_MAXP + 1];
  double sx = 2.0 / (bb[1] - bb[0]), sy = 2.0 / (bb[3] - bb[2]);
  dev_legendre(p, (x - bb[0]) * sx - 1.0, La, dLa);
  dev_legendre(p, (y - bb[2]) * sy - 1.0, Lb, dLb);
  int i = 0;
  for (int d = 0; d <= p; ++d)
    for (int a = d; a >= 0; --a, ++i) {
      int b = d - a;
      g[i] = La[a] * Lb[b];
      if (gx) { gx[i] = dLa[a] * sx * Lb[b]; gy[i] = La[a] * dLb[b] * sy; }
    }
}

// phi = C g (and gradients) for one point
__device__ inline void dev_phi(int p, int n, const double* C, const double* bb, double x, double y, double* phi,
                               double* px, double* py) {
  double g[DGAS_MAXNP], gx[DGAS_MAXNP], gy[DGAS_MAXNP];
  dev_raw(p, bb, x, y, g, px ? gx : nullptr, py ? gy : nullptr);
  for (int a = 0; a < n; ++a) {
    double s = 0, sx = 0, sy = 0;
    for (int b = 0; b <= a; ++b) {  // C is lower triangular
      double c = C[a * n + b];
      s += c * g[b];
      if (px) { sx += c * gx[b]; sy += c * gy[b]; }
    }
    phi[a] = s;
    if (px) { px[a] = sx; py[a] = sy; }
  }
}

__device__ inline double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------- launchers (defined in .cu files)
int setup_kernels_run(dgas_ctx ctx);                 // basis, assembly, local factors, coarse
int coarse_setup_run(dgas_ctx ctx);
int launch_rhs(dgas_ctx ctx, int f_kind, double* b_internal);
void launch_perm(dgas_ctx ctx, const double* in, double* out, int to_internal, cudaStream_t s);
void launch_spmv(dgas_ctx ctx, int mode, const double* x, double* y, PcgState* st, cudaStream_t s);
void launch_restrict(dgas_ctx ctx, int mode, PcgState* st, const double* r, cudaStream_t s);
bool apply_fuses_restrict(dgas_ctx ctx);
int restrict_ctas_per_sm(dgas_ctx ctx);
int prolong_ctas_per_sm(dgas_ctx ctx);
bool panel_is_narrow(dgas_ctx ctx);
void launch_apply(dgas_ctx ctx, int mode, PcgState* st, const double* r, double* z, cudaStream_t s);
void launch_prolong(dgas_ctx ctx, int mode, PcgState* st, const double* r, double* z, cudaStream_t s,
                    cudaGraphConditionalHandle h, int use_handle);
void launch_init_state(dgas_ctx ctx, PcgState* st, int maxit, double rtol, cudaStream_t s);
void launch_pcg_init(dgas_ctx ctx, cudaStream_t s);
void launch_lanczos(dgas_ctx ctx, cudaStream_t s);
int dgas_post_setup(dgas_ctx ctx);
int nd_build(dgas_ctx ctx, const std::vector<int>& pair_h, const std::vector<double>& centroid, int leaf);
int nd_setup_run(dgas_ctx ctx);
void nd_solve_launch(dgas_ctx ctx, int mode, const PcgState* st, cudaStream_t s);
int nd_set_smem(dgas_ctx ctx);
int nd_calibrate(dgas_ctx ctx);
int dense_calibrate(dgas_ctx ctx);
int local_inv_setup(dgas_ctx ctx);
void launch_local_inv(dgas_ctx ctx, int mode, const PcgState* st, const double* r, double* z, cudaStream_t s);
void launch_local_range(dgas_ctx ctx, int sub_begin, int sub_end, const double* r, double* z, cudaStream_t s);
void launch_local_inv_range(dgas_ctx ctx, int sub_begin, int sub_end, const double* r, double* z, cudaStream_t s);
void launch_local_panel_range(dgas_ctx ctx, int sub_begin, int sub_end, const double* r, double* z, cudaStream_t s);
int local_warp_setup(dgas_ctx ctx);
int dedup_setup(dgas_ctx ctx);
int mrhs_setup(dgas_ctx ctx, const std::vector<int>& rep_of);
int spmv_cls_setup(dgas_ctx ctx, const std::vector<int64_t>& dd);
void launch_local_mrhs(dgas_ctx ctx, int mode, const PcgState* st, const double* r, double* z, cudaStream_t s);
void launch_local_warp(dgas_ctx ctx, int mode, const PcgState* st, const double* r, double* z, cudaStream_t s);
void launch_spmv_range(dgas_ctx ctx, int c_begin, int c_end, const double* x, double* y, cudaStream_t s);
void launch_coarse_only(dgas_ctx ctx, cudaStream_t s);
void launch_lanczos(dgas_ctx ctx, cudaStream_t s);
int dgas_post_setup(dgas_ctx ctx);
void shard_free(dgas_ctx ctx);
void launch_a0_diag(dgas_ctx ctx, const int* prow, double* dsc, cudaStream_t s);
void launch_a0_resid(dgas_ctx ctx, const int* prow, const double* b, const double* z, double* res, const PcgState* st,
                     int mode, cudaStream_t s);
void launch_axpy_add(int64_t n, const double* a, double* y, const PcgState* st, int mode, cudaStream_t s);
void launch_coarse_dense(dgas_ctx ctx, int mode, const PcgState* st, const double* r0, double* z0, cudaStream_t s);
void nd_free(dgas_ctx ctx);
int apply_set_smem(dgas_ctx ctx, size_t smem);
size_t apply_smem_bytes(dgas_ctx ctx);
size_t spmv_smem_bytes(dgas_ctx ctx);
int spmv_batch_cells(int p, int ng);
int spmv_gather_cap(int p, int ng);
int spmv_groups_ok(int p);
int local_threads(int p);
void launch_local_only(dgas_ctx ctx, const double* r, double* z, cudaStream_t s);
void launch_coarse_only(dgas_ctx ctx, cudaStream_t s);
int spmv_set_smem(dgas_ctx ctx, size_t smem);
int spmv_ring_configure(dgas_ctx ctx, int nsm);
size_t spmv_ring_smem(dgas_ctx ctx);
void launch_spmv_ring(dgas_ctx ctx, int mode, const double* x, double* y, PcgState* st, cudaStream_t s);
int panel_supported(int p);
int pack_ppw(int np);
int restrict_chunk_threads();
int panel_min_cc(int np, int f32);
int panel_al(int f32);
size_t panel_base_bytes(int max_cells, int np, bool narrow);
int panel_setup(dgas_ctx ctx, const std::vector<int>& sub_ptr, const std::vector<int>& first);
size_t panel_smem_bytes(dgas_ctx ctx);
int panel_set_smem(dgas_ctx ctx);
void launch_local_panel(dgas_ctx ctx, int mode, PcgState* st, const double* r, double* z, cudaStream_t s);

template <typename T>
inline int dev_upload(dgas_ctx ctx, T** d, const std::vector<T>& h) {
  size_t n = std::max<size_t>(h.size(), 1);
  DGAS_CUDA(cudaMalloc((void**)d, n * sizeof(T)));
  if (!h.empty()) DGAS_CUDA(cudaMemcpyAsync(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  return 0;
}
template <typename T>
inline int dev_alloc(dgas_ctx ctx, T** d, size_t n, bool zero = true) {
  n = std::max<size_t>(n, 1);
  DGAS_CUDA(cudaMalloc((void**)d, n * sizeof(T)));
  if (zero) DGAS_CUDA(cudaMemsetAsync(*d, 0, n * sizeof(T), ctx->stream));
  return 0;
}
