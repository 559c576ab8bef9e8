/* include/dgas.h — C ABI of the B200 (sm_100a) additive-Schwarz PCG library for SIPDG on polytopic
 * meshes (arXiv 1903.11357). Shared library: paper_1903_11357_b200/libdgas.so.
 *
 * The library computes, entirely in its own CUDA kernels:
 *   - the SIPDG matrix A of eq:Ah, assembled in the face form of PAPER.md:467-469,
 *     with penalty sigma = C_sigma <rho> p^2 / <h_kappa> (eq:Sigma);
 *   - the two-level non-overlapping additive Schwarz preconditioner
 *         P^-1 = R0^T A0^-1 R0 + sum_i R_i^T A_i^-1 R_i
 *     with exact local solves on the subdomains of T_HH, the L2 prolongation
 *     R0^T (eq:R0T) from the degree-q space on the (possibly non-nested) coarse
 *     partition T_H, and the Galerkin coarse operator A0 = R0 A R0^T (eq:A0);
 *   - PCG (ASPCG) with the Euclidean relative-residual stop of PAPER.md:741 and the Lanczos
 *     extreme-eigenvalue estimate of K(P_ad) from the CG coefficients.
 * Readings where the paper is silent are listed in DESIGN.md (R1..R30).
 *
 * Conventions (all entry points):
 *   - Return an int status: 0 = OK, > 0 = result exists with a warning, < 0 = error (see DGAS_*).
 *     No exception crosses the ABI. dgas_strerror() gives a static message; dgas_error_detail()
 *     the context's last detail string (e.g. which block was not SPD).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Vectors passed to dgas_rhs/spmv/apply/pcg are DEVICE pointers to fp64 arrays of length
 *     N = n_cells * n_p, n_p = (p+1)(p+2)/2, in the CALLER's cell order with the n_p modal
 *     coefficients of one cell contiguous, in the basis order of DESIGN.md R6 (per-cell
 *     L2-orthonormal basis from bbox-scaled Legendre products of total degree <= p, graded order).
 *     The caller owns them. dgas_pcg_host takes HOST pointers instead (pinned memory recommended).
 *   - The context owns every device buffer it allocates (matrix, factors, prolongation, coarse
 *     inverse/factor, work vectors, alpha/beta history). One context = one stream at a time.
 *   - dgas_spmv / dgas_apply / dgas_rhs are asynchronous on `stream`; dgas_setup, dgas_pcg and
 *     dgas_pcg_host synchronise `stream` before returning.
 */
#ifndef DGAS_H
#define DGAS_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  DGAS_OK = 0,
  DGAS_NOT_CONVERGED = 1,     /* pcg: x = last iterate, iters = maxit, cond from the T_k available */
  DGAS_E_INVALID_ARG = -1,    /* p<1, q<1, q>p, p>6, bad partition, kappa<=0/non-finite, penalty<=0, rtol<=0, maxit<1, NULL */
  DGAS_E_MESH = -2,           /* non-manifold edge, non-CCW/zero-area cell, overlap areas != |kappa| (1e-10 rel) */
  DGAS_E_NOT_SPD = -3,        /* Cholesky pivot <= 0 in a local block A_i or in A0 (detail names it) */
  DGAS_E_BREAKDOWN = -4,      /* pcg: p.Ap <= 0, r.z <= 0 or a non-finite scalar */
  DGAS_E_CUDA = -5,           /* a CUDA runtime call failed (detail has the CUDA error string) */
  DGAS_E_NOMEM = -6           /* device allocation failed */
};

typedef struct dgas_ctx_s* dgas_ctx;

/* Fine polytopic mesh T_h. Host arrays, copied by dgas_setup.
 *   xy[2*n_vertices]                vertex coordinates
 *   cell_ptr[n_cells+1], cell_vtx   counter-clockwise vertex loops (cells convex) */
typedef struct {
  int32_t n_vertices;
  const double* xy;
  int32_t n_cells;
  const int32_t* cell_ptr;
  const int32_t* cell_vtx;
} dgas_mesh;

/* Coarse partition T_H for the degree-q coarse space V_0.
 * Nested (T_h is a refinement of T_H): parent[n_cells] gives the coarse element of each fine cell,
 *   and the overlap fields are ignored (R0^T is then the natural injection, Remark 3.2).
 * Non-nested (parent == NULL): the n_overlaps pieces kappa ∩ D_J (generator-made polygons, CCW,
 *   possibly non-convex; ov_xy points ov_ptr[k]..ov_ptr[k+1]-1) define the integrals of eq:R0T.
 *   Pieces of every fine cell must cover it (area check 1e-10 relative, else DGAS_E_MESH). */
typedef struct {
  int32_t n_coarse;
  const int32_t* parent;
  int32_t n_overlaps;
  const int32_t* ov_fine;
  const int32_t* ov_coarse;
  const int32_t* ov_ptr;
  const double* ov_xy;
} dgas_coarse;

typedef struct {
  int64_t N, N0;                 /* fine and coarse dofs */
  int32_t n_cells, n_p, n_q, n_subdomains, n_coarse, n_faces, n_overlaps;
  int32_t coarse_dense;          /* 1: explicit dense A0^-1; 0: banded Cholesky of A0 */
  int32_t coarse_band;           /* half bandwidth of A0 (dofs) */
  int64_t nnz_blocks;            /* stored n_p x n_p blocks of A (full block-CSR) */
  int64_t bytes_A, bytes_U, bytes_Dinv, bytes_G, bytes_coarse; /* device bytes of each operator */
  int64_t alg_bytes_spmv;        /* algorithmic HBM bytes of one q = A p */
  int64_t alg_bytes_apply;       /* algorithmic HBM bytes of one z = P^-1 r */
  int64_t alg_bytes_iter;        /* algorithmic HBM bytes of one PCG iteration */
  int32_t last_iters, last_status;
  double last_cond, last_lmin, last_lmax, last_relres;
  int32_t coarse_mode;           /* 0 dense explicit inverse, 1 band, 2 nested dissection */
  int32_t launches_per_iter;     /* kernel launches of one PCG iteration (graph body) */
  int32_t launches_per_solve;    /* fixed launches of one dgas_pcg besides the iterations */
  int32_t coarse_refine;         /* iterative-refinement steps of the coarse solve (dense or ND; R30 calibration) */
  double coarse_solve_relerr;    /* measured ||z - v|| / ||v|| of one coarse solve of A0 z = A0 v (dense or ND;
                                    refinement steps are added while it exceeds 3e-11) */
  int32_t unroll;                /* PCG iterations per execution of the graph's WHILE body; the last body of a
                                    solve launches its remaining copies as immediate-return kernels */
  int32_t local_kernel;          /* 1: envelope kernel (all subdomains resident); 2: panel kernel (merged
                                    [D | -U] panels, TMA ring); 3: explicit local inverses Z_i = A_i^-1 (one
                                    GEMV per subdomain, L2-resident small configs; NEXT-4) */
  int32_t local_ctas_per_sm;     /* resident local-solve CTAs per SM the panel kernel is sized for */
  int64_t bytes_local;           /* operator bytes one local-solve launch reads (factor; or Z for kernel 3) */
  double local_inv_err;          /* kernel 3: ||Z r - exact solve(r)|| / ||exact solve(r)|| at setup */
  int64_t dedup_A_bytes;         /* bytes of A actually stored when bitwise-identical row-blocks are shared
                                    (exact de-duplication, NEXT-4; 0: not de-duplicated) */
  int64_t dedup_local_bytes;     /* the same for the local factors (merged panels) */
} dgas_info_t;

/* Build the SIPDG operator and the two-level Schwarz preconditioner on the GPU.
 *   p in [1,6] (fine degree), 1 <= q <= p (coarse degree)
 *   partition[n_cells] in [0, n_subdomains) — subdomain Omega_i of each cell (T_HH)
 *   kappa[n_cells] > 0 — piecewise-constant diffusion rho
 *   penalty = C_sigma > 0 (10 in every experiment)
 * All host inputs are copied. On failure *out is NULL and the status says why. */
int dgas_setup(dgas_ctx* out, const dgas_mesh* mesh, int p, const int32_t* partition, int32_t n_subdomains,
               const dgas_coarse* coarse, int q, const double* kappa, double penalty, void* stream);

/* b_a = int_kappa f phi_a (eq:dG) with a fixed collapsed Gauss rule (R10).
 * f_kind: 0 = 2 pi^2 sin(pi x) sin(pi y), 1 = 1, 2 = 2[x(1-x) + y(1-y)]. b: device, length N. */
int dgas_rhs(dgas_ctx ctx, int f_kind, double* b, void* stream);

/* y = A x (device vectors, caller order). Test hook and the per-iteration SpMV kernel. */
int dgas_spmv(dgas_ctx ctx, const double* x, double* y, void* stream);

/* z = P^-1 r = Q A0^-1 Q^T r + sum_i E_i A_i^-1 E_i^T r (device vectors, caller order). */
int dgas_apply(dgas_ctx ctx, const double* r, double* z, void* stream);

/* Which preconditioner dgas_apply and dgas_pcg use (default DGAS_PRECOND_TWO_LEVEL):
 *   TWO_LEVEL  P^-1 = R0^T A0^-1 R0 + sum_i R_i^T A_i^-1 R_i        (eq:Pad)
 *   ONE_LEVEL  P^-1 = sum_i R_i^T A_i^-1 R_i  (no coarse space)
 *   COARSE     P^-1 = R0^T A0^-1 R0           (coarse space only; singular as a preconditioner unless
 *                                              V_H spans V_h, test/diagnostic use)
 *   NONE       P^-1 = I, plain CG: its Lanczos estimate is K(A_h) (Tables of Ex.3)
 * Returns DGAS_E_INVALID_ARG for an unknown mode. Takes effect for the next call on the context. */
enum { DGAS_PRECOND_TWO_LEVEL = 0, DGAS_PRECOND_ONE_LEVEL = 1, DGAS_PRECOND_COARSE = 2, DGAS_PRECOND_NONE = 3 };
int dgas_set_precond(dgas_ctx ctx, int mode);

/* ASPCG: solves A x = b from the initial guess in x (device vectors, caller order); stops when
 * ||b - A x_k||_2 (recursive residual) <= rtol ||b||_2 or after maxit iterations. Writes the
 * iteration count and the Lanczos estimate lambda_max/lambda_min of P^-1 A built from the same
 * run's alpha/beta (R12). Returns DGAS_OK, DGAS_NOT_CONVERGED or an error. Synchronous. */
int dgas_pcg(dgas_ctx ctx, const double* b, double* x, double rtol, int maxit, int* iters, double* lanczos_cond,
             void* stream);

/* Same as dgas_pcg with HOST b / x (copied host->device and back inside the call). */
int dgas_pcg_host(dgas_ctx ctx, const double* b_host, double* x_host, double rtol, int maxit, int* iters,
                  double* lanczos_cond, void* stream);

/* Sizes, byte counts and the last solve's outcome. */
int dgas_info(dgas_ctx ctx, dgas_info_t* info);

/* alpha_k (k < iters) and beta_k (k < iters-1) of the last dgas_pcg (host arrays of length cap). */
int dgas_history(dgas_ctx ctx, double* alphas, double* betas, int cap);

/* Diagnostics (host outputs, caller order): the A block coupling caller cells (i, j) (n_p x n_p,
 * zero if not coupled; returns 1 if stored), the basis coefficients of cell i (n_p x n_p, over the
 * bbox-Legendre products of R6), the assembled A0 = Q^T A Q densely (N0 x N0, row-major; any coarse
 * mode; caller allocates N0*N0 doubles). */
int dgas_debug_block(dgas_ctx ctx, int32_t i, int32_t j, double* out);
int dgas_debug_basis(dgas_ctx ctx, int32_t i, double* out);
int dgas_debug_A0(dgas_ctx ctx, double* out);

/* Bench hook: launch `reps` times, on `stream`, the per-iteration kernel(s) `which` on the context's
 * internal scratch vectors (0 = SpMV q = A p; 1 = full preconditioner apply = restrict + fused
 * coarse||local solve + prolong; 2 = fused coarse||local solve kernel alone). Asynchronous; used
 * by bench.py to time kernels with CUDA events on the launching stream. */
int dgas_bench_kernels(dgas_ctx ctx, int which, int reps, void* stream);

/* ---- Subdomain-sharded multi-GPU solve (PAPER.md:123 any decomposition,
 * PAPER.md:741 "massively parallel"). One process per GPU, each with a full (replicated) context from
 * dgas_setup. dgas_shard gives rank `rank` of `nranks` a contiguous range of subdomains (balanced by cell
 * count); per iteration the rank computes only its own rows, subdomains and cells. The collectives are
 * the CALLER's (sum over ranks; all-gather for the halo), between these calls, on the same stream:
 *   begin -> allreduce(red0) -> precond -> allreduce(red1) -> direction(first=1) -> allgather(hsend)
 *   loop: spmv -> allreduce(red2) -> update -> allreduce(red0) -> [stop if red0[N0] <= rtol^2 red0_begin[N0+1]]
 *         -> precond -> allreduce(red1) -> direction(first=0) -> allgather(hsend)
 *   finish -> allreduce(x)
 * Buffers are caller-owned device arrays of doubles: red0 [N0 + 2] = [Q^T r | r.r | b.b] (begin fills all
 * three parts, update the first two), red1 [1] = r.z, red2 [1] = p.q, hsend [cap] = this rank's border
 * values of p, hall [nranks * cap] = every rank's hsend (all-gathered, rank-major). Asynchronous on
 * `stream` except dgas_shard and dgas_shard_finish. info[6] out: own dof range [info0, info1) in internal
 * order, cap, N, N0, own subdomain count. Errors: DGAS_E_INVALID_ARG (ranks > subdomains, bad rank, no
 * byte-ring SpMV); dgas_shard_finish returns DGAS_E_BREAKDOWN if p.Ap <= 0 or r.z <= 0 was seen. */
int dgas_shard(dgas_ctx ctx, int32_t rank, int32_t nranks, int64_t* info);
/* b: caller order, length N, the full right-hand side on every rank. x = 0, r = b. */
int dgas_shard_begin(dgas_ctx ctx, const double* b, double* red0, void* stream);
/* z0 = A0^-1 r0 with r0 = summed red0[0..N0) (replicated coarse solve), z = own local solves + Q z0 on own
 * cells; red1 = own part of r.z. */
int dgas_shard_precond(dgas_ctx ctx, const double* red0, double* red1, void* stream);
/* beta = summed r.z / previous (first: p = z), p = z + beta p on own dofs; hsend = p on own border cells. */
int dgas_shard_direction(dgas_ctx ctx, const double* red1, double* hsend, int32_t first, void* stream);
/* p on other ranks' border cells from hall; q = A p on own rows (eq:Ah); red2 = own part of p.q. */
int dgas_shard_spmv(dgas_ctx ctx, const double* hall, double* red2, void* stream);
/* alpha = summed r.z / summed p.q; x += alpha p, r -= alpha q (own); red0[0..N0] = own [Q^T r | r.r]. */
int dgas_shard_update(dgas_ctx ctx, const double* red2, double* red0, void* stream);
/* x: caller order, length N: own dofs of the iterate, zero elsewhere (sum over ranks = the solution).
 * lanczos[3] (device) = (lmin, lmax, K) from the first `iters` CG coefficients. */
int dgas_shard_finish(dgas_ctx ctx, int32_t iters, double* x, double* lanczos, void* stream);

/* Frees every device buffer of the context. */
int dgas_destroy(dgas_ctx ctx);

const char* dgas_strerror(int status);
const char* dgas_error_detail(dgas_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif /* DGAS_H */
