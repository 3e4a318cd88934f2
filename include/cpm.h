/*
 * cpm.h — C ABI of the B200-native closest point method (CPM) hot path.
 *
 * The operations follow the problem statement of May, Haynes & Ruuth,
 * "A closest point method library for PDEs on surfaces with parallel domain
 * decomposition solvers and preconditioners" (arXiv:2110.06322), reproduced in
 * PAPER.md; "PAPER.md:N" below cites its line N.  DESIGN.md lists the readings
 * (R1..R15) taken where the paper is silent.
 *
 * Conventions (all entry points):
 *  - Return CPM_OK (0) on success, a negative CPM_ERR_* code otherwise; the
 *    message of the last error on the calling thread is cpm_last_error().
 *    No entry point aborts the process.
 *  - Floating point is IEEE binary64 ("fp64") throughout.
 *  - Vector arguments are plain pointers to nA doubles (nA = number of active
 *    nodes) in BAND ORDER (reading R8: Morton order of 8^3 bricks, then z,y,x
 *    inside a brick).  A pointer may be DEVICE memory (cudaMalloc / torch CUDA
 *    tensor) or HOST memory (pageable or pinned); host pointers are staged
 *    through device buffers owned by the band, with the copies on `stream`.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Calls are asynchronous w.r.t. the host for device pointers, except where
 *    a result must reach the host (cpm_solve statistics, host outputs).
 *  - Handles (cpm_band, cpm_ras, cpm_comm) are owned by the caller and
 *    released with the matching *_free; they own all device memory they use.
 *  - Concurrency: a band (and every cpm_ras / cpm_part built on it) owns ONE
 *    set of scratch buffers (E u bricks, host staging, the GMRES workspace).
 *    Calls on the same band must be issued one stream at a time from one
 *    thread; concurrent calls on one band from different streams or threads
 *    race.  Different bands are independent.
 *  - The partitioned calls (cpm_part_*, cpm_part_ras_*) take DEVICE pointers
 *    only; a host pointer returns CPM_ERR_ARG.
 *  - Only p = 3 (tricubic) interpolation and d = 3 are implemented.
 */
#ifndef CPM_H_
#define CPM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CPM_OK 0
#define CPM_ERR_ARG (-1)      /* invalid argument */
#define CPM_ERR_CUDA (-2)     /* CUDA runtime error (message has the CUDA text) */
#define CPM_ERR_GEOM (-3)     /* closest point undefined in the band / stencil leaves Sigma_A */
#define CPM_ERR_NOMEM (-4)    /* device or host allocation failed */
#define CPM_ERR_NCCL (-5)     /* NCCL error (multi-GPU calls) */
#define CPM_ERR_LIMIT (-6)    /* a size limit of this implementation was exceeded */

/* Surfaces with an analytic closest point function cp_S (Eq. 3). */
#define CPM_SURF_SPHERE 1 /* param[0] = radius R, centred at the origin */
#define CPM_SURF_TORUS 2  /* param[0] = major radius R, param[1] = minor radius r, axis z */

typedef struct cpm_surface {
  int32_t kind;
  double param[4];
} cpm_surface;

typedef struct cpm_band cpm_band;
typedef struct cpm_ras cpm_ras;
typedef struct cpm_comm cpm_comm;

typedef struct cpm_band_info {
  int64_t n_active;   /* |Sigma_A| — the unknowns */
  int64_t n_ghost;    /* |Sigma_G| */
  int64_t n_tiles;    /* occupied 8^3 bricks (apply work units) */
  int64_t n_runs;     /* stencil-box fill runs (apply metadata) */
  int64_t max_box;    /* largest per-tile stencil box, cells */
  int64_t bytes_device; /* device memory held by the band */
  double h, lambda, L;
  int32_t lattice_lo[3], lattice_hi[3]; /* inclusive lattice bounds of Sigma_A u Sigma_G */
  int32_t zero_fill;  /* 1 if some stencil cell is not a source node (sub-bands) */
  int32_t rank, nranks; /* owning rank of a partitioned band (0, 1 otherwise) */
  int64_t n_owned;    /* owned active nodes (== n_active unless partitioned) */
  int64_t n_halo;     /* halo source nodes received from other ranks */
} cpm_band_info;

typedef struct cpm_solve_stats {
  int32_t iterations;  /* Arnoldi steps (operator applications inside cycles) */
  int32_t converged;   /* 1 if |g_{k+1}| <= rtol ||f|| was reached */
  int32_t cycles;      /* restart cycles */
  int32_t breakdown;   /* 1 on happy breakdown */
  double resid_est;    /* Givens residual estimate at exit */
  double resid_true;   /* ||f - A u||_2 recomputed at exit */
  double bnorm;        /* ||f||_2 */
  double seconds;      /* wall time of the call (host clock, includes syncs) */
} cpm_solve_stats;

/* ---------------------------------------------------------------- version / errors */
const char* cpm_version(void);
const char* cpm_last_error(void);

/* ---------------------------------------------------------------- band construction
 * cpm_build_band — north_star item (1); PAPER.md:62 (Sigma_A, Sigma_G),
 * PAPER.md:76 (the (p+1)^d interpolation cubes).
 *   Sigma_A = { x = h (i,j,k), |i|,|j|,|k| <= round(L/h) : |x - cp(x)| <= lambda },
 *   lambda = sqrt(17) h (reading R1); Sigma_G = 6-neighbours of Sigma_A outside it.
 *   For every node of Sigma_A u Sigma_G: cp(x), the stencil base floor(cp/h) - 1
 *   and the fractional offset cp/h - floor(cp/h) (reading R2), plus the bucketed
 *   (8^3-brick) node -> lattice map used by the apply.
 * Arguments: surface (host struct), h > 0 grid spacing, p (must be 3),
 *   L > 0 half-width of the computational box [-L, L]^3, stream, out (receives
 *   the handle).  Device work runs on `stream`; the call synchronises it.
 * Errors: CPM_ERR_ARG (p != 3, h <= 0, unknown surface), CPM_ERR_GEOM (cp
 *   undefined at a band node or a stencil leaves Sigma_A — the band is wider
 *   than the surface's reach), CPM_ERR_LIMIT, CPM_ERR_CUDA. */
int cpm_build_band(const cpm_surface* surface, double h, int p, double L, void* stream,
                   cpm_band** out);
int cpm_band_get_info(const cpm_band* band, cpm_band_info* info);
/* Lattice coordinates (i,j,k) of the active / ghost nodes, in band order, into
 * a HOST int32 array of 3*n entries. */
int cpm_band_active_coords(const cpm_band* band, int32_t* ijk_host);
int cpm_band_ghost_coords(const cpm_band* band, int32_t* ijk_host);
/* Diagnostics of the extend's node order (build.cu k_item_order / k_warp_order;
 * DESIGN.md §Kernels): per tile 6 int32 into tiles_host[6*n_tiles] = e0, e1
 * (eval-node range, padded index space), the order word — item order (the
 * default): 1 << 30 | number of rounds (cpm_band_item_rounds); pair order
 * (CPM_ITEMS=0 at build): np | nd << 16 (np equal-base pairs at e0 + 2p,
 * e0 + 2p + 1; then nd unpaired nodes gathered by lane pairs, the rest one per lane),
 * row stride and plane stride of the tile's stencil box, box cells; and, if
 * eoff_host is not null, the packed stencil-base offsets (low 16 bits: offset
 * in the box, high 16: brick cell) of the padded eval index space [0, e1 of the
 * last tile) into eoff_host.  Read-only; CPM_ERR_ARG on null band/tiles_host. */
int cpm_band_eval_order(const cpm_band* band, int32_t* tiles_host, uint32_t* eoff_host);
/* The item rounds of an item-order band (build.cu k_item_order): 32 uint64 per
 * tile into rounds_host[32*n_tiles] (unused words 0).  Word bits 0-31: lane l's
 * item holds two nodes; 32-47: the round's first node relative to the tile's e0;
 * 48-53: lanes in use.  Lane l's item starts at that node + l + popcount(bits
 * below l).  Read-only; CPM_ERR_ARG on a null argument or a pair-order band. */
int cpm_band_item_rounds(const cpm_band* band, uint64_t* rounds_host);
void cpm_band_free(cpm_band* band);

/* ---------------------------------------------------------------- operator apply
 * cpm_apply — y = (c I - Delta_S^h) u with Delta_S^h of PAPER.md:80-85 (Eq. 4,
 * d = 3) and c of Eq. 2:
 *   y = c u - [ Delta_h E u - (6/h^2)(u - E u) ] = (c + 6/h^2) u - (1/h^2) sum_{6 nbrs} (E u)
 * E is the tricubic barycentric Lagrange extension, applied
 * matrix-free: weights are recomputed from the stored fractional offsets.
 * u, y: nA doubles each (device or host), must not alias.  Asynchronous on
 * `stream` for device pointers; synchronous for host pointers.
 * Errors: CPM_ERR_ARG (null pointers / aliasing), CPM_ERR_CUDA. */
int cpm_apply(const cpm_band* band, double c, const double* u, double* y, void* stream);
/* cpm_apply_async — cpm_apply for PINNED host buffers (cudaMallocHost /
 * cudaHostRegister), pipelined: the call enqueues the copy of u to the device, the
 * apply (on `stream`) and the copy of y back, and returns; y is complete after
 * cpm_apply_sync(band) (or a device synchronise).  Consecutive calls overlap (the
 * copy-in of the next call with the apply and copy-out of this one; two staging
 * slots owned by the band): u and y of a call must stay untouched until then.
 * Device or pageable pointers: exactly cpm_apply (synchronous for host memory).
 * Errors: those of cpm_apply. */
int cpm_apply_async(const cpm_band* band, double c, const double* u, double* y, void* stream);
int cpm_apply_sync(const cpm_band* band);

/* ---------------------------------------------------------------- Krylov solve
 * cpm_solve — solve (c - Delta_S^h) u = f (Eq. 2) by restarted GMRES(restart)
 * (GMRES is the default solver) with classical Gram-Schmidt
 * applied twice (CGS2; without ras in its delayed one-reduction form DCGS2,
 * reading R15), fused dot/axpy/norm kernels, deterministic reductions.
 * Right-preconditioned flexible GMRES when `ras` is not NULL.
 * Convention (reading R5): u holds the initial guess on entry (pass zeros for
 * x0 = 0) and the solution on exit; convergence when the Givens residual
 * estimate <= rtol * ||f||_2; maxit bounds the total Arnoldi steps.
 * f, u: nA doubles (device or host).  stats may be NULL.  Synchronises `stream`.
 * Errors: CPM_ERR_ARG (restart < 1 or > 128, rtol <= 0, f not finite), CPM_ERR_CUDA,
 * CPM_ERR_NOMEM. Not converging within maxit is NOT an error (stats.converged = 0).
 * A restart cycle that completes no Arnoldi step (non-finite x0 or residual) or a
 * non-finite residual estimate ends the solve with stats.breakdown = 1,
 * stats.converged = 0 (never an endless restart loop). */
int cpm_solve(const cpm_band* band, double c, const double* f, double* u, double rtol, int restart,
              int maxit, const cpm_ras* ras, cpm_solve_stats* stats, void* stream);

/* ---------------------------------------------------------------- RAS preconditioner
 * cpm_ras_setup — one-level restricted additive Schwarz, PAPER.md:87-111 with
 * Dirichlet transmission (T_jk = identity; the default,
 * PAPER.md:252).  Disjoint subdomains = n_sub Morton slabs of the band order
 * (reading R8); each grown by `overlap` lattice 6-neighbour layers inside
 * Sigma_A (reading R7).  Local solves: exactly k_inner GMRES steps from zero on
 * A_j = R_j A R_j^T, batched over subdomains on the GPU (reading R6).
 * c: the shift of the operator being preconditioned.
 * Errors: CPM_ERR_ARG (n_sub < 1, overlap < 0, k_inner < 1 or > 64), CPM_ERR_CUDA. */
int cpm_ras_setup(const cpm_band* band, int n_sub, int overlap, int k_inner, double c,
                  void* stream, cpm_ras** out);
/* z = sum_j R~_j^T GMRES_k(A_j, R_j r): r, z nA doubles (device or host), no aliasing. */
int cpm_ras_apply(const cpm_ras* ras, const double* r, double* z, void* stream);
void cpm_ras_free(cpm_ras* ras);

/* ---------------------------------------------------------------- multi-GPU (north_star item 5)
 * One process per GPU.  Every rank builds the same global band (deterministic,
 * cheap) and then its partition: rank r of R owns the band-order slab
 * [floor(r nA/R), floor((r+1) nA/R)) (reading R8); its local operator reads the
 * owned entries of a vector plus a HALO of other ranks' entries (the active nodes
 * in the stencil boxes of the tiles it evaluates).  Before every apply the halo
 * is exchanged with NCCL send/recv; every Krylov reduction is an NCCL allreduce
 * (or, for a communicator from cpm_comm_init_host, the caller's host callbacks).
 * NCCL is loaded at run time (dlopen "libnccl.so.2"); without it the cpm_comm_*
 * calls return CPM_ERR_NCCL and the single-GPU API is unaffected. */
typedef struct cpm_part cpm_part;
typedef struct cpm_part_info {
  int32_t rank, nranks;
  int64_t lo, hi;        /* owned band-order range [lo, hi) */
  int64_t n_owned, n_halo, n_tiles, n_send;
  int64_t n_interior_tiles; /* tiles [0, n_interior_tiles) read no halo node: their extend
                               overlaps the halo exchange */
} cpm_part_info;

/* 128-byte NCCL unique id (rank 0 creates it; broadcast it, e.g. with torch.distributed). */
int cpm_comm_unique_id(void* id_out_128);
int cpm_comm_init(const void* id_128, int rank, int nranks, cpm_comm** out);
/* Host-staged transport (the second transport behind the same cpm_part_* calls):
 * the two data-plane collectives of the partitioned path are delegated to caller
 * callbacks on HOST buffers — used to run several ranks as processes sharing one
 * GPU (NCCL refuses two ranks on one device), e.g. over a torch.distributed gloo
 * group.  The library synchronises `stream`, copies the device data into pinned
 * host staging, calls the callback, and copies the result back.
 *   allreduce_sum(ctx, buf, n): buf[0..n) <- its sum over all ranks (in place).
 *   alltoallv(ctx, send, send_counts, recv, recv_counts): send_counts[q] doubles
 *     to rank q (blocks in rank order in `send`), recv_counts[q] doubles from
 *     rank q (rank order in `recv`); counts have nranks entries, own entry 0.
 * Callbacks return 0 on success; any other value fails the calling entry point
 * with CPM_ERR_NCCL.  The struct is copied; ctx must outlive the communicator. */
typedef struct cpm_host_transport {
  void* ctx;
  int (*allreduce_sum)(void* ctx, double* buf, int64_t n);
  int (*alltoallv)(void* ctx, const double* send, const int64_t* send_counts, double* recv,
                   const int64_t* recv_counts);
} cpm_host_transport;
int cpm_comm_init_host(const cpm_host_transport* transport, int rank, int nranks, cpm_comm** out);
void cpm_comm_free(cpm_comm* comm);

/* Build rank's partition of `band` (device work on stream).  Errors: CPM_ERR_ARG. */
int cpm_part_create(const cpm_band* band, int rank, int nranks, void* stream, cpm_part** out);
int cpm_part_get_info(const cpm_part* part, cpm_part_info* info);
/* Global band-order indices of the halo nodes (sorted ascending, grouped by owner
 * rank) into a HOST int64 array of n_halo entries: what this rank RECEIVES. */
int cpm_part_halo_nodes(const cpm_part* part, int64_t* halo_host);
/* What this rank SENDS: for every peer q (counts[q] entries, peers in rank order)
 * the owned global indices peer q requested (its cpm_part_halo_nodes restricted to
 * this rank's slab, in its order).  HOST arrays; copied.  Errors: CPM_ERR_ARG if an
 * index is not owned. */
int cpm_part_set_send(cpm_part* part, const int64_t* send_global_host, const int64_t* counts_host);
/* y_owned = (c - Delta_S^h) u restricted to the owned rows, halo values given
 * explicitly (u_halo: n_halo doubles in cpm_part_halo_nodes order); no
 * communication.  Device pointers. */
int cpm_part_apply_local(const cpm_part* part, double c, const double* u_owned,
                         const double* u_halo, double* y_owned, void* stream);
/* Halo exchange over `comm` + local apply.  Device pointers (n_owned doubles). */
int cpm_part_apply(const cpm_part* part, const cpm_comm* comm, double c, const double* u_owned,
                   double* y_owned, void* stream);
/* Distributed GMRES(restart) on the owned slices (conventions of cpm_solve); every
 * rank gets identical statistics.  ras: NULL, or this rank's cpm_part_ras_setup
 * preconditioner (flexible GMRES, RAS halo exchanged before every apply). */
int cpm_part_solve(const cpm_part* part, const cpm_comm* comm, double c, const double* f_owned,
                   double* u_owned, double rtol, int restart, int maxit, const cpm_ras* ras,
                   cpm_solve_stats* stats, void* stream);
void cpm_part_free(cpm_part* part);

/* ---------------------------------------------------------------- distributed RAS (items 4 + 5)
 * cpm_part_ras_setup — this rank's share of the one-level RAS preconditioner of
 * cpm_ras_setup for a partitioned band: n_sub Morton-slab subdomains (reading
 * R8), n_sub a multiple of nranks (as in the paper), rank r handles
 * subdomains [r n_sub/R, (r+1) n_sub/R) whose disjoint parts are exactly its
 * owned slab.  The overlap (reading R7) reaches into other ranks' slabs: those
 * members form the RAS HALO, received before every apply (cpm_ras_halo_nodes /
 * cpm_ras_set_send, as for the operator halo); the inner solves and the
 * restricted prolongation are rank-local.  Errors: CPM_ERR_ARG, CPM_ERR_CUDA. */
typedef struct cpm_ras_info {
  int32_t n_sub, sub0, n_sub_local, rank, nranks;
  int64_t n_members;  /* concatenated overlapping subdomains of this rank */
  int64_t n_owned, n_halo, n_send;
} cpm_ras_info;
int cpm_part_ras_setup(const cpm_part* part, int n_sub, int overlap, int k_inner, double c,
                       void* stream, cpm_ras** out);
int cpm_ras_get_info(const cpm_ras* ras, cpm_ras_info* info);
/* Global band-order indices of the RAS halo, sorted (grouped by owner), HOST array. */
int cpm_ras_halo_nodes(const cpm_ras* ras, int64_t* halo_host);
/* What this rank sends to each peer's RAS halo (layout of cpm_part_set_send). */
int cpm_ras_set_send(cpm_ras* ras, const int64_t* send_global_host, const int64_t* counts_host);
/* z_owned = (M r)_owned with the RAS-halo values given explicitly (no communication);
 * r_halo: n_halo doubles in cpm_ras_halo_nodes order.  Device pointers. */
int cpm_part_ras_apply_local(const cpm_ras* ras, const double* r_owned, const double* r_halo,
                             double* z_owned, void* stream);
/* RAS-halo exchange over `comm` + local apply.  Device pointers (n_owned doubles). */
int cpm_part_ras_apply(const cpm_ras* ras, const cpm_comm* comm, const double* r_owned,
                       double* z_owned, void* stream);

/* ---------------------------------------------------------------- problem data
 * cpm_eval_sph — out_i = scale * Y_l^m(cp(x_i)) on the active nodes, real
 * orthonormal spherical harmonics without Condon-Shortley phase (reading R9);
 * the manufactured right-hand sides of BASELINE configs 0, 1, 3.
 * Requires a sphere band.  out: nA doubles (device or host). */
int cpm_eval_sph(const cpm_band* band, int l, int m, double scale, double* out, void* stream);
/* cpm_eval_torus_rhs — out_i = cos(3 th) sin(2 ph) (1 + sum_q a_q sin(k_q . cp))
 * at cp(x_i) of a torus band (BASELINE config 2, reading R10).  coeffs: HOST
 * array of nq rows (a, kx, ky, kz). */
int cpm_eval_torus_rhs(const cpm_band* band, const double* coeffs, int nq, double* out,
                       void* stream);

/* ---------------------------------------------------------------- reaction-diffusion (config 4)
 * cpm_rd_step — one IMEX Euler step of the Schnakenberg system on the surface
 * (BASELINE.json configs[4]; the paper's time-dependent examples treat diffusion
 * implicitly and the nonlinear coupling explicitly):
 *   u_t = mu1 Delta_S u + gamma (a - u + u^2 v),  v_t = mu2 Delta_S v + gamma (b - u^2 v)
 *   (c_i I - Delta_S^h) w1 = c_i (w0 + dt R_w(u0, v0)),  c_i = 1/(dt mu_i)      (reading R14)
 * i.e. two shifted solves of Eq. 2 (GMRES(restart), rtol, warm-started from w0).
 * u, v: DEVICE arrays of nA doubles, updated in place.  su, sv: statistics of the
 * two solves (may be NULL).  Synchronises `stream`.
 * Errors: CPM_ERR_ARG (null / host pointers, dt or mu_i <= 0), those of cpm_solve. */
typedef struct cpm_rd_params {
  double a, b, gamma, mu1, mu2, dt;
  double rtol;
  int32_t restart, maxit;
} cpm_rd_params;
int cpm_rd_step(const cpm_band* band, const cpm_rd_params* params, double* u, double* v,
                cpm_solve_stats* su, cpm_solve_stats* sv, void* stream);

/* cpm_part_rd_step — cpm_rd_step on this rank's owned slices of u and v (DEVICE
 * arrays of n_owned doubles, updated in place): the reaction terms pointwise on the
 * slice, then the two shifted solves by cpm_part_solve (halo exchanges and Krylov
 * allreduces over comm; collective: every rank calls it).  Synchronises `stream`.
 * Errors: those of cpm_rd_step and cpm_part_solve. */
int cpm_part_rd_step(const cpm_part* part, const cpm_comm* comm, const cpm_rd_params* params,
                     double* u_owned, double* v_owned, cpm_solve_stats* su, cpm_solve_stats* sv,
                     void* stream);

/* ---------------------------------------------------------------- profiling
 * When enabled, every kernel launched by the library on the caller's stream is
 * bracketed by CUDA events; cpm_profile_read sums the device time (ms) and the
 * launch count per kernel name since the last reset.  Names: "extend",
 * "laplace", "mdot", "cgs_update", "cgs_final", "axpy", "other". */
int cpm_profile_enable(int on);
int cpm_profile_reset(void);
int cpm_profile_read(const char* name, double* ms, int64_t* launches);
int64_t cpm_kernel_launches(void); /* total kernels launched by the library (all names) */

#ifdef __cplusplus
}
#endif
#endif /* CPM_H_ */
