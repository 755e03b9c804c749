/*
 * ader.h — C ABI of the B200-native ADER-WENO hot path (arXiv:1212.3585).
 *
 * extern "C", FP64 throughout, plain pointers and sizes, no torch types.
 * One context = one rank = one GPU.  A context is single-writer: calls on the
 * same context must not overlap (they may run on different contexts in
 * different threads).  Every call returns an ader_status; on failure
 * ader_last_error(ctx) holds a one-line reason (with cell index, level and
 * time for solver failures, following SPEC S:47/S:88).
 *
 * Citations: P:a-b = PAPER.md lines a..b with the equation label they fall in.
 *
 * What one macro step computes (ader_step), on the active cells of every
 * level:
 *   a1 WENO reconstruction, dimension by dimension
 *   a2 local space-time DG predictor (Picard iteration) P:331-474
 *   a3 space-time Gauss quadrature of the Rusanov flux
 *   a4 one-step finite-volume update                     eq:finite_vol P:147-152
 *   a8 CFL time step dt0 = cfl / max sum_dir s_dir/dx_dir (reading R1)
 * Level-0 cells are partitioned in Cartesian blocks over world_size ranks;
 * ghost layers are exchanged with NCCL (P:794-810 is the paper's MPI form).
 */
#ifndef ADER_H
#define ADER_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define ADER_ABI_VERSION 6

typedef struct ader_ctx ader_ctx;   /* opaque; owns all device memory it allocates */

typedef enum {
  ADER_OK = 0,
  ADER_ERR_ARG = 1,      /* null pointer, capacity too small, bad enum            */
  ADER_ERR_CONFIG = 2,   /* configuration rejected before any allocation  */
  ADER_ERR_SOLVER = 3,   /* inadmissible state (rho<=0 or p<=0) or predictor cap  */
  ADER_ERR_CUDA = 4,     /* CUDA runtime error or no sm_100 device                */
  ADER_ERR_NCCL = 5,     /* NCCL missing or failed                                */
  ADER_ERR_UNSUPPORTED = 6
} ader_status;

typedef enum { ADER_EULER = 0, ADER_MHD_GLM = 1 } ader_system;
typedef enum { ADER_BC_PERIODIC = 0,
               ADER_BC_TRANSMISSIVE = 1,   /* reading R5 */
               ADER_BC_REFLECTIVE = 2,     /* reflecting wall, reading R22 (Euler only) */
               ADER_BC_INFLOW = 3,         /* Dirichlet inflow: the ghost layer keeps the IC cell
                                            * averages (reading R23; uniform grids) */
               ADER_BC_EXACT = 4           /* time-dependent Dirichlet "exact solution prescribed"
                                            * (P:1103-1105): before every step the ghost layer takes
                                            * the cell averages of ic(x - t exact_vel), the initial
                                            * condition translated with the front velocity
                                            * exact_vel (reading R26; uniform grids) */
} ader_bc;
/* Two-point flux of the space-time face quadrature. */
typedef enum { ADER_FLUX_RUSANOV = 0,   /* eqn.rusanov @ P:181-185                  */
               ADER_FLUX_OSHER = 1      /* eqn.osher @ P:186-196, Euler only         */
} ader_flux;

/* Problem statement.  All lengths in cells. */
typedef struct {
  int32_t abi_version;          /* must be ADER_ABI_VERSION                        */
  int32_t dim;                  /* d in {2,3}                                      */
  int32_t system;               /* ader_system: Euler nu = d+2 (2D nu=4), MHD nu=9 */
  int32_t degree;               /* M in {2,3}: order M+1 in space and time         */
  int32_t n0[3];                /* level-0 cells per axis (global); n0[2]=1 if d=2 */
  double  lo[3], hi[3];         /* domain box                                      */
  int32_t bc[6];                /* ader_bc for -x,+x,-y,+y,-z,+z                   */
  int32_t refine_factor;        /* r >= M                              */
  int32_t lmax;                 /* 0 = uniform grid                                */
  double  gamma;                /* ideal-gas adiabatic index                       */
  double  ch;                   /* GLM cleaning speed (MHD only)           */
  double  cfl;                  /* reading R1 (BASELINE: 0.9)                      */
  double  chi_ref, chi_rec, chi_eps;   /* indicator thresholds         */
  int32_t indicator_var;        /* 0 = rho                                 */
  double  pred_tol;             /* Picard stopping tolerance (reading R2), 1e-13   */
  int32_t pred_max_sweeps;      /* cap (reading R2), 32; reaching it = solver error*/
  int32_t ic_quad;              /* GL points per axis for IC cell averages (R6); 0 = M+1 */
  int32_t adapt_every;          /* macro steps between adapts (AMR); 0 = frozen    */
  int32_t rank, world_size;     /* one rank per GPU; world_size=1 => no NCCL       */
  int32_t device;               /* CUDA device ordinal; -1 = current device        */
  uint8_t nccl_id[128];         /* ncclUniqueId from rank 0 (ader_nccl_unique_id)  */
  int32_t flux;                 /* ader_flux; ADER_FLUX_OSHER needs system=EULER   */
  int32_t flux_quad;            /* Gauss-Legendre points of the Osher path integral
                                 * ("at least two"), 1..4; 0 = 3 (R21)   */
  int32_t load_balance;         /* AMR, world_size > 1: 0 = static Cartesian blocks
                                 * (ader_partition); 1 = dynamic: after every adapt the
                                 * level-0 cells are re-cut by ader_rcb_partition on
                                 * their subtrees' local steps when that lowers the
                                 * imbalance (reading R24; the paper's future work,
                                 * P:809-810)                                       */
  int32_t pred_guess;           /* Picard initial guess, uniform grids: 0 = the
                                 * time-constant extension of w_h (reading R3); 1 = the
                                 * previous step's q_h of the cell extrapolated in time,
                                 * q0 = w + q_prev(1 + r tau) - q_prev(1), r = dt_n /
                                 * dt_{n-1} (reading R25; R3 on the first step after
                                 * set_initial / set_cells)                         */
  double  exact_vel[3];         /* ADER_BC_EXACT sides: front velocity of the exact
                                 * solution u(x, t) = ic(x - t exact_vel) (R26)     */
  int32_t fuse_pred_flux;       /* uniform grids: 0 = separate a2 (predictor) and a3
                                 * (face flux) kernels with q_h in HBM (default); 1 = both
                                 * in one tile walk with q_h kept on chip (pred_flux.cu;
                                 * measured slower at C4; ignored with
                                 * pred_guess = 1, which reads the previous q_h).  The
                                 * same fluxes either way (bitwise for Euler).         */
} ader_config;

/* Batched IC callback (host): x[n][3] -> prim[n][9] with
 * prim = (rho, vx, vy, vz, p, Bx, By, Bz, psi).  Euler reads the first five. */
typedef void (*ader_ic_fn)(const double* x, int64_t n, double* prim, void* user);

typedef struct {
  double  t, dt0;                 /* time reached, last level-0 dt                 */
  int64_t macro_steps;            /* level-0 steps taken by this call              */
  int64_t cell_updates;           /* active-cell local steps, this rank*/
  int64_t updates_per_level[8];
  int64_t pred_sweeps_total;      /* Picard sweeps summed over predicted cells     */
  int32_t pred_sweeps_max;
  int32_t rebalances;             /* dynamic load-balancing repartitions (R24)     */
  int64_t pred_cells;             /* cells run through the predictor (incl. halo)  */
  double  cons_total[9];          /* sum of u * cell volume over owned active cells*/
  double  wall_s;
  double  min_threshold_margin;   /* AMR: min over the adapts of this call and their
                                   * active cells of min(|chi - chi_ref| / chi_ref,
                                   * |chi - chi_rec| / chi_rec) — how close a strict
                                   * threshold comparison came to flipping
                                   * a refinement decision; 1e300 if no adapt ran     */
  int64_t pred_flat_cells;        /* of pred_cells: cells whose nodes all carried the same
                                   * reconstruction w bit for bit and that converged in the
                                   * first Picard sweep (eqn.stdg.final P:463-474 with the
                                   * time-constant guess, R3; counted at M = 2) — how much
                                   * of the workload is constant-state streaming (ABI 6)  */
} ader_step_report;

/* One cell as exported by ader_get_cells: parity key (level, idx, status). */
typedef struct {
  int32_t level;
  int32_t status;                 /* 0 active, +1 virtual child, -1 virtual mother */
  int64_t idx[3];                 /* integer index at its level (global)           */
  double  u[9];                   /* cell average (first nu entries valid)         */
} ader_cell;

/* Block of level-0 cells owned by a rank (host-only, no GPU needed). */
typedef struct {
  int32_t dims[3];                /* process grid                                  */
  int32_t coord[3];               /* this rank's coordinate in the process grid    */
  int32_t lo[3], hi[3];           /* owned global cells [lo, hi)                   */
  int32_t nbr[6];                 /* neighbour rank on -x,+x,-y,+y,-z,+z; -1 none  */
  int32_t halo;                   /* ghost-layer width (M+1)                       */
} ader_partition_info;

/* --- lifecycle ------------------------------------------------------------ */
/* Validates cfg before any allocation (ADER_ERR_CONFIG: dim/degree/system out
 * of range, r < M, n0 < 1, world_size not in 1..8, rank out of range).  On
 * success *out owns device memory on cfg->device; release with ader_destroy. */
ader_status ader_create(const ader_config* cfg, ader_ctx** out);
void        ader_destroy(ader_ctx* c);
const char* ader_last_error(const ader_ctx* c);
/* Use the given cudaStream_t for all work (e.g. torch's current stream);
 * NULL restores the context's own stream. */
ader_status ader_set_stream(ader_ctx* c, void* cuda_stream);

/* --- state ---------------------------------------------------------------- */
/* Host-evaluated IC: ic is called on batches of Gauss-Legendre points
 * x = lo + (i + lambda_k) dx (reading R6), the cell averages are formed on
 * the GPU.  Then (lmax > 0) the initial refinement runs up to lmax. */
ader_status ader_set_initial(ader_ctx* c, ader_ic_fn ic, void* user);
/* Owned level-0 cell averages from a host buffer u[cell][nu], cells ordered
 * x fastest then y then z inside the rank's block; n_cells must equal the
 * block size.  Synchronous. */
ader_status ader_set_cells(ader_ctx* c, const double* u_host, int64_t n_cells);
/* Compact copy of the owned level-0 averages into u_host[cell][nu] (same
 * order as ader_set_cells).  Synchronous. */
ader_status ader_get_state(const ader_ctx* c, double* u_host, int64_t capacity_cells);
/* All cells of this rank (every status) sorted by (level, z, y, x);
 * out == NULL => *n = count only.  Synchronous. */
ader_status ader_get_cells(const ader_ctx* c, ader_cell* out, int64_t capacity, int64_t* n);
double      ader_time(const ader_ctx* c);

/* One macro step with the state crossing the host boundary (the e2e path):
 * in_host (optional, [owned cell][nu] like ader_set_cells) is copied in first;
 * out_host receives the owned state after the step ([owned cell][nu], like
 * ader_get_state).  The face fluxes and the update run in slabs along the
 * last axis and each finished slab is copied to out_host on a second stream
 * while the next slabs' fluxes run, so most of the device-to-host copy
 * overlaps the step; the result is bitwise that of ader_set_cells +
 * ader_step(1) + ader_get_state.  in_host may equal out_host.  Host buffers
 * should be pinned for the copies to overlap.  Uniform grids
 * (ADER_ERR_UNSUPPORTED on AMR). */
ader_status ader_step_io(ader_ctx* c, const double* in_host, double* out_host, double t_end, ader_step_report* rep);

/* --- time stepping ---------------------------------------------------------- */
/* Whole level-0 macro steps until t >= t_end or max_macro_steps were taken:
 * dt0 = cfl / max over active cells of sum_dir s_dir/dx_dir (all ranks),
 * clipped to t_end; then a1..a4 on every level in LTS order;
 * adapt every adapt_every macro steps (AMR).  rep may be NULL. */
ader_status ader_step(ader_ctx* c, double t_end, int64_t max_macro_steps, ader_step_report* rep);
/* One adapt pass at synchronized time.  Uniform grids: no-op. */
ader_status ader_refine(ader_ctx* c, ader_step_report* rep);

/* --- multi-GPU plumbing (host only) ---------------------------------------- */
ader_status ader_partition(const ader_config* cfg, int32_t rank, ader_partition_info* out);
/* Ghost-layer plan of one side of one axis for a rank (host only).  Boxes are
 * in the rank's padded coordinates (owned cells start at H = M+1 on every active
 * axis).  Axes are filled in order x, y, z; for axis a, the extent on axes < a
 * covers the full padded range (so edges and corners propagate), on axes > a
 * the owned range.  kind: 0 axis unused, 1 exchange with `peer` (send
 * send_lo..send_hi, receive into recv_lo..recv_hi; NCCL order per peer: send
 * low, recv high, send high, recv low), 2 periodic wrap onto itself, 3
 * transmissive copy of the nearest owned cell (reading R5), 4 reflective
 * mirror of the owned cells with the normal momentum negated (R22), 5 inflow
 * (the ghost cells keep their initial values, R23), 6 exact (the ghost cells
 * are set from the translated initial condition before every step, R26). */
typedef struct {
  int32_t kind, peer;
  int32_t send_lo[3], send_hi[3];
  int32_t recv_lo[3], recv_hi[3];
} ader_halo_desc;
ader_status ader_halo_plan(const ader_config* cfg, int32_t rank, int32_t axis, int32_t side, ader_halo_desc* out);
/* Dynamic load balancing of the AMR level-0 cells (reading R24; host only).
 * Recursive coordinate bisection: the box is cut across its longest axis
 * (lowest axis on ties) at the plane that brings the lower part's weight
 * closest to floor(np/2)/np of the box total (first such plane), leaving at
 * least as many planes as ranks on each side, and both halves recurse; rank
 * p0.. takes the lower part.  weights[n0[0]*n0[1]*n0[2]] (x fastest) are the
 * per-level-0-cell costs (the solver uses sum over active subtree cells of
 * r^level, i.e. local steps per macro step); boxes[world][6] receives lo[3],
 * hi[3] per rank.  ADER_ERR_ARG if an axis is too short to give every rank a
 * plane, or on bad arguments. */
ader_status ader_rcb_partition(int32_t dim, const int32_t n0[3], const int64_t* weights, int32_t world,
                               int32_t* boxes);
/* Collectives of a rank group supplied by the caller on the host (e.g. an MPI
 * or gloo process group) instead of NCCL: the library stages device buffers
 * through pinned host memory and synchronises its stream around every call.
 * Each callback returns 0 on success; any other value fails the step with
 * ADER_ERR_NCCL.
 *   p2p: n entries; to peers[i] send scount[i] doubles from send[i], from
 *        peers[i] receive rcount[i] doubles into recv[i] (counts may be 0).
 *        Messages between one pair of ranks must be matched in entry order
 *        (the library orders its entries so that both sides agree).
 *   allreduce_sum / allreduce_max_u64: in place over all ranks.
 * The pointers passed to the callbacks are valid only during the call. */
typedef struct {
  void* user;
  int32_t (*p2p)(void* user, int32_t n, const int32_t* peers, const double* const* send, const int64_t* scount,
                 double* const* recv, const int64_t* rcount);
  int32_t (*allreduce_sum)(void* user, double* buf, int64_t n);
  int32_t (*allreduce_max_u64)(void* user, uint64_t* buf, int64_t n);
} ader_host_comm;
/* ader_create for rank cfg->rank of a group of cfg->world_size >= 2 processes
 * whose collectives go through *comm (copied; comm->user must outlive the
 * context).  cfg->nccl_id is ignored.  Errors as ader_create; ADER_ERR_ARG if
 * a callback is missing. */
ader_status ader_create_host_comm(const ader_config* cfg, const ader_host_comm* comm, ader_ctx** out);
/* 128-byte ncclUniqueId for rank 0 to broadcast (loads libnccl.so.2 lazily). */
ader_status ader_nccl_unique_id(uint8_t out[128]);

/* --- instrumentation / test hooks ---------------------------------------- */
enum { ADER_K_WENO = 0, ADER_K_PRED = 1, ADER_K_FLUX = 2, ADER_K_UPDATE = 3,
       ADER_K_HALO = 4, ADER_K_OTHER = 5, ADER_K_PRED_FLUX = 6 /* fused a2 + a3 tile walk */,
       ADER_K_COUNT = 7 };
/* When on, every kernel launch is bracketed by CUDA events on the launch
 * stream; ader_kernel_stats returns, per kernel class, total device ms,
 * launch count and the algorithmic FP64 flops of those launches. */
ader_status ader_set_profiling(ader_ctx* c, int32_t on);
ader_status ader_kernel_stats(ader_ctx* c, double ms[ADER_K_COUNT], int64_t launches[ADER_K_COUNT],
                              double flops[ADER_K_COUNT]);
/* Number of kernels this context has launched since ader_create. */
ader_status ader_launch_count(const ader_ctx* c, int64_t* n);
/* Test-only rank group in ONE process on one GPU (no NCCL): creates the n
 * contexts of the partition of cfg (rank i = out[i], world_size = n) whose
 * exchanges (uniform: ghost slabs; AMR: owners' averages into the other ranks'
 * compute bands, the global indicator) are device-to-device copies / host
 * merges; ader_debug_group_set_initial and ader_debug_group_step run all of
 * them in lockstep with the same phases as ader_set_initial / ader_step (the
 * CFL max over ranks is taken on the host).  Used to check that the
 * partitioned path reproduces the one-rank result bitwise.  ader_step,
 * ader_refine (and, for AMR, ader_set_initial) on a group context return
 * ADER_ERR_ARG.  Release each context with ader_destroy.  reps may be NULL or
 * hold n reports.  ader_get_cells of an AMR rank returns its own subtrees. */
ader_status ader_debug_group_create(const ader_config* cfg, int32_t n, ader_ctx** out);
ader_status ader_debug_group_set_initial(ader_ctx** ctxs, int32_t n, ader_ic_fn ic, void* user);
ader_status ader_debug_group_step(ader_ctx** ctxs, int32_t n, double t_end, int64_t max_macro_steps,
                                  ader_step_report* reps);
/* sizeof of the ABI structs as compiled into the library (no GPU needed), so a
 * binding can check its layout: what = 0 ader_config, 1 ader_step_report,
 * 2 ader_cell, 3 ader_partition_info, 4 ader_halo_desc; -1 for other values. */
int64_t ader_sizeof(int32_t what);
/* Test-only dumps of one stage on the current state (state not modified):
 *   what = 0 RECON: w[cell][nu][N^d]           (owned cells, x-fastest nodes)
 *   what = 1 PRED : q[cell][nu][N^(d+1)]       (space fastest, time slowest), step dt
 *   what = 2 FLUX : F[dir][ext cell][nu]        ext box = block + 1 per axis, lower faces
 * capacity in doubles. */
/* Uniform grids only; a loopback group context (ader_debug_group_create) is
 * rejected with ADER_ERR_ARG. */
ader_status ader_debug_dump(ader_ctx* c, int32_t what, double dt, double* out, int64_t capacity);

#ifdef __cplusplus
}
#endif
#endif
