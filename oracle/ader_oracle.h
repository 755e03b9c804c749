/*
 * ader_oracle.h — CPU ORACLE of the ADER-WENO hot path (arXiv:1212.3585).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load, call or link
 * anything under oracle/.  The product path (paper_1212_3585_b200/) never
 * does, and shares no code, header, table or helper with this file.
 *
 * Citation format: "P:a-b" = lines a..b of PAPER.md (the LaTeX source of the
 * paper), with the section / equation label they fall in.
 *
 * All arithmetic is IEEE FP64, single threaded, compiled with
 * -O2 -ffp-contract=off (no FMA contraction, no fast-math).
 */
#ifndef ADER_ORACLE_H
#define ADER_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAXN 5            /* nodes per axis, N = M+1 <= 5                */
#define ORC_MAXV 9            /* conserved variables (MHD-GLM)               */

enum { ORC_EULER = 0, ORC_MHD = 1 };
enum { ORC_BC_PERIODIC = 0, ORC_BC_TRANSMISSIVE = 1, ORC_BC_REFLECTIVE = 2,   /* reflective: Euler only (R22) */
       ORC_BC_INFLOW = 3,     /* Dirichlet inflow: ghost cells keep the IC averages (R23), uniform grids */
       ORC_BC_EXACT = 4 };    /* time-dependent Dirichlet: before every step the ghost cells take the
                               * averages of the exact solution ic(x - t exact_vel) (R26), uniform grids */
enum { ORC_FLUX_RUSANOV = 0, ORC_FLUX_OSHER = 1 };   /* eqn.rusanov / eqn.osher */

typedef struct {
  int32_t dim, system, degree;       /* d in {2,3}; M in {2,3}              */
  int32_t n[3];                      /* level-0 cells per axis (n[2]=1, d=2) */
  double lo[3], hi[3];
  int32_t bc[6];                     /* -x,+x,-y,+y,-z,+z                   */
  double gamma, ch, cfl;
  double pred_tol; int32_t pred_max_sweeps;
  int32_t ic_quad;                   /* GL points per axis for IC averages   */
  /* AMR (used by the AMR oracle; lmax = 0 means uniform grid) */
  int32_t refine_factor, lmax;
  double chi_ref, chi_rec, chi_eps;
  /* numerical flux: ORC_FLUX_RUSANOV or ORC_FLUX_OSHER (Euler
   * only); flux_quad = Gauss-Legendre points of the Osher path integral */
  int32_t flux, flux_quad;
  /* Picard initial guess (uniform grids): 0 = time-constant extension
   * of w_h (reading R3), 1 = the previous step's q_h of the same cell
   * extrapolated in time (reading R25, orc_extrapolate_guess) */
  int32_t pred_guess;
  /* ORC_BC_EXACT sides: the exact solution is the initial condition translated
   * with this constant front velocity, u(x, t) = ic(x - t exact_vel) (R26) */
  double exact_vel[3];
} orc_config;

/* Batched initial-condition callback: x[n][3] -> prim[n][9]
 * prim = (rho, vx, vy, vz, p, Bx, By, Bz, psi); Euler reads the first 5. */
typedef void (*orc_ic_fn)(const double* x, int64_t n, double* prim, void* user);

typedef struct orc_ctx orc_ctx;

typedef struct {
  double t, dt;
  int64_t steps, cell_updates, sweeps_total;
  int32_t sweeps_max;
  int64_t updates_per_level[8];
  /* AMR: min over the adapts of the call and their active cells of
   * min(|chi - chi_ref| / chi_ref, |chi - chi_rec| / chi_rec): how close any
   * strict threshold comparison of P:622-624 came to flipping (1e300 if no
   * adapt ran) */
  double min_threshold_margin;
} orc_report;

/* ---- tables / pure per-cell numerics (for pins) ---------------------- */
int  orc_nvar(int system, int dim);
/* Basis tables for degree M.  Any pointer may be NULL.
 * lam,w [N]; psi0,psi1 [N]; Sigma [N*N]; rec [nS*N*N] (rec[s][p][o]);
 * stencil L,R,lin [nS]; M1,Kx1,K1t [N*N] row-major [test][trial]; returns nS. */
int  orc_basis_tables(int M, double* lam, double* w, double* psi0, double* psi1,
                      double* Sigma, double* rec, int* L, int* R, double* lin,
                      double* M1, double* Kx1, double* K1t);
/* Dense predictor operators (eqn.pde.weak4 @ P:451-459) for (d, M):
 * NST = N^(d+1), NS = N^d.  K1 [NST*NST], Kdir [d][NST*NST], F0 [NST*NS]. */
int  orc_predictor_matrices(int d, int M, double* K1, double* Kdir, double* F0);
void orc_weno_1d(int M, const double* win, double* out);
/* Dimension-by-dimension WENO of one cell from its (2M+1)^d box of cell
 * averages ubox[box][nv] (x fastest) -> w[nv][N^d] (x fastest). */
int  orc_reconstruct_box(int d, int M, int nv, const double* ubox, double* w);
/* Space-time predictor (eqn.stdg.final @ P:463-474): w[nv][N^d] ->
 * q[nv][N^(d+1)] (space fastest, time slowest).  dtdx[d] = dt/dx_dir.
 * Returns 0 on success, 3 on non-convergence or inadmissible state. */
int  orc_predict_cell(int d, int M, int system, double gamma, double ch,
                      const double* w, const double* dtdx, double tol, int max_sweeps,
                      double* q, int* sweeps);
/* orc_predict_cell from the initial guess q0[nv][N^(d+1)] (NULL: R3). */
int  orc_predict_cell_guess(int d, int M, int system, double gamma, double ch,
                            const double* w, const double* dtdx, double tol, int max_sweeps,
                            const double* q0, double* q, int* sweeps);
/* Reading R25 (the extrapolation initial guess of P:472): from the previous
 * step's space-time polynomial qp[nv][N^(d+1)] of the cell over [t^{n-1}, t^n]
 * and the new reconstruction w[nv][N^d] at t^n,
 *   q0(x_node, tau_s) = w(x_node) + qp(x_node, 1 + r tau_s) - qp(x_node, 1),
 * r = dt_n / dt_{n-1}: the old time evolution carried forward, anchored at the
 * new w.  Exact for a solution polynomial of degree <= M in t. */
void orc_extrapolate_guess(int d, int M, int nv, const double* w, const double* qp, double r, double* q0);
/* Space-time face flux (flux:F/G/H @ P:158-172) of the selected two-point flux
 * (eqn.rusanov @ P:181-185 or eqn.osher @ P:186-196)
 * between the left (lower) cell qL and right (upper) cell qR along dir.  At a
 * transmissive boundary face pass NULL for the exterior side: it takes the
 * interior trace (q^+ = q^-, reading R5). */
int  orc_face_flux(int d, int M, int system, double gamma, double ch, int flux, int nq, int dir,
                   const double* qL, const double* qR, double* F);
int  orc_phys_flux(int system, int dim, double gamma, double ch, const double* u, int dir, double* f);
double orc_max_speed(int system, int dim, double gamma, double ch, const double* u, int dir);
int  orc_rusanov(int system, int dim, double gamma, double ch, const double* uL,
                 const double* uR, int dir, double* f);
/* Reflected space-time polynomial across a wall normal to dir (reading R22):
 * node order reversed along dir (the GL nodes are symmetric, lambda_{N-1-a} =
 * 1 - lambda_a) and the normal momentum negated.  q, out [nv][N^(d+1)]. */
void orc_reflect_poly(int d, int M, int nv, int dir, const double* q, double* out);
/* Euler Jacobian A_dir = df_dir/du (analytic, row-major nv x nv). */
int  orc_euler_jacobian(int dim, double gamma, const double* u, int dir, double* A);
/* |A_dir(u)| for Euler by Sylvester's formula over the three distinct
 * eigenvalues v_n - c, v_n, v_n + c (A is diagonalisable). */
int  orc_euler_abs_jacobian(int dim, double gamma, const double* u, int dir, double* absA);
/* eqn.osher @ P:186-196 along the straight path psi(s) = uL + s (uR - uL),
 * the path integral by an nq-point Gauss-Legendre rule (Euler only). */
int  orc_osher(int system, int dim, double gamma, int nq, const double* uL, const double* uR, int dir, double* f);
/* The selected two-point flux: flux = ORC_FLUX_RUSANOV or ORC_FLUX_OSHER. */
int  orc_numflux(int system, int dim, double gamma, double ch, int flux, int nq, const double* uL,
                 const double* uR, int dir, double* f);
void orc_prim_to_cons(int system, int dim, double gamma, const double* prim, double* u);
/* q_h(xi, tau) = theta_p(xi, tau) q_p (eqn.st.q @ P:391-394), q[nv][N^(d+1)]. */
void orc_eval_st(int d, int M, int nv, const double* q, const double* xi, double tau, double* out);
/* w_h(xi) = psi_p(xi) w_p (eqn.weno.z @ P:314-317), w[nv][N^d]. */
void orc_eval_w(int d, int M, int nv, const double* w, const double* xi, double* out);
/* n-point Gauss-Legendre rule on [0,1]. */
void orc_gauss_legendre(int n, double* x, double* w);
/* Space-time two-point flux along dir integrated over the face sub-box of the
 * left cell qL and right cell qR: the face points are given in each cell's
 * reference coordinates by affine maps xi = a + b * eta (eta the fine face /
 * time GL nodes), i.e. for cell X: xi_k = offX[k] + sclX * eta_k on the
 * tangential axes, xi_dir = posX, tau = toffX + tsclX * eta_t.  NULL side =
 * transmissive boundary (interior trace on both sides).  Used by the AMR
 * oracle for same-level and coarse-fine faces. */
int  orc_face_flux_mapped(int d, int M, int system, double gamma, double ch, int flux, int nq, int dir,
                          const double* qL, const double* offL, double sclL, double toffL, double tsclL,
                          const double* qR, const double* offR, double sclR, double toffR, double tsclR,
                          double* F);
/* Projection of a mother cell's polynomial into its child sub-box off[d]
 * (0 <= off_k < r): mean over the child box of w_h (mode 0,
 * poly = w[nv][N^d]) or of q_h(., tau) (mode 1, poly = q[nv][N^(d+1)]). */
void orc_project_subbox(int d, int M, int nv, int r, int mode, const double* poly, const int* off, double tau,
                        double* out);
/* Loehner-type indicator chi of eqn.indicator in the discretised
 * reading R14 from the 3^d same-level box of Phi (x fastest). */
double orc_indicator(int d, const double* phi, double eps);

/* ---- uniform-grid driver --------------------------------------------- */
orc_ctx* orc_create(const orc_config* cfg);
void     orc_destroy(orc_ctx* c);
const char* orc_last_error(const orc_ctx* c);
int  orc_set_initial(orc_ctx* c, orc_ic_fn ic, void* user);
/* IC averages only for the interior cells of the box [blo, bhi). */
int  orc_set_initial_box(orc_ctx* c, orc_ic_fn ic, void* user, const int32_t* blo, const int32_t* bhi);
/* Interior cell averages, u[cell][nv], cells x fastest then y then z. */
int  orc_set_cells(orc_ctx* c, const double* u);
int  orc_get_cells(const orc_ctx* c, double* u);
double orc_time(const orc_ctx* c);
int64_t orc_num_cells(const orc_ctx* c);
/* CFL time step of the current state (O2), before clipping. */
double orc_compute_dt(orc_ctx* c);
/* Whole steps until t_end or max_steps. */
int  orc_step(orc_ctx* c, double t_end, int64_t max_steps, orc_report* rep);
/* One step of size dt computed only for the interior box [blo,bhi) (cell
 * indices); writes the new averages of the box to out[box cells][nv]
 * (x fastest) and leaves the state untouched.  Used for sampled parity. */
int  orc_advance_box(orc_ctx* c, double dt, const int32_t* blo, const int32_t* bhi,
                     double* out, orc_report* rep);
/* Distributed emulation (tests of the multi-rank host logic): the padded
 * grid [pad cell][nv] with ghost width M+1 (x fastest), and a switch that
 * makes the driver use the ghost cells as given instead of filling them. */
int64_t orc_num_padded(const orc_ctx* c);
int  orc_get_padded(const orc_ctx* c, double* u);
int  orc_set_padded(orc_ctx* c, const double* u);
void orc_set_external_ghosts(orc_ctx* c, int on);
/* Debug: reconstruction / predictor of the interior cells with the current
 * state and step dt.  w[cell][nv][N^d], q[cell][nv][N^(d+1)]. */
int  orc_dump_recon(orc_ctx* c, double* w);
int  orc_dump_pred(orc_ctx* c, double dt, double* q);
/* Debug: face fluxes F[dir][cell][nv] on the lower face of every interior
 * cell, plus the upper boundary faces at index n[dir] (array sized
 * d * (n0+1)(n1+1)(n2+1) * nv, cell index over the (n+1) extended box). */
int  orc_dump_flux(orc_ctx* c, double dt, double* F);

#ifdef __cplusplus
}
#endif
#endif
