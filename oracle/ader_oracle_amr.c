/*
 * ader_oracle_amr.c — CPU ORACLE of the cell-by-cell AMR with time-accurate
 * local time stepping (arXiv:1212.3585 Sect. 3).  TEST INFRASTRUCTURE ONLY
 * (same rules as ader_oracle.c: only tests/, smoke() and bench.py's CPU legs
 * may load it; it shares nothing with paper_1212_3585_b200/).
 *
 * Followed literally, in the paper's order:
 *   tree rules 1-7 (status 0 active, +1 virtual child, -1 virtual mother,
 *     r^d consecutive children, Voronoi closure, <=1 level jump, recoarsening)
 *                                                          P:520-584
 *   refinement indicator (reading R14 of eqn.indicator)
 *   update criterion / r^l substeps, finest level first
 *   coarse-fine fluxes with flux memory (eqn.memory.sum)
 *   projection of the mother's q_h into virtual children
 *   averaging of virtual mothers (eqn.average)
 * Readings: R15 recursive LTS order (predict level l at the start
 * of its step, update it at the end), R16 ghost refresh before every level
 * step, R17 order-independent adapt (closure to the least fixed point, then
 * simultaneous rule-7 recoarsening that the closure may revert, then GC),
 * R18 new active children take sub-box averages of the mother's WENO
 * polynomial at t^{n+1} (conservative), R19 adapt every macro step, R20 the
 * initial hierarchy refines the IC level by level and evaluates the IC on
 * new children.
 */
#include "ader_oracle.h"
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define LMAXX 8
#define VMAX ORC_MAXV

static int g_sched[4096];     /* level update order of the last step (test hook) */
static int g_nsched = 0;

typedef struct {
  int level, status, alive, isnew;
  int64_t idx[3];
  int mother, child;          /* child = first of r^d consecutive ids */
  double u[VMAX];
  double mem[6][VMAX];        /* flux memory on faces -x,+x,-y,+y,-z,+z */
  double* q;                  /* predictor dofs of the current level step */
  double* w;                  /* WENO dofs (adapt) */
  double chi;
} acell;

typedef struct {
  orc_config cfg;
  int d, M, N, nv, NS, NST, r, lmax, rd;
  int64_t n[LMAXX][3];
  int32_t* map[LMAXX];
  double dx[LMAXX][3];
  acell* c;
  int ncap, nused;
  int* freel; int nfree;
  double t;
  orc_ic_fn ic; void* user;
  char err[512];
  int64_t steps, updates[LMAXX], sweeps;
  int sweeps_max;
  double gq[8], gw[8];        /* N-point GL rule for projections */
  double margin;              /* min threshold margin since the last reset (orc_report) */
} amr_t;

/* ---- storage ------------------------------------------------------------ */
static int64_t lin_idx(const amr_t* A, int l, const int64_t* ix) {
  return (ix[2] * A->n[l][1] + ix[1]) * A->n[l][0] + ix[0];
}

static int alloc_block(amr_t* A, int cnt) {
  /* cnt consecutive ids (children must be consecutive) */
  if (A->nused + cnt > A->ncap) {
    int nc = A->ncap * 2 + cnt + 1024;
    A->c = (acell*)realloc(A->c, sizeof(acell) * nc);
    memset(A->c + A->ncap, 0, sizeof(acell) * (nc - A->ncap));
    A->ncap = nc;
  }
  int id = A->nused;
  A->nused += cnt;
  for (int i = 0; i < cnt; ++i) { memset(&A->c[id + i], 0, sizeof(acell)); A->c[id + i].alive = 1; A->c[id + i].mother = -1; A->c[id + i].child = -1; }
  return id;
}

/* Cell at level l and (possibly out-of-domain) index ix: periodic wrap or
 * transmissive clamp per axis (reading R5), reflective mirror (R22: the
 * caller negates the momentum of the axes flagged in *flip), -1 if missing. */
static int lookup_flip(const amr_t* A, int l, const int64_t* ix0, int* flip) {
  int64_t ix[3] = {ix0[0], ix0[1], ix0[2]};
  int fl = 0;
  for (int k = 0; k < A->d; ++k) {
    int64_t n = A->n[l][k];
    if (ix[k] < 0 || ix[k] >= n) {
      int side = ix[k] < 0 ? 0 : 1;
      if (A->cfg.bc[2 * k + side] == ORC_BC_PERIODIC) ix[k] = ((ix[k] % n) + n) % n;
      else if (A->cfg.bc[2 * k + side] == ORC_BC_REFLECTIVE) { ix[k] = ix[k] < 0 ? -1 - ix[k] : 2 * n - 1 - ix[k]; fl |= 1 << k; }
      else ix[k] = ix[k] < 0 ? 0 : n - 1;
    }
  }
  if (A->d == 2) ix[2] = 0;
  if (flip) *flip = fl;
  return A->map[l][lin_idx(A, l, ix)];
}
static int lookup(const amr_t* A, int l, const int64_t* ix0) { return lookup_flip(A, l, ix0, NULL); }

static int outside(const amr_t* A, int l, const int64_t* ix) {
  for (int k = 0; k < A->d; ++k)
    if (ix[k] < 0 || ix[k] >= A->n[l][k]) return 1;
  return 0;
}

static void cell_center_lo(const amr_t* A, int id, double* lo) {
  const acell* C = &A->c[id];
  for (int k = 0; k < 3; ++k) lo[k] = (k < A->d) ? A->cfg.lo[k] + (double)C->idx[k] * A->dx[C->level][k] : 0.0;
}

/* create the r^d children of cell m with a given status */
static int make_children(amr_t* A, int m, int status) {
  int r = A->r, d = A->d, l = A->c[m].level + 1;
  int id = alloc_block(A, A->rd);
  acell* M = &A->c[m];
  M->child = id;
  for (int q = 0; q < A->rd; ++q) {
    acell* C = &A->c[id + q];
    int off[3] = {q % r, (q / r) % r, (d == 3) ? q / (r * r) : 0};
    C->level = l; C->status = status; C->mother = m;
    for (int k = 0; k < 3; ++k) C->idx[k] = (k < d) ? M->idx[k] * r + off[k] : 0;
    A->map[l][lin_idx(A, l, C->idx)] = id + q;
  }
  return id;
}

static void destroy_children(amr_t* A, int m) {
  int ch = A->c[m].child;
  if (ch < 0) return;
  for (int q = 0; q < A->rd; ++q) {
    acell* C = &A->c[ch + q];
    if (C->child >= 0) destroy_children(A, ch + q);
    A->map[C->level][lin_idx(A, C->level, C->idx)] = -1;
    free(C->q); free(C->w);
    memset(C, 0, sizeof(*C));
  }
  A->c[m].child = -1;
}

/* ---- IC --------------------------------------------------------------- */
static void ic_cells(amr_t* A, const int* ids, int cnt) {
  int Q = A->cfg.ic_quad, d = A->d, nv = A->nv;
  double qx[16], qw[16];
  orc_gauss_legendre(Q, qx, qw);
  int nq = 1;
  for (int k = 0; k < d; ++k) nq *= Q;
  double* x = (double*)malloc(sizeof(double) * (size_t)cnt * nq * 3);
  double* pr = (double*)calloc((size_t)cnt * nq * 9, sizeof(double));
  for (int i = 0; i < cnt; ++i) {
    const acell* C = &A->c[ids[i]];
    for (int g = 0; g < nq; ++g) {
      int gi[3] = {g % Q, (g / Q) % Q, g / (Q * Q)};
      for (int k = 0; k < 3; ++k)
        x[((size_t)i * nq + g) * 3 + k] = (k < d) ? A->cfg.lo[k] + ((double)C->idx[k] + qx[gi[k]]) * A->dx[C->level][k] : 0.0;
    }
  }
  A->ic(x, (int64_t)cnt * nq, pr, A->user);
  for (int i = 0; i < cnt; ++i) {
    double acc[VMAX] = {0};
    for (int g = 0; g < nq; ++g) {
      int gi[3] = {g % Q, (g / Q) % Q, g / (Q * Q)};
      double wg = 1.0;
      for (int k = 0; k < d; ++k) wg *= qw[gi[k]];
      double uu[VMAX];
      orc_prim_to_cons(A->cfg.system, d, A->cfg.gamma, &pr[((size_t)i * nq + g) * 9], uu);
      for (int v = 0; v < nv; ++v) acc[v] += wg * uu[v];
    }
    memcpy(A->c[ids[i]].u, acc, sizeof(double) * nv);
  }
  free(x); free(pr);
}

/* ---- per-cell numerics on the tree ------------------------------------ */
static int gather_box(const amr_t* A, int id, double* box) {
  const acell* C = &A->c[id];
  int M = A->M, nv = A->nv, b = 0;
  int zl = (A->d == 3) ? -M : 0, zh = (A->d == 3) ? M : 0;
  for (int dz = zl; dz <= zh; ++dz)
    for (int dy = -M; dy <= M; ++dy)
      for (int dx = -M; dx <= M; ++dx, ++b) {
        int64_t ix[3] = {C->idx[0] + dx, C->idx[1] + dy, C->idx[2] + dz};
        int fl = 0;
        int n = lookup_flip(A, C->level, ix, &fl);
        if (n < 0) return -1;
        memcpy(&box[b * nv], A->c[n].u, sizeof(double) * nv);
        for (int k = 0; k < A->d; ++k)
          if (fl & (1 << k)) box[b * nv + 1 + k] = -box[b * nv + 1 + k];   /* R22 mirror */
      }
  return 0;
}

static int reconstruct(amr_t* A, int id) {
  int W = 2 * A->M + 1, nb = (A->d == 3) ? W * W * W : W * W;
  double* box = (double*)malloc(sizeof(double) * nb * A->nv);
  if (gather_box(A, id, box)) {
    free(box);
    snprintf(A->err, sizeof(A->err), "missing stencil cell around level %d cell (%lld,%lld,%lld)", A->c[id].level,
             (long long)A->c[id].idx[0], (long long)A->c[id].idx[1], (long long)A->c[id].idx[2]);
    return 3;
  }
  if (!A->c[id].w) A->c[id].w = (double*)malloc(sizeof(double) * A->nv * A->NS);
  orc_reconstruct_box(A->d, A->M, A->nv, box, A->c[id].w);
  free(box);
  return 0;
}

/* Projection of a mother polynomial into the child sub-box `off`:
 * the child's cell average (1/|child|) int_child poly d x, i.e. the mean over
 * xi in prod_k [off_k/r, (off_k+1)/r] of the mother's WENO polynomial w_h
 * (mode 0) or of its space-time polynomial q_h at time fraction tau (mode 1),
 * by the N-point Gauss-Legendre rule on the child box (exact: degree <= M per
 * axis).  Exported for the pins in tests/test_oracle_pins_r2.py. */
void orc_project_subbox(int d, int M, int nv, int r, int mode, const double* poly, const int* off, double tau,
                        double* out) {
  int N = M + 1, np = 1;
  double gq[8], gw[8];
  orc_gauss_legendre(N, gq, gw);
  for (int k = 0; k < d; ++k) np *= N;
  for (int v = 0; v < nv; ++v) out[v] = 0.0;
  for (int g = 0; g < np; ++g) {
    int gi[3] = {g % N, (g / N) % N, g / (N * N)};
    double xi[3], wg = 1.0, val[VMAX];
    for (int k = 0; k < d; ++k) { xi[k] = (off[k] + gq[gi[k]]) / r; wg *= gw[gi[k]]; }
    if (mode == 0) orc_eval_w(d, M, nv, poly, xi, val);
    else orc_eval_st(d, M, nv, poly, xi, tau, val);
    for (int v = 0; v < nv; ++v) out[v] += wg * val[v];
  }
}

/* cell average over child sub-box `off` of the polynomial (mode 0: WENO w,
 * mode 1: space-time q at tau) of cell m */
static void subbox_average(const amr_t* A, int m, const int* off, int mode, double tau, double* out) {
  orc_project_subbox(A->d, A->M, A->nv, A->r, mode, mode == 0 ? A->c[m].w : A->c[m].q, off, tau, out);
}

static void child_off(const amr_t* A, int id, int* off) {
  const acell* C = &A->c[id];
  for (int k = 0; k < 3; ++k) off[k] = (k < A->d) ? (int)(C->idx[k] - A->c[C->mother].idx[k] * A->r) : 0;
}

/* averaging (eqn.average @ P:750-753), children current, recursively */
static void average_into(amr_t* A, int m) {
  acell* Mc = &A->c[m];
  for (int v = 0; v < A->nv; ++v) {
    double s = 0.0;
    for (int q = 0; q < A->rd; ++q) s += A->c[Mc->child + q].u[v];
    Mc->u[v] = s / (double)A->rd;
  }
}

/* ghost refresh of level l at fraction tau of the parent step (R16):
 * virtual mothers of levels >= l by averaging (finest first), virtual
 * children of level l by projection of the mother's q_h. */
static void fill_level(amr_t* A, int l, double tau) {
  for (int lv = A->lmax - 1; lv >= l; --lv)
    for (int i = 0; i < A->nused; ++i)
      if (A->c[i].alive && A->c[i].level == lv && A->c[i].status == -1) average_into(A, i);
  if (l == 0) return;
  for (int i = 0; i < A->nused; ++i) {
    acell* C = &A->c[i];
    if (!C->alive || C->level != l || C->status != 1) continue;
    int off[3];
    child_off(A, i, off);
    if (A->c[C->mother].q) subbox_average(A, C->mother, off, 1, tau, C->u);
  }
}

static int predict(amr_t* A, int id, double dt) {
  int l = A->c[id].level, sw = 0;
  double dtdx[3];
  for (int k = 0; k < A->d; ++k) dtdx[k] = dt / A->dx[l][k];
  if (reconstruct(A, id)) return 3;
  if (!A->c[id].q) A->c[id].q = (double*)malloc(sizeof(double) * A->nv * A->NST);
  int rc = orc_predict_cell(A->d, A->M, A->cfg.system, A->cfg.gamma, A->cfg.ch, A->c[id].w, dtdx,
                            A->cfg.pred_tol, A->cfg.pred_max_sweeps, A->c[id].q, &sw);
  A->sweeps += sw;
  if (sw > A->sweeps_max) A->sweeps_max = sw;
  if (rc) snprintf(A->err, sizeof(A->err), "predictor failed at level %d cell (%lld,%lld,%lld) t=%.17g", l,
                   (long long)A->c[id].idx[0], (long long)A->c[id].idx[1], (long long)A->c[id].idx[2], A->t);
  return rc;
}

/* flux through the face (dir, side) of active cell id at level l in substep
 * m of the parent step.  F is the + direction flux. */
static int cell_face_flux(amr_t* A, int id, int dir, int side, int m, double* F) {
  const acell* C = &A->c[id];
  int l = C->level, d = A->d, nv = A->nv;
  int64_t ix[3] = {C->idx[0], C->idx[1], C->idx[2]};
  ix[dir] += side ? 1 : -1;
  double zero[3] = {0, 0, 0}, offC[3] = {0, 0, 0};
  offC[dir] = side ? 1.0 : 0.0;
  if (outside(A, l, ix) && A->cfg.bc[2 * dir + side] == ORC_BC_REFLECTIVE) {
    /* R22: the wall faces the reflected polynomial of the cell itself */
    double* qr = (double*)malloc(sizeof(double) * nv * A->NST);
    orc_reflect_poly(d, A->M, nv, dir, C->q, qr);
    double offR[3] = {0, 0, 0};
    offR[dir] = side ? 0.0 : 1.0;
    int rc = side ? orc_face_flux_mapped(d, A->M, A->cfg.system, A->cfg.gamma, A->cfg.ch, A->cfg.flux, A->cfg.flux_quad, dir, C->q, offC, 1.0, 0.0, 1.0,
                                         qr, offR, 1.0, 0.0, 1.0, F)
                  : orc_face_flux_mapped(d, A->M, A->cfg.system, A->cfg.gamma, A->cfg.ch, A->cfg.flux, A->cfg.flux_quad, dir, qr, offR, 1.0, 0.0, 1.0,
                                         C->q, offC, 1.0, 0.0, 1.0, F);
    free(qr);
    return rc;
  }
  if (outside(A, l, ix) && A->cfg.bc[2 * dir + side] == ORC_BC_TRANSMISSIVE) {
    /* R5: interior trace on both sides */
    return side ? orc_face_flux_mapped(d, A->M, A->cfg.system, A->cfg.gamma, A->cfg.ch, A->cfg.flux, A->cfg.flux_quad, dir, C->q, offC, 1.0, 0.0, 1.0,
                                       NULL, zero, 0, 0, 0, F)
                : orc_face_flux_mapped(d, A->M, A->cfg.system, A->cfg.gamma, A->cfg.ch, A->cfg.flux, A->cfg.flux_quad, dir, NULL, zero, 0, 0, 0,
                                       C->q, offC, 1.0, 0.0, 1.0, F);
  }
  int nb = lookup(A, l, ix);
  if (nb < 0) { snprintf(A->err, sizeof(A->err), "missing face neighbour"); return 3; }
  const acell* Nb = &A->c[nb];
  if (Nb->status == 0) {
    double offN[3] = {0, 0, 0};
    offN[dir] = side ? 0.0 : 1.0;
    return side ? orc_face_flux_mapped(d, A->M, A->cfg.system, A->cfg.gamma, A->cfg.ch, A->cfg.flux, A->cfg.flux_quad, dir, C->q, offC, 1.0, 0.0, 1.0,
                                       Nb->q, offN, 1.0, 0.0, 1.0, F)
                : orc_face_flux_mapped(d, A->M, A->cfg.system, A->cfg.gamma, A->cfg.ch, A->cfg.flux, A->cfg.flux_quad, dir, Nb->q, offN, 1.0, 0.0, 1.0,
                                       C->q, offC, 1.0, 0.0, 1.0, F);
  }
  if (Nb->status == 1) {
    /* coarse-fine: the virtual neighbour scales the coarse mother's q_h down
     * to the fine face and the fine time step */
    int K = Nb->mother, r = A->r;
    const acell* Kc = &A->c[K];
    /* fine face in K's reference coordinates: K's lower face if K lies on the
     * + side of C, its upper face otherwise; tangential offset = position of
     * the fine cell inside K's r^(d-1) sub-faces (also across periodic wraps) */
    double offK[3] = {0, 0, 0};
    for (int k = 0; k < d; ++k) offK[k] = (double)(C->idx[k] % r) / r;
    offK[dir] = side ? 0.0 : 1.0;
    (void)Kc;
    double toff = (double)m / r, tscl = 1.0 / r;
    int rc = side ? orc_face_flux_mapped(d, A->M, A->cfg.system, A->cfg.gamma, A->cfg.ch, A->cfg.flux, A->cfg.flux_quad, dir, C->q, offC, 1.0, 0.0, 1.0,
                                         Kc->q, offK, 1.0 / r, toff, tscl, F)
                  : orc_face_flux_mapped(d, A->M, A->cfg.system, A->cfg.gamma, A->cfg.ch, A->cfg.flux, A->cfg.flux_quad, dir, Kc->q, offK, 1.0 / r, toff, tscl,
                                         C->q, offC, 1.0, 0.0, 1.0, F);
    if (rc) return rc;
    /* memory variable of the virtual neighbour */
    acell* Nw = &A->c[nb];
    int face = 2 * dir + (side ? 0 : 1);   /* Nb's face toward C */
    for (int v = 0; v < nv; ++v) Nw->mem[face][v] += F[v];
    return 0;
  }
  /* Nb is a virtual mother: sum the memory of C's own virtual children on this
   * face (eqn.memory.sum @ P:693-709), then clear it */
  if (C->child < 0) { snprintf(A->err, sizeof(A->err), "coarse cell without virtual children next to a finer level"); return 3; }
  for (int v = 0; v < nv; ++v) F[v] = 0.0;
  int r = A->r;
  for (int q = 0; q < A->rd; ++q) {
    acell* Vc = &A->c[C->child + q];
    int off[3] = {q % r, (q / r) % r, (d == 3) ? q / (r * r) : 0};
    if (off[dir] != (side ? r - 1 : 0)) continue;
    for (int v = 0; v < nv; ++v) { F[v] += Vc->mem[2 * dir + side][v]; Vc->mem[2 * dir + side][v] = 0.0; }
  }
  for (int v = 0; v < nv; ++v) F[v] = F[v] / (double)A->rd;
  return 0;
}

static int advance(amr_t* A, int l, int m, double dt0) {
  double dt = dt0;
  for (int k = 0; k < l; ++k) dt /= A->r;
  fill_level(A, l, (double)m / A->r);
  for (int i = 0; i < A->nused; ++i)
    if (A->c[i].alive && A->c[i].level == l && A->c[i].status == 0)
      if (predict(A, i, dt)) return 3;
  if (l < A->lmax) {
    int any = 0;
    for (int i = 0; i < A->nused && !any; ++i) any = A->c[i].alive && A->c[i].level == l + 1;
    if (any)
      for (int k = 0; k < A->r; ++k)
        if (advance(A, l + 1, k, dt0)) return 3;
  }
  /* fluxes + update of the active cells of level l (eq:finite_vol) */
  int nv = A->nv;
  double* unew = (double*)malloc(sizeof(double) * (size_t)A->nused * nv);
  for (int i = 0; i < A->nused; ++i) {
    acell* C = &A->c[i];
    if (!C->alive || C->level != l || C->status != 0) continue;
    for (int v = 0; v < nv; ++v) unew[(size_t)i * nv + v] = C->u[v];
    for (int dir = 0; dir < A->d; ++dir) {
      double Fm[VMAX], Fp[VMAX];
      if (cell_face_flux(A, i, dir, 0, m, Fm) || cell_face_flux(A, i, dir, 1, m, Fp)) {
        if (!A->err[0])
          snprintf(A->err, sizeof(A->err), "inadmissible face state at level %d cell (%lld,%lld,%lld) t=%.17g", l,
                   (long long)C->idx[0], (long long)C->idx[1], (long long)C->idx[2], A->t);
        free(unew);
        return 3;
      }
      for (int v = 0; v < nv; ++v) unew[(size_t)i * nv + v] = unew[(size_t)i * nv + v] - dt / A->dx[l][dir] * (Fp[v] - Fm[v]);
    }
    A->updates[l]++;
  }
  if (g_nsched < 4096) g_sched[g_nsched++] = l;
  for (int i = 0; i < A->nused; ++i) {
    acell* C = &A->c[i];
    if (C->alive && C->level == l && C->status == 0) memcpy(C->u, &unew[(size_t)i * nv], sizeof(double) * nv);
  }
  free(unew);
  return 0;
}

/* ======================================================================== */
/* adapt (rules 1-7; indicator P:614-632)                        */
/* ======================================================================== */

static const int kMaxVor = 26;

/* same-level Voronoi neighbours (3^d - 1), -1 where missing / outside */
static int voronoi(const amr_t* A, int id, int* out) {
  const acell* C = &A->c[id];
  int n = 0, zl = (A->d == 3) ? -1 : 0, zh = (A->d == 3) ? 1 : 0;
  for (int dz = zl; dz <= zh; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        if (!dx && !dy && !dz) continue;
        int64_t ix[3] = {C->idx[0] + dx, C->idx[1] + dy, C->idx[2] + dz};
        int o = 0;
        for (int k = 0; k < A->d; ++k)
          if ((ix[k] < 0 || ix[k] >= A->n[C->level][k]) && A->cfg.bc[2 * k + (ix[k] < 0 ? 0 : 1)] != ORC_BC_PERIODIC) o = 1;
        out[n++] = o ? -1 : lookup(A, C->level, ix);
      }
  return n;
}

static double indicator(const amr_t* A, int id) {
  const acell* C = &A->c[id];
  double phi[27];
  int b = 0, zl = (A->d == 3) ? -1 : 0, zh = (A->d == 3) ? 1 : 0;
  for (int dz = zl; dz <= zh; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx, ++b) {
        int64_t ix[3] = {C->idx[0] + dx, C->idx[1] + dy, C->idx[2] + dz};
        int n = lookup(A, C->level, ix);
        phi[b] = (n >= 0) ? A->c[n].u[0] : A->c[id].u[0];   /* Phi = rho */
      }
  return orc_indicator(A->d, phi, A->cfg.chi_eps);
}

/* new active children: IC (t = 0, R20) or sub-box averages of the mother's
 * WENO polynomial at t^{n+1} (R18) */
static void init_new_children(amr_t* A, int m, int at_t0) {
  int ch = A->c[m].child;
  if (!at_t0 && !A->c[m].w) reconstruct(A, m);   /* mother activated during this adapt */
  if (at_t0) {
    int ids[512];
    for (int q = 0; q < A->rd; ++q) ids[q] = ch + q;
    ic_cells(A, ids, A->rd);
    return;
  }
  for (int q = 0; q < A->rd; ++q) {
    int off[3];
    child_off(A, ch + q, off);
    subbox_average(A, m, off, 0, 0.0, A->c[ch + q].u);
  }
}

/* activate or create the children of active cell c (c becomes a virtual mother) */
static void refine_cell(amr_t* A, int c, int at_t0) {
  acell* C = &A->c[c];
  if (C->child < 0) make_children(A, c, 0);
  else
    for (int q = 0; q < A->rd; ++q) { A->c[C->child + q].status = 0; memset(A->c[C->child + q].mem, 0, sizeof(A->c[0].mem)); }
  C = &A->c[c];
  C->status = -1;
  for (int q = 0; q < A->rd; ++q) A->c[C->child + q].isnew = 1;
  init_new_children(A, c, at_t0);
}

/* virtual children of active cell v (status +1) */
static void virtually_refine(amr_t* A, int v, int at_t0) {
  int ch = make_children(A, v, 1);
  if (at_t0) {
    int ids[512];
    for (int q = 0; q < A->rd; ++q) ids[q] = ch + q;
    ic_cells(A, ids, A->rd);
  } else if (A->c[v].q) {
    for (int q = 0; q < A->rd; ++q) {
      int off[3];
      child_off(A, ch + q, off);
      subbox_average(A, v, off, 1, 1.0, A->c[ch + q].u);
    }
  }
}

/* rules 4 and 5 to the least fixed point (monotone, hence order-independent) */
static int closure(amr_t* A, int at_t0) {
  int changed = 1, iters = 0;
  int nb[kMaxVor];
  while (changed) {
    changed = 0;
    ++iters;
    int nu = A->nused;
    for (int i = 0; i < nu; ++i) {
      if (!A->c[i].alive || A->c[i].status != -1) continue;
      int k = voronoi(A, i, nb);
      for (int j = 0; j < k; ++j) {
        int v = nb[j];
        if (v < 0 || A->c[v].child >= 0) continue;
        if (A->c[v].status == 0) { virtually_refine(A, v, at_t0); changed = 1; }
        else if (A->c[v].status == 1) {
          int K = A->c[v].mother;            /* rule 5 cascade (Fig. 1 right) */
          refine_cell(A, K, at_t0);
          changed = 1;
        }
      }
    }
  }
  return iters;
}

/* destroy virtual children nobody needs any more (R17 GC) */
static void garbage_collect(amr_t* A) {
  int nb[kMaxVor];
  for (int i = 0; i < A->nused; ++i) {
    acell* C = &A->c[i];
    if (!C->alive || C->status != 0 || C->child < 0) continue;
    int k = voronoi(A, i, nb), need = 0;
    for (int j = 0; j < k && !need; ++j)
      if (nb[j] >= 0 && A->c[nb[j]].status == -1) need = 1;
    if (!need) destroy_children(A, i);
  }
}

/* deep copy of the tree (for the revert loop of the recoarsening) */
typedef struct { acell* c; int nused, ncap; int32_t* map[LMAXX]; } snap_t;
static void snap_take(const amr_t* A, snap_t* S) {
  memset(S, 0, sizeof(*S));
  S->nused = A->nused; S->ncap = A->ncap;
  S->c = (acell*)malloc(sizeof(acell) * A->ncap);
  memcpy(S->c, A->c, sizeof(acell) * A->ncap);
  for (int i = 0; i < A->nused; ++i) { S->c[i].q = NULL; S->c[i].w = NULL; }
  for (int l = 0; l <= A->lmax; ++l) {
    size_t n = (size_t)A->n[l][0] * A->n[l][1] * A->n[l][2];
    S->map[l] = (int32_t*)malloc(sizeof(int32_t) * n);
    memcpy(S->map[l], A->map[l], sizeof(int32_t) * n);
  }
}
static void snap_restore(amr_t* A, const snap_t* S) {
  /* q / w pointers stay with the live cells of the same id where possible */
  for (int i = S->nused; i < A->nused; ++i) { free(A->c[i].q); free(A->c[i].w); }
  if (A->ncap < S->ncap) { A->c = (acell*)realloc(A->c, sizeof(acell) * S->ncap); A->ncap = S->ncap; }
  double** qs = (double**)calloc(S->nused, sizeof(double*));
  double** ws = (double**)calloc(S->nused, sizeof(double*));
  for (int i = 0; i < S->nused && i < A->nused; ++i) { qs[i] = A->c[i].q; ws[i] = A->c[i].w; }
  memcpy(A->c, S->c, sizeof(acell) * S->nused);
  memset(A->c + S->nused, 0, sizeof(acell) * (A->ncap - S->nused));
  for (int i = 0; i < S->nused; ++i) { A->c[i].q = qs[i]; A->c[i].w = ws[i]; }
  free(qs); free(ws);
  A->nused = S->nused;
  for (int l = 0; l <= A->lmax; ++l) {
    size_t n = (size_t)A->n[l][0] * A->n[l][1] * A->n[l][2];
    memcpy(A->map[l], S->map[l], sizeof(int32_t) * n);
  }
}
static void snap_free(snap_t* S) {
  free(S->c);
  for (int l = 0; l < LMAXX; ++l) free(S->map[l]);
  memset(S, 0, sizeof(*S));
}

static int adapt(amr_t* A, int at_t0) {
  int nb[kMaxVor];
  /* 1. ghost refresh at the synchronized time, indicator on active cells */
  if (!at_t0) fill_level(A, 0, 1.0);
  if (!at_t0)
    for (int l = 1; l <= A->lmax; ++l)
      for (int i = 0; i < A->nused; ++i) {
        acell* C = &A->c[i];
        if (!C->alive || C->level != l || C->status != 1) continue;
        int off[3];
        child_off(A, i, off);
        if (A->c[C->mother].q) subbox_average(A, C->mother, off, 1, 1.0, C->u);
      }
  for (int i = 0; i < A->nused; ++i) {
    A->c[i].isnew = 0;
    if (A->c[i].status != 0) { free(A->c[i].w); A->c[i].w = NULL; }
    if (A->c[i].alive && A->c[i].status == 0) {
      double chi = indicator(A, i);
      A->c[i].chi = chi;
      /* distance of chi to the strict thresholds, relative */
      double m1 = fabs(chi - A->cfg.chi_ref) / A->cfg.chi_ref, m2 = fabs(chi - A->cfg.chi_rec) / A->cfg.chi_rec;
      double m = m1 < m2 ? m1 : m2;
      if (m < A->margin) A->margin = m;
    }
  }
  /* WENO polynomials at t^{n+1} of every active cell (mothers of new children, R18) */
  if (!at_t0)
    for (int i = 0; i < A->nused; ++i)
      if (A->c[i].alive && A->c[i].status == 0)
        if (reconstruct(A, i)) return 3;
  /* 2. refinement marks R = {active, chi > chi_ref, level < lmax} */
  int nu = A->nused;
  int* mark = (int*)calloc((size_t)(nu > 0 ? nu : 1), sizeof(int));
  for (int i = 0; i < nu; ++i)
    mark[i] = A->c[i].alive && A->c[i].status == 0 && A->c[i].level < A->lmax && A->c[i].chi > A->cfg.chi_ref;
  for (int i = 0; i < nu; ++i)
    if (mark[i]) refine_cell(A, i, at_t0);
  /* 3. closure (rules 4, 5) */
  closure(A, at_t0);
  if (!at_t0) {
    /* 4. recoarsening candidates: virtual mothers whose children are all
     * unmarked, not new, active leaves with chi < chi_rec (rule 7) */
    int nu2 = A->nused;
    int* cand = (int*)calloc(nu2, sizeof(int));
    for (int i = 0; i < nu2; ++i) {
      acell* C = &A->c[i];
      if (!C->alive || C->status != -1) continue;
      int ok = 1;
      for (int q = 0; q < A->rd && ok; ++q) {
        const acell* K = &A->c[C->child + q];
        int kid = C->child + q;
        if (K->status != 0 || K->child >= 0 || K->isnew || !(K->chi < A->cfg.chi_rec) || (kid < nu && mark[kid])) ok = 0;
      }
      cand[i] = ok;
    }
    for (;;) {
      snap_t S;
      snap_take(A, &S);
      /* simultaneous rule 7 against the post-closure state */
      int* destroy = (int*)calloc(nu2, sizeof(int));
      for (int i = 0; i < nu2; ++i) {
        if (!cand[i]) continue;
        int k = voronoi(A, i, nb), busy = 0;
        for (int j = 0; j < k && !busy; ++j)
          if (nb[j] >= 0 && A->c[nb[j]].status == -1) busy = 1;
        destroy[i] = !busy;
      }
      for (int i = 0; i < nu2; ++i) {
        if (!cand[i]) continue;
        average_into(A, i);                       /* eqn.average */
        if (destroy[i]) destroy_children(A, i);
        else
          for (int q = 0; q < A->rd; ++q) A->c[A->c[i].child + q].status = 1;
        A->c[i].status = 0;
      }
      free(destroy);
      closure(A, 0);
      int reverted = 0;
      for (int i = 0; i < nu2; ++i)
        if (cand[i] && A->c[i].status == -1) { cand[i] = 0; reverted = 1; }
      if (!reverted) { snap_free(&S); break; }
      snap_restore(A, &S);                        /* closure wins: retry without them */
      snap_free(&S);
    }
    free(cand);
  }
  free(mark);
  /* 5. garbage collection of unneeded virtual children */
  garbage_collect(A);
  for (int i = 0; i < A->nused; ++i) A->c[i].isnew = 0;
  return 0;
}

/* ======================================================================== */
/* public API                                                               */
/* ======================================================================== */

typedef struct {
  int32_t level, status;
  int64_t idx[3];
  double u[9];
} orc_amr_cell;

void* orc_amr_create(const orc_config* cfg) {
  if (!cfg || (cfg->dim != 2 && cfg->dim != 3) || cfg->degree < 2 || cfg->degree > 3) return NULL;
  if (cfg->lmax < 0 || cfg->lmax >= LMAXX || cfg->refine_factor < cfg->degree) return NULL;
  if (cfg->flux == ORC_FLUX_OSHER && cfg->system != ORC_EULER) return NULL;   /* Osher: Euler only */
  if (cfg->pred_guess != 0) return NULL;   /* R25 guess: uniform grids only */
  for (int k = 0; k < 2 * cfg->dim; ++k) {
    if (cfg->bc[k] == ORC_BC_REFLECTIVE && (cfg->system != ORC_EULER || cfg->n[k / 2] < cfg->degree + 1)) return NULL;
    if (cfg->bc[k] == ORC_BC_INFLOW || cfg->bc[k] == ORC_BC_EXACT) return NULL;   /* R23, R26: uniform grids only */
  }
  amr_t* A = (amr_t*)calloc(1, sizeof(amr_t));
  A->cfg = *cfg;
  A->d = cfg->dim; A->M = cfg->degree; A->N = A->M + 1;
  A->nv = orc_nvar(cfg->system, A->d);
  A->NS = 1;
  for (int k = 0; k < A->d; ++k) A->NS *= A->N;
  A->NST = A->NS * A->N;
  A->r = cfg->refine_factor; A->lmax = cfg->lmax;
  A->margin = 1e300;
  A->rd = 1;
  for (int k = 0; k < A->d; ++k) A->rd *= A->r;
  if (A->cfg.pred_tol <= 0) A->cfg.pred_tol = 1e-13;
  if (A->cfg.pred_max_sweeps <= 0) A->cfg.pred_max_sweeps = 32;
  if (A->cfg.ic_quad <= 0) A->cfg.ic_quad = A->N;
  if (A->cfg.flux_quad <= 0) A->cfg.flux_quad = 3;   /* reading R21 */
  orc_gauss_legendre(A->N, A->gq, A->gw);
  for (int l = 0; l <= A->lmax; ++l) {
    int64_t s = 1;
    for (int k = 0; k < 3; ++k) {
      A->n[l][k] = (k < A->d) ? cfg->n[k] * (int64_t)pow(A->r, l) : 1;
      A->dx[l][k] = (k < A->d) ? (cfg->hi[k] - cfg->lo[k]) / (double)A->n[l][k] : 1.0;
      s *= A->n[l][k];
    }
    A->map[l] = (int32_t*)malloc(sizeof(int32_t) * s);
    for (int64_t i = 0; i < s; ++i) A->map[l][i] = -1;
  }
  int64_t n0 = A->n[0][0] * A->n[0][1] * A->n[0][2];
  int id = alloc_block(A, (int)n0);
  for (int64_t i = 0; i < n0; ++i) {
    acell* C = &A->c[id + i];
    C->level = 0; C->status = 0;
    C->idx[0] = i % A->n[0][0]; C->idx[1] = (i / A->n[0][0]) % A->n[0][1]; C->idx[2] = i / (A->n[0][0] * A->n[0][1]);
    A->map[0][i] = (int32_t)(id + i);
  }
  return A;
}

void orc_amr_destroy(void* h) {
  amr_t* A = (amr_t*)h;
  if (!A) return;
  for (int i = 0; i < A->nused; ++i) { free(A->c[i].q); free(A->c[i].w); }
  free(A->c);
  for (int l = 0; l < LMAXX; ++l) free(A->map[l]);
  free(A);
}

const char* orc_amr_last_error(void* h) { return ((amr_t*)h)->err; }
double orc_amr_time(void* h) { return ((amr_t*)h)->t; }

/* IC on level 0, then the initial hierarchy up to lmax (R20) */
int orc_amr_set_initial(void* h, orc_ic_fn ic, void* user) {
  amr_t* A = (amr_t*)h;
  A->ic = ic; A->user = user;
  int n = 0;
  int* ids = (int*)malloc(sizeof(int) * A->nused);
  for (int i = 0; i < A->nused; ++i) if (A->c[i].alive) ids[n++] = i;
  ic_cells(A, ids, n);
  free(ids);
  for (int l = 0; l < A->lmax; ++l)
    if (adapt(A, 1)) return 3;
  A->t = 0.0;
  return 0;
}

double orc_amr_compute_dt(void* h) {
  amr_t* A = (amr_t*)h;
  double smax = 0.0;
  for (int i = 0; i < A->nused; ++i) {
    const acell* C = &A->c[i];
    if (!C->alive || C->status != 0) continue;
    double s = 0.0;
    for (int k = 0; k < A->d; ++k)
      s += orc_max_speed(A->cfg.system, A->d, A->cfg.gamma, A->cfg.ch, C->u, k) / A->dx[0][k];
    if (!(s <= smax)) smax = s;
  }
  return A->cfg.cfl / smax;   /* R1 with level-0 spacing (dt_l / dx_l = dt_0 / dx_0) */
}

int orc_amr_step(void* h, double t_end, int64_t max_steps, int adapt_every, orc_report* rep) {
  amr_t* A = (amr_t*)h;
  orc_report R; memset(&R, 0, sizeof(R));
  A->margin = 1e300;
  for (int l = 0; l < LMAXX; ++l) A->updates[l] = 0;
  A->sweeps = 0; A->sweeps_max = 0;
  g_nsched = 0;
  while (R.steps < max_steps && A->t < t_end) {
    double dt = orc_amr_compute_dt(A);
    if (!(dt > 0.0) || !isfinite(dt)) { snprintf(A->err, sizeof(A->err), "invalid dt"); return 3; }
    if (A->t + dt > t_end) dt = t_end - A->t;
    if (advance(A, 0, 0, dt)) return 3;
    A->t += dt;
    R.dt = dt;
    R.steps++;
    if (adapt_every > 0 && R.steps % adapt_every == 0)
      if (adapt(A, 0)) return 3;
  }
  R.t = A->t;
  for (int l = 0; l < LMAXX; ++l) { R.updates_per_level[l] = A->updates[l]; R.cell_updates += A->updates[l]; }
  R.sweeps_total = A->sweeps;
  R.sweeps_max = A->sweeps_max;
  R.min_threshold_margin = A->margin;
  if (rep) *rep = R;
  return 0;
}

int orc_amr_adapt(void* h) {
  ((amr_t*)h)->margin = 1e300;
  return adapt((amr_t*)h, 0);
}
/* min threshold margin of the adapts since the last orc_amr_step / orc_amr_adapt */
double orc_amr_margin(void* h) { return ((amr_t*)h)->margin; }

/* all cells sorted by (level, z, y, x); out == NULL -> count */
int64_t orc_amr_get_cells(void* h, orc_amr_cell* out) {
  amr_t* A = (amr_t*)h;
  int64_t n = 0;
  for (int l = 0; l <= A->lmax; ++l) {
    int64_t s = A->n[l][0] * A->n[l][1] * A->n[l][2];
    for (int64_t i = 0; i < s; ++i) {
      int id = A->map[l][i];
      if (id < 0) continue;
      if (out) {
        const acell* C = &A->c[id];
        out[n].level = C->level; out[n].status = C->status;
        for (int k = 0; k < 3; ++k) out[n].idx[k] = C->idx[k];
        for (int v = 0; v < 9; ++v) out[n].u[v] = (v < A->nv) ? C->u[v] : 0.0;
      }
      ++n;
    }
  }
  return n;
}

/* does cell a's closed box touch cell b's (b one level finer)? */
static int touches(const amr_t* A, int a, int b) {
  const acell* Ca = &A->c[a];
  const acell* Cb = &A->c[b];
  for (int k = 0; k < A->d; ++k) {
    int64_t lo = Ca->idx[k] * A->r, hi = lo + A->r;       /* a in b's index units */
    int64_t n = A->n[Cb->level][k];
    int64_t bl = Cb->idx[k], bh = bl + 1;
    int ok = (bh >= lo && bl <= hi);
    if (!ok && A->cfg.bc[2 * k] == ORC_BC_PERIODIC)      /* across the periodic seam */
      ok = (bh + n >= lo && bl + n <= hi) || (bh - n >= lo && bl - n <= hi);
    if (!ok) return 0;
  }
  return 1;
}

/* rules 1-7 invariant scan; returns 0 if all hold */
int orc_amr_check(void* h, char* msg, int cap) {
  amr_t* A = (amr_t*)h;
  int nb[kMaxVor];
  for (int i = 0; i < A->nused; ++i) {
    const acell* C = &A->c[i];
    if (!C->alive) continue;
    if (C->level > A->lmax) { snprintf(msg, cap, "rule 6 violated"); return 6; }
    if (C->child >= 0)
      for (int q = 0; q < A->rd; ++q)
        if (A->c[C->child + q].mother != i) { snprintf(msg, cap, "rule 1/3: children not consecutive"); return 1; }
    if (C->status == 1 && (C->mother < 0 || A->c[C->mother].status != 0)) { snprintf(msg, cap, "rule 2: virtual child without active mother"); return 2; }
    if (C->status == 1 && C->child >= 0) { snprintf(msg, cap, "rule 2: refined virtual child"); return 2; }
    if (C->status == 0 && C->level > 0 && A->c[C->mother].status != -1) { snprintf(msg, cap, "rule 2: active cell with non-virtual-mother mother"); return 2; }
    if (C->status == -1) {
      if (C->child < 0) { snprintf(msg, cap, "virtual mother without children"); return 2; }
      for (int q = 0; q < A->rd; ++q)
        if (A->c[C->child + q].status > 0) { snprintf(msg, cap, "rule 2: virtual mother with virtual children"); return 2; }
    }
    /* rule 4: a cell with children of status <= 0 has no Voronoi neighbour
     * without children (and all its same-level neighbours exist) */
    if (C->status == -1) {
      int k = voronoi(A, i, nb);
      for (int j = 0; j < k; ++j) {
        int zl = (A->d == 3) ? -1 : 0;
        (void)zl;
        if (nb[j] >= 0 && A->c[nb[j]].child < 0) {
          snprintf(msg, cap, "rule 4: neighbour of a refined level-%d cell has no children", C->level);
          return 4;
        }
      }
    }
    /* rule 5: an active cell never touches an active cell two levels finer */
    if (C->status == 0) {
      int k = voronoi(A, i, nb);
      for (int j = 0; j < k; ++j) {
        if (nb[j] < 0 || A->c[nb[j]].status != -1) continue;
        const acell* Nn = &A->c[nb[j]];
        for (int q = 0; q < A->rd; ++q) {
          int kid = Nn->child + q;
          if (A->c[kid].status == -1 && touches(A, i, kid)) {
            snprintf(msg, cap, "rule 5: level %d active cell touches level %d refined cell", C->level, C->level + 1);
            return 5;
          }
        }
      }
    }
  }
  return 0;
}

/* test hook: refine one active cell (rules 4/5 closure included), t = 0 style */
int orc_amr_refine_cell(void* h, int level, const int64_t* idx) {
  amr_t* A = (amr_t*)h;
  int64_t ix[3] = {idx[0], idx[1], A->d == 3 ? idx[2] : 0};
  int id = A->map[level][lin_idx(A, level, ix)];
  if (id < 0 || A->c[id].status != 0 || level >= A->lmax) return 1;
  refine_cell(A, id, 1);
  closure(A, 1);
  garbage_collect(A);
  return 0;
}

/* level update order of the last orc_amr_step (P:651-653 schedule) */
int orc_amr_schedule(int* out, int cap) {
  int n = g_nsched < cap ? g_nsched : cap;
  memcpy(out, g_sched, sizeof(int) * n);
  return g_nsched;
}

