/*
 * ader_oracle.c — CPU ORACLE of the ADER-WENO hot path (arXiv:1212.3585).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or execute this.
 * It shares no code, header, table or helper with paper_1212_3585_b200/.
 *
 * The oracle is the algorithm written step by step in the paper's order and
 * notation, plain loops, single thread, FP64, no FMA contraction:
 *   - nodal Gauss-Legendre Lagrange basis on [0,1]
 *   - WENO stencils / reconstruction / oscillation indicator
 *       eqn.stencildef @ P:212-225, eqn.rec.x @ P:244-250,
 *       eqn.omegas @ P:260-264, eqn.sigmas @ P:266-273, P:274 constants,
 *       y and z sweeps per degree of freedom @ P:279-322
 *   - local space-time DG predictor as the dense weak form
 *       K1, K^xi, M, F0 integrals @ P:434-449, system eqn.pde.weak4
 *       @ P:451-459, Picard iteration eqn.stdg.final @ P:463-474
 *       (S = 0: neither Euler nor GLM-MHD has a source)
 *   - space-time Gauss quadrature of the two-point flux
 *       Rusanov eqn.rusanov @ P:181-185, Osher-type eqn.osher @ P:186-196
 *       (|A| by Sylvester's formula, path by Gauss-Legendre)
 *   - one-step finite-volume update eq:finite_vol
 *   - Euler system eq:Euler-system
 *   - ideal MHD with GLM cleaning, Gaussian units
 * Readings where the paper is silent or garbled are listed in DESIGN.md
 * ("Readings"); the ones used here: R1 CFL rule, R2 predictor stopping rule,
 * R3 time-constant initial guess, R4 s_max = max of both states, R5 ghost
 * cells (periodic wrap / transmissive copy), R6 IC by Q-point GL averages.
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu") tie each function to closed
 * forms, exactness properties and brute force; see DESIGN.md "Oracle pins".
 */
#include "ader_oracle.h"
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define NMAX ORC_MAXN
#define VMAX ORC_MAXV

/* ====================================================================== */
/* 1. Gauss-Legendre nodes and the nodal Lagrange basis        */
/* ====================================================================== */

/* Legendre P_n and derivative at x in [-1,1] by the three-term recurrence. */
static void legendre(int n, double x, double* p, double* dp) {
  double p0 = 1.0, p1 = x;
  if (n == 0) { *p = 1.0; *dp = 0.0; return; }
  for (int k = 2; k <= n; ++k) {
    double pk = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
    p0 = p1; p1 = pk;
  }
  *p = p1;
  *dp = n * (x * p1 - p0) / (x * x - 1.0);
}

/* n-point Gauss-Legendre rule mapped to [0,1], nodes increasing. */
static void gauss_legendre01(int n, double* x, double* w) {
  for (int i = 0; i < n; ++i) {
    double z = cos(M_PI * (i + 0.75) / (n + 0.5)), p, dp;
    for (int it = 0; it < 100; ++it) {
      legendre(n, z, &p, &dp);
      double dz = p / dp;
      z -= dz;
      if (fabs(dz) < 1e-16) break;
    }
    legendre(n, z, &p, &dp);
    /* z_i decreases with i; x = (1+z)/2 on [0,1], weight 2/((1-z^2)P'^2) / 2 */
    x[n - 1 - i] = 0.5 * (1.0 + z);
    w[n - 1 - i] = 1.0 / ((1.0 - z * z) * dp * dp);
  }
}

typedef struct {
  int M, N, nS;
  double lam[NMAX], w[NMAX];
  double mono[NMAX][NMAX];          /* psi_p(xi) = sum_j mono[p][j] xi^j      */
  int L[4], R[4];
  double lin[4];                    /* lambda_s of eqn.omegas                 */
  double rec[4][NMAX][NMAX];        /* Rec_s = A_s^-1: dofs_p = sum_o rec[s][p][o] u_o */
  double Sigma[NMAX][NMAX];         /* oscillation indicator matrix           */
  double M1[NMAX][NMAX], Kx1[NMAX][NMAX], K1t[NMAX][NMAX];
  double psi0[NMAX], psi1[NMAX];
} basis_t;

/* psi_p(xi) by the Lagrange product formula (exact at the nodes). */
static double psi_val(const basis_t* B, int p, double xi) {
  double v = 1.0;
  for (int k = 0; k < B->N; ++k)
    if (k != p) v *= (xi - B->lam[k]) / (B->lam[p] - B->lam[k]);
  return v;
}

/* alpha-th derivative of psi_p from its monomial coefficients. */
static double psi_der(const basis_t* B, int p, int alpha, double xi) {
  double s = 0.0;
  for (int j = B->N - 1; j >= alpha; --j) {
    double c = B->mono[p][j];
    for (int k = 0; k < alpha; ++k) c *= (double)(j - k);
    s = s * xi + c;
  }
  return s;
}

/* High-order (16-point) Gauss rule for the 1D integrals of the tables. */
static double QX[16], QW[16];
static int q_init = 0;
static void quad_init(void) { if (!q_init) { gauss_legendre01(16, QX, QW); q_init = 1; } }

/* Gauss-Jordan inverse with partial pivoting, n x n row-major. */
static int mat_inverse(int n, const double* A, double* Ai) {
  double* a = (double*)malloc(sizeof(double) * n * n * 2);
  int w2 = 2 * n;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < w2; ++j)
      a[i * w2 + j] = (j < n) ? A[i * n + j] : (j - n == i ? 1.0 : 0.0);
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (fabs(a[r * w2 + c]) > fabs(a[piv * w2 + c])) piv = r;
    if (a[piv * w2 + c] == 0.0) { free(a); return -1; }
    if (piv != c)
      for (int j = 0; j < w2; ++j) { double t = a[c * w2 + j]; a[c * w2 + j] = a[piv * w2 + j]; a[piv * w2 + j] = t; }
    double d = a[c * w2 + c];
    for (int j = 0; j < w2; ++j) a[c * w2 + j] /= d;
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      double f = a[r * w2 + c];
      if (f != 0.0)
        for (int j = 0; j < w2; ++j) a[r * w2 + j] -= f * a[c * w2 + j];
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) Ai[i * n + j] = a[i * w2 + n + j];
  free(a);
  return 0;
}

static basis_t g_basis[NMAX + 1];
static int g_basis_ok[NMAX + 1];

static const basis_t* basis_get(int M) {
  if (M < 1 || M + 1 > NMAX) return NULL;
  if (g_basis_ok[M]) return &g_basis[M];
  quad_init();
  basis_t* B = &g_basis[M];
  memset(B, 0, sizeof(*B));
  B->M = M; B->N = M + 1;
  int N = B->N;
  /* Gauss-Legendre nodes lambda_k of the nodal basis */
  gauss_legendre01(N, B->lam, B->w);
  /* monomial coefficients of psi_p = prod_{k!=p} (xi - lam_k)/(lam_p - lam_k) */
  for (int p = 0; p < N; ++p) {
    double c[NMAX + 1] = {0};
    c[0] = 1.0;
    int deg = 0;
    for (int k = 0; k < N; ++k) {
      if (k == p) continue;
      double den = B->lam[p] - B->lam[k];
      double nc[NMAX + 1] = {0};
      for (int j = 0; j <= deg; ++j) {
        nc[j + 1] += c[j] / den;
        nc[j] += -B->lam[k] * c[j] / den;
      }
      ++deg;
      memcpy(c, nc, sizeof(nc));
    }
    for (int j = 0; j < N; ++j) B->mono[p][j] = c[j];
  }
  /* stencils, eqn.stencildef @ P:212-225 */
  if (M % 2 == 0) {
    B->nS = 3;
    B->L[0] = M / 2; B->R[0] = M / 2; B->lin[0] = 1e5;   /* central s=1       */
    B->L[1] = M;     B->R[1] = 0;     B->lin[1] = 1.0;   /* left-sided s=2    */
    B->L[2] = 0;     B->R[2] = M;     B->lin[2] = 1.0;   /* right-sided s=3   */
  } else {
    B->nS = 4;
    B->L[0] = M / 2 + 1; B->R[0] = M / 2;     B->lin[0] = 1e5;  /* central s=0 */
    B->L[1] = M / 2;     B->R[1] = M / 2 + 1; B->lin[1] = 1e5;  /* central s=1 */
    B->L[2] = M;         B->R[2] = 0;         B->lin[2] = 1.0;
    B->L[3] = 0;         B->R[3] = M;         B->lin[3] = 1.0;
  }
  /* eqn.rec.x @ P:244-250: A_s[o][p] = int_{o}^{o+1} psi_p(xi) dxi over the
   * stencil cells e = i-L..i+R (reference coordinate of cell e is xi - (e-i));
   * Rec_s = A_s^{-1}, precomputed once on the reference element. */
  for (int s = 0; s < B->nS; ++s) {
    double A[NMAX * NMAX], Ai[NMAX * NMAX];
    for (int o = -B->L[s]; o <= B->R[s]; ++o)
      for (int p = 0; p < N; ++p) {
        double acc = 0.0;
        for (int q = 0; q < 16; ++q) acc += QW[q] * psi_val(B, p, o + QX[q]);
        A[(o + B->L[s]) * N + p] = acc;
      }
    mat_inverse(N, A, Ai);
    for (int p = 0; p < N; ++p)
      for (int o = 0; o < N; ++o) B->rec[s][p][o] = Ai[p * N + o];
  }
  /* oscillation indicator matrix */
  for (int p = 0; p < N; ++p)
    for (int m = 0; m < N; ++m) {
      double acc = 0.0;
      for (int a = 1; a <= M; ++a)
        for (int q = 0; q < 16; ++q)
          acc += QW[q] * psi_der(B, p, a, QX[q]) * psi_der(B, m, a, QX[q]);
      B->Sigma[p][m] = acc;
    }
  /* 1D factors of the predictor integrals */
  for (int a = 0; a < N; ++a) {
    B->psi0[a] = psi_val(B, a, 0.0);
    B->psi1[a] = psi_val(B, a, 1.0);
  }
  for (int a = 0; a < N; ++a)
    for (int b = 0; b < N; ++b) {
      double m = 0.0, kx = 0.0, kt = 0.0;
      for (int q = 0; q < 16; ++q) {
        m  += QW[q] * psi_val(B, a, QX[q]) * psi_val(B, b, QX[q]);       /* int psi_a psi_b    */
        kx += QW[q] * psi_val(B, a, QX[q]) * psi_der(B, b, 1, QX[q]);    /* int psi_a psi_b'   */
        kt += QW[q] * psi_der(B, a, 1, QX[q]) * psi_val(B, b, QX[q]);    /* int psi_a' psi_b   */
      }
      B->M1[a][b] = m;
      B->Kx1[a][b] = kx;
      B->K1t[a][b] = B->psi1[a] * B->psi1[b] - kt;
    }
  g_basis_ok[M] = 1;
  return B;
}

int orc_basis_tables(int M, double* lam, double* w, double* psi0, double* psi1,
                     double* Sigma, double* rec, int* L, int* R, double* lin,
                     double* M1, double* Kx1, double* K1t) {
  const basis_t* B = basis_get(M);
  if (!B) return -1;
  int N = B->N;
  for (int i = 0; i < N; ++i) {
    if (lam) lam[i] = B->lam[i];
    if (w) w[i] = B->w[i];
    if (psi0) psi0[i] = B->psi0[i];
    if (psi1) psi1[i] = B->psi1[i];
    for (int j = 0; j < N; ++j) {
      if (Sigma) Sigma[i * N + j] = B->Sigma[i][j];
      if (M1) M1[i * N + j] = B->M1[i][j];
      if (Kx1) Kx1[i * N + j] = B->Kx1[i][j];
      if (K1t) K1t[i * N + j] = B->K1t[i][j];
    }
  }
  for (int s = 0; s < B->nS; ++s) {
    if (L) L[s] = B->L[s];
    if (R) R[s] = B->R[s];
    if (lin) lin[s] = B->lin[s];
    if (rec)
      for (int p = 0; p < N; ++p)
        for (int o = 0; o < N; ++o) rec[(s * N + p) * N + o] = B->rec[s][p][o];
  }
  return B->nS;
}

/* ====================================================================== */
/* 2. Physics: Euler (eq:Euler-system @ P:838-869) and GLM-MHD*/
/* ====================================================================== */

int orc_nvar(int system, int dim) {
  if (system == ORC_MHD) return 9;
  return dim + 2;    /* rho, rho v (d comps), E  (reading R7: nu=4 in 2D) */
}

void orc_prim_to_cons(int system, int dim, double gamma, const double* prim, double* u) {
  double rho = prim[0], vx = prim[1], vy = prim[2], vz = prim[3], p = prim[4];
  if (system == ORC_MHD) {
    double Bx = prim[5], By = prim[6], Bz = prim[7];
    u[0] = rho; u[1] = rho * vx; u[2] = rho * vy; u[3] = rho * vz;
    /* p = (gamma-1)(E - rho v^2/2 - B^2/8pi) */
    u[4] = p / (gamma - 1.0) + 0.5 * rho * (vx * vx + vy * vy + vz * vz)
         + (Bx * Bx + By * By + Bz * Bz) / (8.0 * M_PI);
    u[5] = Bx; u[6] = By; u[7] = Bz; u[8] = prim[8];
    return;
  }
  /* E = p/(gamma-1) + rho (vx^2+vy^2+vz^2)/2 */
  double vv[3] = {vx, vy, vz};
  u[0] = rho;
  double ke = 0.0;
  for (int k = 0; k < dim; ++k) { u[1 + k] = rho * vv[k]; ke += vv[k] * vv[k]; }
  u[1 + dim] = p / (gamma - 1.0) + 0.5 * rho * ke;
}

/* Primitive state of a conserved vector; returns 0 if admissible (rho>0, p>0). */
static int cons_to_prim(int system, int dim, double gamma, const double* u,
                        double* rho, double v[3], double* p, double B[3]) {
  *rho = u[0];
  v[0] = v[1] = v[2] = 0.0;
  B[0] = B[1] = B[2] = 0.0;
  if (!(u[0] > 0.0)) return -1;
  if (system == ORC_MHD) {
    for (int k = 0; k < 3; ++k) { v[k] = u[1 + k] / u[0]; B[k] = u[5 + k]; }
    double vv = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
    double bb = B[0] * B[0] + B[1] * B[1] + B[2] * B[2];
    *p = (gamma - 1.0) * (u[4] - 0.5 * u[0] * vv - bb / (8.0 * M_PI));
  } else {
    double vv = 0.0;
    for (int k = 0; k < dim; ++k) { v[k] = u[1 + k] / u[0]; vv += v[k] * v[k]; }
    *p = (gamma - 1.0) * (u[1 + dim] - 0.5 * u[0] * vv);
  }
  return (*p > 0.0) ? 0 : -1;
}

int orc_phys_flux(int system, int dim, double gamma, double ch, const double* u, int dir, double* f) {
  double rho, v[3], p, B[3];
  if (cons_to_prim(system, dim, gamma, u, &rho, v, &p, B)) return -1;
  if (system == ORC_MHD) {
    /* flux tensor row dir of F = (rho v; rho v v + (p + B^2/8pi) I - B B/4pi;
     * v (E + p + B^2/8pi) - B (v.B)/4pi; v B - B v + Psi I; ch^2 B) */
    double bb = B[0] * B[0] + B[1] * B[1] + B[2] * B[2];
    double vB = v[0] * B[0] + v[1] * B[1] + v[2] * B[2];
    double pt = p + bb / (8.0 * M_PI);
    f[0] = rho * v[dir];
    for (int k = 0; k < 3; ++k)
      f[1 + k] = rho * v[dir] * v[k] + (k == dir ? pt : 0.0) - B[dir] * B[k] / (4.0 * M_PI);
    f[4] = v[dir] * (u[4] + pt) - B[dir] * vB / (4.0 * M_PI);
    for (int k = 0; k < 3; ++k)
      f[5 + k] = v[dir] * B[k] - B[dir] * v[k] + (k == dir ? u[8] : 0.0);
    f[8] = ch * ch * B[dir];
    return 0;
  }
  /* eq:Euler-system @ P:838-867 */
  f[0] = rho * v[dir];
  for (int k = 0; k < dim; ++k) f[1 + k] = rho * v[dir] * v[k] + (k == dir ? p : 0.0);
  f[1 + dim] = v[dir] * (u[1 + dim] + p);
  return 0;
}

/* Largest |eigenvalue| of A_dir = df/du.  Euler: |v_n| + c.
 * MHD (Gaussian units): max(|v_n| + c_f, c_h), c_f the fast speed. */
double orc_max_speed(int system, int dim, double gamma, double ch, const double* u, int dir) {
  double rho, v[3], p, B[3];
  if (cons_to_prim(system, dim, gamma, u, &rho, v, &p, B)) return NAN;
  double a2 = gamma * p / rho;
  if (system == ORC_MHD) {
    double b2 = (B[0] * B[0] + B[1] * B[1] + B[2] * B[2]) / (4.0 * M_PI * rho);
    double bn2 = B[dir] * B[dir] / (4.0 * M_PI * rho);
    double s = a2 + b2;
    double disc = s * s - 4.0 * a2 * bn2;
    if (disc < 0.0) disc = 0.0;
    double cf = sqrt(0.5 * (s + sqrt(disc)));
    double sp = fabs(v[dir]) + cf;
    return sp > ch ? sp : ch;
  }
  return fabs(v[dir]) + sqrt(a2);
}

/* eqn.rusanov @ P:181-185; s_max = max over both states (reading R4). */
int orc_rusanov(int system, int dim, double gamma, double ch, const double* uL,
                const double* uR, int dir, double* f) {
  int nv = orc_nvar(system, dim);
  double fL[VMAX], fR[VMAX];
  if (orc_phys_flux(system, dim, gamma, ch, uL, dir, fL)) return -1;
  if (orc_phys_flux(system, dim, gamma, ch, uR, dir, fR)) return -1;
  double sL = orc_max_speed(system, dim, gamma, ch, uL, dir);
  double sR = orc_max_speed(system, dim, gamma, ch, uR, dir);
  double smax = sL > sR ? sL : sR;
  for (int v = 0; v < nv; ++v) f[v] = 0.5 * (fL[v] + fR[v]) - 0.5 * fabs(smax) * (uR[v] - uL[v]);
  return 0;
}

/* A = df_dir/du of eq:Euler-system differentiated by hand in the
 * conserved variables u = (rho, m_1..m_d, E), v = m/rho,
 * p = (gamma-1)(E - rho |v|^2/2), H = (E + p)/rho:
 *   f_0     = m_n
 *   f_{1+k} = m_n m_k / rho + p delta_kn
 *   f_{1+d} = v_n (E + p)                                                   */
int orc_euler_jacobian(int dim, double gamma, const double* u, int dir, double* A) {
  double rho, v[3], p, B[3];
  if (cons_to_prim(ORC_EULER, dim, gamma, u, &rho, v, &p, B)) return -1;
  const int nv = dim + 2, n = dir;
  const double g1 = gamma - 1.0;
  double vv = 0.0;
  for (int k = 0; k < dim; ++k) vv += v[k] * v[k];
  const double H = (u[1 + dim] + p) / rho;
  for (int i = 0; i < nv * nv; ++i) A[i] = 0.0;
  A[0 * nv + 1 + n] = 1.0;
  for (int k = 0; k < dim; ++k) {
    double* row = A + (1 + k) * nv;
    row[0] = -v[n] * v[k] + (k == n ? 0.5 * g1 * vv : 0.0);
    for (int j = 0; j < dim; ++j)
      row[1 + j] = (j == n ? v[k] : 0.0) + (j == k ? v[n] : 0.0) - (k == n ? g1 * v[j] : 0.0);
    row[1 + dim] = (k == n) ? g1 : 0.0;
  }
  double* row = A + (1 + dim) * nv;
  row[0] = v[n] * (0.5 * g1 * vv - H);
  for (int j = 0; j < dim; ++j) row[1 + j] = (j == n ? H : 0.0) - g1 * v[n] * v[j];
  row[1 + dim] = gamma * v[n];
  return 0;
}

static void matmul(int n, const double* X, const double* Y, double* Z) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int k = 0; k < n; ++k) s += X[i * n + k] * Y[k * n + j];
      Z[i * n + j] = s;
    }
}

/* |A| = sum_i |lambda_i| prod_{j != i} (A - lambda_j I) / (lambda_i - lambda_j)
 * (Sylvester's formula for a diagonalisable A with the distinct eigenvalues
 * lambda = v_n - c, v_n, v_n + c of the Euler Jacobian, c^2 = gamma p / rho). */
int orc_euler_abs_jacobian(int dim, double gamma, const double* u, int dir, double* absA) {
  double rho, v[3], p, B[3];
  if (cons_to_prim(ORC_EULER, dim, gamma, u, &rho, v, &p, B)) return -1;
  const int nv = dim + 2;
  const double c = sqrt(gamma * p / rho);
  const double lam[3] = {v[dir] - c, v[dir], v[dir] + c};
  double A[VMAX * VMAX], S[3][VMAX * VMAX], P[VMAX * VMAX];
  if (orc_euler_jacobian(dim, gamma, u, dir, A)) return -1;
  for (int i = 0; i < 3; ++i) {
    for (int e = 0; e < nv * nv; ++e) S[i][e] = A[e];
    for (int e = 0; e < nv; ++e) S[i][e * nv + e] -= lam[i];   /* S_i = A - lambda_i I */
  }
  for (int e = 0; e < nv * nv; ++e) absA[e] = 0.0;
  for (int i = 0; i < 3; ++i) {
    const int j0 = (i == 0) ? 1 : 0, j1 = (i == 2) ? 1 : 2;
    matmul(nv, S[j0], S[j1], P);
    const double coef = fabs(lam[i]) / ((lam[i] - lam[j0]) * (lam[i] - lam[j1]));
    for (int e = 0; e < nv * nv; ++e) absA[e] += coef * P[e];
  }
  return 0;
}

/* eqn.osher @ P:186-196: f = (f(uL) + f(uR))/2 - (1/2) (int_0^1 |A(psi(s))| ds)
 * (uR - uL), psi(s) = uL + s (uR - uL), the integral by nq-point Gauss-Legendre
 * ("at least two quadrature points"). */
int orc_osher(int system, int dim, double gamma, int nq, const double* uL, const double* uR, int dir, double* f) {
  if (system != ORC_EULER || nq < 1 || nq > 16) return -2;
  const int nv = dim + 2;
  double fL[VMAX], fR[VMAX], sq[16], wq[16], du[VMAX], absA[VMAX * VMAX], D[VMAX];
  if (orc_phys_flux(system, dim, gamma, 0.0, uL, dir, fL)) return -1;
  if (orc_phys_flux(system, dim, gamma, 0.0, uR, dir, fR)) return -1;
  gauss_legendre01(nq, sq, wq);
  for (int v = 0; v < nv; ++v) { du[v] = uR[v] - uL[v]; D[v] = 0.0; }
  for (int g = 0; g < nq; ++g) {
    double ps[VMAX];
    for (int v = 0; v < nv; ++v) ps[v] = uL[v] + sq[g] * du[v];
    if (orc_euler_abs_jacobian(dim, gamma, ps, dir, absA)) return -1;
    for (int a = 0; a < nv; ++a) {
      double s = 0.0;
      for (int b = 0; b < nv; ++b) s += absA[a * nv + b] * du[b];
      D[a] += wq[g] * s;
    }
  }
  for (int v = 0; v < nv; ++v) f[v] = 0.5 * (fL[v] + fR[v]) - 0.5 * D[v];
  return 0;
}

int orc_numflux(int system, int dim, double gamma, double ch, int flux, int nq, const double* uL,
                const double* uR, int dir, double* f) {
  if (flux == ORC_FLUX_OSHER) return orc_osher(system, dim, gamma, nq, uL, uR, dir, f);
  return orc_rusanov(system, dim, gamma, ch, uL, uR, dir, f);
}

/* ====================================================================== */
/* 3. WENO reconstruction                                     */
/* ====================================================================== */

/* One 1D problem: win[0..2M] = averages of cells i-M..i+M (or the dofs of
 * the previous sweep), out[N] = nodal dofs of the WENO polynomial. */
void orc_weno_1d(int M, const double* win, double* out) {
  const basis_t* B = basis_get(M);
  int N = B->N;
  double ws[4][NMAX], wt[4], sum = 0.0;
  for (int s = 0; s < B->nS; ++s) {
    /* eqn.rec.x: w^s = Rec_s * (u_{i-L} .. u_{i+R}) */
    for (int p = 0; p < N; ++p) {
      double acc = 0.0;
      for (int o = 0; o < N; ++o) acc += B->rec[s][p][o] * win[M - B->L[s] + o];
      ws[s][p] = acc;
    }
    /* eqn.sigmas: sigma_s = Sigma_pm w_p w_m with Sigma_pm of P:271-273, i.e.
     * sigma_s = sum_alpha int_0^1 (d^alpha w_h^s / dxi^alpha)^2 dxi.  Evaluated in
     * this integral form (reading R13): the quadratic form in nodal
     * coefficients cancels O(|w|^2 |Sigma| 1e-16) ~ 1e-13 of round-off, more
     * than eps = 1e-14, which would leave the weights undetermined in FP64. */
    double sig = 0.0;
    for (int a = 1; a <= M; ++a)
      for (int q = 0; q < 16; ++q) {
        double dv = 0.0;
        for (int p = 0; p < N; ++p) dv += ws[s][p] * psi_der(B, p, a, QX[q]);
        sig += QW[q] * dv * dv;
      }
    /* eqn.omegas with eps = 1e-14, r = 8 */
    wt[s] = B->lin[s] / pow(sig + 1e-14, 8.0);
    sum += wt[s];
  }
  for (int p = 0; p < N; ++p) {
    double acc = 0.0;
    for (int s = 0; s < B->nS; ++s) acc += (wt[s] / sum) * ws[s][p];
    out[p] = acc;   /* eqn.weno */
  }
}

static int ipow(int b, int e) { int r = 1; while (e--) r *= b; return r; }

int orc_reconstruct_box(int d, int M, int nv, const double* ubox, double* w) {
  const basis_t* B = basis_get(M);
  if (!B || d < 2 || d > 3) return -1;
  int N = B->N, W = 2 * M + 1;
  double win[2 * NMAX + 1];
  if (d == 2) {
    /* x sweep on rows jy = -M..M: wx[jy][v][a] */
    double* wx = (double*)malloc(sizeof(double) * W * nv * N);
    for (int jy = 0; jy < W; ++jy)
      for (int v = 0; v < nv; ++v) {
        for (int i = 0; i < W; ++i) win[i] = ubox[(jy * W + i) * nv + v];
        orc_weno_1d(M, win, &wx[(jy * nv + v) * N]);
      }
    /* y sweep for each x dof a */
    for (int v = 0; v < nv; ++v)
      for (int a = 0; a < N; ++a) {
        double out[NMAX];
        for (int j = 0; j < W; ++j) win[j] = wx[(j * nv + v) * N + a];
        orc_weno_1d(M, win, out);
        for (int b = 0; b < N; ++b) w[v * N * N + a + N * b] = out[b];
      }
    free(wx);
    return 0;
  }
  /* d = 3: x sweep on the (2M+1)^2 rows, y sweep on the W z-layers, z sweep */
  double* wx = (double*)malloc(sizeof(double) * W * W * nv * N);
  double* wxy = (double*)malloc(sizeof(double) * W * nv * N * N);
  for (int jz = 0; jz < W; ++jz)
    for (int jy = 0; jy < W; ++jy)
      for (int v = 0; v < nv; ++v) {
        for (int i = 0; i < W; ++i) win[i] = ubox[((jz * W + jy) * W + i) * nv + v];
        orc_weno_1d(M, win, &wx[((jz * W + jy) * nv + v) * N]);
      }
  for (int jz = 0; jz < W; ++jz)
    for (int v = 0; v < nv; ++v)
      for (int a = 0; a < N; ++a) {
        double out[NMAX];
        for (int j = 0; j < W; ++j) win[j] = wx[((jz * W + j) * nv + v) * N + a];
        orc_weno_1d(M, win, out);
        for (int b = 0; b < N; ++b) wxy[((jz * nv + v) * N + a) * N + b] = out[b];
      }
  for (int v = 0; v < nv; ++v)
    for (int a = 0; a < N; ++a)
      for (int b = 0; b < N; ++b) {
        double out[NMAX];
        for (int k = 0; k < W; ++k) win[k] = wxy[((k * nv + v) * N + a) * N + b];
        orc_weno_1d(M, win, out);
        for (int c = 0; c < N; ++c) w[v * N * N * N + a + N * b + N * N * c] = out[c];
      }
  free(wx); free(wxy);
  return 0;
}

/* ====================================================================== */
/* 4. Local space-time DG predictor                            */
/* ====================================================================== */

typedef struct {
  int d, M, N, NS, NST;
  double* K1inv;     /* [NST][NST] */
  double* Kdir[3];   /* [NST][NST] */
  double* F0;        /* [NST][NS]  */
} pred_t;

static pred_t g_pred[4][NMAX + 1];

/* multi-index decode, index = i0 + N i1 + N^2 i2 (+ N^d s), i0 = x fastest */
static void decode(int idx, int N, int n, int* out) {
  for (int k = 0; k < n; ++k) { out[k] = idx % N; idx /= N; }
}

static int build_pred(int d, int M, double* K1, double* Kd, double* F0) {
  const basis_t* B = basis_get(M);
  int N = B->N, NS = ipow(N, d), NST = NS * N;
  int qi[4], pi[4];
  for (int q = 0; q < NST; ++q) {
    decode(q, N, d + 1, qi);
    for (int p = 0; p < NST; ++p) {
      decode(p, N, d + 1, pi);
      /* K1_qp = int theta_q(xi,1) theta_p(xi,1) dxi - int int (d/dtau theta_q) theta_p */
      double ms = 1.0;
      for (int k = 0; k < d; ++k) ms *= B->M1[qi[k]][pi[k]];
      K1[q * NST + p] = ms * B->K1t[qi[d]][pi[d]];
      /* K^dir_qp = int theta_q d/dxi_dir theta_p */
      for (int dir = 0; dir < d; ++dir) {
        double v = 1.0;
        for (int k = 0; k < d; ++k) v *= (k == dir) ? B->Kx1[qi[k]][pi[k]] : B->M1[qi[k]][pi[k]];
        v *= B->M1[qi[d]][pi[d]];
        Kd[(size_t)dir * NST * NST + q * NST + p] = v;
      }
    }
    /* F0_qm = int theta_q(xi,0) psi_m(xi) dxi */
    for (int m = 0; m < NS; ++m) {
      decode(m, N, d, pi);
      double v = B->psi0[qi[d]];
      for (int k = 0; k < d; ++k) v *= B->M1[qi[k]][pi[k]];
      F0[q * NS + m] = v;
    }
  }
  return NST;
}

int orc_predictor_matrices(int d, int M, double* K1, double* Kdir, double* F0) {
  if (d < 1 || d > 3 || !basis_get(M)) return -1;
  build_pred(d, M, K1, Kdir, F0);
  return 0;
}

static const pred_t* pred_get(int d, int M) {
  pred_t* P = &g_pred[d][M];
  if (P->K1inv) return P;
  const basis_t* B = basis_get(M);
  int N = B->N, NS = ipow(N, d), NST = NS * N;
  double* K1 = (double*)malloc(sizeof(double) * NST * NST);
  double* Kd = (double*)malloc(sizeof(double) * d * NST * NST);
  P->F0 = (double*)malloc(sizeof(double) * NST * NS);
  build_pred(d, M, K1, Kd, P->F0);
  P->K1inv = (double*)malloc(sizeof(double) * NST * NST);
  /* "K1 can be easily inverted once and for all on the reference element" P:472-474 */
  mat_inverse(NST, K1, P->K1inv);
  for (int dir = 0; dir < d; ++dir) {
    P->Kdir[dir] = (double*)malloc(sizeof(double) * NST * NST);
    memcpy(P->Kdir[dir], Kd + (size_t)dir * NST * NST, sizeof(double) * NST * NST);
  }
  free(K1); free(Kd);
  P->d = d; P->M = M; P->N = N; P->NS = NS; P->NST = NST;
  return P;
}

int orc_predict_cell(int d, int M, int system, double gamma, double ch,
                     const double* w, const double* dtdx, double tol, int max_sweeps,
                     double* q, int* sweeps) {
  return orc_predict_cell_guess(d, M, system, gamma, ch, w, dtdx, tol, max_sweeps, NULL, q, sweeps);
}

void orc_extrapolate_guess(int d, int M, int nv, const double* w, const double* qp, double r, double* q0) {
  const basis_t* B = basis_get(M);
  int N = B->N, NS = ipow(N, d), NST = NS * N;
  for (int v = 0; v < nv; ++v)
    for (int x = 0; x < NS; ++x) {
      /* the node's old time polynomial at tau = 1 */
      double end = 0.0;
      for (int a = 0; a < N; ++a) end += psi_val(B, a, 1.0) * qp[v * NST + a * NS + x];
      for (int s = 0; s < N; ++s) {
        double tau = 1.0 + r * B->lam[s], val = 0.0;
        for (int a = 0; a < N; ++a) val += psi_val(B, a, tau) * qp[v * NST + a * NS + x];
        q0[v * NST + s * NS + x] = w[v * NS + x] + (val - end);
      }
    }
}

int orc_predict_cell_guess(int d, int M, int system, double gamma, double ch,
                           const double* w, const double* dtdx, double tol, int max_sweeps,
                           const double* q0, double* q, int* sweeps) {
  const pred_t* P = pred_get(d, M);
  int nv = orc_nvar(system, d), NS = P->NS, NST = P->NST;
  double* qo = (double*)malloc(sizeof(double) * nv * NST);
  double* fs = (double*)malloc(sizeof(double) * 3 * nv * NST);
  double* rhs = (double*)malloc(sizeof(double) * NST);
  /* initial guess: time-constant extension of w_h (reading R3), or
   * the caller's (reading R25) */
  if (q0) memcpy(q, q0, sizeof(double) * nv * NST);
  else
    for (int v = 0; v < nv; ++v)
      for (int p = 0; p < NST; ++p) q[v * NST + p] = w[v * NS + p % NS];
  int k, rc = 3;
  for (k = 1; k <= max_sweeps; ++k) {
    memcpy(qo, q, sizeof(double) * nv * NST);
    /* nodal fluxes f*_p = (dt/dx) f(q_p), eqn.nodal.eval @ P:405-412 */
    for (int p = 0; p < NST; ++p) {
      double up[VMAX], f[VMAX];
      for (int v = 0; v < nv; ++v) up[v] = qo[v * NST + p];
      for (int dir = 0; dir < d; ++dir) {
        if (orc_phys_flux(system, d, gamma, ch, up, dir, f)) { rc = 3; goto done_fail; }
        for (int v = 0; v < nv; ++v) fs[(dir * nv + v) * NST + p] = dtdx[dir] * f[v];
      }
    }
    /* K1 q^{k+1} = F0 w - sum_dir K^dir f*^k   (eqn.stdg.final, S = 0) */
    double dmax = 0.0, qmax = 0.0;
    for (int v = 0; v < nv; ++v) {
      for (int r = 0; r < NST; ++r) {
        double acc = 0.0;
        for (int m = 0; m < NS; ++m) acc += P->F0[r * NS + m] * w[v * NS + m];
        for (int dir = 0; dir < d; ++dir)
          for (int p = 0; p < NST; ++p) acc -= P->Kdir[dir][r * NST + p] * fs[(dir * nv + v) * NST + p];
        rhs[r] = acc;
      }
      for (int p = 0; p < NST; ++p) {
        double acc = 0.0;
        for (int r = 0; r < NST; ++r) acc += P->K1inv[p * NST + r] * rhs[r];
        q[v * NST + p] = acc;
        double dd = fabs(acc - qo[v * NST + p]);
        if (dd > dmax) dmax = dd;
        if (fabs(acc) > qmax) qmax = fabs(acc);
      }
    }
    /* stopping rule (reading R2): max|dq| <= tol (1 + max|q|) */
    if (dmax <= tol * (1.0 + qmax)) { rc = 0; break; }
  }
  if (k > max_sweeps) k = max_sweeps;
done_fail:
  if (sweeps) *sweeps = k;
  free(qo); free(fs); free(rhs);
  return rc;
}

/* ====================================================================== */
/* 5. Space-time face flux (flux:F/G/H @ P:158-172)                        */
/* ====================================================================== */

/* q_h(xi, tau) = theta_p(xi, tau) q_p  (eqn.st.q @ P:391-394) */
static void eval_st(const basis_t* B, int d, int nv, const double* q, const double* xi, double tau, double* out) {
  int N = B->N, NST = ipow(N, d + 1);
  for (int v = 0; v < nv; ++v) out[v] = 0.0;
  int pi[4];
  for (int p = 0; p < NST; ++p) {
    decode(p, N, d + 1, pi);
    double th = psi_val(B, pi[d], tau);
    for (int k = 0; k < d; ++k) th *= psi_val(B, pi[k], xi[k]);
    for (int v = 0; v < nv; ++v) out[v] += th * q[v * NST + p];
  }
}

int orc_face_flux(int d, int M, int system, double gamma, double ch, int flux, int nq, int dir,
                  const double* qL, const double* qR, double* F) {
  const basis_t* B = basis_get(M);
  int N = B->N, nv = orc_nvar(system, d);
  for (int v = 0; v < nv; ++v) F[v] = 0.0;
  /* tangential directions */
  int tdir[2], nt = 0;
  for (int k = 0; k < d; ++k) if (k != dir) tdir[nt++] = k;
  int npt = ipow(N, d - 1);
  for (int s = 0; s < N; ++s)
    for (int t = 0; t < npt; ++t) {
      int ti[2] = {t % N, t / N};
      double xl[3], xr[3], wgt = B->w[s];
      for (int k = 0; k < nt; ++k) { xl[tdir[k]] = xr[tdir[k]] = B->lam[ti[k]]; wgt *= B->w[ti[k]]; }
      xl[dir] = 1.0; xr[dir] = 0.0;
      double um[VMAX], up[VMAX], ft[VMAX];
      /* q_h^- at x_{i+1/2} from the left cell, q_h^+ from the right cell; at a
       * transmissive boundary face the missing side is NULL and takes the
       * interior trace, q^+ = q^- (reading R5) */
      if (qL) eval_st(B, d, nv, qL, xl, B->lam[s], um);
      if (qR) eval_st(B, d, nv, qR, xr, B->lam[s], up);
      if (!qL) memcpy(um, up, sizeof(double) * nv);
      if (!qR) memcpy(up, um, sizeof(double) * nv);
      if (orc_numflux(system, d, gamma, ch, flux, nq, um, up, dir, ft)) return 3;
      for (int v = 0; v < nv; ++v) F[v] += wgt * ft[v];
    }
  return 0;
}

void orc_eval_st(int d, int M, int nv, const double* q, const double* xi, double tau, double* out) {
  eval_st(basis_get(M), d, nv, q, xi, tau, out);
}

void orc_eval_w(int d, int M, int nv, const double* w, const double* xi, double* out) {
  const basis_t* B = basis_get(M);
  int N = B->N, NS = ipow(N, d), pi[3];
  for (int v = 0; v < nv; ++v) out[v] = 0.0;
  for (int p = 0; p < NS; ++p) {
    decode(p, N, d, pi);
    double th = 1.0;
    for (int k = 0; k < d; ++k) th *= psi_val(B, pi[k], xi[k]);
    for (int v = 0; v < nv; ++v) out[v] += th * w[v * NS + p];
  }
}

void orc_gauss_legendre(int n, double* x, double* w) { gauss_legendre01(n, x, w); }

int orc_face_flux_mapped(int d, int M, int system, double gamma, double ch, int flux, int nq, int dir,
                         const double* qL, const double* offL, double sclL, double toffL, double tsclL,
                         const double* qR, const double* offR, double sclR, double toffR, double tsclR,
                         double* F) {
  const basis_t* B = basis_get(M);
  int N = B->N, nv = orc_nvar(system, d);
  for (int v = 0; v < nv; ++v) F[v] = 0.0;
  int tdir[2], nt = 0;
  for (int k = 0; k < d; ++k) if (k != dir) tdir[nt++] = k;
  int npt = ipow(N, d - 1);
  for (int s = 0; s < N; ++s)
    for (int t = 0; t < npt; ++t) {
      int ti[2] = {t % N, t / N};
      double xl[3], xr[3], wgt = B->w[s];
      for (int k = 0; k < nt; ++k) {
        const int a = tdir[k];
        const double eta = B->lam[ti[k]];
        if (qL) xl[a] = offL[a] + sclL * eta;
        if (qR) xr[a] = offR[a] + sclR * eta;
        wgt *= B->w[ti[k]];
      }
      double um[VMAX], up[VMAX], ft[VMAX];
      if (qL) { xl[dir] = offL[dir]; eval_st(B, d, nv, qL, xl, toffL + tsclL * B->lam[s], um); }
      if (qR) { xr[dir] = offR[dir]; eval_st(B, d, nv, qR, xr, toffR + tsclR * B->lam[s], up); }
      if (!qL) memcpy(um, up, sizeof(double) * nv);
      if (!qR) memcpy(up, um, sizeof(double) * nv);
      if (orc_numflux(system, d, gamma, ch, flux, nq, um, up, dir, ft)) return 3;
      for (int v = 0; v < nv; ++v) F[v] += wgt * ft[v];
    }
  return 0;
}

/* Reading R14 of the garbled eqn.indicator: with unit
 * offsets +-k on the same-level 3^d box,
 *   N_kk = P(+k) - 2P(0) + P(-k)
 *   E_kk = |P(+k)-P(0)| + |P(0)-P(-k)| + eps (|P(+k)| + 2|P(0)| + |P(-k)|)
 *   N_kl = 1/4 [P(+k+l) - P(+k-l) - P(-k+l) + P(-k-l)]                 k != l
 *   E_kl = 1/2 [|P(+k+l)-P(-k+l)| + |P(+k-l)-P(-k-l)|]
 *          + eps/4 [|P(+k+l)| + |P(+k-l)| + |P(-k+l)| + |P(-k-l)|]
 *   chi  = sqrt(sum N^2 / sum E^2) over ordered pairs (k outer, l inner),
 *   chi = 0 if the denominator vanishes.  The loop order and the explicit
 *   left-to-right sums are part of the reading (bit-exact flags, H2). */
double orc_indicator(int d, const double* phi, double eps) {
  int W = 3, st[3] = {1, 3, 9};
  int c = 0;
  for (int k = 0; k < d; ++k) c += st[k];
  double num = 0.0, den = 0.0;
  for (int k = 0; k < d; ++k)
    for (int l = 0; l < d; ++l) {
      double n, e;
      if (k == l) {
        double pp = phi[c + st[k]], p0 = phi[c], pm = phi[c - st[k]];
        n = (pp - 2.0 * p0) + pm;
        e = (fabs(pp - p0) + fabs(p0 - pm)) + eps * ((fabs(pp) + 2.0 * fabs(p0)) + fabs(pm));
      } else {
        double a = phi[c + st[k] + st[l]], b = phi[c + st[k] - st[l]];
        double cc = phi[c - st[k] + st[l]], dd = phi[c - st[k] - st[l]];
        n = 0.25 * (((a - b) - cc) + dd);
        e = 0.5 * (fabs(a - cc) + fabs(b - dd)) + 0.25 * eps * (((fabs(a) + fabs(b)) + fabs(cc)) + fabs(dd));
      }
      num = num + n * n;
      den = den + e * e;
    }
  (void)W;
  if (den == 0.0) return 0.0;
  return sqrt(num / den);
}

/* ====================================================================== */
/* 6. Uniform-grid driver (eq:finite_vol @ P:147-152)                      */
/* ====================================================================== */

struct orc_ctx {
  orc_config cfg;
  int d, M, N, nv, NS, NST, G;
  int n[3], np[3];
  int64_t npad;
  double dx[3];
  double* u;          /* padded grid [pad cell][nv], ghosts of width G */
  double t;
  /* reading R25 (pred_guess = 1): q_h of every predicted cell of the last
   * orc_step step (padded index) and that step's dt; qnext collects the
   * current step's */
  double *qprev, *qnext;
  double dtprev;
  int have_prev;
  orc_ic_fn ic;       /* the problem's initial condition (ORC_BC_EXACT sides, R26) */
  void* ic_user;
  int ext_ghosts;
  char err[512];
};

static int64_t pidx(const orc_ctx* c, int i, int j, int k) {
  return ((int64_t)(k + (c->d == 3 ? c->G : 0)) * c->np[1] + (j + c->G)) * c->np[0] + (i + c->G);
}

orc_ctx* orc_create(const orc_config* cfg) {
  if (!cfg || (cfg->dim != 2 && cfg->dim != 3) || cfg->degree < 1 || cfg->degree + 1 > NMAX) return NULL;
  if (cfg->flux == ORC_FLUX_OSHER && cfg->system != ORC_EULER) return NULL;   /* Osher: Euler only */
  for (int k = 0; k < 2 * cfg->dim; ++k)
    if (cfg->bc[k] == ORC_BC_REFLECTIVE && (cfg->system != ORC_EULER || cfg->n[k / 2] < cfg->degree + 1)) return NULL;
  orc_ctx* c = (orc_ctx*)calloc(1, sizeof(orc_ctx));
  c->cfg = *cfg;
  c->d = cfg->dim; c->M = cfg->degree; c->N = c->M + 1;
  c->nv = orc_nvar(cfg->system, c->d);
  c->NS = ipow(c->N, c->d); c->NST = c->NS * c->N;
  c->G = c->M + 1;   /* update needs q of face neighbours, q needs a (2M+1)^d box */
  for (int k = 0; k < 3; ++k) {
    c->n[k] = (k < c->d) ? cfg->n[k] : 1;
    if (c->n[k] < 1) { free(c); return NULL; }
    c->np[k] = (k < c->d) ? c->n[k] + 2 * c->G : 1;
    c->dx[k] = (k < c->d) ? (cfg->hi[k] - cfg->lo[k]) / c->n[k] : 1.0;
  }
  c->npad = (int64_t)c->np[0] * c->np[1] * c->np[2];
  c->u = (double*)calloc((size_t)c->npad * c->nv, sizeof(double));
  if (c->cfg.pred_max_sweeps <= 0) c->cfg.pred_max_sweeps = 32;
  if (c->cfg.pred_tol <= 0) c->cfg.pred_tol = 1e-13;
  if (c->cfg.ic_quad <= 0) c->cfg.ic_quad = c->N;
  if (c->cfg.flux_quad <= 0) c->cfg.flux_quad = 3;   /* reading R21 */
  basis_get(c->M);
  pred_get(c->d, c->M);
  return c;
}

void orc_destroy(orc_ctx* c) { if (c) { free(c->u); free(c->qprev); free(c->qnext); free(c); } }
const char* orc_last_error(const orc_ctx* c) { return c ? c->err : "null ctx"; }
double orc_time(const orc_ctx* c) { return c->t; }
int64_t orc_num_cells(const orc_ctx* c) { return (int64_t)c->n[0] * c->n[1] * c->n[2]; }

int orc_set_initial(orc_ctx* c, orc_ic_fn ic, void* user) {
  /* the box reaches into the ghost layer on inflow sides (clipped there) */
  int32_t lo[3] = {-c->G, -c->G, -c->G}, hi[3] = {c->n[0] + c->G, c->n[1] + c->G, c->n[2] + c->G};
  return orc_set_initial_box(c, ic, user, lo, hi);
}

/* cell averages of ic(x - shift) on the cells bl + [0, be) of the padded
 * grid (cell index space, ghosts negative), by the ic_quad^d Gauss-Legendre
 * rule (reading R6) */
static void ic_average_box(orc_ctx* c, orc_ic_fn ic, void* user, const int* bl, const int* be, const double* shift) {
  int Q = c->cfg.ic_quad, d = c->d, nv = c->nv;
  double qx[16], qw[16];
  gauss_legendre01(Q, qx, qw);
  int nq = ipow(Q, d);
  int64_t ncell = (int64_t)be[0] * be[1] * be[2];
  const int64_t chunk = 4096;
  double* x = (double*)malloc(sizeof(double) * chunk * nq * 3);
  double* pr = (double*)malloc(sizeof(double) * chunk * nq * 9);
  for (int64_t c0 = 0; c0 < ncell; c0 += chunk) {
    int64_t nc = (ncell - c0 < chunk) ? ncell - c0 : chunk;
    for (int64_t ci = 0; ci < nc; ++ci) {
      int64_t lin = c0 + ci;
      int ii[3] = {bl[0] + (int)(lin % be[0]), bl[1] + (int)((lin / be[0]) % be[1]), bl[2] + (int)(lin / ((int64_t)be[0] * be[1]))};
      for (int g = 0; g < nq; ++g) {
        int gi[3] = {g % Q, (g / Q) % Q, g / (Q * Q)};
        double* xp = &x[(ci * nq + g) * 3];
        for (int k = 0; k < 3; ++k)
          xp[k] = (k < d) ? (c->cfg.lo[k] + ((double)ii[k] + qx[gi[k]]) * c->dx[k]) - shift[k] : 0.0;
      }
    }
    for (int64_t i = 0; i < nc * nq * 9; ++i) pr[i] = 0.0;
    ic(x, nc * nq, pr, user);
    for (int64_t ci = 0; ci < nc; ++ci) {
      int64_t lin = c0 + ci;
      int ii[3] = {bl[0] + (int)(lin % be[0]), bl[1] + (int)((lin / be[0]) % be[1]), bl[2] + (int)(lin / ((int64_t)be[0] * be[1]))};
      double acc[VMAX] = {0};
      /* u_bar = sum_g (prod_k w_gk) cons(ic(x_g)) , z outer, y, x inner (reading R6) */
      for (int g = 0; g < nq; ++g) {
        int gi[3] = {g % Q, (g / Q) % Q, g / (Q * Q)};
        double wg = 1.0;
        for (int k = 0; k < d; ++k) wg *= qw[gi[k]];
        double uu[VMAX];
        orc_prim_to_cons(c->cfg.system, d, c->cfg.gamma, &pr[(ci * nq + g) * 9], uu);
        for (int v = 0; v < nv; ++v) acc[v] += wg * uu[v];
      }
      double* dst = &c->u[pidx(c, ii[0], ii[1], ii[2]) * nv];
      for (int v = 0; v < nv; ++v) dst[v] = acc[v];
    }
  }
  free(x); free(pr);
}

int orc_set_initial_box(orc_ctx* c, orc_ic_fn ic, void* user, const int32_t* blo, const int32_t* bhi) {
  int d = c->d;
  c->have_prev = 0;
  c->ic = ic;
  c->ic_user = user;
  int bl[3], be[3];
  for (int k = 0; k < 3; ++k) {
    /* inflow and exact sides (R23, R26): the ghost layer takes IC averages too */
    const int lo_g = k < d && (c->cfg.bc[2 * k] == ORC_BC_INFLOW || c->cfg.bc[2 * k] == ORC_BC_EXACT);
    const int hi_g = k < d && (c->cfg.bc[2 * k + 1] == ORC_BC_INFLOW || c->cfg.bc[2 * k + 1] == ORC_BC_EXACT);
    const int glo = lo_g ? -c->G : 0;
    const int ghi = hi_g ? c->n[k] + c->G : c->n[k];
    bl[k] = (k < d) ? (blo[k] < glo ? glo : blo[k]) : 0;
    int h = (k < d) ? (bhi[k] > ghi ? ghi : bhi[k]) : 1;
    be[k] = h > bl[k] ? h - bl[k] : 0;
  }
  const double zero[3] = {0, 0, 0};
  ic_average_box(c, ic, user, bl, be, zero);
  c->t = 0.0;
  return 0;
}

/* Reading R26 (the "exact solution prescribed" boundaries of P:1103-1105):
 * before every step the ghost layer of each ORC_BC_EXACT side, over the full
 * padded extent of the other axes, takes the averages of the exact solution
 * at the step's start time, u(x, t) = ic(x - t exact_vel). */
static void refresh_exact(orc_ctx* c) {
  if (!c->ic) return;
  const int d = c->d, G = c->G;
  const double shift[3] = {c->t * c->cfg.exact_vel[0], c->t * c->cfg.exact_vel[1], c->t * c->cfg.exact_vel[2]};
  for (int a = 0; a < d; ++a)
    for (int side = 0; side < 2; ++side) {
      if (c->cfg.bc[2 * a + side] != ORC_BC_EXACT) continue;
      int bl[3], be[3];
      for (int k = 0; k < 3; ++k) {
        bl[k] = (k < d) ? -G : 0;
        be[k] = (k < d) ? c->n[k] + 2 * G : 1;
      }
      bl[a] = side ? c->n[a] : -G;
      be[a] = G;
      ic_average_box(c, c->ic, c->ic_user, bl, be, shift);
    }
}

int orc_set_cells(orc_ctx* c, const double* u) {
  int64_t lin = 0;
  c->have_prev = 0;   /* R25: a new state has no previous step */
  for (int k = 0; k < c->n[2]; ++k)
    for (int j = 0; j < c->n[1]; ++j)
      for (int i = 0; i < c->n[0]; ++i, ++lin)
        memcpy(&c->u[pidx(c, i, j, k) * c->nv], &u[lin * c->nv], sizeof(double) * c->nv);
  return 0;
}

int orc_get_cells(const orc_ctx* c, double* u) {
  int64_t lin = 0;
  for (int k = 0; k < c->n[2]; ++k)
    for (int j = 0; j < c->n[1]; ++j)
      for (int i = 0; i < c->n[0]; ++i, ++lin)
        memcpy(&u[lin * c->nv], &c->u[pidx(c, i, j, k) * c->nv], sizeof(double) * c->nv);
  return 0;
}

/* Ghost cells (reading R5): periodic wrap, or transmissive copy of the
 * nearest interior cell (index clamped per axis); reflective walls (R22) take
 * the mirror cell (index -1-i / 2n-1-i) with the normal momentum negated. */
static int ghost_src(const orc_ctx* c, int axis, int i) {
  int n = c->n[axis];
  if (i >= 0 && i < n) return i;
  int side = (i < 0) ? 0 : 1;
  if (c->cfg.bc[2 * axis + side] == ORC_BC_PERIODIC) return ((i % n) + n) % n;
  if (c->cfg.bc[2 * axis + side] == ORC_BC_REFLECTIVE) return (i < 0) ? -1 - i : 2 * n - 1 - i;
  if (c->cfg.bc[2 * axis + side] == ORC_BC_INFLOW) return i;   /* R23: the ghost keeps its IC average */
  if (c->cfg.bc[2 * axis + side] == ORC_BC_EXACT) return i;    /* R26: set by refresh_exact */
  return (i < 0) ? 0 : n - 1;
}
static int ghost_reflected(const orc_ctx* c, int axis, int i) {
  if (i >= 0 && i < c->n[axis]) return 0;
  return c->cfg.bc[2 * axis + (i < 0 ? 0 : 1)] == ORC_BC_REFLECTIVE;
}

void orc_reflect_poly(int d, int M, int nv, int dir, const double* q, double* out) {
  int N = M + 1, NST = ipow(N, d + 1), pi[4];
  for (int p = 0; p < NST; ++p) {
    decode(p, N, d + 1, pi);
    pi[dir] = N - 1 - pi[dir];
    int src = 0;
    for (int k = d; k >= 0; --k) src = src * N + pi[k];
    for (int v = 0; v < nv; ++v) out[v * NST + p] = (v == 1 + dir ? -1.0 : 1.0) * q[v * NST + src];
  }
}

int64_t orc_num_padded(const orc_ctx* c) { return c->npad; }
int orc_get_padded(const orc_ctx* c, double* u) { memcpy(u, c->u, sizeof(double) * c->npad * c->nv); return 0; }
int orc_set_padded(orc_ctx* c, const double* u) { memcpy(c->u, u, sizeof(double) * c->npad * c->nv); return 0; }
void orc_set_external_ghosts(orc_ctx* c, int on) { c->ext_ghosts = on; }

static void fill_ghosts(orc_ctx* c) {
  if (c->ext_ghosts) return;   /* ghost cells provided by the caller (distributed emulation) */
  int G = c->G;
  int lo[3], hi[3];
  for (int k = 0; k < 3; ++k) { lo[k] = (k < c->d) ? -G : 0; hi[k] = (k < c->d) ? c->n[k] + G : 1; }
  for (int k = lo[2]; k < hi[2]; ++k)
    for (int j = lo[1]; j < hi[1]; ++j)
      for (int i = lo[0]; i < hi[0]; ++i) {
        int si = ghost_src(c, 0, i), sj = ghost_src(c, 1, j), sk = (c->d == 3) ? ghost_src(c, 2, k) : 0;
        if (si == i && sj == j && sk == k) continue;
        double* g = &c->u[pidx(c, i, j, k) * c->nv];
        memcpy(g, &c->u[pidx(c, si, sj, sk) * c->nv], sizeof(double) * c->nv);
        const int ii[3] = {i, j, k};
        for (int a = 0; a < c->d; ++a)
          if (ghost_reflected(c, a, ii[a])) g[1 + a] = -g[1 + a];
      }
}

/* Reading R1: dt = CFL / max_cells sum_dir s_dir(u)/dx_dir. */
double orc_compute_dt(orc_ctx* c) {
  double smax = 0.0;
  for (int k = 0; k < c->n[2]; ++k)
    for (int j = 0; j < c->n[1]; ++j)
      for (int i = 0; i < c->n[0]; ++i) {
        const double* u = &c->u[pidx(c, i, j, k) * c->nv];
        double s = 0.0;
        for (int dir = 0; dir < c->d; ++dir)
          s += orc_max_speed(c->cfg.system, c->d, c->cfg.gamma, c->cfg.ch, u, dir) / c->dx[dir];
        if (!(s <= smax)) smax = s;   /* NaN propagates */
      }
  return c->cfg.cfl / smax;
}

/* Gather the (2M+1)^d box of cell (i,j,k) from the padded grid. */
static void gather_box(const orc_ctx* c, int i, int j, int k, double* box) {
  int M = c->M, W = 2 * M + 1, nv = c->nv;
  int zl = (c->d == 3) ? -M : 0, zh = (c->d == 3) ? M : 0;
  int b = 0;
  for (int dz = zl; dz <= zh; ++dz)
    for (int dy = -M; dy <= M; ++dy)
      for (int dx = -M; dx <= M; ++dx, ++b)
        memcpy(&box[b * nv], &c->u[pidx(c, i + dx, j + dy, k + dz) * nv], sizeof(double) * nv);
  (void)W;
}

/* Ghost cell beyond a transmissive or reflective boundary (its predictor is
 * never used: boundary faces use the interior trace, R5, or its reflection, R22). */
static int beyond_transmissive(const orc_ctx* c, int i, int j, int k) {
  const int ii[3] = {i, j, k};
  for (int a = 0; a < c->d; ++a) {
    const int lo = c->cfg.bc[2 * a], hi = c->cfg.bc[2 * a + 1];
    if (ii[a] < 0 && (lo == ORC_BC_TRANSMISSIVE || lo == ORC_BC_REFLECTIVE)) return 1;
    if (ii[a] >= c->n[a] && (hi == ORC_BC_TRANSMISSIVE || hi == ORC_BC_REFLECTIVE)) return 1;
  }
  return 0;
}

/* Reconstruct + predict cell (i,j,k) (may be a ghost cell of depth 1). */
static int cell_predict(orc_ctx* c, int i, int j, int k, double dt, double* q, int* sweeps) {
  int M = c->M, W = 2 * M + 1, nv = c->nv;
  int nb = (c->d == 3) ? W * W * W : W * W;
  double* box = (double*)malloc(sizeof(double) * nb * nv);
  double* w = (double*)malloc(sizeof(double) * nv * c->NS);
  gather_box(c, i, j, k, box);
  orc_reconstruct_box(c->d, M, nv, box, w);
  double dtdx[3];
  for (int dir = 0; dir < c->d; ++dir) dtdx[dir] = dt / c->dx[dir];
  double* q0 = NULL;
  const int64_t pc = pidx(c, i, j, k);
  if (c->cfg.pred_guess == 1 && c->have_prev && c->dtprev > 0.0 && dt > 0.0) {
    q0 = (double*)malloc(sizeof(double) * nv * c->NST);
    orc_extrapolate_guess(c->d, M, nv, w, &c->qprev[pc * nv * c->NST], dt / c->dtprev, q0);
  }
  int rc = orc_predict_cell_guess(c->d, M, c->cfg.system, c->cfg.gamma, c->cfg.ch, w, dtdx,
                                  c->cfg.pred_tol, c->cfg.pred_max_sweeps, q0, q, sweeps);
  if (c->qnext && rc == 0) memcpy(&c->qnext[pc * nv * c->NST], q, sizeof(double) * nv * c->NST);
  free(q0);
  if (rc)
    snprintf(c->err, sizeof(c->err), "predictor failed (non-convergence or inadmissible state) in cell (%d,%d,%d), level 0, t=%.17g", i, j, k, c->t);
  free(box); free(w);
  return rc;
}

int orc_advance_box(orc_ctx* c, double dt, const int32_t* blo, const int32_t* bhi,
                    double* out, orc_report* rep) {
  int d = c->d, nv = c->nv, NST = c->NST;
  if (!c->ext_ghosts) refresh_exact(c);
  fill_ghosts(c);
  int lo[3], hi[3], ext[3];
  for (int k = 0; k < 3; ++k) {
    lo[k] = (k < d) ? blo[k] : 0; hi[k] = (k < d) ? bhi[k] : 1;
    ext[k] = hi[k] - lo[k] + ((k < d) ? 2 : 0);   /* box + 1 layer (face neighbours) */
  }
  int64_t next = (int64_t)ext[0] * ext[1] * ext[2];
  double* q = (double*)calloc((size_t)next * nv * NST, sizeof(double));
  double qref[VMAX * 256], qref2[VMAX * 256];   /* reflected polynomials (N^(d+1) <= 256) */
  int64_t sw_tot = 0; int sw_max = 0;
  int off = 1;
  /* 1. reconstruction + predictor on the box and its face neighbours */
  for (int k = 0; k < ext[2]; ++k)
    for (int j = 0; j < ext[1]; ++j)
      for (int i = 0; i < ext[0]; ++i) {
        int ci = lo[0] + i - off, cj = lo[1] + j - off, ck = (d == 3) ? lo[2] + k - off : 0;
        int outside = (ci < lo[0] || ci >= hi[0]) + (cj < lo[1] || cj >= hi[1]) +
                      ((d == 3) && (ck < lo[2] || ck >= hi[2]));
        if (outside > 1) continue;   /* only face neighbours are needed */
        if (beyond_transmissive(c, ci, cj, ck)) continue;   /* R5: not used */
        int sw = 0;
        int64_t e = ((int64_t)k * ext[1] + j) * ext[0] + i;
        if (cell_predict(c, ci, cj, ck, dt, &q[e * nv * NST], &sw)) { free(q); return 3; }
        sw_tot += sw; if (sw > sw_max) sw_max = sw;
      }
  /* 2. face fluxes and 3. update (eq:finite_vol) */
  int64_t o = 0;
  for (int k = lo[2]; k < hi[2]; ++k)
    for (int j = lo[1]; j < hi[1]; ++j)
      for (int i = lo[0]; i < hi[0]; ++i, ++o) {
        double unew[VMAX];
        const double* u0 = &c->u[pidx(c, i, j, k) * nv];
        for (int v = 0; v < nv; ++v) unew[v] = u0[v];
        int ei = i - lo[0] + off, ej = j - lo[1] + off, ek = (d == 3) ? k - lo[2] + off : 0;
        int64_t e0 = ((int64_t)ek * ext[1] + ej) * ext[0] + ei;
        double Fm[VMAX], Fp[VMAX];
        for (int dir = 0; dir < d; ++dir) {
          int64_t stride = (dir == 0) ? 1 : (dir == 1) ? ext[0] : (int64_t)ext[0] * ext[1];
          const int ic[3] = {i, j, k};
          const double* qc = &q[e0 * nv * NST];
          /* R5: a transmissive boundary face takes the interior trace on both
           * sides; R22: a reflective wall faces the reflected polynomial */
          const double* qm = &q[(e0 - stride) * nv * NST];
          const double* qp = &q[(e0 + stride) * nv * NST];
          if (ic[dir] == 0 && c->cfg.bc[2 * dir] == ORC_BC_TRANSMISSIVE) qm = NULL;
          if (ic[dir] == c->n[dir] - 1 && c->cfg.bc[2 * dir + 1] == ORC_BC_TRANSMISSIVE) qp = NULL;
          if (ic[dir] == 0 && c->cfg.bc[2 * dir] == ORC_BC_REFLECTIVE) {
            orc_reflect_poly(d, c->M, nv, dir, qc, qref);
            qm = qref;
          }
          if (ic[dir] == c->n[dir] - 1 && c->cfg.bc[2 * dir + 1] == ORC_BC_REFLECTIVE) {
            orc_reflect_poly(d, c->M, nv, dir, qc, qref2);
            qp = qref2;
          }
          if (orc_face_flux(d, c->M, c->cfg.system, c->cfg.gamma, c->cfg.ch, c->cfg.flux, c->cfg.flux_quad, dir, qm, qc, Fm) ||
              orc_face_flux(d, c->M, c->cfg.system, c->cfg.gamma, c->cfg.ch, c->cfg.flux, c->cfg.flux_quad, dir, qc, qp, Fp)) {
            snprintf(c->err, sizeof(c->err), "inadmissible face state at cell (%d,%d,%d) t=%.17g", i, j, k, c->t);
            free(q); return 3;
          }
          for (int v = 0; v < nv; ++v) unew[v] = unew[v] - dt / c->dx[dir] * (Fp[v] - Fm[v]);
        }
        memcpy(&out[o * nv], unew, sizeof(double) * nv);
      }
  if (rep) {
    rep->sweeps_total += sw_tot;
    if (sw_max > rep->sweeps_max) rep->sweeps_max = sw_max;
    rep->cell_updates += o;
  }
  free(q);
  return 0;
}

int orc_step(orc_ctx* c, double t_end, int64_t max_steps, orc_report* rep) {
  orc_report r; memset(&r, 0, sizeof(r));
  int64_t ncell = orc_num_cells(c);
  double* un = (double*)malloc(sizeof(double) * ncell * c->nv);
  int32_t blo[3] = {0, 0, 0}, bhi[3] = {c->n[0], c->n[1], c->n[2]};
  int rc = 0;
  if (c->cfg.pred_guess == 1 && !c->qprev) {
    c->qprev = (double*)calloc((size_t)c->npad * c->nv * c->NST, sizeof(double));
    c->qnext = (double*)calloc((size_t)c->npad * c->nv * c->NST, sizeof(double));
  }
  while (r.steps < max_steps && c->t < t_end) {
    double dt = orc_compute_dt(c);
    if (!(dt > 0.0) || !isfinite(dt)) { snprintf(c->err, sizeof(c->err), "invalid dt %g", dt); rc = 3; break; }
    if (c->t + dt > t_end) dt = t_end - c->t;
    rc = orc_advance_box(c, dt, blo, bhi, un, &r);
    if (rc) break;
    orc_set_cells(c, un);
    if (c->qnext) {   /* R25: this step's q_h become the next step's guess source */
      double* tmp = c->qprev; c->qprev = c->qnext; c->qnext = tmp;
      c->dtprev = dt;
      c->have_prev = 1;
    }
    c->t += dt;
    r.dt = dt;
    r.steps++;
  }
  r.t = c->t;
  r.updates_per_level[0] = r.cell_updates;
  r.min_threshold_margin = 1e300;   /* no adapt on a uniform grid */
  if (rep) *rep = r;
  free(un);
  return rc;
}

int orc_dump_recon(orc_ctx* c, double* w) {
  fill_ghosts(c);
  int M = c->M, W = 2 * M + 1, nv = c->nv;
  int nb = (c->d == 3) ? W * W * W : W * W;
  double* box = (double*)malloc(sizeof(double) * nb * nv);
  int64_t lin = 0;
  for (int k = 0; k < c->n[2]; ++k)
    for (int j = 0; j < c->n[1]; ++j)
      for (int i = 0; i < c->n[0]; ++i, ++lin) {
        gather_box(c, i, j, k, box);
        orc_reconstruct_box(c->d, M, nv, box, &w[lin * nv * c->NS]);
      }
  free(box);
  return 0;
}

int orc_dump_pred(orc_ctx* c, double dt, double* q) {
  fill_ghosts(c);
  int64_t lin = 0;
  for (int k = 0; k < c->n[2]; ++k)
    for (int j = 0; j < c->n[1]; ++j)
      for (int i = 0; i < c->n[0]; ++i, ++lin) {
        int sw;
        if (cell_predict(c, i, j, k, dt, &q[lin * c->nv * c->NST], &sw)) return 3;
      }
  return 0;
}

int orc_dump_flux(orc_ctx* c, double dt, double* F) {
  fill_ghosts(c);
  int d = c->d, nv = c->nv, NST = c->NST;
  int e[3] = {c->n[0] + 1, c->n[1] + 1, (d == 3) ? c->n[2] + 1 : 1};
  int64_t nf = (int64_t)e[0] * e[1] * e[2];
  double* qa = (double*)malloc(sizeof(double) * nv * NST);
  double* qb = (double*)malloc(sizeof(double) * nv * NST);
  for (int dir = 0; dir < d; ++dir)
    for (int k = 0; k < e[2]; ++k)
      for (int j = 0; j < e[1]; ++j)
        for (int i = 0; i < e[0]; ++i) {
          int64_t f = ((int64_t)k * e[1] + j) * e[0] + i;
          double* Fo = &F[((int64_t)dir * nf + f) * nv];
          for (int v = 0; v < nv; ++v) Fo[v] = 0.0;
          /* lower face of cell (i,j,k) along dir; skip faces not on the grid */
          int ii[3] = {i, j, k};
          int ok = 1;
          for (int a = 0; a < d; ++a)
            if (a != dir && ii[a] >= c->n[a]) ok = 0;
          if (!ok) continue;
          int im[3] = {i, j, k};
          im[dir] -= 1;
          int sw;
          const int lob = (i == 0 && dir == 0) || (j == 0 && dir == 1) || (k == 0 && dir == 2);
          const int hib = ii[dir] == c->n[dir];
          const int tlo = lob && c->cfg.bc[2 * dir] == ORC_BC_TRANSMISSIVE;
          const int thi = hib && c->cfg.bc[2 * dir + 1] == ORC_BC_TRANSMISSIVE;
          const int rlo = lob && c->cfg.bc[2 * dir] == ORC_BC_REFLECTIVE;
          const int rhi = hib && c->cfg.bc[2 * dir + 1] == ORC_BC_REFLECTIVE;
          if (!tlo && !rlo && cell_predict(c, im[0], im[1], im[2], dt, qa, &sw)) goto fail;
          if (!thi && !rhi && cell_predict(c, i, j, k, dt, qb, &sw)) goto fail;
          if (rlo) orc_reflect_poly(d, c->M, nv, dir, qb, qa);   /* R22 */
          if (rhi) orc_reflect_poly(d, c->M, nv, dir, qa, qb);
          if (orc_face_flux(d, c->M, c->cfg.system, c->cfg.gamma, c->cfg.ch, c->cfg.flux, c->cfg.flux_quad, dir, tlo ? NULL : qa, thi ? NULL : qb, Fo)) goto fail;
        }
  free(qa); free(qb);
  return 0;
fail:
  free(qa); free(qb);
  return 3;
}
