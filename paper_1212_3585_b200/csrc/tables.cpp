// tables.cpp — host construction of the reference-element constants used by the
// CUDA kernels.  See tables.h.  Citations: P:n = PAPER.md line n.
#include "tables.h"

#include <cmath>
#include <cstring>

namespace ader {
namespace {

// Gauss-Legendre nodes / weights on [0,1] in closed form (N = 1..4).
bool gl_closed_form(int N, double* x, double* w) {
  if (N == 1) {
    x[0] = 0.5; w[0] = 1.0;
    return true;
  }
  if (N == 2) {
    const double h = std::sqrt(3.0) / 6.0;
    x[0] = 0.5 - h; x[1] = 0.5 + h;
    w[0] = w[1] = 0.5;
    return true;
  }
  if (N == 3) {
    const double h = std::sqrt(15.0) / 10.0;
    x[0] = 0.5 - h; x[1] = 0.5; x[2] = 0.5 + h;
    w[0] = 5.0 / 18.0; w[1] = 4.0 / 9.0; w[2] = 5.0 / 18.0;
    return true;
  }
  if (N == 4) {
    const double r = 2.0 / 7.0 * std::sqrt(6.0 / 5.0);
    const double a = 0.5 * std::sqrt(3.0 / 7.0 - r), b = 0.5 * std::sqrt(3.0 / 7.0 + r);
    const double wa = (18.0 + std::sqrt(30.0)) / 72.0, wb = (18.0 - std::sqrt(30.0)) / 72.0;
    x[0] = 0.5 - b; x[1] = 0.5 - a; x[2] = 0.5 + a; x[3] = 0.5 + b;
    w[0] = wb; w[1] = wa; w[2] = wa; w[3] = wb;
    return true;
  }
  return false;
}

// Solve A X = B in place (A n x n, B n x m, row-major) by LU with row pivoting.
bool solve(int n, int m, double* A, double* B) {
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(A[i * n + k]) > std::fabs(A[p * n + k])) p = i;
    if (A[p * n + k] == 0.0) return false;
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(A[k * n + j], A[p * n + j]);
      for (int j = 0; j < m; ++j) std::swap(B[k * m + j], B[p * m + j]);
    }
    for (int i = k + 1; i < n; ++i) {
      const double l = A[i * n + k] / A[k * n + k];
      for (int j = k; j < n; ++j) A[i * n + j] -= l * A[k * n + j];
      for (int j = 0; j < m; ++j) B[i * m + j] -= l * B[k * m + j];
    }
  }
  for (int k = n - 1; k >= 0; --k)
    for (int j = 0; j < m; ++j) {
      double s = B[k * m + j];
      for (int i = k + 1; i < n; ++i) s -= A[k * n + i] * B[i * m + j];
      B[k * m + j] = s / A[k * n + k];
    }
  return true;
}

struct Lagrange {
  int N;
  double x[kMaxN], bw[kMaxN];
  // psi_p(t) via the barycentric formula; exact Kronecker delta at the nodes
  double val(int p, double t) const {
    for (int k = 0; k < N; ++k)
      if (t == x[k]) return p == k ? 1.0 : 0.0;
    double num = 0.0, den = 0.0;
    for (int k = 0; k < N; ++k) {
      const double c = bw[k] / (t - x[k]);
      den += c;
      if (k == p) num = c;
    }
    return num / den;
  }
};

}  // namespace

bool build_tables(int M, DevTables* t) {
  const int N = M + 1;
  if (M < 2 || N > kMaxN) return false;
  std::memset(t, 0, sizeof(*t));
  Lagrange L;
  L.N = N;
  if (!gl_closed_form(N, L.x, t->w)) return false;
  for (int k = 0; k < N; ++k) {
    t->lam[k] = L.x[k];
    double prod = 1.0;
    for (int j = 0; j < N; ++j)
      if (j != k) prod *= (L.x[k] - L.x[j]);
    L.bw[k] = 1.0 / prod;
  }
  // differentiation matrix D[k][b] = psi_b'(x_k) (barycentric form)
  for (int k = 0; k < N; ++k) {
    double diag = 0.0;
    for (int b = 0; b < N; ++b) {
      if (b == k) continue;
      t->D[k][b] = (L.bw[b] / L.bw[k]) / (L.x[k] - L.x[b]);
      diag -= t->D[k][b];
    }
    t->D[k][k] = diag;
  }
  for (int a = 0; a < N; ++a) {
    t->psi0[a] = L.val(a, 0.0);
    t->psi1[a] = L.val(a, 1.0);
  }
  // time operator: K1t[a][b] = psi_a(1) psi_b(1) - int psi_a' psi_b
  //   (GL quadrature exact for degree 2M-1: int psi_a' psi_b = w_b D[b][a]),
  // T = K1t^{-1} diag(w) so that q = w_h - T G  (nodal form of eqn.stdg.final)
  {
    double K[kMaxN * kMaxN], B[kMaxN * kMaxN];
    for (int a = 0; a < N; ++a)
      for (int b = 0; b < N; ++b) {
        K[a * N + b] = t->psi1[a] * t->psi1[b] - t->w[b] * t->D[b][a];
        B[a * N + b] = (a == b) ? t->w[a] : 0.0;
      }
    if (!solve(N, N, K, B)) return false;
    for (int a = 0; a < N; ++a) {
      double rs = 0.0;
      for (int b = 0; b < N; ++b) { t->T[a][b] = B[a * N + b]; rs += B[a * N + b]; }
      t->Tsum[a] = rs;
    }
  }
  // WENO stencils (eqn.stencildef @ P:220-224): offsets -L..R
  int nS, Ls[4];
  if (M % 2 == 0) {
    nS = 3; Ls[0] = M / 2; Ls[1] = M; Ls[2] = 0;
    t->lin[0] = 1e5; t->lin[1] = 1.0; t->lin[2] = 1.0;
  } else {
    nS = 4; Ls[0] = M / 2 + 1; Ls[1] = M / 2; Ls[2] = M; Ls[3] = 0;
    t->lin[0] = 1e5; t->lin[1] = 1e5; t->lin[2] = 1.0; t->lin[3] = 1.0;
  }
  for (int s = 0; s < nS; ++s) {
    // A[o][p] = int_{o}^{o+1} psi_p = sum_k w_k psi_p(o + x_k)  (exact, degree M)
    double A[kMaxN * kMaxN], I[kMaxN * kMaxN];
    for (int r = 0; r < N; ++r) {
      const int o = r - Ls[s];
      for (int p = 0; p < N; ++p) {
        double acc = 0.0;
        for (int k = 0; k < N; ++k) acc += t->w[k] * L.val(p, o + L.x[k]);
        A[r * N + p] = acc;
        I[r * N + p] = (r == p) ? 1.0 : 0.0;
      }
    }
    if (!solve(N, N, A, I)) return false;
    for (int p = 0; p < N; ++p)
      for (int o = 0; o < N; ++o) t->rec[s][p][o] = I[p * N + o];
  }
  // Sigma_pm = sum_{alpha=1..M} int psi_p^(alpha) psi_m^(alpha): nodal values of
  // the alpha-th derivative are rows of D^alpha; N-point GL is exact here.
  {
    double Dk[kMaxN][kMaxN], tmp[kMaxN][kMaxN];
    std::memcpy(Dk, t->D, sizeof(Dk));
    for (int alpha = 1; alpha <= M; ++alpha) {
      for (int p = 0; p < N; ++p)
        for (int m = 0; m < N; ++m) {
          double acc = 0.0;
          for (int k = 0; k < N; ++k) acc += t->w[k] * Dk[k][p] * Dk[k][m];
          t->sigma[p][m] += acc;
        }
      for (int i = 0; i < N; ++i)
        for (int j = 0; j < N; ++j) {
          double acc = 0.0;
          for (int k = 0; k < N; ++k) acc += t->D[i][k] * Dk[k][j];
          tmp[i][j] = acc;
        }
      std::memcpy(Dk, tmp, sizeof(Dk));
    }
  }
  return true;
}

bool build_osher_quadrature(int nq, DevTables* t) {
  if (nq < 1 || nq > kMaxN) return false;
  t->oq_n = nq;
  return gl_closed_form(nq, t->oq_x, t->oq_w);
}

}  // namespace ader
