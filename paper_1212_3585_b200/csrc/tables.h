// tables.h — reference-element constants of the nodal ADER-WENO scheme for the
// CUDA path (computed on the host once per context, passed to every kernel by
// value as a __grid_constant__ parameter, i.e. read through the constant bank).
//
// Independent of oracle/: different construction (closed-form Gauss-Legendre
// nodes, barycentric differentiation matrix, node-based Gauss quadrature).
#pragma once

namespace ader {

constexpr int kMaxN = 4;   // N = M+1 <= 4 (M in {2,3})

struct DevTables {
  double lam[kMaxN];              // Gauss-Legendre nodes on [0,1]
  double w[kMaxN];                // Gauss-Legendre weights
  double psi0[kMaxN], psi1[kMaxN];// psi_a(0), psi_a(1): boundary traces
  double D[kMaxN][kMaxN];         // D[k][b] = psi_b'(lam_k)
  double T[kMaxN][kMaxN];         // T_tau = K1t^{-1} diag(w): nodal time integration
  double rec[4][kMaxN][kMaxN];    // rec[s][p][o]: stencil inverse (eqn.rec.x)
  double sigma[kMaxN][kMaxN];     // oscillation indicator matrix
  double lin[4];                  // linear weights lambda_s
  double Tsum[kMaxN];             // row sums of T_tau (first Picard sweep, time-constant guess)
  double oq_x[kMaxN], oq_w[kMaxN];// Gauss-Legendre rule of the Osher path integral
  int oq_n;                       // its number of points (1..4)
  int flux;                       // two-point flux: 0 Rusanov (eqn.rusanov), 1 Osher (eqn.osher)
};

// Fills t for degree M (2 or 3).  Returns false for an unsupported degree.
bool build_tables(int M, DevTables* t);
// Fills the nq-point path rule of eqn.osher (nq in 1..4).  Returns false otherwise.
bool build_osher_quadrature(int nq, DevTables* t);

}  // namespace ader
