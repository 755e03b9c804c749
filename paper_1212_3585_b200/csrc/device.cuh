// device.cuh — device-side physics and the 1D WENO building block.
// Citations: P:n = PAPER.md line n.
#pragma once
#include <cstdint>

#include "tables.h"

namespace ader {

// Reciprocal and square root from the MUFU approximations refined by Newton
// steps to ~1 ulp: the IEEE-exact div/sqrt sequences (slow-path branches
// included) dominated the pointwise flux evaluations.  Inputs here are
// positive, normal numbers (densities, squared sound speeds); the
// admissibility checks run on the unmodified values.  The MUFU seeds are good
// to ~2^-20 (relative), each Newton step squares the error: two steps for the
// reciprocal (2^-80), one for 1/sqrt (2^-39) followed by one correction of
// s = a/sqrt(a) (2^-78) — fewer dependent FP64 operations on the flux
// evaluations' critical path than the three-step forms of round 1.
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ double fast_sqrt(double a) {
  if (!(a > 0.0)) return 0.0;
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  // Newton on 1/sqrt(a): y <- y (3 - a y^2) / 2; then s = a y with one correction
  const double h = 0.5 * a;
  y = y * fma(-h * y, y, 1.5);
  const double s = a * y;
  const double r = fma(-s, s, a);
  return fma(0.5 * y, r, s);
}

// ---------------------------------------------------------------------------
// Physics.  Euler (eq:Euler-system @ P:838-869): nu = D+2 (rho, rho v, E) —
// reading R7 drops the identically-zero v_z row in 2D.  GLM-MHD in Gaussian
// units: nu = 9 (rho, rho v[3], E, B[3], psi).
// All functions return false when the state is inadmissible (rho<=0, p<=0).
// ---------------------------------------------------------------------------
template <int SYS, int D> struct Phys;

template <int D> struct Phys<0, D> {
  static constexpr int NV = D + 2;
  // fluxes f_dir(u) for every direction at once (predictor nodes)
  __device__ __forceinline__ static bool fluxes(const double (&u)[NV], double gamma, double /*ch*/,
                                                double (&f)[D][NV]) {
    const double rho = u[0];
    const double ir = fast_rcp(rho);
    double v[D], ke = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) { v[k] = u[1 + k] * ir; ke += v[k] * u[1 + k]; }
    const double p = (gamma - 1.0) * (u[D + 1] - 0.5 * ke);
    const double ep = u[D + 1] + p;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      f[d][0] = u[1 + d];
#pragma unroll
      for (int k = 0; k < D; ++k) f[d][1 + k] = u[1 + d] * v[k];
      f[d][1 + d] += p;
      f[d][D + 1] = v[d] * ep;
    }
    return rho > 0.0 && p > 0.0;
  }
  // flux along one direction + max |eigenvalue|: |v_n| + sqrt(gamma p / rho)
  template <int DIR>
  __device__ __forceinline__ static bool flux_speed(const double (&u)[NV], double gamma, double /*ch*/,
                                                    double (&f)[NV], double& s) {
    const double rho = u[0];
    const double ir = fast_rcp(rho);
    double v[D], ke = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) { v[k] = u[1 + k] * ir; ke += v[k] * u[1 + k]; }
    const double p = (gamma - 1.0) * (u[D + 1] - 0.5 * ke);
    f[0] = u[1 + DIR];
#pragma unroll
    for (int k = 0; k < D; ++k) f[1 + k] = u[1 + DIR] * v[k];
    f[1 + DIR] += p;
    f[D + 1] = v[DIR] * (u[D + 1] + p);
    const bool ok = rho > 0.0 && p > 0.0;
    s = fabs(v[DIR]) + fast_sqrt(gamma * p * ir);
    return ok;
  }
  // sum_dir s_dir(u) * inv_dx[dir]  (CFL, reading R1)
  __device__ __forceinline__ static bool cfl_speed(const double (&u)[NV], double gamma, double /*ch*/,
                                                   const double (&inv_dx)[3], double& s) {
    const double rho = u[0];
    const double ir = fast_rcp(rho);
    double v[D], ke = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) { v[k] = u[1 + k] * ir; ke += v[k] * u[1 + k]; }
    const double p = (gamma - 1.0) * (u[D + 1] - 0.5 * ke);
    const double c = fast_sqrt(gamma * p * ir);
    s = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) s += (fabs(v[k]) + c) * inv_dx[k];
    return rho > 0.0 && p > 0.0;
  }
  __device__ __forceinline__ static void prim_to_cons(const double* pr, double gamma, double (&u)[NV]) {
    const double rho = pr[0];
    double ke = 0.0;
    u[0] = rho;
#pragma unroll
    for (int k = 0; k < D; ++k) { u[1 + k] = rho * pr[1 + k]; ke += pr[1 + k] * pr[1 + k]; }
    u[D + 1] = pr[4] / (gamma - 1.0) + 0.5 * rho * ke;
  }
  // acc += wq |A_DIR(u)| du with the closed-form eigenvectors of the Euler
  // Jacobian (used by the Osher path integral, eqn.osher @ P:186-196):
  //   |A| du = |v_n| du + (|v_n - c| - |v_n|) a1 r1 + (|v_n + c| - |v_n|) a3 r3,
  //   dp = (gamma-1)(|v|^2 drho / 2 - v.dm + dE),  rho dv_n = dm_n - v_n drho,
  //   a1,3 = (dp -+ c rho dv_n) / (2 c^2),  r1,3 = (1, v -+ c e_n, H -+ v_n c)
  // (the shear and entropy waves share the eigenvalue v_n, so they enter only
  // through |v_n| du).
  template <int DIR>
  __device__ __forceinline__ static bool abs_jacobian_apply(const double (&u)[NV], const double (&du)[NV],
                                                            double gamma, double wq, double (&acc)[NV]) {
    const double rho = u[0];
    const double ir = fast_rcp(rho);
    double v[D], ke = 0.0, vdm = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) { v[k] = u[1 + k] * ir; ke += v[k] * u[1 + k]; vdm += v[k] * du[1 + k]; }
    const double p = (gamma - 1.0) * (u[D + 1] - 0.5 * ke);
    const double gp = gamma * p;
    const double c = fast_sqrt(gp * ir);
    const double h2c2 = 0.5 * rho * fast_rcp(gp);   // 1 / (2 c^2)
    const double H = (u[D + 1] + p) * ir;
    const double vn = v[DIR];
    const double dp = (gamma - 1.0) * (0.5 * (ke * ir) * du[0] - vdm + du[D + 1]);
    const double rdv = du[1 + DIR] - vn * du[0];
    const double an = fabs(vn);
    const double k1 = wq * (fabs(vn - c) - an) * ((dp - c * rdv) * h2c2);
    const double k3 = wq * (fabs(vn + c) - an) * ((dp + c * rdv) * h2c2);
    const double wa = wq * an;
    acc[0] += wa * du[0] + (k1 + k3);
#pragma unroll
    for (int k = 0; k < D; ++k) acc[1 + k] += wa * du[1 + k] + (k1 + k3) * v[k];
    acc[1 + DIR] += c * (k3 - k1);
    acc[D + 1] += wa * du[D + 1] + (k1 + k3) * H + (k3 - k1) * (vn * c);
    return rho > 0.0 && p > 0.0;
  }
};

// Osher-type dissipation (eqn.osher @ P:186-196, Euler only): dis =
// sum_g w_g |A(psi(s_g))| (up - um) along psi(s) = um + s (up - um), with the
// path rule of DevTables (oq_n Gauss-Legendre points).
template <int D, int DIR>
__device__ __forceinline__ bool osher_dissipation(const double (&um)[D + 2], const double (&up)[D + 2], double gamma,
                                                  const DevTables& T, double (&dis)[D + 2]) {
  constexpr int NV = D + 2;
  double du[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) { du[v] = up[v] - um[v]; dis[v] = 0.0; }
  bool ok = true;
#pragma unroll 1
  for (int g = 0; g < T.oq_n; ++g) {
    const double sg = T.oq_x[g];
    double ps[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) ps[v] = um[v] + sg * du[v];
    ok &= Phys<0, D>::template abs_jacobian_apply<DIR>(ps, du, gamma, T.oq_w[g], dis);
  }
  return ok;
}

template <int D> struct Phys<1, D> {
  static constexpr int NV = 9;
  static constexpr double k4pi = 0.07957747154594767;   // 1/(4 pi)
  static constexpr double k8pi = 0.039788735772973836;  // 1/(8 pi)
  __device__ __forceinline__ static bool prim(const double (&u)[NV], double gamma, double (&v)[3],
                                              double& p, double& bb, double& vb) {
    const double ir = fast_rcp(u[0]);
    v[0] = u[1] * ir; v[1] = u[2] * ir; v[2] = u[3] * ir;
    const double ke = v[0] * u[1] + v[1] * u[2] + v[2] * u[3];
    bb = u[5] * u[5] + u[6] * u[6] + u[7] * u[7];
    vb = v[0] * u[5] + v[1] * u[6] + v[2] * u[7];
    p = (gamma - 1.0) * (u[4] - 0.5 * ke - bb * k8pi);
    return u[0] > 0.0 && p > 0.0;
  }
  template <int DIR>
  __device__ __forceinline__ static void flux_dir(const double (&u)[NV], double ch, const double (&v)[3],
                                                  double p, double bb, double vb, double (&f)[NV]) {
    const double pt = p + bb * k8pi;
    const double Bn = u[5 + DIR];
    f[0] = u[1 + DIR];
#pragma unroll
    for (int k = 0; k < 3; ++k) f[1 + k] = u[1 + DIR] * v[k] - Bn * u[5 + k] * k4pi;
    f[1 + DIR] += pt;
    f[4] = v[DIR] * (u[4] + pt) - Bn * vb * k4pi;
#pragma unroll
    for (int k = 0; k < 3; ++k) f[5 + k] = v[DIR] * u[5 + k] - Bn * v[k];
    f[5 + DIR] += u[8];
    f[8] = ch * ch * Bn;
  }
  __device__ __forceinline__ static double fast_speed(const double (&u)[NV], double gamma, double ch,
                                                      const double (&v)[3], double p, double bb, int dir) {
    const double ir = fast_rcp(u[0]);
    const double a2 = gamma * p * ir;
    const double b2 = bb * k4pi * ir;
    const double bn2 = u[5 + dir] * u[5 + dir] * k4pi * ir;
    const double s = a2 + b2;
    const double disc = fmax(s * s - 4.0 * a2 * bn2, 0.0);
    const double cf = fast_sqrt(0.5 * (s + fast_sqrt(disc)));
    return fmax(fabs(v[dir]) + cf, ch);
  }
  __device__ __forceinline__ static bool fluxes(const double (&u)[NV], double gamma, double ch,
                                                double (&f)[D][NV]) {
    double v[3], p, bb, vb;
    const bool ok = prim(u, gamma, v, p, bb, vb);
    flux_dir<0>(u, ch, v, p, bb, vb, f[0]);
    flux_dir<1>(u, ch, v, p, bb, vb, f[1]);
    if constexpr (D == 3) flux_dir<2>(u, ch, v, p, bb, vb, f[2]);
    return ok;
  }
  template <int DIR>
  __device__ __forceinline__ static bool flux_speed(const double (&u)[NV], double gamma, double ch,
                                                    double (&f)[NV], double& s) {
    double v[3], p, bb, vb;
    const bool ok = prim(u, gamma, v, p, bb, vb);
    flux_dir<DIR>(u, ch, v, p, bb, vb, f);
    s = fast_speed(u, gamma, ch, v, fmax(p, 0.0), bb, DIR);
    return ok;
  }
  __device__ __forceinline__ static bool cfl_speed(const double (&u)[NV], double gamma, double ch,
                                                   const double (&inv_dx)[3], double& s) {
    double v[3], p, bb, vb;
    const bool ok = prim(u, gamma, v, p, bb, vb);
    s = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) s += fast_speed(u, gamma, ch, v, fmax(p, 0.0), bb, k) * inv_dx[k];
    return ok;
  }
  __device__ __forceinline__ static void prim_to_cons(const double* pr, double gamma, double (&u)[NV]) {
    const double rho = pr[0];
    u[0] = rho; u[1] = rho * pr[1]; u[2] = rho * pr[2]; u[3] = rho * pr[3];
    const double bb = pr[5] * pr[5] + pr[6] * pr[6] + pr[7] * pr[7];
    u[4] = pr[4] / (gamma - 1.0) + 0.5 * rho * (pr[1] * pr[1] + pr[2] * pr[2] + pr[3] * pr[3]) + bb * k8pi;
    u[5] = pr[5]; u[6] = pr[6]; u[7] = pr[7]; u[8] = pr[8];
  }
};

// ---------------------------------------------------------------------------
// WENO, one 1D problem: win[0..2M] are the cell averages of cells
// i-M..i+M (or previous-sweep dofs); out[N] the nodal dofs.
// ---------------------------------------------------------------------------
template <int M> struct Stencils {
  static constexpr int N = M + 1;
  static constexpr int NS = (M % 2 == 0) ? 3 : 4;
  __host__ __device__ static constexpr int L(int s) {
    return (M % 2 == 0) ? (s == 0 ? M / 2 : (s == 1 ? M : 0))
                        : (s == 0 ? M / 2 + 1 : (s == 1 ? M / 2 : (s == 2 ? M : 0)));
  }
};

template <int M>
__device__ __forceinline__ void weno1d(const DevTables& T, const double (&win)[2 * M + 1], double (&out)[M + 1]) {
  constexpr int N = M + 1;
  constexpr int NS = Stencils<M>::NS;
  // constant data: every stencil polynomial is that constant (rec reproduces
  // constants), so the WENO polynomial is exactly the constant
  bool flat = true;
#pragma unroll
  for (int o = 1; o < 2 * M + 1; ++o) flat &= win[o] == win[0];
  if (flat) {
#pragma unroll
    for (int p = 0; p < N; ++p) out[p] = win[0];
    return;
  }
  double ws[NS][N], om[NS];
  double sum = 0.0;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    constexpr int dummy = 0; (void)dummy;
#pragma unroll
    for (int p = 0; p < N; ++p) {
      double acc = 0.0;
#pragma unroll
      for (int o = 0; o < N; ++o) acc += T.rec[s][p][o] * win[M - Stencils<M>::L(s) + o];
      ws[s][p] = acc;
    }
    // sigma_s = Sigma_pm w_p w_m (eqn.sigmas).  Sigma annihilates constants, so
    // the dofs are shifted by the centre average first (reading R13): the
    // unshifted quadratic form loses ~|w|^2 |Sigma| 1e-16 > eps to cancellation.
    const double c0 = win[M];
    double sig = 0.0;
#pragma unroll
    for (int p = 0; p < N; ++p) {
      double acc = 0.0;
#pragma unroll
      for (int m = 0; m < N; ++m) acc += T.sigma[p][m] * (ws[s][m] - c0);
      sig += acc * (ws[s][p] - c0);
    }
    // omega~ = lambda_s / (sigma + 1e-14)^8 by three squarings
    double x = sig + 1e-14;
    x = x * x; x = x * x; x = x * x;
    om[s] = T.lin[s] * fast_rcp(x);
    sum += om[s];
  }
  const double isum = fast_rcp(sum);
#pragma unroll
  for (int p = 0; p < N; ++p) {
    double acc = 0.0;
#pragma unroll
    for (int s = 0; s < NS; ++s) acc += (om[s] * isum) * ws[s][p];
    out[p] = acc;
  }
}

}  // namespace ader
