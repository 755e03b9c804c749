// flux_point.cuh — one space-time quadrature point of the two-point face flux
// (flux:F/G/H @ P:158-172; eqn.rusanov @ P:181-185, eqn.osher @ P:186-196),
// shared by the face-flux kernels of the uniform path (kernels.cu, flux_tma.cu).
#pragma once
#include <cstdint>

#include "device.cuh"

namespace ader {

constexpr int ipow_c(int b, int e) { return e == 0 ? 1 : b * ipow_c(b, e - 1); }
constexpr int pow2_at_least(int x) { return x <= 1 ? 1 : 2 * pow2_at_least((x + 1) / 2); }

template <bool GLOBAL>
__device__ __forceinline__ double ldq(const double* p) {
  if constexpr (GLOBAL) return __ldg(p);
  else return *p;
}

// Trace of a cell block [NV][N^(D+1)] (space fastest, time slowest) on the face
// normal to DIR at the face's space-time point p (p = (tangential nodes, time
// node), tangential axes in increasing order, time slowest):
//   out[v] = sum_a psi[a] q[v][... node a along DIR ...]
// psi = psi1 (xi = 1, the lower cell's side of a face) or psi0 (xi = 0).
template <int D, int M, int NV, int DIR, bool GL>
__device__ __forceinline__ void face_trace(const double* q0, int p, const double (&psi)[kMaxN], double (&out)[NV]) {
  constexpr int N = M + 1, NS = ipow_c(N, D), NST = NS * N, NT = NS / N;
  const int s = p / NT, t = p - s * NT;
  const int t1 = t % N, t2 = t / N;
  constexpr int ax0 = (DIR == 0) ? 1 : 0;
  constexpr int ax1 = (DIR == 2) ? 1 : 2;
  constexpr int sn = ipow_c(N, DIR);
  const int base = s * NS + t1 * ipow_c(N, ax0) + (D == 3 ? t2 * ipow_c(N, ax1) : 0);
  const double* q = q0 + base;
  if constexpr (GL && DIR == 0 && (N == 3 || N == 4)) {
    // x faces: the N nodes along the normal are contiguous in the block, so each
    // lane loads them with 16-byte loads (N = 4: two; N = 3: one 16-byte and one
    // 8-byte load, which half of the lanes issue from the other end of their
    // pencil since the pencils alternate in 16-byte alignment).  The 27 lanes
    // of a warp load span the same lines as before, so this cuts the L1
    // wavefronts of the x faces (the kernel's limiter) by 1/3
    // (N = 3) or 1/2 (N = 4).  Same values, same arithmetic order.
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const double* pc = q + v * NST;
      double x[N];
      if constexpr (N == 4) {   // blocks, variables and pencils start at even offsets
        const double2 lo = __ldg(reinterpret_cast<const double2*>(pc));
        const double2 hi = __ldg(reinterpret_cast<const double2*>(pc + 2));
        x[0] = lo.x; x[1] = lo.y; x[2] = hi.x; x[3] = hi.y;
      } else {
        const bool odd = (reinterpret_cast<uintptr_t>(pc) & 8) != 0;
        const double2 pr = __ldg(reinterpret_cast<const double2*>(pc + (odd ? 1 : 0)));
        const double sg = __ldg(pc + (odd ? 0 : 2));
        x[0] = odd ? sg : pr.x;
        x[1] = odd ? pr.x : pr.y;
        x[2] = odd ? pr.y : sg;
      }
      double a = psi[0] * x[0];
#pragma unroll
      for (int k = 1; k < N; ++k) a += psi[k] * x[k];
      out[v] = a;
    }
  } else {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double a = psi[0] * ldq<GL>(&q[v * NST]);
#pragma unroll
      for (int k = 1; k < N; ++k) a += psi[k] * ldq<GL>(&q[v * NST + k * sn]);
      out[v] = a;
    }
  }
}

// Both x traces of a block at the face point p: out0 = sum_a psi0[a] q[..a..]
// (xi = 0) and out1 = sum_a psi1[a] q[..a..] (xi = 1) from ONE set of loads —
// the same loads, products and order as face_trace<.., 0, true> gives for each.
template <int D, int M, int NV>
__device__ __forceinline__ void face_trace_x_both(const double* q0, int p, const double (&psi0)[kMaxN],
                                                  const double (&psi1)[kMaxN], double (&out0)[NV],
                                                  double (&out1)[NV]) {
  constexpr int N = M + 1, NS = ipow_c(N, D), NST = NS * N, NT = NS / N;
  const int s = p / NT, t = p - s * NT;
  const int t1 = t % N, t2 = t / N;
  const double* q = q0 + s * NS + t1 * N + (D == 3 ? t2 * N * N : 0);
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const double* pc = q + v * NST;
    double x[N];
    if constexpr (N == 4) {
      const double2 lo = __ldg(reinterpret_cast<const double2*>(pc));
      const double2 hi = __ldg(reinterpret_cast<const double2*>(pc + 2));
      x[0] = lo.x; x[1] = lo.y; x[2] = hi.x; x[3] = hi.y;
    } else if constexpr (N == 3) {
      const bool odd = (reinterpret_cast<uintptr_t>(pc) & 8) != 0;
      const double2 pr = __ldg(reinterpret_cast<const double2*>(pc + (odd ? 1 : 0)));
      const double sg = __ldg(pc + (odd ? 0 : 2));
      x[0] = odd ? sg : pr.x;
      x[1] = odd ? pr.x : pr.y;
      x[2] = odd ? pr.y : sg;
    } else {
#pragma unroll
      for (int k = 0; k < N; ++k) x[k] = __ldg(pc + k);
    }
    double a = psi0[0] * x[0], b = psi1[0] * x[0];
#pragma unroll
    for (int k = 1; k < N; ++k) { a += psi0[k] * x[k]; b += psi1[k] * x[k]; }
    out0[v] = a;
    out1[v] = b;
  }
}

// The two-point flux of one face point from the raw traces a (q_h^-, xi = 1 of
// the lower cell) and b (q_h^+, xi = 0 of the upper cell), with the boundary
// flags of the face, times the quadrature weight wt.
// (INTERIOR: the caller knows that none of the four boundary flags is set — no selects)
template <int D, int SYS, int DIR, int FLUX, bool INTERIOR = false>
__device__ __forceinline__ bool point_flux_states(const double (&a)[Phys<SYS, D>::NV], const double (&b)[Phys<SYS, D>::NV],
                                                  bool tlo, bool thi, bool rlo, bool rhi, double wt, double gamma,
                                                  double ch, const DevTables& T, double* val) {
  using PH = Phys<SYS, D>;
  constexpr int NV = PH::NV;
  double um[NV], up[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    um[v] = (!INTERIOR && (tlo || rlo)) ? b[v] : a[v];   // transmissive boundary: interior trace on both sides (R5)
    up[v] = (!INTERIOR && (thi || rhi)) ? a[v] : b[v];
  }
  // reflective wall (R22): the exterior state is the interior trace with the
  // normal momentum negated
  if (!INTERIOR && rlo) um[1 + DIR] = -um[1 + DIR];
  if (!INTERIOR && rhi) up[1 + DIR] = -up[1 + DIR];
  // equal traces (e.g. inside a constant region): eqn.rusanov and eqn.osher
  // reduce exactly to f(q) — 0.5 (f + f) = f and the dissipation term is 0 — so one flux
  // evaluation gives the bitwise-identical result
  bool same = true;
#pragma unroll
  for (int v = 0; v < NV; ++v) same &= um[v] == up[v];
  if (same) {
    double f[NV], s0;
    const bool ok = PH::template flux_speed<DIR>(um, gamma, ch, f, s0);
#pragma unroll
    for (int v = 0; v < NV; ++v) val[v] = wt * f[v];
    return ok;
  }
  double fL[NV], fR[NV], sL, sR;
  bool ok = PH::template flux_speed<DIR>(um, gamma, ch, fL, sL);
  ok &= PH::template flux_speed<DIR>(up, gamma, ch, fR, sR);
  if constexpr (FLUX == 1 && SYS == 0) {
    double dis[NV];
    ok &= osher_dissipation<D, DIR>(um, up, gamma, T, dis);
#pragma unroll
    for (int v = 0; v < NV; ++v) val[v] = wt * (0.5 * (fL[v] + fR[v]) - 0.5 * dis[v]);   // eqn.osher
  } else {
    const double smax = fmax(sL, sR);   // reading R4
    const double hw = 0.5 * wt;         // eqn.rusanov with the 1/2 folded into the quadrature weight
#pragma unroll
    for (int v = 0; v < NV; ++v) val[v] = hw * ((fL[v] + fR[v]) - smax * (up[v] - um[v]));
  }
  return ok;
}

// One space-time quadrature point of the face between the cell blocks qL0
// (lower side) and qR0 (upper side), [NV][N^(D+1)] each, in global (GL_L,
// GL_R) or shared memory.
template <int D, int M, int SYS, int DIR, int FLUX, bool GL_L, bool GL_R = GL_L, bool INTERIOR = false>
__device__ __forceinline__ bool point_flux_blocks(const double* qL0, const double* qR0, int p, bool fok, bool tlo,
                                                  bool thi, bool rlo, bool rhi, double wt, double gamma, double ch,
                                                  const DevTables& T, double* val) {
  constexpr int NV = Phys<SYS, D>::NV;
#pragma unroll
  for (int v = 0; v < NV; ++v) val[v] = 0.0;
  if (!fok) return true;
  // both traces unpredicated (the padded grid holds a ghost layer on every
  // side, so the far-side reads stay in bounds; their values are discarded at
  // transmissive boundaries)
  double a[NV], b[NV];
  face_trace<D, M, NV, DIR, GL_L>(qL0, p, T.psi1, a);   // q_h^- (xi = 1 of the left cell)
  face_trace<D, M, NV, DIR, GL_R>(qR0, p, T.psi0, b);   // q_h^+ (xi = 0 of the right cell)
  return point_flux_states<D, SYS, DIR, FLUX, INTERIOR>(a, b, tlo, thi, rlo, rhi, wt, gamma, ch, T, val);
}

}  // namespace ader
