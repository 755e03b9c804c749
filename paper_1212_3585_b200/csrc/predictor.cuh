// predictor.cuh — the element-local space-time DG predictor of one cell (a2),
// nodal Picard form of eqn.stdg.final:
//   q = w - T_tau sum_dir D_dir f*_dir(q),   f*_dir = (dt/dx_dir) f_dir(q)
// executed by a lane group of G >= N^D lanes inside one warp, one lane per
// spatial node holding the node's time pencil q[NV][N] in registers.  Used by
// the stand-alone predictor kernel (kernels.cu: uniform box and AMR id lists)
// and by the fused WENO + predictor tile walk (weno_pred.cu).
#pragma once
#include <type_traits>

#include "device.cuh"
#include "flux_point.cuh"

namespace ader {

// PERS: the f* scratch holds one time level at a time (the sweep stores a
// level's fluxes, contracts them, then the next level), D NV N^D doubles per
// cell instead of D NV N^(D+1); the same arithmetic in the same order.
template <int D, int M, int SYS, bool PERS = false>
struct PredCfg {
  static constexpr int NV = Phys<SYS, D>::NV, N = M + 1, NS = ipow_c(N, D), NST = NS * N;
  static constexpr int G = (NS <= 8) ? 8 : (NS <= 16 ? 16 : 32);   // lanes per cell
  static constexpr int CPW = 32 / G;
  static_assert(NS <= 32, "one cell must fit in a warp");
  // shared-memory layout of f*_d: lines along axis d stored contiguously (axis d
  // fastest, padded to LP = 4 doubles), so the D_d contraction reads a line
  // with two 16-byte loads: Fs[((d*NV + v)*N + s)*NL + line_d][pos_d]
  // (used for N = 4; for N = 3 the padding costs occupancy and bank
  // conflicts, and the natural node-major layout is kept)
  static constexpr bool LINES = (N == 4);
  static constexpr int LP = LINES ? 4 : N, NL = NS / N;
  static constexpr int FSZ = D * NV * (PERS ? 1 : N) * NL * LP + 8;   // +8: bank offset between cells
};

// per-lane constants of a lane group: node, its coordinates, line indices and
// rows of the differentiation matrix D[ia_d][j]
template <int D, int M, int SYS>
struct PredLane {
  using C = PredCfg<D, M, SYS>;
  int node;
  bool lane_ok;
  int ia[3], line[3];
  double Drow[D][M + 1];
  __device__ __forceinline__ void init(int node0, const DevTables& T) {
    constexpr int N = M + 1;
    lane_ok = node0 < C::NS;
    node = lane_ok ? node0 : C::NS - 1;
    ia[0] = node % N;
    ia[1] = (node / N) % N;
    ia[2] = node / (N * N);
    // index of the node's line along each axis (the other two coordinates)
    line[0] = ia[1] + N * ia[2];
    line[1] = ia[0] + N * ia[2];
    line[2] = ia[0] + N * ia[1];
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int j = 0; j < N; ++j) Drow[d][j] = T.D[ia[d]][j];
  }
};

// Flat cell (every node carries the same w): G = sum_dir D_dir f*_dir at the node
// whose rows of the differentiation matrix are Drow — f*_dir is one value per
// variable and direction, contracted in the order of the general path.  The
// predictor's flat first sweep and the face-flux kernel (which rebuilds a flat
// cell's q_h = w - Tsum[s] G from w instead of reading it) both call this.
template <int D, int M, int SYS>
__device__ __forceinline__ bool flat_cell_G(const double (&w)[Phys<SYS, D>::NV], const double (&Drow)[D][M + 1],
                                            const double (&dtdx)[3], double gamma, double ch,
                                            double (&G)[Phys<SYS, D>::NV]) {
  using PH = Phys<SYS, D>;
  constexpr int NV = PH::NV, N = M + 1;
  double f[D][NV];
  const bool ok = PH::fluxes(w, gamma, ch, f);
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double g = 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const double fs = dtdx[d] * f[d][v];
#pragma unroll
      for (int j = 0; j < N; ++j) g = fma(Drow[d][j], fs, g);
    }
    G[v] = g;
  }
  return ok;
}
// time level s of a flat cell's first-sweep iterate: q^1_s = w - Tsum[s] G
__device__ __forceinline__ double flat_cell_q(double w, double tsum, double G) { return fma(-tsum, G, w); }

// Picard iteration of one cell per lane group (all 32 lanes of the warp call
// it together, with the same from_guess; cell_ok false for a lane group without a cell).  wv: this
// node's w (eqn.weno.z); on return qv holds the node's time pencil, nsw the
// sweeps, conv the convergence flag (reading R2), bad an inadmissible state.
// Sweep 1 starts from the time-constant guess q^0 = w (R3): all N time levels
// carry the same flux, so it is evaluated once and q^1_s = w - (sum_s' T_ss') G.
// x contraction of one (variable, time level) by the FP64 tensor-core MMA
// (mma.sync m8n8k4 f64, 2D M = 3): with the node-per-lane layout lane L =
// ix + 4 iy of a 16-lane cell group is exactly A[row L/4][col L%4] of the
// 8x4 A fragment, row = the x line (iy; the warp's second cell holds rows
// 4-7), col = the node along it; B[k][n] = D[n/2][k] (each row of D twice),
// so C[line][n] = sum_j D[n/2][j] f*_x[j] and the lane's first accumulator
// register c0 = C[iy][2 ix] is its own G_x = sum_j D[ix][j] f*_x[line, j].
// The f*_x values never touch shared memory; the rows of a cell are
// independent, so a converged cell's stale values do not reach the other.
__device__ __forceinline__ double dmma_x(double a, double b) {
  double c0, c1;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
               : "=d"(c0), "=d"(c1)
               : "d"(a), "d"(b), "d"(0.0), "d"(0.0));
  (void)c1;
  return c0;
}

template <int D, int M, int SYS, bool PERS = false, bool XMMA = false>
__device__ __forceinline__ void predictor_cell(const double (&wv)[Phys<SYS, D>::NV],
                                               double (&qv)[Phys<SYS, D>::NV][M + 1], double* Fs,
                                               const PredLane<D, M, SYS>& L, const double (&dtdx)[3], bool cell_ok,
                                               double gamma, double ch, double tol, int max_sweeps,
                                               const DevTables& T, int& nsw, bool& conv, bool& bad,
                                               bool from_guess = false, bool flat_en = false,
                                               bool* was_flat = nullptr) {
  using PH = Phys<SYS, D>;
  using C = PredCfg<D, M, SYS, PERS>;
  constexpr int NV = C::NV, N = C::N, NS = C::NS, G = C::G;
  constexpr bool LINES = C::LINES;
  constexpr int LP = C::LP, NL = C::NL;
  const int node = L.node;
  const bool lane_ok = L.lane_ok;
  static_assert(!XMMA || (D == 2 && N == 4 && G == 16 && LINES), "DMMA x contraction: 2D, M = 3");
  // B fragment of dmma_x: B[k = lane % 4][n = lane / 4] = D[n / 2][k]
  const int lane32 = threadIdx.x & 31;
  const double bD = XMMA ? T.D[(lane32 >> 3) & 3][lane32 & 3] : 0.0;
  conv = !cell_ok;
  bad = false;
  nsw = 0;
  // Flat cells (flat_en): if every node of every cell of the warp carries the
  // same w (bit for bit; the WENO flat-window shortcut makes constant regions
  // exactly so), the first sweep's f*_dir is one value per variable and
  // direction, identical on every lane, so each lane contracts its own copy
  // in the order of the general path — the same numbers in the same order
  // (bitwise the same G) without the shared-memory round trip.
  // (M = 2 only: at M = 3 the extra live state spills registers, and the 2D M = 3 workloads
  // have no constant regions to gain from)
  bool flat_warp = false;
  if (M == 2 && flat_en && !from_guess) {
    const int lead = (threadIdx.x & 31) & ~(G - 1);
    bool same = true;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const long long mine = __double_as_longlong(wv[v]);
      same &= mine == __shfl_sync(0xffffffffu, mine, lead);
    }
    flat_warp = __all_sync(0xffffffffu, same || !(cell_ok && lane_ok));
  }
  if (was_flat) *was_flat = flat_warp && max_sweeps >= 1;
  // one Picard sweep; FIRST: the iterate is the time-constant guess (one flux level)
  auto sweep_once = [&](auto first_tag) {
    constexpr bool FIRST = decltype(first_tag)::value;
    const bool live = !conv && nsw < max_sweeps;   // this cell still iterates
    constexpr int NT = FIRST ? 1 : N;                          // distinct time levels of the iterate
    constexpr int SL = PERS ? 1 : N;                           // time levels held by the scratch
    // nodal fluxes f*_dir = (dt/dx_dir) f_dir(q) (eqn.nodal.eval @ P:405-412) of level s
    auto store_fluxes = [&](int s) {
      const int sl = PERS ? 0 : s;
      double uu[NV], f[D][NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) uu[v] = FIRST ? wv[v] : qv[v][s];
      bad |= !PH::fluxes(uu, gamma, ch, f);
#pragma unroll
      for (int d = 0; d < D; ++d)
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          if constexpr (LINES) Fs[(((d * NV + v) * SL + sl) * NL + L.line[d]) * LP + L.ia[d]] = dtdx[d] * f[d][v];
          else Fs[((d * NV + v) * SL + sl) * NS + node] = dtdx[d] * f[d][v];
        }
    };
    // G = sum_dir D_dir f*_dir of variable v, level s
    auto contract = [&](int v, int s, double g) -> double {
      const int sl = PERS ? 0 : s;
#pragma unroll
      for (int d = XMMA ? 1 : 0; d < D; ++d) {
        if constexpr (LINES) {
          const double2* fb = reinterpret_cast<const double2*>(Fs + (((d * NV + v) * SL + sl) * NL + L.line[d]) * LP);
          const double2 f01 = fb[0], f23 = fb[1];
          g += L.Drow[d][0] * f01.x;
          g += L.Drow[d][1] * f01.y;
          g += L.Drow[d][2] * f23.x;
          g += L.Drow[d][N - 1] * f23.y;
        } else {
          const int sd = (d == 0) ? 1 : (d == 1 ? N : N * N);
          const double* fb = Fs + ((d * NV + v) * SL + sl) * NS + node - L.ia[d] * sd;
#pragma unroll
          for (int j = 0; j < N; ++j) g += L.Drow[d][j] * fb[j * sd];
        }
      }
      return g;
    };
    double Gs[NV][NT];
    // XMMA: the fluxes of level s with f*_y stored and G_x = D_x f*_x formed
    // by dmma_x in registers (all 32 lanes execute the MMA)
    auto xmma_level = [&](int s) {
      const int sl = PERS ? 0 : s;
      double fx[NV];
      if (live && lane_ok) {
        double uu[NV], f[D][NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) uu[v] = FIRST ? wv[v] : qv[v][s];
        bad |= !PH::fluxes(uu, gamma, ch, f);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          fx[v] = dtdx[0] * f[0][v];
          Fs[(((1 * NV + v) * SL + sl) * NL + L.line[1]) * LP + L.ia[1]] = dtdx[1] * f[1][v];
        }
      } else {
#pragma unroll
        for (int v = 0; v < NV; ++v) fx[v] = 0.0;
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) Gs[v][s] = dmma_x(fx[v], bD);
    };
    if (M == 2 && FIRST && flat_warp) {
      if (live && lane_ok) {
        double g[NV];
        bad |= !flat_cell_G<D, M, SYS>(wv, L.Drow, dtdx, gamma, ch, g);
#pragma unroll
        for (int v = 0; v < NV; ++v) Gs[v][0] = g[v];
      }
    } else if constexpr (XMMA) {
#pragma unroll
      for (int s = 0; s < NT; ++s) {
        xmma_level(s);
        if constexpr (PERS) {
          __syncwarp();
          if (live && lane_ok) {
#pragma unroll
            for (int v = 0; v < NV; ++v) Gs[v][s] = contract(v, s, Gs[v][s]);
          }
          __syncwarp();
        }
      }
      if constexpr (!PERS) {
        __syncwarp();
        if (live && lane_ok) {
#pragma unroll
          for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int s = 0; s < NT; ++s) Gs[v][s] = contract(v, s, Gs[v][s]);
        }
      }
    } else if constexpr (PERS) {
#pragma unroll
      for (int s = 0; s < NT; ++s) {
        if (live && lane_ok) store_fluxes(s);
        __syncwarp();
        if (live && lane_ok) {
#pragma unroll
          for (int v = 0; v < NV; ++v) Gs[v][s] = contract(v, s, 0.0);
        }
        __syncwarp();
      }
    } else {
      if (live && lane_ok) {
#pragma unroll
        for (int s = 0; s < NT; ++s) store_fluxes(s);
      }
      __syncwarp();
      if (live && lane_ok) {
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
          for (int s = 0; s < NT; ++s) Gs[v][s] = contract(v, s, 0.0);
      }
    }
    // convergence bookkeeping on the high words of |dq| and |q| (monotone in
    // the value for non-negative doubles): max hi(|dq|) + 1 bounds |dq| from
    // above, max hi(|q|) with a zero low word bounds |q| from below, so a
    // passed test implies the exact FP64 test (R2); 32-bit integer max and
    // shuffles instead of FP64 -> FP32 conversions
    unsigned dmax = 0u, qmax = 0u;
    if (live && lane_ok) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
#pragma unroll
        for (int s = 0; s < N; ++s) {
          double acc;
          if (FIRST) {
            acc = flat_cell_q(wv[v], T.Tsum[s], Gs[v][0]);   // = w - Tsum[s] G, one rounding
          } else {
            acc = wv[v];
#pragma unroll
            for (int s2 = 0; s2 < NT; ++s2) acc -= T.T[s][s2] * Gs[v][s2];
          }
          const double prev = FIRST ? wv[v] : qv[v][s];
          dmax = max(dmax, (unsigned)__double2hiint(fabs(acc - prev)));
          qmax = max(qmax, (unsigned)__double2hiint(fabs(acc)));
          qv[v][s] = acc;
        }
      }
    }
    // per-cell max over the lane group (segmented butterfly)
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      dmax = max(dmax, __shfl_xor_sync(0xffffffffu, dmax, o, G));
      qmax = max(qmax, __shfl_xor_sync(0xffffffffu, qmax, o, G));
    }
    if (live) {
      ++nsw;
      const double dup = __hiloint2double((int)(dmax + 1u), 0), qlo = __hiloint2double((int)qmax, 0);
      // (a non-finite |dq| or |q| — high word >= 0x7FF00000 — never converges;
      // the cap then reports the cell)
      if (dmax < 0x7FF00000u && qmax < 0x7FF00000u && dup <= tol * (1.0 + qlo)) conv = true;   // reading R2
    }
  };
  // (from_guess: qv holds the caller's initial guess (reading R25), whose time
  // levels differ, so every sweep is a full one)
  if (max_sweeps >= 1 && !from_guess) sweep_once(std::integral_constant<bool, true>());
  // every lane takes part in the vote (lane groups of a warp may stop at
  // different sweep counts)
  while (!__all_sync(0xffffffffu, conv || nsw >= max_sweeps)) {
    __syncwarp();
    sweep_once(std::integral_constant<bool, false>());
  }
}

}  // namespace ader
