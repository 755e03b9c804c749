// kernels.cu — sm_100a kernels of the ADER-WENO hot path (FP64).
//
//   k_weno      a1 WENO reconstruction, one sweep
//   k_predictor a2 local space-time DG predictor, nodal Picard form of
//               eqn.stdg.final: q = w - T_tau sum_dir D_dir f*_dir(q)
//   k_face_flux_cells a3 space-time Gauss quadrature of the two-point flux,
//               Rusanov (eqn.rusanov @ P:181-185) or Osher (eqn.osher @ P:186-196)
//   k_update    a4 one-step FV update (eq:finite_vol @ P:147-152) fused with the
//               CFL speed of the new state (reading R1)
// plus ghost fill / pack / IC / gather helpers.  Layouts: see launch.h.
// Citations: P:n = PAPER.md line n.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "device.cuh"
#include "flux_point.cuh"
#include "launch.h"
#include "predictor.cuh"

namespace ader {


__device__ __forceinline__ long long box_cell(const Box& R, long long r, long long sy, long long sz) {
  const long long x = R.lo[0] + r % R.ext[0];
  const long long t = r / R.ext[0];
  const long long y = R.lo[1] + t % R.ext[1];
  const long long z = R.lo[2] + t / R.ext[1];
  return x + y * sy + z * sz;
}

__device__ __forceinline__ int box_coord(const Box& R, long long r, int axis) {
  if (axis == 0) return R.lo[0] + (int)(r % R.ext[0]);
  const long long t = r / R.ext[0];
  if (axis == 1) return R.lo[1] + (int)(t % R.ext[1]);
  return R.lo[2] + (int)(t / R.ext[1]);
}

__device__ __forceinline__ void record_error(DevCounters* c, int code, int stage, long long cell) {
  if (atomicCAS(&c->err_code, 0, code) == 0) {
    c->err_stage = stage;
    c->err_cell = (unsigned long long)cell;
  }
}

// ===========================================================================
// a1: WENO sweep K (axis K).  Thread per (cell, variable, previous-sweep dof).
// src [cell][NV][N^K], dst [cell][NV][N^(K+1)] with the new axis slowest.
// ===========================================================================
// The z sweep (K = 2) visits cells x fastest, then y inside chunks of YC rows,
// then z, then the chunk: the 2M+1 source planes it reads then span a few MB
// of L2 instead of 5 full planes (~120 MB at 256^3, re-read from HBM).
// G3: the (y, z) row comes from blockIdx.y / .z (y inside the chunk and z in
// blockIdx.y, the chunk in blockIdx.z: the same traversal) and only x and the
// dof from the thread index, so no thread divides by a run-time extent (the
// index arithmetic was more than half of the z sweep's instructions).
template <int M, int K, int NV, int YC, bool G3 = false>
__global__ void __launch_bounds__(256) k_weno(const double* __restrict__ src, double* __restrict__ dst,
                                              const Box R, const long long sy, const long long sz,
                                              const long long astride, const __grid_constant__ DevTables T) {
  constexpr int N = M + 1;
  constexpr int NT = ipow_c(N, K);
  constexpr int NIN = NV * NT;
  const unsigned ex = (unsigned)R.ext[0], ey = (unsigned)R.ext[1], ez = (unsigned)R.ext[2];
  unsigned x, y, z;
  int inner;
  if constexpr (G3) {
    const unsigned gx = blockIdx.x * blockDim.x + threadIdx.x;
    x = gx / NIN;
    inner = (int)(gx - x * NIN);
    if (x >= ex) return;
    if constexpr (YC > 1) {
      z = blockIdx.y / YC;
      y = blockIdx.z * YC + (blockIdx.y - z * YC);
      if (y >= ey) return;
    } else {
      y = blockIdx.y;
      z = blockIdx.z;
    }
  } else {
  // 32-bit index decomposition (the launcher guarantees < 2^32 threads)
  const unsigned gid = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned r = gid / NIN;
  inner = (int)(gid - r * NIN);
  const unsigned ty = r / ex;
  x = r - ty * ex;
  if constexpr (YC > 1) {
    const unsigned t2 = ty / YC;
    const unsigned yb = t2 / ez;
    z = t2 - yb * ez;
    y = yb * YC + (ty % YC);
    if (yb >= (ey + YC - 1) / YC || y >= ey) return;
  } else {
    z = ty / ey;
    y = ty - z * ey;
    if (z >= ez) return;
  }
  }
  const long long cell = (long long)(R.lo[0] + (int)x) + (long long)(R.lo[1] + (int)y) * sy +
                         (long long)(R.lo[2] + (int)z) * sz;
  double win[2 * M + 1];
#pragma unroll
  for (int o = -M; o <= M; ++o) win[o + M] = __ldg(&src[(cell + o * astride) * NIN + inner]);
  double out[N];
  weno1d<M>(T, win, out);
  const int v = inner / NT, t = inner - v * NT;
  double* d = dst + cell * (NIN * N) + v * NT * N + t;
#pragma unroll
  for (int a = 0; a < N; ++a) d[NT * a] = out[a];
}

// ===========================================================================
// a2: predictor.  One lane per (cell, spatial node); the lane keeps the node's
// time pencil q[NV][N] in registers.  A cell owns a power-of-two lane group
// (G >= N^D) inside one warp, so the Picard loop needs only __syncwarp and
// segmented shuffles; each cell stops at its own convergence (R2), which makes
// the result independent of how cells are grouped into CTAs.
// Sweep 1 starts from the time-constant guess q^0 = w (R3): all N time levels
// carry the same flux, so it is evaluated once and q^1_s = w - (sum_s' T_ss') G.
// ===========================================================================

template <int D, int M, int SYS, int WARPS, bool XM = false>
__global__ void __launch_bounds__(WARPS * 32, (SYS == 0) ? 4 : 2) k_predictor(
    const double* __restrict__ w, double* __restrict__ q, const Box R, const long long sy, const long long sz,
    const double dtdx0, const double dtdx1, const double dtdx2, const double gamma, const double ch,
    const double tol, const int max_sweeps, DevCounters* __restrict__ cnt, const int* __restrict__ list,
    const long long nlist, const unsigned char* __restrict__ emask, const double* __restrict__ dtdx_dev,
    const long long qs, const int guess, const StepState* __restrict__ gst, const double guess_r,
    const int* __restrict__ rows, const int flat, unsigned char* __restrict__ qflat,
    const __grid_constant__ DevTables T) {
  using C = PredCfg<D, M, SYS>;
  constexpr int NV = C::NV, N = C::N, NS = C::NS, NST = C::NST, G = C::G, CPW = C::CPW, FSZ = C::FSZ;
  extern __shared__ double smem[];
  // reading R25: extrapolation coefficients c[s][a] = psi_a(1 + r lambda_s) - psi_a(1)
  // of the previous step's time pencil (Lagrange basis on the GL nodes)
  double* gc = smem + WARPS * CPW * FSZ;                      // [N][N]
  double r = 0.0;
  if (guess) {
    r = gst ? ((gst->prev_dt > 0.0 && gst->dt > 0.0) ? gst->dt / gst->prev_dt : 0.0) : guess_r;
    if (threadIdx.x < N * N) {
      const int s = threadIdx.x / N, a = threadIdx.x % N;
      const double tau = 1.0 + r * T.lam[s];
      double pt = 1.0, p1 = 1.0;
      for (int m = 0; m < N; ++m)
        if (m != a) {
          const double den = T.lam[a] - T.lam[m];
          pt *= (tau - T.lam[m]) / den;
          p1 *= (1.0 - T.lam[m]) / den;
        }
      gc[threadIdx.x] = pt - p1;
    }
    __syncthreads();
  }
  const bool use_guess = guess && r > 0.0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = lane / G, node0 = lane - slot * G;
  PredLane<D, M, SYS> L;
  L.init(node0, T);
  const bool lane_ok = L.lane_ok;
  const int node = L.node;
  double* Fs = smem + (warp * CPW + slot) * FSZ;
  // cells of a box (uniform grid) or of an id list (AMR level)
  const long long count = list ? nlist : R.count();
  // (32-bit index decomposition: a rank's box holds < 2^31 cells)
  const unsigned bx = (unsigned)R.ext[0], by = (unsigned)R.ext[1];
  const double dtdx[3] = {dtdx_dev ? dtdx_dev[0] : dtdx0, dtdx_dev ? dtdx_dev[1] : dtdx1,
                          dtdx_dev ? dtdx_dev[2] : dtdx2};

  // persistent warps: the warp walks cell groups with a stride of the whole
  // grid and prefetches the next group's w while it iterates on the current one.
  // Box mode advances the group's box coordinates by the decomposed stride
  // (add with carry) instead of dividing the linear index in every iteration
  // (two 32-bit divisions were 11 % of the kernel's stall samples at 256^3).
  const long long wstride = (long long)gridDim.x * WARPS;
  long long wb = (long long)blockIdx.x * WARPS + warp;        // warp-uniform iteration index
  unsigned px, py, pz, sx_, sy_, sz_;                         // next cell's box coordinates, stride
  {
    const unsigned r0 = (unsigned)(wb * CPW + slot), t0 = r0 / bx;
    px = r0 - t0 * bx; pz = t0 / by; py = t0 - pz * by;
    const unsigned dr = (unsigned)(wstride * CPW), t1 = dr / bx;
    sx_ = dr - t1 * bx; sz_ = t1 / by; sy_ = t1 - sz_ * by;
  }
  auto cell_at = [&](long long r) -> long long {   // cell of index r, whose box coordinates are (px, py, pz)
    if (list) return (long long)list[r];
    return (long long)(R.lo[0] + (int)px) + (long long)(R.lo[1] + (int)py) * sy + (long long)(R.lo[2] + (int)pz) * sz;
  };
  auto advance = [&]() {
    px += sx_;
    const unsigned cx = px >= bx ? 1u : 0u;
    px -= cx * bx;
    py += sy_ + cx;
    const unsigned cy = py >= by ? 1u : 0u;
    py -= cy * by;
    pz += sz_ + cy;
  };
  double wn[NV];
  long long celln, drown;
  {
    const long long r0 = wb * CPW + slot;
    celln = r0 < count ? cell_at(r0) : 0;
    drown = rows ? (long long)rows[celln] : celln;   // row of w / q
#pragma unroll
    for (int v = 0; v < NV; ++v) wn[v] = r0 < count ? __ldg(&w[drown * (NV * NS) + v * NS + node]) : 1.0;
  }
  unsigned long long acc_sweeps = 0, acc_cells = 0, acc_flat = 0;
  int acc_max = 0;
  for (; wb * CPW < count; wb += wstride) {
  const long long rc = wb * CPW + slot;
  const bool cell_ok = rc < count;
  const bool active = cell_ok && lane_ok;
  const long long cell = celln;
  const long long drow = drown;
  double wv[NV], qv[NV][N];
#pragma unroll
  for (int v = 0; v < NV; ++v) wv[v] = wn[v];
  {
    const long long rn = (wb + wstride) * CPW + slot;
    advance();
    celln = rn < count ? cell_at(rn) : 0;
    drown = rows ? (long long)rows[celln] : celln;
#pragma unroll
    for (int v = 0; v < NV; ++v) wn[v] = rn < count ? __ldg(&w[drown * (NV * NS) + v * NS + node]) : 1.0;
  }
  bool conv, bad;
  int nsw;
  if (use_guess && cell_ok && lane_ok) {
    // q0 = w + sum_a c[s][a] q_prev[a] (the cell's previous q, read in place)
    const double* qp = q + drow * qs + node;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double old[N];
#pragma unroll
      for (int a = 0; a < N; ++a) old[a] = qp[v * NST + a * NS];
#pragma unroll
      for (int s2 = 0; s2 < N; ++s2) {
        double acc = wv[v];
#pragma unroll
        for (int a = 0; a < N; ++a) acc += gc[s2 * N + a] * old[a];
        qv[v][s2] = acc;
      }
    }
  }
  bool was_flat = false;
  predictor_cell<D, M, SYS, false, XM>(wv, qv, Fs, L, dtdx, cell_ok, gamma, ch, tol, max_sweeps, T, nsw, conv, bad,
                                        use_guess, flat != 0, &was_flat);
  // qflat (uniform boxes): a flat cell that converged in its first sweep is fully described
  // by its w — q_h[v][s][node] = w_v - Tsum[s] G_v(node) — so only a flag is stored and the
  // face-flux kernel rebuilds the traces from w (flat_cell_G): no 3.2 KB q_h block written
  // here and read there for the constant regions
  const bool skipq = qflat && was_flat && conv && !bad && nsw == 1;
  if (qflat && active && node == 0) qflat[cell] = skipq ? 1 : 0;
  if (active && (!emask || emask[cell])) {   // emask: cells whose errors count (multi-rank AMR: owned)
    if (bad) record_error(cnt, 1, 1, cell);
    else if (!conv) record_error(cnt, 2, 1, cell);
  }
  if (active) {
    if (!skipq) {
      double* qo = q + drow * qs + node;   // qs: block stride (>= NV * NST)
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int s = 0; s < N; ++s) qo[v * NST + s * NS] = qv[v][s];
    }
    if (node == 0) {
      acc_sweeps += (unsigned long long)nsw;
      acc_cells += 1ull;
      acc_flat += (was_flat && conv && !bad && nsw == 1) ? 1ull : 0ull;
      acc_max = nsw > acc_max ? nsw : acc_max;
    }
  }
  __syncwarp();
  }
  // one set of counter atomics per warp (same-address atomics per cell serialise in L2)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc_sweeps += __shfl_xor_sync(0xffffffffu, acc_sweeps, o);
    acc_cells += __shfl_xor_sync(0xffffffffu, acc_cells, o);
    acc_flat += __shfl_xor_sync(0xffffffffu, acc_flat, o);
    acc_max = max(acc_max, __shfl_xor_sync(0xffffffffu, acc_max, o));
  }
  if (lane == 0 && acc_cells) {
    atomicAdd(&cnt->sweeps, acc_sweeps);
    atomicAdd(&cnt->cells, acc_cells);
    if (acc_flat) atomicAdd(&cnt->flat_cells, acc_flat);
    atomicMax(&cnt->sweeps_max, acc_max);
  }
}

// ---------------------------------------------------------------------------
// a3 (cell-grouped): one lane group (power of two >= N^D lanes, a lane per
// space-time quadrature point) computes ALL lower faces of one cell, reading the
// cell's q once for the D faces.  Cells are visited x fastest, then y inside
// chunks of YC rows, then z, then the y chunk, so that the -y and -z
// neighbours' q (read for the same cell) were touched a few MB earlier and are
// still in L2 (the plain x-y-z order re-reads the -z neighbour from HBM).
// The D faces are evaluated together (independent dependency chains) and the
// D*NV point sums are formed through shared memory in a fixed order
// (deterministic).
// ---------------------------------------------------------------------------
template <int D, int M, int SYS, int DIR, int FLUX>
__device__ __forceinline__ bool point_flux(const double* __restrict__ q, long long cR, long long sd, int p, bool fok,
                                           bool tlo, bool thi, bool rlo, bool rhi, double wt, double gamma,
                                           double ch, const DevTables& T, double* val) {
  constexpr int BLK = Phys<SYS, D>::NV * ipow_c(M + 1, D + 1);
  return point_flux_blocks<D, M, SYS, DIR, FLUX, true>(q + (cR - sd) * BLK, q + cR * BLK, p, fok, tlo, thi, rlo, rhi,
                                                       wt, gamma, ch, T, val);
}


template <int D, int M, int SYS, int WARPS, int YC, int FLUX>
__global__ void __launch_bounds__(WARPS * 32, (FLUX == 1) ? 5 : (SYS == 1 ? 4 : (D == 3 ? 7 : 8))) k_face_flux_cells(const double* __restrict__ q, double* __restrict__ F,
                                                                const Box E, const int H, const int n0, const int n1,
                                                                const int n2, const long long sy, const long long sz,
                                                                const long long ncell, const double gamma,
                                                                const double ch, const int bmask, const int rmask,
                                                                DevCounters* __restrict__ cnt, const long long QSB,
                                                                const __grid_constant__ DevTables T) {
  using PH = Phys<SYS, D>;
  constexpr int NV = PH::NV, N = M + 1, NS = ipow_c(N, D), NT = NS / N;
  constexpr int G = (NS <= 8) ? 8 : (NS <= 16 ? 16 : 32);
  constexpr int CPW = 32 / G;
  constexpr int KP = pow2_at_least(D * NV);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = lane & (G - 1);
  // 32-bit index decomposition (the launcher guarantees < 2^32 cell groups)
  const unsigned r = (blockIdx.x * WARPS + warp) * CPW + lane / G;
  const unsigned ex = (unsigned)E.ext[0], ez = (unsigned)E.ext[2];
  const unsigned t = r / ex;
  const int x = (int)(r - t * ex);
  const int yi = (int)(t % YC);
  const unsigned t2 = t / YC;
  const unsigned yb = t2 / ez;
  const int z = (int)(t2 - yb * ez);
  const int y = (int)(yb * YC + yi);
  const bool ok = y < E.ext[1];
  const int cx = E.lo[0] + x, cy = E.lo[1] + y, cz = E.lo[2] + z;
  const long long cR = ok ? cx + cy * sy + cz * sz : 0;
  const int zH = (D == 3) ? H : 0;
  const bool inx = cx < H + n0, iny = cy < H + n1, inz = (D == 2) || cz < zH + n2;
  const bool pok = p < NS;
  bool fok[3] = {ok && iny && inz && pok, ok && inx && inz && pok, ok && inx && iny && pok};
  // quadrature weight of this lane's point (same (s, t1, t2) decomposition on every face)
  const int ps = pok ? p : 0;
  const int s = ps / NT, tt = ps - (ps / NT) * NT;
  double wt = T.w[s] * T.w[tt % N];
  if (D == 3) wt *= T.w[tt / N];
  double v[NV];
  bool good = true;
  constexpr int K = D * NV;
  const long long BLK = QSB;   // block stride
  // point sums through shared memory: lane p stores its K = D*NV weighted
  // point fluxes in column p — each direction's as soon as they are formed, so
  // no K-value accumulator stays live across the faces — then lane i sums row
  // i over the NS points in order (rows padded to G+1 doubles: conflict-free
  // column writes and row reads)
  __shared__ double red[WARPS * CPW][K][G + 1];
  double(*rb)[G + 1] = red[warp * CPW + lane / G];
  auto put = [&](int row0) {
    if (pok) {
#pragma unroll
      for (int i = 0; i < NV; ++i) rb[row0 + i][p] = v[i];
    }
  };
  // (tried and removed: staging the cell's own block in shared memory (1.6x
  // slower, bank conflicts) and an L1 prefetch of the D+1 blocks (8 % slower))
  const double* qown = q + cR * BLK;
  // (a face none of whose boundary flags is set takes the point flux without the boundary selects)
  const int bm = bmask | rmask;
  if (!(((bm & 1) && cx == H) || ((bm & 2) && cx == H + n0)))
    good &= point_flux_blocks<D, M, SYS, 0, FLUX, true, true, true>(q + (cR - 1) * BLK, qown, ps, fok[0], false, false,
                                                                    false, false, wt, gamma, ch, T, v);
  else
    good &= point_flux_blocks<D, M, SYS, 0, FLUX, true>(
        q + (cR - 1) * BLK, qown, ps, fok[0], (bmask & 1) && cx == H, (bmask & 2) && cx == H + n0,
        (rmask & 1) && cx == H, (rmask & 2) && cx == H + n0, wt, gamma, ch, T, v);
  put(0);
  if (!(((bm & 4) && cy == H) || ((bm & 8) && cy == H + n1)))
    good &= point_flux_blocks<D, M, SYS, 1, FLUX, true, true, true>(q + (cR - sy) * BLK, qown, ps, fok[1], false, false,
                                                                    false, false, wt, gamma, ch, T, v);
  else
    good &= point_flux_blocks<D, M, SYS, 1, FLUX, true>(
        q + (cR - sy) * BLK, qown, ps, fok[1], (bmask & 4) && cy == H, (bmask & 8) && cy == H + n1,
        (rmask & 4) && cy == H, (rmask & 8) && cy == H + n1, wt, gamma, ch, T, v);
  put(NV);
  if constexpr (D == 3) {
    if (!(((bm & 16) && cz == zH) || ((bm & 32) && cz == zH + n2)))
      good &= point_flux_blocks<D, M, SYS, 2, FLUX, true, true, true>(q + (cR - sz) * BLK, qown, ps, fok[2], false,
                                                                      false, false, false, wt, gamma, ch, T, v);
    else
      good &= point_flux_blocks<D, M, SYS, 2, FLUX, true>(
          q + (cR - sz) * BLK, qown, ps, fok[2], (bmask & 16) && cz == zH, (bmask & 32) && cz == zH + n2,
          (rmask & 16) && cz == zH, (rmask & 32) && cz == zH + n2, wt, gamma, ch, T, v);
    put(2 * NV);
  }
  if (!good) record_error(cnt, 1, 2, cR);
  __syncwarp();
  for (int i = p; i < K; i += G) {
    double acc = rb[i][0];
#pragma unroll
    for (int j = 1; j < NS; ++j) acc += rb[i][j];
    const int dir = i / NV, var = i - dir * NV;
    const bool face_ok = dir == 0 ? (ok && iny && inz) : (dir == 1 ? (ok && inx && inz) : (ok && inx && iny));
    if (face_ok) F[((long long)dir * ncell + cR) * NV + var] = acc;
  }
}

// ---------------------------------------------------------------------------
// a3 by x runs (D = 3, M = 2, Euler, Rusanov: the default there): a warp walks RL
// consecutive cells along x and carries the xi = 1 trace of the cell it just
// finished — the lower side of the next cell's x face — formed from the loads
// that cell made anyway (face_trace_x_both), so only the first cell of a run
// reads its -x neighbour: one of the four blocks a cell reads less, and the
// index decomposition once per run.  Each direction's point fluxes go to shared
// memory as soon as they are formed (no 15-value accumulator held across the
// three faces).  Same loads, products and order per trace as k_face_flux_cells:
// F bitwise equal; C4 flux 29.3 -> 26.9 ms at 5 CTAs/SM (28.1 at 7, 27.0 at 6).
template <int D, int M, int SYS, int WARPS, int YC, int FLUX, int RL, int MB>
__global__ void __launch_bounds__(WARPS * 32, MB) k_face_flux_runs(
    const double* __restrict__ q, double* __restrict__ F, const Box E, const int H, const int n0, const int n1,
    const int n2, const long long sy, const long long sz, const long long ncell, const double gamma, const double ch,
    const int bmask, const int rmask, DevCounters* __restrict__ cnt, const long long QSB, const unsigned nrx,
    const __grid_constant__ DevTables T) {
  using PH = Phys<SYS, D>;
  constexpr int NV = PH::NV, N = M + 1, NS = ipow_c(N, D), NT = NS / N;
  static_assert(D == 3 && NS <= 32 && NS > 16, "one cell per warp");
  constexpr int G = 32, K = D * NV;
  const int warp = threadIdx.x >> 5, p = threadIdx.x & 31;
  const unsigned r = blockIdx.x * WARPS + warp;
  const unsigned ez = (unsigned)E.ext[2];
  const unsigned t = r / nrx;
  const int x0 = (int)(r - t * nrx) * RL;
  const int yi = (int)(t % YC);
  const unsigned t2 = t / YC;
  const unsigned yb = t2 / ez;
  const int z = (int)(t2 - yb * ez);
  const int y = (int)(yb * YC + yi);
  const bool rowok = y < E.ext[1];
  const int cy = E.lo[1] + y, cz = E.lo[2] + z;
  const int zH = H;
  const bool iny = cy < H + n1, inz = cz < zH + n2;
  const bool pok = p < NS;
  const int ps = pok ? p : 0;
  const int s = ps / NT, tt = ps - (ps / NT) * NT;
  double wt = T.w[s] * T.w[tt % N];
  wt *= T.w[tt / N];
  const long long BLK = QSB;
  __shared__ double red[WARPS][K][G + 1];
  double(*rb)[G + 1] = red[warp];
  double ax[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) ax[i] = 0.0;
  const long long row = cy * sy + cz * sz;
  // a boundary flag applies on the y / z faces of this row (uniform over the run)
  const bool ybnd = (((bmask | rmask) & 4) && cy == H) || (((bmask | rmask) & 8) && cy == H + n1);
  const bool zbnd = (((bmask | rmask) & 16) && cz == zH) || (((bmask | rmask) & 32) && cz == zH + n2);
#pragma unroll 1
  for (int c = 0; c < RL; ++c) {
    const int x = x0 + c;
    const bool ok = rowok && x < E.ext[0];
    const int cx = E.lo[0] + x;
    const long long cR = ok ? cx + row : 0;
    const bool inx = cx < H + n0;
    const double* qown = q + cR * BLK;
    bool good = true;
    double val[NV];
    {
      const bool fok = ok && iny && inz && pok;
#pragma unroll
      for (int i = 0; i < NV; ++i) val[i] = 0.0;
      if (fok) {
        double b[NV], an[NV];
        if (c == 0) face_trace<D, M, NV, 0, true>(q + (cR - 1) * BLK, ps, T.psi1, ax);
        face_trace_x_both<D, M, NV>(qown, ps, T.psi0, T.psi1, b, an);
        const bool xlo = cx == H, xhi = cx == H + n0;
        if (!(((bmask | rmask) & 1) && xlo) && !(((bmask | rmask) & 2) && xhi))   // interior face: no selects
          good &= point_flux_states<D, SYS, 0, FLUX, true>(ax, b, false, false, false, false, wt, gamma, ch, T, val);
        else
          good &= point_flux_states<D, SYS, 0, FLUX>(ax, b, (bmask & 1) && xlo, (bmask & 2) && xhi, (rmask & 1) && xlo,
                                                     (rmask & 2) && xhi, wt, gamma, ch, T, val);
#pragma unroll
        for (int i = 0; i < NV; ++i) ax[i] = an[i];
      }
      if (pok) {
#pragma unroll
        for (int i = 0; i < NV; ++i) rb[i][p] = val[i];
      }
    }
    if (!ybnd)
      good &= point_flux_blocks<D, M, SYS, 1, FLUX, true, true, true>(q + (cR - sy) * BLK, qown, ps, ok && inx && inz && pok,
                                                                      false, false, false, false, wt, gamma, ch, T, val);
    else
      good &= point_flux_blocks<D, M, SYS, 1, FLUX, true>(
          q + (cR - sy) * BLK, qown, ps, ok && inx && inz && pok, (bmask & 4) && cy == H, (bmask & 8) && cy == H + n1,
          (rmask & 4) && cy == H, (rmask & 8) && cy == H + n1, wt, gamma, ch, T, val);
    if (pok) {
#pragma unroll
      for (int i = 0; i < NV; ++i) rb[NV + i][p] = val[i];
    }
    if (!zbnd)
      good &= point_flux_blocks<D, M, SYS, 2, FLUX, true, true, true>(q + (cR - sz) * BLK, qown, ps, ok && inx && iny && pok,
                                                                      false, false, false, false, wt, gamma, ch, T, val);
    else
      good &= point_flux_blocks<D, M, SYS, 2, FLUX, true>(
          q + (cR - sz) * BLK, qown, ps, ok && inx && iny && pok, (bmask & 16) && cz == zH,
          (bmask & 32) && cz == zH + n2, (rmask & 16) && cz == zH, (rmask & 32) && cz == zH + n2, wt, gamma, ch, T, val);
    if (pok) {
#pragma unroll
      for (int i = 0; i < NV; ++i) rb[2 * NV + i][p] = val[i];
    }
    if (!good) record_error(cnt, 1, 2, cR);
    __syncwarp();
    for (int i = p; i < K; i += G) {
      double acc = rb[i][0];
#pragma unroll
      for (int j = 1; j < NS; ++j) acc += rb[i][j];
      const int dir = i / NV, var = i - dir * NV;
      const bool face_ok = dir == 0 ? (ok && iny && inz) : (dir == 1 ? (ok && inx && inz) : (ok && inx && iny));
      if (face_ok) F[((long long)dir * ncell + cR) * NV + var] = acc;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// a3 with flat cells rebuilt from w (D = 3, M = 2; one cell per warp).  A cell
// flagged by the predictor (qflat) has no q block: its q_h[v][s][node] =
// w_v - Tsum[s] G_v(node) with G the predictor's flat first sweep
// (flat_cell_G, the same code, so bitwise the value the predictor would have
// stored).  Lane p builds G of node p into a shared table per cell (own; a
// flat lower neighbour with the same w bit for bit — the rule inside a
// constant region — shares it, another flat neighbour gets a second table),
// and the trace contractions of flagged cells read the table instead of
// gathering from a q block.  Unflagged cells go through face_trace as in
// k_face_flux_cells; same trace arithmetic, point flux and point-sum order.
template <int D, int M, int NV, int DIR>
__device__ __forceinline__ void flat_trace(const double* __restrict__ tab, const double (&w)[NV], int p,
                                           const double (&psi)[kMaxN], const DevTables& T, double (&out)[NV]) {
  constexpr int N = M + 1, NS = ipow_c(N, D), NT = NS / N;
  const int s = p / NT, t = p - s * NT;
  const int t1 = t % N, t2 = t / N;
  constexpr int ax0 = (DIR == 0) ? 1 : 0;
  constexpr int ax1 = (DIR == 2) ? 1 : 2;
  constexpr int sn = ipow_c(N, DIR);
  const int base = t1 * ipow_c(N, ax0) + (D == 3 ? t2 * ipow_c(N, ax1) : 0);
  const double ts = T.Tsum[s];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double a = psi[0] * flat_cell_q(w[v], ts, tab[v * NS + base]);
#pragma unroll
    for (int k = 1; k < N; ++k) a += psi[k] * flat_cell_q(w[v], ts, tab[v * NS + base + k * sn]);
    out[v] = a;
  }
}

template <int D, int M, int SYS, int WARPS, int YC, int FLUX>
__global__ void __launch_bounds__(WARPS * 32, (FLUX == 1) ? 4 : (SYS == 1 ? 3 : 6)) k_face_flux_cells_flat(
    const double* __restrict__ q, double* __restrict__ F, const Box E, const int H, const int n0, const int n1,
    const int n2, const long long sy, const long long sz, const long long ncell, const double gamma, const double ch,
    const int bmask, const int rmask, DevCounters* __restrict__ cnt, const long long QSB,
    const unsigned char* __restrict__ qflat, const double* __restrict__ w, const double dtdx0, const double dtdx1,
    const double dtdx2, const double* __restrict__ dtdx_dev, const __grid_constant__ DevTables T) {
  using PH = Phys<SYS, D>;
  constexpr int NV = PH::NV, N = M + 1, NS = ipow_c(N, D), NT = NS / N;
  static_assert(D == 3 && NS <= 32 && NS > 16, "one cell per warp");
  constexpr int G = 32;
  constexpr int KP = pow2_at_least(D * NV);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = lane;
  const unsigned r = blockIdx.x * WARPS + warp;
  const unsigned ex = (unsigned)E.ext[0], ez = (unsigned)E.ext[2];
  const unsigned t = r / ex;
  const int x = (int)(r - t * ex);
  const int yi = (int)(t % YC);
  const unsigned t2 = t / YC;
  const unsigned yb = t2 / ez;
  const int z = (int)(t2 - yb * ez);
  const int y = (int)(yb * YC + yi);
  const bool ok = y < E.ext[1];
  const int cx = E.lo[0] + x, cy = E.lo[1] + y, cz = E.lo[2] + z;
  const long long cR = ok ? cx + cy * sy + cz * sz : 0;
  const int zH = H;
  const bool inx = cx < H + n0, iny = cy < H + n1, inz = cz < zH + n2;
  const bool pok = p < NS;
  const bool fok[3] = {ok && iny && inz && pok, ok && inx && inz && pok, ok && inx && iny && pok};
  const int ps = pok ? p : 0;
  const int s = ps / NT, tt = ps - (ps / NT) * NT;
  double wt = T.w[s] * T.w[tt % N];
  wt *= T.w[tt / N];
  constexpr int K = D * NV;
  const long long BLK = QSB;
  __shared__ double red[WARPS][K][G + 1];
  __shared__ double tabs[WARPS][2][NV * NS];
  double(*rb)[G + 1] = red[warp];
  double* tab0 = tabs[warp][0];
  double* tab1 = tabs[warp][1];
  const double dtdx[3] = {dtdx_dev ? dtdx_dev[0] : dtdx0, dtdx_dev ? dtdx_dev[1] : dtdx1,
                          dtdx_dev ? dtdx_dev[2] : dtdx2};
  const long long nstr[3] = {1, sy, sz};
  // flags of the cell and its three lower neighbours (warp-uniform)
  const bool fo = ok && qflat[cR] != 0;
  bool fnb[3];
#pragma unroll
  for (int d = 0; d < D; ++d) fnb[d] = ok && qflat[cR - nstr[d]] != 0;
  // G of node p of a flat cell with state ws into a table
  auto build = [&](double* tab, const double (&ws)[NV]) -> bool {
    bool okb = true;
    if (pok) {
      const int ia[3] = {p % N, (p / N) % N, p / (N * N)};
      double Drow[D][N], g[NV];
#pragma unroll
      for (int d = 0; d < D; ++d)
#pragma unroll
        for (int j = 0; j < N; ++j) Drow[d][j] = T.D[ia[d]][j];
      okb = flat_cell_G<D, M, SYS>(ws, Drow, dtdx, gamma, ch, g);
#pragma unroll
      for (int v = 0; v < NV; ++v) tab[v * NS + p] = g[v];
    }
    return okb;
  };
  double wo[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) wo[v] = fo ? __ldg(w + cR * (NV * NS) + v * NS) : 0.0;
  if (fo) (void)build(tab0, wo);   // (an inadmissible w was already reported by the predictor)
  __syncwarp();
  double v[KP];
  bool good = true;
  const double* qown = q + cR * BLK;
  auto face = [&](auto dirc, bool tlo, bool thi, bool rlo, bool rhi, double* val) {
    constexpr int DIR = decltype(dirc)::value;
    const long long cN = cR - nstr[DIR];
    double wn[NV];
    bool shared_tab = false;
    if (fnb[DIR]) {
      bool same = fo;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        wn[i] = __ldg(w + cN * (NV * NS) + i * NS);
        same &= __double_as_longlong(wn[i]) == __double_as_longlong(wo[i]);
      }
      shared_tab = same;
      if (!same) {
        __syncwarp();            // the previous face's reads of tab1 are done
        (void)build(tab1, wn);
        __syncwarp();
      }
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) val[i] = 0.0;
    if (!fok[DIR]) return;
    double a[NV], b[NV];
    if (fnb[DIR]) flat_trace<D, M, NV, DIR>(shared_tab ? tab0 : tab1, wn, ps, T.psi1, T, a);
    else face_trace<D, M, NV, DIR, true>(q + cN * BLK, ps, T.psi1, a);
    if (fo) flat_trace<D, M, NV, DIR>(tab0, wo, ps, T.psi0, T, b);
    else face_trace<D, M, NV, DIR, true>(qown, ps, T.psi0, b);
    good &= point_flux_states<D, SYS, DIR, FLUX>(a, b, tlo, thi, rlo, rhi, wt, gamma, ch, T, val);
  };
  face(std::integral_constant<int, 0>{}, (bmask & 1) && cx == H, (bmask & 2) && cx == H + n0, (rmask & 1) && cx == H,
       (rmask & 2) && cx == H + n0, v);
  face(std::integral_constant<int, 1>{}, (bmask & 4) && cy == H, (bmask & 8) && cy == H + n1, (rmask & 4) && cy == H,
       (rmask & 8) && cy == H + n1, v + NV);
  face(std::integral_constant<int, 2>{}, (bmask & 16) && cz == zH, (bmask & 32) && cz == zH + n2,
       (rmask & 16) && cz == zH, (rmask & 32) && cz == zH + n2, v + 2 * NV);
  if (!good) record_error(cnt, 1, 2, cR);
  if (pok) {
#pragma unroll
    for (int i = 0; i < K; ++i) rb[i][p] = v[i];
  }
  __syncwarp();
  for (int i = p; i < K; i += G) {
    double acc = rb[i][0];
#pragma unroll
    for (int j = 1; j < NS; ++j) acc += rb[i][j];
    const int dir = i / NV, var = i - dir * NV;
    const bool face_ok = dir == 0 ? (ok && iny && inz) : (dir == 1 ? (ok && inx && inz) : (ok && inx && iny));
    if (face_ok) F[((long long)dir * ncell + cR) * NV + var] = acc;
  }
}

// ===========================================================================
// a4: FV update + next CFL speed (block max, then one atomicMax per block).
// ===========================================================================
__device__ __forceinline__ void block_max_to(double s, unsigned long long* dst) {
  __shared__ double sm[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sm[warp] = s;
  __syncthreads();
  if (warp == 0) {
    s = (lane < (int)(blockDim.x >> 5)) ? sm[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
    if (lane == 0) atomicMax(dst, (unsigned long long)__double_as_longlong(s));
  }
}

template <int D, int SYS>
__global__ void __launch_bounds__(256) k_update(double* __restrict__ u, const double* __restrict__ F, const Box R,
                                                const long long sy, const long long sz, const long long ncell,
                                                const double dtdx0, const double dtdx1, const double dtdx2,
                                                const double idx0, const double idx1, const double idx2,
                                                const double gamma, const double ch, DevCounters* __restrict__ cnt,
                                                const double* __restrict__ dtdx_dev) {
  using PH = Phys<SYS, D>;
  constexpr int NV = PH::NV;
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0.0;
  if (r < R.count()) {
    const long long c = box_cell(R, r, sy, sz);
    const double dtdx[3] = {dtdx_dev ? dtdx_dev[0] : dtdx0, dtdx_dev ? dtdx_dev[1] : dtdx1,
                            dtdx_dev ? dtdx_dev[2] : dtdx2};
    const long long st[3] = {1, sy, sz};
    double uu[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) uu[v] = u[c * NV + v];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const double* Fm = F + ((long long)d * ncell + c) * NV;
      const double* Fp = F + ((long long)d * ncell + c + st[d]) * NV;
#pragma unroll
      for (int v = 0; v < NV; ++v) uu[v] = uu[v] - dtdx[d] * (Fp[v] - Fm[v]);
    }
    const double inv_dx[3] = {idx0, idx1, idx2};
    if (!PH::cfl_speed(uu, gamma, ch, inv_dx, s)) record_error(cnt, 1, 3, c);
#pragma unroll
    for (int v = 0; v < NV; ++v) u[c * NV + v] = uu[v];
  }
  block_max_to(s, &cnt->speed_bits);
}

template <int D, int SYS>
__global__ void __launch_bounds__(256) k_cfl_speed(const double* __restrict__ u, const Box R, const long long sy,
                                                   const long long sz, const double idx0, const double idx1,
                                                   const double idx2, const double gamma, const double ch,
                                                   DevCounters* __restrict__ cnt) {
  using PH = Phys<SYS, D>;
  constexpr int NV = PH::NV;
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0.0;
  if (r < R.count()) {
    const long long c = box_cell(R, r, sy, sz);
    double uu[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) uu[v] = u[c * NV + v];
    const double inv_dx[3] = {idx0, idx1, idx2};
    if (!PH::cfl_speed(uu, gamma, ch, inv_dx, s)) record_error(cnt, 1, 4, c);
  }
  block_max_to(s, &cnt->speed_bits);
}

// ===========================================================================
// helpers
// ===========================================================================
// dt of the next step from the reduced CFL speed (reading R1), on the device
__global__ void k_step_dt(DevCounters* __restrict__ cnt, StepState* __restrict__ st, const double cfl,
                          const double t_end, const double dx0, const double dx1, const double dx2, const int d) {
  const unsigned long long b = cnt->speed_bits;
  const double speed = __longlong_as_double((long long)b);
  double dt = cfl / speed;
  if (!(dt > 0.0) || !isfinite(dt)) {
    if (atomicCAS(&cnt->err_code, 0, 3) == 0) { cnt->err_stage = 4; cnt->err_cell = 0; }
    dt = 0.0;
  }
  const double t = st->t;
  if (!(t < t_end)) dt = 0.0;             // past t_end: the step is a no-op
  else if (t + dt > t_end) dt = t_end - t;
  const double dx[3] = {dx0, dx1, dx2};
  st->prev_dt = st->dt;   // the previous step's dt (predictor guess, R25)
  st->dt = dt;
  for (int k = 0; k < 3; ++k) st->dtdx[k] = k < d ? dt / dx[k] : 0.0;
  st->t = t + dt;
  if (dt > 0.0) { st->steps += 1; st->last_dt = dt; }
}

__global__ void k_set_dt(StepState* __restrict__ st, const double dt, const double dx0, const double dx1,
                         const double dx2, const int d) {
  const double dx[3] = {dx0, dx1, dx2};
  st->dt = dt;
  for (int k = 0; k < 3; ++k) st->dtdx[k] = k < d ? dt / dx[k] : 0.0;
}

__global__ void k_fill_axis(double* __restrict__ u, const Box R, const long long sy, const long long sz, const int nv,
                            const int axis, const int mode, const int H, const int n) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= R.count() * nv) return;
  const long long r = gid / nv;
  const int v = (int)(gid - r * nv);
  int c[3];
  c[0] = R.lo[0] + (int)(r % R.ext[0]);
  const long long t = r / R.ext[0];
  c[1] = R.lo[1] + (int)(t % R.ext[1]);
  c[2] = R.lo[2] + (int)(t / R.ext[1]);
  int i = c[axis] - H;
  if (mode == 0) i = ((i % n) + n) % n;                      // periodic wrap
  else if (mode == 2) i = i < 0 ? -1 - i : (i >= n ? 2 * n - 1 - i : i);   // reflective mirror (R22)
  else i = i < 0 ? 0 : (i >= n ? n - 1 : i);                 // transmissive copy (R5)
  int s[3] = {c[0], c[1], c[2]};
  s[axis] = i + H;
  const long long dst = c[0] + c[1] * sy + c[2] * sz;
  const long long src = s[0] + s[1] * sy + s[2] * sz;
  const double val = u[src * nv + v];
  u[dst * nv + v] = (mode == 2 && v == 1 + axis) ? -val : val;   // wall: normal momentum negated
}

__global__ void k_pack(const double* __restrict__ src, const Box R, const long long sy, const long long sz,
                       const int stride, double* __restrict__ out, const int to_buf) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= R.count() * stride) return;
  const long long r = gid / stride;
  const int v = (int)(gid - r * stride);
  const long long c = box_cell(R, r, sy, sz);
  if (to_buf) out[gid] = src[c * stride + v];
  else const_cast<double*>(src)[c * stride + v] = out[gid];
}

template <int D, int SYS>
__global__ void k_ic_average(double* __restrict__ u, const double* __restrict__ prim, const double* __restrict__ wq,
                             const int nq, const long long first, const long long ncells, const int n0, const int n1,
                             const int H, const long long sy, const long long sz, const double gamma,
                             const int o0, const int o1, const int o2) {
  using PH = Phys<SYS, D>;
  constexpr int NV = PH::NV;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncells) return;
  const long long lin = first + i;
  const long long x = lin % n0, y = (lin / n0) % n1, z = lin / ((long long)n0 * n1);
  double acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = 0.0;
  for (int g = 0; g < nq; ++g) {
    double uu[NV];
    PH::prim_to_cons(prim + (i * nq + g) * 9, gamma, uu);
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] += wq[g] * uu[v];
  }
  const long long c = (x + o0 + H) + (y + o1 + H) * sy + (D == 3 ? (z + o2 + H) : z) * sz;
#pragma unroll
  for (int v = 0; v < NV; ++v) u[c * NV + v] = acc[v];
}

__global__ void k_cons_partials(const double* __restrict__ u, const Box R, const long long sy, const long long sz,
                                const int nv, const double vol, double* __restrict__ partial) {
  __shared__ double sm[256 * 9];
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (int v = 0; v < nv; ++v) sm[v * 256 + threadIdx.x] = 0.0;
  if (r < R.count()) {
    const long long c = box_cell(R, r, sy, sz);
    for (int v = 0; v < nv; ++v) sm[v * 256 + threadIdx.x] = u[c * nv + v] * vol;
  }
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o)
      for (int v = 0; v < nv; ++v) sm[v * 256 + threadIdx.x] += sm[v * 256 + threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int v = 0; v < nv; ++v) partial[(long long)blockIdx.x * nv + v] = sm[v * 256];
}

// ===========================================================================
// launchers
// ===========================================================================
namespace {
inline unsigned grid_for(long long n, int bs) { return (unsigned)((n + bs - 1) / bs); }
inline void count_launch(const KCtx& k) { if (k.launches) ++*k.launches; }

#define ADER_DISPATCH(D_, M_, SYS_, ...)                                          \
  do {                                                                             \
    if (D_ == 2 && M_ == 2 && SYS_ == 0) { constexpr int D = 2, M = 2, SYS = 0; __VA_ARGS__; } \
    else if (D_ == 2 && M_ == 3 && SYS_ == 0) { constexpr int D = 2, M = 3, SYS = 0; __VA_ARGS__; } \
    else if (D_ == 3 && M_ == 2 && SYS_ == 0) { constexpr int D = 3, M = 2, SYS = 0; __VA_ARGS__; } \
    else if (D_ == 2 && M_ == 2 && SYS_ == 1) { constexpr int D = 2, M = 2, SYS = 1; __VA_ARGS__; } \
    else if (D_ == 2 && M_ == 3 && SYS_ == 1) { constexpr int D = 2, M = 3, SYS = 1; __VA_ARGS__; } \
    else if (D_ == 3 && M_ == 2 && SYS_ == 1) { constexpr int D = 3, M = 2, SYS = 1; __VA_ARGS__; } \
  } while (0)

constexpr int kPredWarps = 4;
constexpr int kFluxWarps = 4;

template <int D, int M, int SYS>
size_t pred_smem() {
  constexpr int NV = Phys<SYS, D>::NV, N = M + 1, NS = ipow_c(N, D);
  constexpr int G = (NS <= 8) ? 8 : (NS <= 16 ? 16 : 32), CPW = 32 / G;
  constexpr int LP = (N == 4) ? 4 : N;
  return sizeof(double) * ((size_t)kPredWarps * CPW * (D * NV * N * (NS / N) * LP + 8) + N * N);   // + R25 coefficients
}

// ADER_PRED_FLAT=0: no flat-cell first sweep (A/B; bitwise the same q either way)
bool pred_flat_enabled() {
  static const bool on = !(std::getenv("ADER_PRED_FLAT") && std::getenv("ADER_PRED_FLAT")[0] == '0');
  return on;
}

bool pred_dmma_enabled() {
  static const bool on = !(std::getenv("ADER_PRED_DMMA") && std::getenv("ADER_PRED_DMMA")[0] == '0');
  return on;
}
}  // namespace

bool supported(int D, int M, int SYS) {
  bool ok = false;
  ADER_DISPATCH(D, M, SYS, ok = true);
  return ok;
}

template <int M, int K>
static void weno_sweep_nv(const KCtx& k, const double* src, double* dst, const Box& R, long long astride) {
  constexpr int N = M + 1;
  constexpr int YC = (K == 2) ? 16 : 1;
  const long long per = ipow_c(N, K);
  if (R.count() == 0) return;
  const long long rows = (YC > 1) ? (long long)R.ext[0] * ((R.ext[1] + YC - 1) / YC) * YC * R.ext[2] : R.count();
  const long long threads = rows * k.NV * per;
  if (threads >= (1LL << 32) - 256) return;   // guarded at ader_create (32-bit thread indexing)
  const unsigned g = grid_for(threads, 256);
  count_launch(k);
  // ADER_WENO_G3=0: linear thread index decomposed by division (A/B; the same dofs)
  static const bool g3 = !(std::getenv("ADER_WENO_G3") && std::getenv("ADER_WENO_G3")[0] == '0');
  const long long gy = (YC > 1) ? (long long)YC * R.ext[2] : R.ext[1];
  const long long gz = (YC > 1) ? (R.ext[1] + YC - 1) / YC : R.ext[2];
  if (g3 && gy <= 65535 && gz <= 65535) {
    const dim3 grid(grid_for((long long)R.ext[0] * k.NV * per, 256), (unsigned)gy, (unsigned)gz);
    switch (k.NV) {
      case 4: k_weno<M, K, 4, YC, true><<<grid, 256, 0, k.stream>>>(src, dst, R, k.sy, k.sz, astride, k.tab); break;
      case 5: k_weno<M, K, 5, YC, true><<<grid, 256, 0, k.stream>>>(src, dst, R, k.sy, k.sz, astride, k.tab); break;
      case 9: k_weno<M, K, 9, YC, true><<<grid, 256, 0, k.stream>>>(src, dst, R, k.sy, k.sz, astride, k.tab); break;
      default: break;
    }
    return;
  }
  switch (k.NV) {
    case 4: k_weno<M, K, 4, YC><<<g, 256, 0, k.stream>>>(src, dst, R, k.sy, k.sz, astride, k.tab); break;
    case 5: k_weno<M, K, 5, YC><<<g, 256, 0, k.stream>>>(src, dst, R, k.sy, k.sz, astride, k.tab); break;
    case 9: k_weno<M, K, 9, YC><<<g, 256, 0, k.stream>>>(src, dst, R, k.sy, k.sz, astride, k.tab); break;
    default: break;
  }
}

void launch_weno_sweep(const KCtx& k, int sweep, const double* src, double* dst, const Box& region) {
  const long long astride = sweep == 0 ? 1 : (sweep == 1 ? k.sy : k.sz);
  if (k.M == 2) {
    if (sweep == 0) weno_sweep_nv<2, 0>(k, src, dst, region, astride);
    else if (sweep == 1) weno_sweep_nv<2, 1>(k, src, dst, region, astride);
    else weno_sweep_nv<2, 2>(k, src, dst, region, astride);
  } else if (k.M == 3) {
    if (sweep == 0) weno_sweep_nv<3, 0>(k, src, dst, region, astride);
    else if (sweep == 1) weno_sweep_nv<3, 1>(k, src, dst, region, astride);
    else weno_sweep_nv<3, 2>(k, src, dst, region, astride);
  }
}

void launch_predictor(const KCtx& k, const double* w, double* q, const Box& region, const double dtdx[3],
                      double tol, int max_sweeps, DevCounters* cnt, const double* dtdx_dev, long long qs, bool guess,
                      const StepState* gst, double guess_r, unsigned char* qflat) {
  launch_predictor_list(k, w, q, region, nullptr, 0, dtdx, tol, max_sweeps, cnt, nullptr, dtdx_dev, qs, guess, gst,
                        guess_r, nullptr, qflat);
}

void launch_predictor_list(const KCtx& k, const double* w, double* q, const Box& region, const int* list,
                           long long nlist, const double dtdx[3], double tol, int max_sweeps, DevCounters* cnt,
                           const unsigned char* emask, const double* dtdx_dev, long long qs, bool guess,
                           const StepState* gst, double guess_r, const int* slot, unsigned char* qflat) {
  const long long count = list ? nlist : region.count();
  if (count == 0) return;
  ADER_DISPATCH(k.D, k.M, k.SYS, {
    constexpr int N = M + 1;
    constexpr int NS = ipow_c(N, D);
    constexpr int CPW = 32 / ((NS <= 8) ? 8 : (NS <= 16 ? 16 : 32));
    const size_t sm = pred_smem<D, M, SYS>();
    // 2D M = 3: the x contraction on the FP64 tensor cores (dmma_x); ADER_PRED_DMMA=0 selects the
    // shared-memory contraction (A/B)
    constexpr bool XMC = (D == 2 && M == 3);
    auto kern = (XMC && pred_dmma_enabled()) ? k_predictor<D, M, SYS, kPredWarps, XMC> : k_predictor<D, M, SYS, kPredWarps>;
    int dev = 0;
    cudaGetDevice(&dev);
    static int attr_dev_mask = 0;   // the attribute is per device (and kernel variant)
    const int abit = 1 << ((dev & 15) * 2 + (kern == k_predictor<D, M, SYS, kPredWarps> ? 0 : 1));
    if (!(attr_dev_mask & abit)) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      attr_dev_mask |= abit;
    }
    const long long qstride = qs > 0 ? qs : (long long)Phys<SYS, D>::NV * NS * N;
    // persistent grid: enough CTAs for every SM at full occupancy, a few times over
    const unsigned need = grid_for(count, kPredWarps * CPW);
    const unsigned g = need < 148u * 16u ? need : 148u * 16u;
    count_launch(k);
    kern<<<g, kPredWarps * 32, sm, k.stream>>>(w, q, region, k.sy, k.sz, dtdx[0], dtdx[1], dtdx[2], k.gamma,
                                                k.ch, tol, max_sweeps, cnt, list, nlist, emask, dtdx_dev, qstride, guess ? 1 : 0,
                                                gst, guess_r, slot, pred_flat_enabled() ? 1 : 0, (pred_flat_enabled() && !guess) ? qflat : nullptr,
                                                k.tab);
  });
}

namespace {
template <int D, int M, int SYS>
void flux_cells_for(const KCtx& k, const double* q, double* F, const Box& ext, int H, const int n[3], int bmask,
                    int rmask, DevCounters* cnt, long long qs, const unsigned char* qflat, const double* w,
                    const double* dtdx, const double* dtdx_dev) {
  constexpr int YC = 16;
  if constexpr (D == 3 && M == 2 && SYS == 0) {
    static const int runs = [] {
      const char* e = std::getenv("ADER_FLUX_RUNS");
      return (e && e[0]) ? std::atoi(e) : 5;
    }();
    // x runs of 8 cells (default; ADER_FLUX_RUNS=0: k_face_flux_cells, 5..7: CTAs/SM of the register budget)
    if (runs > 0 && !qflat && k.tab.flux == 0) {
      static const int rl = [] {
        const char* e = std::getenv("ADER_FLUX_RL");
        return (e && e[0]) ? std::atoi(e) : 8;
      }();
      const int RLv = rl >= 16 ? 16 : 8;
      const unsigned nrx = (unsigned)((ext.ext[0] + RLv - 1) / RLv);
      const long long ychr = (ext.ext[1] + YC - 1) / YC;
      const long long groupsr = (long long)nrx * ychr * YC * ext.ext[2];
      count_launch(k);
      const unsigned gr = grid_for(groupsr, kFluxWarps);
#define ADER_RUNS(RL_, MB_)                                                                                     \
  k_face_flux_runs<D, M, SYS, kFluxWarps, YC, 0, RL_, MB_><<<gr, kFluxWarps * 32, 0, k.stream>>>(               \
      q, F, ext, H, n[0], n[1], n[2], k.sy, k.sz, k.ncell, k.gamma, k.ch, bmask, rmask, cnt, qs, nrx, k.tab)
      if (RLv == 16) { if (runs <= 4) ADER_RUNS(16, 4); else ADER_RUNS(16, 5); }
      else if (runs >= 7) ADER_RUNS(8, 7);
      else if (runs == 6) ADER_RUNS(8, 6);
      else if (runs == 5) ADER_RUNS(8, 5);
      else ADER_RUNS(8, 4);
#undef ADER_RUNS
      return;
    }
  }
  if constexpr (D == 3 && M == 2) {
    if (qflat) {   // flat cells rebuilt from w (one cell per warp)
      const long long ychf = (ext.ext[1] + YC - 1) / YC;
      const long long groupsf = (long long)ext.ext[0] * ychf * YC * ext.ext[2];
      count_launch(k);
      const unsigned gf = grid_for(groupsf, kFluxWarps);
      const double d0 = dtdx ? dtdx[0] : 0.0, d1 = dtdx ? dtdx[1] : 0.0, d2 = dtdx ? dtdx[2] : 0.0;
      if constexpr (SYS == 0) {
        if (k.tab.flux == 1) {
          k_face_flux_cells_flat<D, M, SYS, kFluxWarps, YC, 1><<<gf, kFluxWarps * 32, 0, k.stream>>>(
              q, F, ext, H, n[0], n[1], n[2], k.sy, k.sz, k.ncell, k.gamma, k.ch, bmask, rmask, cnt, qs, qflat, w, d0,
              d1, d2, dtdx_dev, k.tab);
          return;
        }
      }
      k_face_flux_cells_flat<D, M, SYS, kFluxWarps, YC, 0><<<gf, kFluxWarps * 32, 0, k.stream>>>(
          q, F, ext, H, n[0], n[1], n[2], k.sy, k.sz, k.ncell, k.gamma, k.ch, bmask, rmask, cnt, qs, qflat, w, d0, d1,
          d2, dtdx_dev, k.tab);
      return;
    }
  }
  constexpr int NS = ipow_c(M + 1, D);
  constexpr int CPW = 32 / ((NS <= 8) ? 8 : (NS <= 16 ? 16 : 32));
  const long long ych = (ext.ext[1] + YC - 1) / YC;
  const long long groups = (long long)ext.ext[0] * ych * YC * ext.ext[2];
  count_launch(k);
  const unsigned g = grid_for(groups, kFluxWarps * CPW);
  if constexpr (SYS == 0) {
    if (k.tab.flux == 1) {   // eqn.osher (Euler only, checked at ader_create)
      k_face_flux_cells<D, M, SYS, kFluxWarps, YC, 1><<<g, kFluxWarps * 32, 0, k.stream>>>(
          q, F, ext, H, n[0], n[1], n[2], k.sy, k.sz, k.ncell, k.gamma, k.ch, bmask, rmask, cnt, qs, k.tab);
      return;
    }
  }
  k_face_flux_cells<D, M, SYS, kFluxWarps, YC, 0><<<g, kFluxWarps * 32, 0, k.stream>>>(
      q, F, ext, H, n[0], n[1], n[2], k.sy, k.sz, k.ncell, k.gamma, k.ch, bmask, rmask, cnt, qs, k.tab);
}
}  // namespace

void launch_face_flux_cells(const KCtx& k, const double* q, double* F, const Box& ext, int H, const int n[3],
                            int bmask, int rmask, DevCounters* cnt, long long qs, const unsigned char* qflat,
                            const double* w, const double* dtdx, const double* dtdx_dev) {
  if (ext.count() == 0) return;
  ADER_DISPATCH(k.D, k.M, k.SYS,
                (flux_cells_for<D, M, SYS>(k, q, F, ext, H, n, bmask, rmask, cnt, qs, qflat, w, dtdx, dtdx_dev)));
}

void launch_update(const KCtx& k, double* u, const double* F, const Box& R, const double dtdx[3],
                   const double inv_dx[3], DevCounters* cnt, const double* dtdx_dev) {
  if (R.count() == 0) return;
  const unsigned g = grid_for(R.count(), 256);
  count_launch(k);
#define UPD(D_, S_)                                                                                   \
  k_update<D_, S_><<<g, 256, 0, k.stream>>>(u, F, R, k.sy, k.sz, k.ncell, dtdx[0], dtdx[1], dtdx[2], \
                                             inv_dx[0], inv_dx[1], inv_dx[2], k.gamma, k.ch, cnt, dtdx_dev)
  if (k.D == 2 && k.SYS == 0) UPD(2, 0);
  else if (k.D == 3 && k.SYS == 0) UPD(3, 0);
  else if (k.D == 2 && k.SYS == 1) UPD(2, 1);
  else if (k.D == 3 && k.SYS == 1) UPD(3, 1);
#undef UPD
}

void launch_cfl_speed(const KCtx& k, const double* u, const Box& R, const double inv_dx[3], DevCounters* cnt) {
  if (R.count() == 0) return;
  const unsigned g = grid_for(R.count(), 256);
  count_launch(k);
#define SPD(D_, S_) \
  k_cfl_speed<D_, S_><<<g, 256, 0, k.stream>>>(u, R, k.sy, k.sz, inv_dx[0], inv_dx[1], inv_dx[2], k.gamma, k.ch, cnt)
  if (k.D == 2 && k.SYS == 0) SPD(2, 0);
  else if (k.D == 3 && k.SYS == 0) SPD(3, 0);
  else if (k.D == 2 && k.SYS == 1) SPD(2, 1);
  else if (k.D == 3 && k.SYS == 1) SPD(3, 1);
#undef SPD
}

void launch_step_dt(const KCtx& k, DevCounters* cnt, StepState* st, double cfl, double t_end, const double dx[3]) {
  count_launch(k);
  k_step_dt<<<1, 1, 0, k.stream>>>(cnt, st, cfl, t_end, dx[0], dx[1], dx[2], k.D);
}

void launch_set_dt(const KCtx& k, StepState* st, double dt, const double dx[3]) {
  count_launch(k);
  k_set_dt<<<1, 1, 0, k.stream>>>(st, dt, dx[0], dx[1], dx[2], k.D);
}

void launch_fill_axis(const KCtx& k, double* u, const Box& region, int axis, int mode, int H, int n) {
  const long long total = region.count() * k.NV;
  if (total == 0) return;
  count_launch(k);
  k_fill_axis<<<grid_for(total, 256), 256, 0, k.stream>>>(u, region, k.sy, k.sz, k.NV, axis, mode, H, n);
}

void launch_pack(const KCtx& k, const double* u, const Box& b, double* buf) {
  const long long total = b.count() * k.NV;
  if (total == 0) return;
  count_launch(k);
  k_pack<<<grid_for(total, 256), 256, 0, k.stream>>>(u, b, k.sy, k.sz, k.NV, buf, 1);
}

void launch_unpack(const KCtx& k, double* u, const Box& b, const double* buf) {
  const long long total = b.count() * k.NV;
  if (total == 0) return;
  count_launch(k);
  k_pack<<<grid_for(total, 256), 256, 0, k.stream>>>(u, b, k.sy, k.sz, k.NV, const_cast<double*>(buf), 0);
}

void launch_gather(const KCtx& k, const double* src, int stride, const Box& b, double* out) {
  const long long total = b.count() * stride;
  if (total == 0) return;
  count_launch(k);
  k_pack<<<grid_for(total, 256), 256, 0, k.stream>>>(src, b, k.sy, k.sz, stride, out, 1);
}

void launch_scatter(const KCtx& k, double* dst, int stride, const Box& b, const double* in) {
  const long long total = b.count() * stride;
  if (total == 0) return;
  count_launch(k);
  k_pack<<<grid_for(total, 256), 256, 0, k.stream>>>(dst, b, k.sy, k.sz, stride, const_cast<double*>(in), 0);
}

void launch_ic_average(const KCtx& k, double* u, const double* prim, const double* wq, int nq, long long first,
                       long long ncells, const int n[3], int H, const int off[3]) {
  if (ncells == 0) return;
  const unsigned g = grid_for(ncells, 128);
  count_launch(k);
#define ICA(D_, S_) \
  k_ic_average<D_, S_><<<g, 128, 0, k.stream>>>(u, prim, wq, nq, first, ncells, n[0], n[1], H, k.sy, k.sz, k.gamma, \
                                                 off[0], off[1], off[2])
  if (k.D == 2 && k.SYS == 0) ICA(2, 0);
  else if (k.D == 3 && k.SYS == 0) ICA(3, 0);
  else if (k.D == 2 && k.SYS == 1) ICA(2, 1);
  else if (k.D == 3 && k.SYS == 1) ICA(3, 1);
#undef ICA
}

int launch_cons_partials(const KCtx& k, const double* u, const Box& b, double vol, double* partial, int max_blocks) {
  const unsigned g = grid_for(b.count(), 256);
  if ((int)g > max_blocks || g == 0) return 0;
  count_launch(k);
  k_cons_partials<<<g, 256, 0, k.stream>>>(u, b, k.sy, k.sz, k.NV, vol, partial);
  return (int)g;
}

}  // namespace ader
