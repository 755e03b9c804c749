// pred_flux.cu — a2 the space-time predictor fused with a3 the space-time face
// flux on the uniform grid: the predictor dofs q never touch HBM.
//
//   a2 nodal Picard iteration of eqn.stdg.final, predictor.cuh
//   a3 space-time Gauss quadrature of the two-point flux on every lower face
//      (flux:F/G/H @ P:158-172, eqn.rusanov @ P:181-185 / eqn.osher @ P:186-196)
//
// Why: the separate kernels write every cell's q (nu N^(d+1) doubles, 3240 B at
// d=3, M=2) and read it back for the faces — 116 GB per step at 256^3, two
// thirds of the step's HBM traffic.  Here a CTA owns a tile of TX x TY cells
// (3D: x, y; 2D: TX cells along x) and walks it along the last axis W (z in
// 3D, y in 2D) over a segment of LS levels.  Per level:
//   A. its lane groups run the predictor of the level's cells (w read from
//      HBM, q kept in shared memory in the block layout [nu][N time][N^d space]);
//   B. every cell's lower faces: in-tile faces read both q blocks from shared
//      memory, the W face takes the upper-W trace of the level below carried in
//      shared memory; the cell's own upper-W trace is carried to the next level.
// Faces between tiles (and between W segments) cannot see both q blocks: the
// cells on both sides write their face trace ([nu][N^d] doubles, psi(1) side of
// the lower cell, psi(0) side of the upper cell) to a face buffer, and
// k_flux_tile_faces evaluates those faces afterwards (about 1/TX + 1/TY + 1/LS
// of the faces).  Per cell HBM traffic drops from w + 2 q + F (7.7 KB at C4) to
// w + F + ~1 KB of traces.
//
// Bitwise the same F as launch_predictor + launch_face_flux_cells: the same
// predictor_cell (its one-time-level scratch variant does the same arithmetic
// in the same order), the same face_trace / point_flux_states, and the same
// point-sum order (lane i sums row i over the N^d points in order).
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"
#include "flux_point.cuh"
#include "launch.h"
#include "predictor.cuh"

namespace ader {

namespace {

__device__ __forceinline__ void rec_err(DevCounters* c, int code, int stage, long long cell) {
  if (atomicCAS(&c->err_code, 0, code) == 0) {
    c->err_stage = stage;
    c->err_cell = (unsigned long long)cell;
  }
}

template <int D, int M, int SYS>
struct PF {
  using P = PredCfg<D, M, SYS, true>;   // one time level of f* scratch per cell
  static constexpr int NV = P::NV, N = M + 1, NS = P::NS, NST = NS * N, NT = NS / N, G = P::G, CPW = P::CPW;
  static constexpr int W = D - 1;
  static constexpr int TX = (D == 3) ? 4 : 8;
  static constexpr int TY = (D == 3) ? 4 : 1;
  static constexpr int CELLS = TX * TY;
  static constexpr int WARPS = (D == 3) ? 8 : 4;
  static constexpr int GROUPS = WARPS * CPW;
  static_assert(CELLS % GROUPS == 0, "every lane group takes the same number of cells per level");
  static constexpr int QS = NV * NST + ((NV * NST) & 1);   // q block stride in shared memory
  static constexpr int TR = NV * NS;                       // one face trace [nu][N^d]
  static constexpr int KR = D * NV;                        // point-sum rows of a cell
  static constexpr int RED = KR * (G + 1);
  static constexpr int SCR = (P::FSZ > RED) ? P::FSZ : RED;   // predictor scratch, then point sums
  static constexpr size_t smem_bytes() {
    return sizeof(double) * ((size_t)CELLS * QS + (size_t)CELLS * TR + (size_t)GROUPS * SCR);
  }
  static_assert(smem_bytes() <= 227 * 1024, "shared memory of one CTA");
  static constexpr int MINB = (SYS == 0) ? ((D == 3) ? 2 : 4) : ((D == 3) ? 1 : 2);
};

// Geometry shared by the walk and the tile-face kernel.  RG: the walked region
// (predictor region PR along every axis at the low end, the face box's upper
// layer at the high end), tiles of TX (x) x TY (y, 3D) cells, segments of LS
// levels along W.  Face buffers of direction d hold, per inter-tile (or
// inter-segment) face, the lower cell's psi(1) trace (L) and the upper cell's
// psi(0) trace (R).
struct WalkGeo {
  Box RG;
  int H, n[3];
  int ntx, nty, LS, nseg;
  long long nf[3];          // inter-tile faces per direction
};

// face index of the face whose upper cell is (cx, cy, cz) and lies at the start
// of tile / segment k >= 1 along d
template <int D>
__device__ __forceinline__ long long face_index(const WalkGeo& g, int d, int cx, int cy, int cz, int k) {
  const int EX = g.RG.ext[0], EY = (D == 3) ? g.RG.ext[1] : 1;
  constexpr int W = D - 1;
  const int xr = cx - g.RG.lo[0], yr = (D == 3) ? cy - g.RG.lo[1] : 0;
  const int wr = ((D == 3) ? cz : cy) - g.RG.lo[W];
  if (d == W) return ((long long)(k - 1) * EY + yr) * EX + xr;
  if (d == 0) return ((long long)wr * EY + yr) * (g.ntx - 1) + (k - 1);
  return ((long long)wr * EX + xr) * (g.nty - 1) + (k - 1);   // d == 1 (3D)
}

// which lower faces of cell (cx, cy, cz) the step needs (the face box of
// launch_face_flux_cells: ext = owned + 1 upper layer, face d needs the other
// axes inside the owned block), and their boundary flags
template <int D>
__device__ __forceinline__ void face_flags(const WalkGeo& g, int bmask, int rmask, int cx, int cy, int cz,
                                           bool (&fok)[3], bool (&tlo)[3], bool (&thi)[3], bool (&rlo)[3],
                                           bool (&rhi)[3]) {
  const int H = g.H, zH = (D == 3) ? H : 0;
  const int c[3] = {cx, cy, cz};
  const int lo[3] = {H, H, zH};
  bool in_ext = true, inn[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (a < D) {
      in_ext &= c[a] >= lo[a] && c[a] <= lo[a] + g.n[a];
      inn[a] = c[a] < lo[a] + g.n[a];
    } else {
      inn[a] = true;
    }
  }
  fok[0] = in_ext && inn[1] && inn[2];
  fok[1] = in_ext && inn[0] && inn[2];
  fok[2] = in_ext && inn[0] && inn[1];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const bool first = c[a] == lo[a], last = c[a] == lo[a] + g.n[a];
    tlo[a] = (bmask & (1 << (2 * a))) && first;
    thi[a] = (bmask & (2 << (2 * a))) && last;
    rlo[a] = (rmask & (1 << (2 * a))) && first;
    rhi[a] = (rmask & (2 << (2 * a))) && last;
  }
}

template <int D, int M, int SYS, int DIR>
__device__ __forceinline__ void store_trace(const double* qb, int ps, const double (&psi)[kMaxN], double* dst) {
  constexpr int NV = Phys<SYS, D>::NV, NS = ipow_c(M + 1, D);
  double a[NV];
  face_trace<D, M, NV, DIR, false>(qb, ps, psi, a);
#pragma unroll
  for (int i = 0; i < NV; ++i) dst[i * NS + ps] = a[i];
}

template <int D, int M, int SYS, int FLUX>
__global__ void __launch_bounds__(PF<D, M, SYS>::WARPS * 32, PF<D, M, SYS>::MINB)
    k_pred_flux(const double* __restrict__ w, double* __restrict__ F, double* __restrict__ bnd0,
                double* __restrict__ bnd1, double* __restrict__ bnd2, const Box PR, const WalkGeo g,
                const long long sy, const long long sz, const long long ncell, const double gamma, const double ch,
                const double tol, const int max_sweeps, const int bmask, const int rmask,
                DevCounters* __restrict__ cnt, const double* __restrict__ dtdx_dev, const double dtdx0,
                const double dtdx1, const double dtdx2, const int ntiles, const __grid_constant__ DevTables T) {
  using C = PF<D, M, SYS>;
  constexpr int NV = C::NV, N = C::N, NS = C::NS, NST = C::NST, NT = C::NT, G = C::G, CPW = C::CPW;
  constexpr int TX = C::TX, TY = C::TY, CELLS = C::CELLS, QS = C::QS, TR = C::TR, KR = C::KR, W = C::W;
  extern __shared__ __align__(16) double smem[];
  double* QB = smem;                          // [CELLS][QS]   q of the level's cells
  double* TRC = QB + CELLS * QS;              // [CELLS][TR]   upper-W traces of the level below
  double* SCRb = TRC + CELLS * TR;            // [GROUPS][SCR] predictor scratch / point sums
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = lane / G, p = lane & (G - 1);
  PredLane<D, M, SYS> L;
  L.init(p, T);
  double* scr = SCRb + (warp * CPW + slot) * C::SCR;
  const bool pok = p < NS;
  const int ps = pok ? p : 0;
  // quadrature weight of this lane's face point (same decomposition on every face)
  const int s_ = ps / NT, tt = ps - (ps / NT) * NT;
  double wt = T.w[s_] * T.w[tt % N];
  if (D == 3) wt *= T.w[tt / N];
  const double dtdx[3] = {dtdx_dev ? dtdx_dev[0] : dtdx0, dtdx_dev ? dtdx_dev[1] : dtdx1,
                          dtdx_dev ? dtdx_dev[2] : dtdx2};
  double* bndL[3] = {bnd0, bnd1, bnd2};
  const int nsegW = g.nseg;
  unsigned long long acc_sweeps = 0, acc_cells = 0;
  int acc_max = 0;
  auto in_pr = [&](int x, int y, int z) {
    return x >= PR.lo[0] && x < PR.lo[0] + PR.ext[0] && y >= PR.lo[1] && y < PR.lo[1] + PR.ext[1] &&
           z >= PR.lo[2] && z < PR.lo[2] + PR.ext[2];
  };

  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int tx = t % g.ntx;
    const int rest = t / g.ntx;
    const int ty = (D == 3) ? rest % g.nty : 0;
    const int seg = (D == 3) ? rest / g.nty : rest;
    const int x0 = g.RG.lo[0] + tx * TX;
    const int nvx = min(TX, g.RG.lo[0] + g.RG.ext[0] - x0);
    const int y0 = (D == 3) ? g.RG.lo[1] + ty * TY : 0;
    const int nvy = (D == 3) ? min(TY, g.RG.lo[1] + g.RG.ext[1] - y0) : 1;
    const int wb = g.RG.lo[W] + seg * g.LS;
    const int we = min(wb + g.LS, g.RG.lo[W] + g.RG.ext[W]);
    for (int lev = wb; lev < we; ++lev) {
      // ---- A: predictor of the level's cells, q -> shared memory
      for (int jb = warp * CPW; jb < CELLS; jb += C::WARPS * CPW) {
        const int j = jb + slot;
        const int cxi = j % TX, cyi = j / TX;
        const bool in_tile = cxi < nvx && cyi < nvy;
        const int cx = x0 + cxi, cy = (D == 3) ? y0 + cyi : lev, cz = (D == 3) ? lev : 0;
        const bool pred_ok = in_tile && in_pr(cx, cy, cz);
        const long long cell = (long long)cx + (long long)cy * sy + (long long)cz * sz;
        double wv[NV], qv[NV][N];
#pragma unroll
        for (int v = 0; v < NV; ++v) wv[v] = pred_ok ? __ldg(&w[cell * (NV * NS) + v * NS + L.node]) : 1.0;
        bool conv, bad;
        int nsw;
        predictor_cell<D, M, SYS, true>(wv, qv, scr, L, dtdx, pred_ok, gamma, ch, tol, max_sweeps, T, nsw, conv,
                                        bad);
        if (pred_ok && L.lane_ok) {
          if (bad) rec_err(cnt, 1, 1, cell);
          else if (!conv) rec_err(cnt, 2, 1, cell);
          double* qo = QB + j * QS + L.node;
#pragma unroll
          for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int s = 0; s < N; ++s) qo[v * NST + s * NS] = qv[v][s];
          if (L.node == 0) {
            acc_sweeps += (unsigned long long)nsw;
            acc_cells += 1ull;
            acc_max = nsw > acc_max ? nsw : acc_max;
          }
        }
        __syncwarp();
      }
      __syncthreads();
      // ---- B: the lower faces of the level's cells
      for (int jb = warp * CPW; jb < CELLS; jb += C::WARPS * CPW) {
        const int j = jb + slot;
        const int cxi = j % TX, cyi = j / TX;
        const bool in_tile = cxi < nvx && cyi < nvy;
        const int cx = x0 + cxi, cy = (D == 3) ? y0 + cyi : lev, cz = (D == 3) ? lev : 0;
        const long long cell = (long long)cx + (long long)cy * sy + (long long)cz * sz;
        const double* qown = QB + j * QS;
        bool fok[3], tlo[3], thi[3], rlo[3], rhi[3];
        face_flags<D>(g, bmask, rmask, cx, cy, cz, fok, tlo, thi, rlo, rhi);
        bool here[3] = {false, false, false};   // face evaluated in this kernel (F stored below)
        // lane p stores its weighted point fluxes of direction d in column p of
        // rows d*NV.. (k_face_flux_cells' point-sum layout), one direction at a time
        double(*rb)[G + 1] = reinterpret_cast<double(*)[G + 1]>(scr);
        bool good = true;
        if (in_tile) {
          // in-plane directions (x; y in 3D)
#pragma unroll
          for (int d = 0; d < W; ++d) {
            const int pos = (d == 0) ? cxi : cyi;
            const int org = (d == 0) ? x0 : y0;
            const int tl = (d == 0) ? TX : TY;
            const int kt = (d == 0) ? tx : ty;
            const int step = (d == 0) ? 1 : TX;
            if (fok[d]) {
              if (pos > 0 || org == g.RG.lo[d]) {
                // in-tile face, or the region's first cell (its lower neighbour is
                // beyond a transmissive side / wall: only the own trace is used)
                const double* ql = pos > 0 ? qown - step * QS : qown;
                double val[NV];
                if (d == 0)
                  good &= point_flux_blocks<D, M, SYS, 0, FLUX, false>(ql, qown, ps, pok, tlo[0], thi[0], rlo[0],
                                                                       rhi[0], wt, gamma, ch, T, val);
                else
                  good &= point_flux_blocks<D, M, SYS, (D == 3 ? 1 : 0), FLUX, false>(
                      ql, qown, ps, pok, tlo[1], thi[1], rlo[1], rhi[1], wt, gamma, ch, T, val);
                if (pok) {
#pragma unroll
                  for (int i = 0; i < NV; ++i) rb[d * NV + i][p] = val[i];
                }
                here[d] = true;
              } else if (pok) {   // inter-tile face: the own psi(0) trace to the face buffer
                const long long f = face_index<D>(g, d, cx, cy, cz, kt);
                double* dst = bndL[d] + (g.nf[d] + f) * TR;
                if (d == 0) store_trace<D, M, SYS, 0>(qown, ps, T.psi0, dst);
                else store_trace<D, M, SYS, (D == 3 ? 1 : 0)>(qown, ps, T.psi0, dst);
              }
            }
            // the psi(1) trace for the next tile's first cell
            if (pos == tl - 1 && org + tl < g.RG.lo[d] + g.RG.ext[d] && pok) {
              bool fo[3], a1[3], a2[3], a3[3], a4[3];
              face_flags<D>(g, bmask, rmask, cx + (d == 0), cy + (d == 1), cz, fo, a1, a2, a3, a4);
              if (fo[d]) {
                const long long f = face_index<D>(g, d, cx + (d == 0), cy + (d == 1), cz, kt + 1);
                double* dst = bndL[d] + f * TR;
                if (d == 0) store_trace<D, M, SYS, 0>(qown, ps, T.psi1, dst);
                else store_trace<D, M, SYS, (D == 3 ? 1 : 0)>(qown, ps, T.psi1, dst);
              }
            }
          }
          // W direction: the carried upper trace of the level below
          if (pok) {
            double a[NV], b[NV];
            face_trace<D, M, NV, W, false>(qown, ps, T.psi0, b);
            if (fok[W]) {
              if (lev > wb || seg == 0) {
                if (lev > wb) {
#pragma unroll
                  for (int i = 0; i < NV; ++i) a[i] = TRC[j * TR + i * NS + ps];
                } else {
#pragma unroll
                  for (int i = 0; i < NV; ++i) a[i] = b[i];   // region start: beyond a side / wall
                }
                double val[NV];
                good &= point_flux_states<D, SYS, W, FLUX>(a, b, tlo[W], thi[W], rlo[W], rhi[W], wt, gamma, ch, T,
                                                           val);
#pragma unroll
                for (int i = 0; i < NV; ++i) rb[W * NV + i][p] = val[i];
              } else {   // first level of a later segment: own psi(0) trace to the face buffer
                double* dst = bndL[W] + (g.nf[W] + face_index<D>(g, W, cx, cy, cz, seg)) * TR;
#pragma unroll
                for (int i = 0; i < NV; ++i) dst[i * NS + ps] = b[i];
              }
            }
            // this level's psi(1) trace: carried to the next level, or to the
            // face buffer at the segment's last level
            face_trace<D, M, NV, W, false>(qown, ps, T.psi1, a);
            if (lev + 1 < we) {
#pragma unroll
              for (int i = 0; i < NV; ++i) TRC[j * TR + i * NS + ps] = a[i];
            } else if (seg + 1 < nsegW) {
              bool fo[3], a1[3], a2[3], a3[3], a4[3];
              face_flags<D>(g, bmask, rmask, cx, (D == 3) ? cy : lev + 1, (D == 3) ? lev + 1 : 0, fo, a1, a2, a3,
                            a4);
              if (fo[W]) {
                double* dst = bndL[W] + face_index<D>(g, W, cx, cy, cz, seg + 1) * TR;
#pragma unroll
                for (int i = 0; i < NV; ++i) dst[i * NS + ps] = a[i];
              }
            }
          }
          here[W] = fok[W] && (lev > wb || seg == 0);
        }
        if (!good) rec_err(cnt, 1, 2, cell);
        // point sums (the order of k_face_flux_cells): lane i sums row i in point order
        __syncwarp();
        for (int i = p; i < KR; i += G) {
          double acc = rb[i][0];
#pragma unroll
          for (int jj = 1; jj < NS; ++jj) acc += rb[i][jj];
          const int dir = i / NV, var = i - dir * NV;
          if (here[dir]) F[((long long)dir * ncell + cell) * NV + var] = acc;
        }
        __syncwarp();
      }
      __syncthreads();   // q slots and carried traces are rewritten by the next level
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc_sweeps += __shfl_xor_sync(0xffffffffu, acc_sweeps, o);
    acc_cells += __shfl_xor_sync(0xffffffffu, acc_cells, o);
    acc_max = max(acc_max, __shfl_xor_sync(0xffffffffu, acc_max, o));
  }
  if (lane == 0 && acc_cells) {
    atomicAdd(&cnt->sweeps, acc_sweeps);
    atomicAdd(&cnt->cells, acc_cells);
    atomicMax(&cnt->sweeps_max, acc_max);
  }
}

// The faces between tiles (DIR in-plane) or between W segments (DIR = W): one
// lane group per face, the two traces from the face buffer, the same point
// flux and point-sum order as every other face.
template <int D, int M, int SYS, int DIR, int FLUX>
__global__ void __launch_bounds__(128) k_flux_tile_faces(const double* __restrict__ bnd, double* __restrict__ F,
                                                         const WalkGeo g, const long long sy, const long long sz,
                                                         const long long ncell, const double gamma, const double ch,
                                                         const int bmask, const int rmask,
                                                         DevCounters* __restrict__ cnt,
                                                         const __grid_constant__ DevTables T) {
  using PH = Phys<SYS, D>;
  constexpr int NV = PH::NV, N = M + 1, NS = ipow_c(N, D), NT = NS / N;
  constexpr int G = (NS <= 8) ? 8 : (NS <= 16 ? 16 : 32), CPW = 32 / G, W = D - 1;
  constexpr int TX = PF<D, M, SYS>::TX, TY = PF<D, M, SYS>::TY, TR = NV * NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, p = lane & (G - 1);
  const long long f = ((long long)blockIdx.x * 4 + warp) * CPW + lane / G;
  const bool fin = f < g.nf[DIR];
  const long long ff = fin ? f : 0;
  // decode the face's upper cell
  int cx, cy, cz;
  const int EX = g.RG.ext[0], EY = (D == 3) ? g.RG.ext[1] : 1;
  if (DIR == W) {
    const int xr = (int)(ff % EX);
    const long long r = ff / EX;
    const int yr = (D == 3) ? (int)(r % EY) : 0;
    const int k = (int)(r / EY) + 1;
    const int wl = g.RG.lo[W] + k * g.LS;
    cx = g.RG.lo[0] + xr;
    cy = (D == 3) ? g.RG.lo[1] + yr : wl;
    cz = (D == 3) ? wl : 0;
  } else if (DIR == 0) {
    const int k = (int)(ff % (g.ntx - 1)) + 1;
    const long long r = ff / (g.ntx - 1);
    const int yr = (D == 3) ? (int)(r % EY) : 0;
    const int wr = (D == 3) ? (int)(r / EY) : (int)r;
    cx = g.RG.lo[0] + k * TX;
    cy = (D == 3) ? g.RG.lo[1] + yr : g.RG.lo[1] + wr;
    cz = (D == 3) ? g.RG.lo[2] + wr : 0;
  } else {
    const int k = (int)(ff % (g.nty - 1)) + 1;
    const long long r = ff / (g.nty - 1);
    const int xr = (int)(r % EX), wr = (int)(r / EX);
    cx = g.RG.lo[0] + xr;
    cy = g.RG.lo[1] + k * TY;
    cz = g.RG.lo[2] + wr;
  }
  bool fok[3], tlo[3], thi[3], rlo[3], rhi[3];
  face_flags<D>(g, bmask, rmask, cx, cy, cz, fok, tlo, thi, rlo, rhi);
  const bool ok = fin && fok[DIR];
  const bool pok = p < NS;
  const int ps = pok ? p : 0;
  const int s_ = ps / NT, tt = ps - (ps / NT) * NT;
  double wt = T.w[s_] * T.w[tt % N];
  if (D == 3) wt *= T.w[tt / N];
  double v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = 0.0;
  const long long cell = (long long)cx + (long long)cy * sy + (long long)cz * sz;
  if (ok && pok) {
    double a[NV], b[NV];
    const double* sa = bnd + ff * TR;
    const double* sb = bnd + (g.nf[DIR] + ff) * TR;
#pragma unroll
    for (int i = 0; i < NV; ++i) { a[i] = __ldg(&sa[i * NS + ps]); b[i] = __ldg(&sb[i * NS + ps]); }
    if (!point_flux_states<D, SYS, DIR, FLUX>(a, b, tlo[DIR], thi[DIR], rlo[DIR], rhi[DIR], wt, gamma, ch, T, v))
      rec_err(cnt, 1, 2, cell);
  }
  __shared__ double red[4 * CPW][NV][G + 1];
  double(*rb)[G + 1] = red[warp * CPW + lane / G];
  if (pok) {
#pragma unroll
    for (int i = 0; i < NV; ++i) rb[i][p] = v[i];
  }
  __syncwarp();
  if (ok && p < NV) {
    double acc = rb[p][0];
#pragma unroll
    for (int jj = 1; jj < NS; ++jj) acc += rb[p][jj];
    F[((long long)DIR * ncell + cell) * NV + p] = acc;
  }
}

template <int D, int M, int SYS>
WalkGeo walk_geo(const Box& PR, int H, const int n[3], int slots) {
  using C = PF<D, M, SYS>;
  constexpr int W = D - 1;
  WalkGeo g{};
  g.H = H;
  g.n[0] = n[0]; g.n[1] = n[1]; g.n[2] = n[2];
  const int zH = (D == 3) ? H : 0;
  const int lo[3] = {H, H, zH};
  // RG: from the predictor region's start to the face box's end (owned + 1)
  int rlo[3], rhi[3];
  for (int a = 0; a < 3; ++a) {
    if (a < D) { rlo[a] = PR.lo[a]; rhi[a] = lo[a] + n[a] + 1; }
    else { rlo[a] = 0; rhi[a] = 1; }
  }
  for (int a = 0; a < 3; ++a) { g.RG.lo[a] = rlo[a]; g.RG.ext[a] = rhi[a] - rlo[a]; }
  g.ntx = (g.RG.ext[0] + C::TX - 1) / C::TX;
  g.nty = (D == 3) ? (g.RG.ext[1] + C::TY - 1) / C::TY : 1;
  const long long cols = (long long)g.ntx * g.nty;
  // segments along W: at least 8 tiles per CTA slot, segments of >= 8 levels
  const int EW = g.RG.ext[W];
  int nseg = 1;
  while (cols * nseg < 8LL * slots && EW / (nseg + 1) >= 8) ++nseg;
  g.LS = (EW + nseg - 1) / nseg;
  g.nseg = (EW + g.LS - 1) / g.LS;
  const long long EX = g.RG.ext[0], EY = (D == 3) ? g.RG.ext[1] : 1;
  g.nf[0] = (long long)(g.ntx - 1) * EY * EW;
  g.nf[1] = (D == 3) ? (long long)(g.nty - 1) * EX * EW : 0;
  g.nf[2] = 0;
  g.nf[W] = (long long)(g.nseg - 1) * EX * EY;
  return g;
}

template <int D, int M, int SYS>
int pf_slots() {
  using C = PF<D, M, SYS>;
  auto kern = k_pred_flux<D, M, SYS, 0>;
  int dev = 0, per_sm = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes());
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::WARPS * 32, C::smem_bytes());
  if (per_sm < 1) per_sm = 1;
  return per_sm * nsm;
}

template <int D, int M, int SYS, int FLUX>
void launch_pf_t(const KCtx& k, const double* w, double* F, double* bnd, const Box& PR, const int H, const int n[3],
                 int bmask, int rmask, double tol, int max_sweeps, DevCounters* cnt, const double dtdx[3],
                 const double* dtdx_dev) {
  using C = PF<D, M, SYS>;
  constexpr int W = D - 1, TR = C::TR;
  auto kern = k_pred_flux<D, M, SYS, FLUX>;
  const size_t sm = C::smem_bytes();
  int dev = 0;
  cudaGetDevice(&dev);
  static int attr_dev_mask = 0;   // the attribute is per device
  if (!(attr_dev_mask & (1 << (dev & 31)))) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr_dev_mask |= 1 << (dev & 31);
  }
  static int slots = 0;
  if (!slots) slots = pf_slots<D, M, SYS>();
  const WalkGeo g = walk_geo<D, M, SYS>(PR, H, n, slots);
  double* b[3] = {nullptr, nullptr, nullptr};
  size_t off = 0;
  for (int d = 0; d < D; ++d) { b[d] = bnd + off; off += (size_t)2 * g.nf[d] * TR; }
  const int ntiles = g.ntx * g.nty * g.nseg;
  const int grid = ntiles < slots ? ntiles : slots;
  if (k.launches) ++*k.launches;
  kern<<<grid, C::WARPS * 32, sm, k.stream>>>(w, F, b[0], b[1], b[2], PR, g, k.sy, k.sz, k.ncell, k.gamma, k.ch, tol,
                                              max_sweeps, bmask, rmask, cnt, dtdx_dev, dtdx[0], dtdx[1], dtdx[2],
                                              ntiles, k.tab);
  constexpr int CPW = C::CPW;
  auto faces = [&](auto dir_tag) {
    constexpr int DIR = decltype(dir_tag)::value;
    if (g.nf[DIR] == 0) return;
    const long long groups = g.nf[DIR];
    const unsigned gr = (unsigned)((groups + 4 * CPW - 1) / (4 * CPW));
    if (k.launches) ++*k.launches;
    k_flux_tile_faces<D, M, SYS, DIR, FLUX><<<gr, 128, 0, k.stream>>>(b[DIR], F, g, k.sy, k.sz, k.ncell, k.gamma, k.ch,
                                                                      bmask, rmask, cnt, k.tab);
  };
  faces(std::integral_constant<int, 0>());
  if constexpr (D == 3) faces(std::integral_constant<int, 1>());
  faces(std::integral_constant<int, W>());
}

template <int D, int M, int SYS>
void pf_for(const KCtx& k, const double* w, double* F, double* bnd, const Box& PR, const int H, const int n[3],
            int bmask, int rmask, double tol, int max_sweeps, DevCounters* cnt, const double dtdx[3],
            const double* dtdx_dev) {
  if constexpr (SYS == 0) {
    if (k.tab.flux == 1) {   // eqn.osher (Euler only, checked at ader_create)
      launch_pf_t<D, M, SYS, 1>(k, w, F, bnd, PR, H, n, bmask, rmask, tol, max_sweeps, cnt, dtdx, dtdx_dev);
      return;
    }
  }
  launch_pf_t<D, M, SYS, 0>(k, w, F, bnd, PR, H, n, bmask, rmask, tol, max_sweeps, cnt, dtdx, dtdx_dev);
}

}  // namespace

long long pred_flux_buffer_doubles(int D, int M, int SYS, const Box& PR, int H, const int n[3]) {
  long long out = -1;
#define ADER_PFB(D_, M_, S_)                                                    \
  if (D == D_ && M == M_ && SYS == S_) {                                        \
    const WalkGeo g = walk_geo<D_, M_, S_>(PR, H, n, pf_slots<D_, M_, S_>());   \
    out = 0;                                                                    \
    for (int d = 0; d < D_; ++d) out += 2 * g.nf[d] * PF<D_, M_, S_>::TR;       \
  }
  ADER_PFB(2, 2, 0) ADER_PFB(2, 3, 0) ADER_PFB(3, 2, 0) ADER_PFB(2, 2, 1) ADER_PFB(2, 3, 1) ADER_PFB(3, 2, 1)
#undef ADER_PFB
  return out;
}

void launch_pred_flux(const KCtx& k, const double* w, double* F, double* bnd, const Box& PR, int H, const int n[3],
                      int bmask, int rmask, double tol, int max_sweeps, DevCounters* cnt, const double dtdx[3],
                      const double* dtdx_dev) {
  if (PR.count() == 0) return;
#define ADER_PF(D_, M_, S_)                                                                              \
  if (k.D == D_ && k.M == M_ && k.SYS == S_) {                                                           \
    pf_for<D_, M_, S_>(k, w, F, bnd, PR, H, n, bmask, rmask, tol, max_sweeps, cnt, dtdx, dtdx_dev);      \
    return;                                                                                              \
  }
  ADER_PF(2, 2, 0) ADER_PF(2, 3, 0) ADER_PF(3, 2, 0) ADER_PF(2, 2, 1) ADER_PF(2, 3, 1) ADER_PF(3, 2, 1)
#undef ADER_PF
}

}  // namespace ader
