// weno_pred.cu — a1 WENO reconstruction fused with a2 the space-time predictor
// on the uniform grid: w_x, w_xy and w never leave the SM.
//
//   a1 dimension-by-dimension WENO: x sweep on the cell averages,
//      y sweep on the x-sweep dofs, z sweep on those (3D)
//   a2 nodal Picard iteration of eqn.stdg.final, predictor.cuh
//
// A CTA owns a tile of TX x TY cells (3D; 2D: TX cells along x) of the
// predictor region and walks it along the last axis W (z in 3D, y in 2D) over a
// segment of levels.  Level L enters a ring of 2M+1 levels in shared memory: its
// cell averages (the tile + M halo cells in x and y) are prefetched one step
// ahead with cp.async, the x sweep (and in 3D the y sweep) runs on them.  Once
// level L + M has entered, level L is complete: its last sweep (along W) reads
// the 2M+1 ring levels and writes w of the tile's cells to shared memory, and
// the predictor lane groups take w from there and stream q to HBM.  Compared
// with separate sweep kernels this removes w_x, w_xy (3D) and w from HBM: per
// cell the kernel reads the averages (with halo) and writes q.
//
// The WENO arithmetic is weno1d on the same windows and the predictor is
// predictor_cell, so q is bitwise identical to the unfused path.
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"
#include "flux_point.cuh"
#include "launch.h"
#include "predictor.cuh"

namespace ader {

namespace {

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void record_error_pred(DevCounters* c, int code, long long cell) {
  if (atomicCAS(&c->err_code, 0, code) == 0) {
    c->err_stage = 1;
    c->err_cell = (unsigned long long)cell;
  }
}

template <int D, int M, int SYS>
struct WenoPred {
  using P = PredCfg<D, M, SYS, true>;   // one time level of f* scratch per cell
  static constexpr int NV = P::NV, N = M + 1, NS = P::NS, G = P::G, CPW = P::CPW;
  static constexpr int WARPS = 8, THREADS = WARPS * 32;
  static constexpr int TX = (D == 3) ? 4 : 16;
  static constexpr int TY = (D == 3) ? 4 : 1;
  static constexpr int CELLS = TX * TY;
  static constexpr int HX = TX + 2 * M;                       // slab extent in x
  static constexpr int HY = (D == 3) ? TY + 2 * M : 1;        // slab extent in y
  static constexpr int SLAB = HX * HY * NV;                   // cell averages of one level
  static constexpr int WXN = (D == 3) ? HY * TX * NV * N : 0; // x-sweep dofs of one level (3D)
  static constexpr int LV = ipow_c(N, D - 1);                 // dofs per variable before the last sweep
  static constexpr int NR = 2 * M + 1;                        // ring levels
  static constexpr int RING = NR * CELLS * NV * LV;
  static constexpr int WH = CELLS * NV * NS;                  // w of one level
  static constexpr int FS = WARPS * CPW * P::FSZ;
  static constexpr size_t smem_bytes() { return sizeof(double) * (2 * (size_t)SLAB + WXN + RING + WH + FS); }
  static_assert(smem_bytes() <= 227 * 1024, "shared memory of one CTA");
  static constexpr int MINB = (SYS == 0) ? 2 : 1;
};

template <int D, int M, int SYS>
__global__ void __launch_bounds__(WenoPred<D, M, SYS>::THREADS, WenoPred<D, M, SYS>::MINB)
    k_weno_predictor(const double* __restrict__ u, double* __restrict__ q, const Box R, const long long sy,
                     const long long sz, const long long qs, const double dtdx0, const double dtdx1,
                     const double dtdx2, const double gamma, const double ch, const double tol, const int max_sweeps,
                     DevCounters* __restrict__ cnt, const double* __restrict__ dtdx_dev, const int ntx, const int nty,
                     const int LS, const int nseg, const int ntiles, const __grid_constant__ DevTables T) {
  using C = WenoPred<D, M, SYS>;
  using PH = Phys<SYS, D>;
  constexpr int NV = C::NV, N = C::N, NS = C::NS, NST = NS * N, G = C::G, CPW = C::CPW;
  constexpr int TX = C::TX, TY = C::TY, HX = C::HX, HY = C::HY, CELLS = C::CELLS, LV = C::LV, NR = C::NR;
  constexpr int W = D - 1;
  extern __shared__ __align__(16) double smem[];
  double* slab = smem;                              // [2][HY][HX][NV]
  double* wx = slab + 2 * C::SLAB;                  // [HY][TX][NV][N]  (3D)
  double* ring = wx + C::WXN;                       // [NR][CELLS][NV][LV]
  double* wh = ring + C::RING;                      // [CELLS][NV][NS]
  double* fsm = wh + C::WH;                         // predictor scratch
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int slot = lane / G, node0 = lane - slot * G;
  PredLane<D, M, SYS> L;
  L.init(node0, T);
  double* Fs = fsm + (warp * CPW + slot) * C::P::FSZ;
  const double dtdx[3] = {dtdx_dev ? dtdx_dev[0] : dtdx0, dtdx_dev ? dtdx_dev[1] : dtdx1,
                          dtdx_dev ? dtdx_dev[2] : dtdx2};
  const long long sW = (D == 3) ? sz : sy;
  unsigned long long acc_sweeps = 0, acc_cells = 0;
  int acc_max = 0;

  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int tx = t % ntx;
    const int rest = t / ntx;
    const int ty = (D == 3) ? rest % nty : 0;
    const int seg = (D == 3) ? rest / nty : rest;
    const int x0 = R.lo[0] + tx * TX;
    const int nvx = min(TX, R.lo[0] + R.ext[0] - x0);
    const int y0 = (D == 3) ? R.lo[1] + ty * TY : 0;
    const int nvy = (D == 3) ? min(TY, R.lo[1] + R.ext[1] - y0) : 1;
    const int w0 = R.lo[W] + seg * LS;
    const int nvw = min(LS, R.lo[W] + R.ext[W] - w0);
    const int nsteps = nvw + 2 * M;
    // cell averages of level lv (tile + M halo in x and y) -> slab buffer b
    auto prefetch = [&](int lv, int b) {
      double* dst = slab + b * C::SLAB;
      const int hx = nvx + 2 * M, hy = (D == 3) ? nvy + 2 * M : 1;
      for (int i = tid; i < hx * hy * NV; i += C::THREADS) {
        const int v = i % NV, c = i / NV;
        const int xx = c % hx, yy = c / hx;
        const long long cell = (long long)(x0 - M + xx) + (D == 3 ? (long long)(y0 - M + yy) * sy : 0) +
                               (long long)lv * sW;
        cp_async8(dst + (yy * HX + xx) * NV + v, u + cell * NV + v);
      }
      cp_async_commit();
    };
    prefetch(w0 - M, 0);
    cp_async_wait_all();
    __syncthreads();
    for (int j = 0; j < nsteps; ++j) {
      const int lin = w0 - M + j;                   // level entering the ring
      const double* sl = slab + (j & 1) * C::SLAB;
      if (j + 1 < nsteps) prefetch(lin + 1, (j + 1) & 1);
      const int rs = ((lin % NR) + NR) % NR;
      double* rg = ring + rs * (CELLS * NV * LV);
      // ---- x sweep of level lin
      if constexpr (D == 3) {
        const int np = (nvy + 2 * M) * nvx * NV;
        for (int i = tid; i < np; i += C::THREADS) {
          const int v = i % NV, c = i / NV;
          const int xx = c % nvx, yy = c / nvx;
          double win[2 * M + 1], out[N];
#pragma unroll
          for (int o = 0; o <= 2 * M; ++o) win[o] = sl[(yy * HX + xx + o) * NV + v];
          weno1d<M>(T, win, out);
#pragma unroll
          for (int a = 0; a < N; ++a) wx[((yy * TX + xx) * NV + v) * N + a] = out[a];
        }
        __syncthreads();
        // ---- y sweep: new axis slowest, w_xy[v][ynode][xnode]
        const int nq = nvy * nvx * NV * N;
        for (int i = tid; i < nq; i += C::THREADS) {
          const int a = i % N, r = i / N;
          const int v = r % NV, c = r / NV;
          const int xx = c % nvx, yy = c / nvx;
          double win[2 * M + 1], out[N];
#pragma unroll
          for (int o = 0; o <= 2 * M; ++o) win[o] = wx[(((yy + o) * TX + xx) * NV + v) * N + a];
          weno1d<M>(T, win, out);
          double* d = rg + ((yy * TX + xx) * NV + v) * LV + a;
#pragma unroll
          for (int b = 0; b < N; ++b) d[b * N] = out[b];
        }
      } else {
        const int np = nvx * NV;
        for (int i = tid; i < np; i += C::THREADS) {
          const int v = i % NV, xx = i / NV;
          double win[2 * M + 1], out[N];
#pragma unroll
          for (int o = 0; o <= 2 * M; ++o) win[o] = sl[(xx + o) * NV + v];
          weno1d<M>(T, win, out);
#pragma unroll
          for (int a = 0; a < N; ++a) rg[(xx * NV + v) * LV + a] = out[a];
        }
      }
      __syncthreads();
      if (j >= 2 * M) {
        const int lout = lin - M;                   // level complete
        // ---- last sweep along W: w[v][a_W][t], t = previous dofs
        const int nq = nvy * nvx * NV * LV;
        for (int i = tid; i < nq; i += C::THREADS) {
          const int tt = i % LV, r = i / LV;
          const int v = r % NV, c = r / NV;
          const int xx = c % nvx, yy = c / nvx;
          const int cl = yy * TX + xx;
          double win[2 * M + 1], out[N];
#pragma unroll
          for (int o = 0; o <= 2 * M; ++o) {
            const int ls = (((lout - M + o) % NR) + NR) % NR;
            win[o] = ring[((ls * CELLS + cl) * NV + v) * LV + tt];
          }
          weno1d<M>(T, win, out);
          double* d = wh + (cl * NV + v) * NS + tt;
#pragma unroll
          for (int b = 0; b < N; ++b) d[b * LV] = out[b];
        }
        __syncthreads();
        // ---- predictor of the level's cells (lane group per cell)
        const int ncell = nvx * nvy;
        for (int cb = warp * CPW; cb < ncell; cb += C::WARPS * CPW) {
          const int cidx = cb + slot;
          const bool cell_ok = cidx < ncell;
          const int xx = cell_ok ? cidx % nvx : 0, yy = cell_ok ? cidx / nvx : 0;
          const int cl = yy * TX + xx;
          double wv[NV], qv[NV][N];
#pragma unroll
          for (int v = 0; v < NV; ++v) wv[v] = cell_ok ? wh[(cl * NV + v) * NS + L.node] : 1.0;
          bool conv, bad;
          int nsw;
          predictor_cell<D, M, SYS, true>(wv, qv, Fs, L, dtdx, cell_ok, gamma, ch, tol, max_sweeps, T, nsw, conv,
                                          bad);
          const long long cell = (long long)(x0 + xx) + (D == 3 ? (long long)(y0 + yy) * sy : 0) +
                                 (long long)lout * sW;
          if (cell_ok && L.lane_ok) {
            if (bad) record_error_pred(cnt, 1, cell);
            else if (!conv) record_error_pred(cnt, 2, cell);
            double* qo = q + cell * qs + L.node;
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
      }
      cp_async_wait_all();
      __syncthreads();
    }
  }
  // one set of counter atomics per warp
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
  (void)PH::NV;
}

template <int D, int M, int SYS>
void launch_weno_pred_t(const KCtx& k, const double* u, double* q, const Box& R, long long qs, const double dtdx[3],
                        double tol, int max_sweeps, DevCounters* cnt, const double* dtdx_dev) {
  using C = WenoPred<D, M, SYS>;
  auto kern = k_weno_predictor<D, M, SYS>;
  const size_t sm = C::smem_bytes();
  int dev = 0;
  cudaGetDevice(&dev);
  static int attr_dev_mask = 0;   // the attribute is per device
  if (!(attr_dev_mask & (1 << (dev & 31)))) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr_dev_mask |= 1 << (dev & 31);
  }
  constexpr int W = D - 1;
  const int ntx = (R.ext[0] + C::TX - 1) / C::TX;
  const int nty = (D == 3) ? (R.ext[1] + C::TY - 1) / C::TY : 1;
  int per_sm = 0, nsm = 148;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, sm);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (per_sm < 1) per_sm = 1;
  const int slots = per_sm * nsm;
  // segments along W: enough tiles for every CTA slot a few times over, but
  // segments of at least 8 levels (each segment re-enters 2M halo levels)
  int nseg = 1;
  while ((long long)ntx * nty * nseg < 4LL * slots && R.ext[W] / (nseg + 1) >= 8 * M) ++nseg;
  const int LS = (R.ext[W] + nseg - 1) / nseg;
  nseg = (R.ext[W] + LS - 1) / LS;
  const int ntiles = ntx * nty * nseg;
  const int g = ntiles < slots ? ntiles : slots;
  if (k.launches) ++*k.launches;
  kern<<<g, C::THREADS, sm, k.stream>>>(u, q, R, k.sy, k.sz, qs, dtdx[0], dtdx[1], dtdx[2], k.gamma, k.ch, tol,
                                        max_sweeps, cnt, dtdx_dev, ntx, nty, LS, nseg, ntiles, k.tab);
}

}  // namespace

void launch_weno_predictor(const KCtx& k, const double* u, double* q, const Box& R, long long qs, const double dtdx[3],
                           double tol, int max_sweeps, DevCounters* cnt, const double* dtdx_dev) {
  if (R.count() == 0) return;
#define ADER_WP(D_, M_, S_)                                                                   \
  if (k.D == D_ && k.M == M_ && k.SYS == S_) {                                                \
    launch_weno_pred_t<D_, M_, S_>(k, u, q, R, qs, dtdx, tol, max_sweeps, cnt, dtdx_dev); \
    return;                                                                                   \
  }
  ADER_WP(2, 2, 0) ADER_WP(2, 3, 0) ADER_WP(3, 2, 0) ADER_WP(2, 2, 1) ADER_WP(2, 3, 1) ADER_WP(3, 2, 1)
#undef ADER_WP
}

}  // namespace ader
