// flux_tma.cu — a3 space-time face flux of the uniform path (flux:F/G/H @
// P:158-172 with eqn.rusanov @ P:181-185 or eqn.osher @ P:186-196), with the
// predictor blocks streamed into shared memory by the Blackwell bulk-copy
// engine (cp.async.bulk + mbarrier transaction counts).
//
// Why: every face point needs, per variable, an N-term contraction of one
// cell block along the face normal (the trace q_h at xi = 0 or 1).  Read
// straight from global memory those loads are 8-byte gathers with a stride of
// N^dir doubles, so one warp load touches ~7 L1 lines and the round-1 kernel
// ran at 0.30 of HBM bandwidth, bound by L1 wavefronts.  A cell's block is a
// contiguous [nu][N^(d+1)] array and a run of cells along x is a contiguous
// range of blocks, so a CTA copies, per run of LX cells at (y, z):
//   own row  cells x0-1 .. x0+LX-1  (LX+1 blocks: the cells and their -x neighbour)
//   -y row   cells x0   .. x0+LX-1  (one block per cell)
//   -z row   cells x0   .. x0+LX-1  (3D)
// with one bulk copy per row into a stage of a two-stage ring, and the trace
// contractions read shared memory.  The block stride QS is the block size
// rounded up to an even number of doubles, so every block starts 16-byte
// aligned (the bulk copy's requirement).
//
// Work split: a lane group of G >= N^d lanes (one lane per space-time point of
// a face) computes ONE face (dir) of one cell; the warps of a CTA cover the LX
// cells x d directions of a run, with dir uniform per warp.  The point
// arithmetic (point_flux_blocks) and the order of the point sums are those of
// k_face_flux_cells, so both kernels produce bitwise-identical F.
// Runs are visited x-run fastest, then y inside chunks of YC rows, then z, then
// the chunk (as the round-1 kernel), so the -y and -z rows a CTA copies were
// copied as own rows a few MB earlier by another CTA and come from L2.
#include <cuda_runtime.h>

#include <cstdint>

#include "flux_point.cuh"
#include "launch.h"

namespace ader {

namespace {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// arrive (count 1) and add `bytes` to the transaction count of the current phase
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      " .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (16-byte aligned, size a multiple of 16) that
// completes `bytes` transactions on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void record_error_flux(DevCounters* c, long long cell) {
  if (atomicCAS(&c->err_code, 0, 1) == 0) {   // 1 = inadmissible state, stage 2 = face flux
    c->err_stage = 2;
    c->err_cell = (unsigned long long)cell;
  }
}

// Tile walk: a CTA owns a tile of TX x TY cells (3D: x, y; 2D: TX cells along
// x, TY = 1) and walks it along the last axis W (z in 3D, y in 2D).  Per step
// (one level w) it copies the tile's rows plus the -x column and (3D) the -y row
// into a stage of a three-stage ring: TY+1 rows (3D; 1 row in 2D) of TX+1
// consecutive blocks, one bulk copy per row.  The -W neighbour is the previous
// level: its upper-W traces were computed one step earlier and are carried in
// shared memory, so no block is copied twice along W.  Step 0 of a tile loads
// the level below the first face level and only computes those traces.
template <int D, int M, int SYS>
struct FluxWalk {
  static constexpr int NV = Phys<SYS, D>::NV, N = M + 1, NS = ipow_c(N, D);
  static constexpr int BLK = NV * NS * N;           // doubles per cell block
  static constexpr int QS = BLK + (BLK & 1);        // block stride: 16-byte aligned blocks
  static constexpr int G = (NS <= 8) ? 8 : (NS <= 16 ? 16 : 32);
  static constexpr int CPW = 32 / G;                // lane groups per warp
  static constexpr int TX = (D == 3) ? (SYS == 1 ? 2 : 4) : 8;
  static constexpr int TY = (D == 3) ? 2 : 1;
  static constexpr int CELLS = TX * TY;
  static constexpr int GROUPS = CELLS * D;          // (cell, face dir) lane groups
  static constexpr int WARPS = GROUPS / CPW;
  static_assert(CELLS % CPW == 0, "a warp's lane groups share one direction");
  static constexpr int ROWS = (D == 3) ? TY + 1 : 1;
  static constexpr int RB = TX + 1;                 // blocks per row
  static constexpr int NSTAGE = 3;
  static constexpr int STAGE = ROWS * RB * QS;      // doubles per stage
  static constexpr int TRC = CELLS * NV * NS;       // carried upper-W traces of one level
  static constexpr int RED = NV * (G + 1);          // point-sum buffer per lane group
  static constexpr int K = (G / NV) < 1 ? 1 : (G / NV);   // partial sums per variable
  static constexpr int CH = (NS + K - 1) / K;             // points per partial sum
  static constexpr size_t smem_bytes() {
    return sizeof(double) * ((size_t)NSTAGE * STAGE + 2 * (size_t)TRC + (size_t)GROUPS * RED) +
           NSTAGE * sizeof(unsigned long long);
  }
  static_assert(smem_bytes() <= 227 * 1024, "shared memory of one CTA");
  static constexpr int MINB = (D == 3) ? 1 : 2;     // CTAs per SM the registers are sized for
};

template <int D, int M, int SYS, int FLUX>
__global__ void __launch_bounds__(FluxWalk<D, M, SYS>::WARPS * 32, FluxWalk<D, M, SYS>::MINB)
    k_face_flux_walk(const double* __restrict__ q, double* __restrict__ F, const Box E, const int H, const int n0,
                     const int n1, const int n2, const long long sy, const long long sz, const long long ncell,
                     const double gamma, const double ch, const int bmask, const int rmask,
                     DevCounters* __restrict__ cnt, const int ntx, const int nty, const int ntiles,
                     const __grid_constant__ DevTables T) {
  using C = FluxWalk<D, M, SYS>;
  constexpr int NV = C::NV, N = C::N, NS = C::NS, NT = NS / N, QS = C::QS, G = C::G, CPW = C::CPW;
  constexpr int TX = C::TX, TY = C::TY, RB = C::RB, W = D - 1;
  extern __shared__ __align__(128) double smem[];
  double* trc = smem + C::NSTAGE * C::STAGE;              // [2][CELLS][NV][NS]
  double* red = trc + 2 * C::TRC;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(red + C::GROUPS * C::RED);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nsteps = E.ext[W] + 1;                        // + the level below the first face level
  const long long ssW = (D == 3) ? sz : sy;               // stride along W
  const long long total = (long long)((ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x) * nsteps;

  // tile t: tiles are numbered in patches of 12 x 12 (x fastest inside a patch,
  // patches row by row, partial patches at the edges), so the tiles a round of
  // CTAs walks together are compact and the halo rows / columns they copy from
  // each other stay in L2
  auto tile_xy = [&](int t, int& tx, int& ty) {
    const int pyi = t / (12 * ntx);
    const int hy = min(12, nty - 12 * pyi);
    const int r = t - pyi * 12 * ntx;
    const int pxi = r / (12 * hy);
    const int r2 = r - pxi * 12 * hy;
    const int wx = min(12, ntx - 12 * pxi);
    tx = 12 * pxi + r2 % wx;
    ty = 12 * pyi + r2 / wx;
  };
  // geometry of CTA step g: tile origin, valid extent, level
  auto geom = [&](long long g, int& x0, int& y0, int& nvx, int& nvy, int& k) -> bool {
    const int it = (int)(g / nsteps);
    k = (int)(g - (long long)it * nsteps);
    int tx, ty;
    tile_xy((int)blockIdx.x + it * (int)gridDim.x, tx, ty);
    if (ty >= nty) return false;
    x0 = E.lo[0] + tx * TX;
    nvx = min(TX, E.lo[0] + E.ext[0] - x0);
    if (D == 3) {
      y0 = E.lo[1] + ty * TY;
      nvy = min(TY, E.lo[1] + E.ext[1] - y0);
    } else {
      y0 = 0;
      nvy = 1;
    }
    return true;
  };
  // producer: the rows of step g into stage s
  auto issue = [&](long long g, int s) {
    unsigned long long* bar = bars + s;
    int x0, y0, nvx, nvy, k;
    if (g >= total || !geom(g, x0, y0, nvx, nvy, k)) {
      mbar_arrive_expect_tx(bar, 0u);
      return;
    }
    const int w = E.lo[W] - 1 + k;                       // level of this step
    double* sb = smem + s * C::STAGE;
    const unsigned rowb = (unsigned)((nvx + 1) * QS * sizeof(double));
    if constexpr (D == 3) {
      mbar_arrive_expect_tx(bar, rowb * (unsigned)(nvy + 1));
      for (int r = 0; r <= nvy; ++r) {
        const long long c0 = (long long)(x0 - 1) + (long long)(y0 - 1 + r) * sy + (long long)w * sz;
        bulk_g2s(sb + r * RB * QS, q + c0 * QS, rowb, bar);
      }
    } else {
      mbar_arrive_expect_tx(bar, rowb);
      bulk_g2s(sb, q + ((long long)(x0 - 1) + (long long)w * sy) * QS, rowb, bar);
    }
  };

  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < C::NSTAGE; ++i) mbar_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int i = 0; i < C::NSTAGE; ++i) issue(i, i);

  // lane group: (cell ci, face dir); dir uniform per warp
  const int grp = warp * CPW + lane / G;
  const int dir = grp / C::CELLS;
  const int ci = grp - dir * C::CELLS;
  const int cxi = ci % TX, cyi = ci / TX;
  const int p = lane & (G - 1);
  const bool pok = p < NS;
  const int ps = pok ? p : 0;
  const int s_ = ps / NT, tt = ps - (ps / NT) * NT;
  double wt = T.w[s_] * T.w[tt % N];
  if (D == 3) wt *= T.w[tt / N];
  double* rb = red + grp * C::RED;                        // [NV][G+1]
  const int zH = (D == 3) ? H : 0;
  const int lvl_hi = (D == 3) ? zH + n2 : H + n1;          // last face level along W

  for (long long g = 0; g < total; ++g) {
    const int s = (int)(g % C::NSTAGE);
    mbar_wait_parity(bars + s, (unsigned)((g / C::NSTAGE) & 1));
    int x0, y0, nvx, nvy, k;
    if (geom(g, x0, y0, nvx, nvy, k)) {
      const double* sb = smem + s * C::STAGE;
      const int w = E.lo[W] - 1 + k;
      const bool cell_in = cxi < nvx && cyi < nvy;
      const int cx = x0 + cxi, cy = (D == 3) ? y0 + cyi : w, cz = (D == 3) ? w : 0;
      const int row = (D == 3) ? cyi + 1 : 0;
      const double* qown = sb + (row * RB + cxi + 1) * QS;
      double* tw = trc + (k & 1) * C::TRC + ci * NV * NS;          // this level's upper-W traces
      const double* tr = trc + ((k + 1) & 1) * C::TRC + ci * NV * NS;   // the level below
      if (k == 0) {
        // the level below the first face level: its upper-W traces only
        if (dir == W && cell_in && pok) {
          double a[NV];
          face_trace<D, M, NV, W, false>(qown, ps, T.psi1, a);
#pragma unroll
          for (int v = 0; v < NV; ++v) tw[v * NS + ps] = a[v];
        }
      } else if (cell_in) {
        const long long cR = (long long)cx + cy * sy + (long long)cz * sz;
        const bool inx = cx < H + n0, iny = cy < H + n1, inz = (D == 2) || cz < zH + n2;
        double v[NV];
        bool face_ok, good = true;
        if (dir == 0) {
          face_ok = iny && inz;
          good = point_flux_blocks<D, M, SYS, 0, FLUX, false>(
              qown - QS, qown, ps, face_ok && pok, (bmask & 1) && cx == H, (bmask & 2) && cx == H + n0,
              (rmask & 1) && cx == H, (rmask & 2) && cx == H + n0, wt, gamma, ch, T, v);
        } else if (D == 3 && dir == 1) {
          face_ok = inx && inz;
          good = point_flux_blocks<D, M, SYS, (D == 3 ? 1 : 0), FLUX, false>(
              qown - RB * QS, qown, ps, face_ok && pok, (bmask & 4) && cy == H, (bmask & 8) && cy == H + n1,
              (rmask & 4) && cy == H, (rmask & 8) && cy == H + n1, wt, gamma, ch, T, v);
        } else {
          // the W face: lower side = carried upper trace of the level below;
          // then this level's upper traces for the next step
          face_ok = (D == 3) ? (inx && iny) : inx;
          const bool tlo = (bmask & (1 << (2 * W))) && w == (D == 3 ? zH : H);
          const bool thi = (bmask & (2 << (2 * W))) && w == lvl_hi;
          const bool rlo = (rmask & (1 << (2 * W))) && w == (D == 3 ? zH : H);
          const bool rhi = (rmask & (2 << (2 * W))) && w == lvl_hi;
#pragma unroll
          for (int i = 0; i < NV; ++i) v[i] = 0.0;
          if (pok) {
            double a[NV], b[NV];
            face_trace<D, M, NV, W, false>(qown, ps, T.psi1, a);   // this level's upper trace first
#pragma unroll
            for (int i = 0; i < NV; ++i) tw[i * NS + ps] = a[i];
#pragma unroll
            for (int i = 0; i < NV; ++i) a[i] = tr[i * NS + ps];
            face_trace<D, M, NV, W, false>(qown, ps, T.psi0, b);
            if (face_ok) good = point_flux_states<D, SYS, W, FLUX>(a, b, tlo, thi, rlo, rhi, wt, gamma, ch, T, v);
          }
        }
        if (!good) record_error_flux(cnt, cR);
        // point sums: K partial sums of CH consecutive points per variable,
        // then the K partials in order (fixed order: deterministic)
        if (pok) {
#pragma unroll
          for (int i = 0; i < NV; ++i) rb[i * (G + 1) + p] = v[i];
        }
        __syncwarp(__activemask());
        double part = 0.0;
        const int var = p / C::K, chunk = p - var * C::K;
        if (var < NV) {
          const double* row = rb + var * (G + 1);
          const int j0 = chunk * C::CH, j1 = min(NS, j0 + C::CH);
          if (j0 < j1) {
            part = row[j0];
            for (int j = j0 + 1; j < j1; ++j) part += row[j];
          }
        }
        // gather the partials of each variable in lane var*K (lanes of this group)
        const int gbase = lane & ~(G - 1);
        double acc = part;
#pragma unroll
        for (int c = 1; c < C::K; ++c) {
          const double o = __shfl_sync(__activemask(), part, gbase + (var < NV ? var : 0) * C::K + c);
          acc += o;
        }
        if (var < NV && chunk == 0 && face_ok) F[((long long)dir * ncell + cR) * NV + var] = acc;
        __syncwarp(__activemask());
      }
    }
    __syncthreads();   // every warp is done with stage s (and with the traces of level k-1)
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(g + C::NSTAGE, s);
    }
  }
}

template <int D, int M, int SYS, int FLUX>
void launch_flux_walk_t(const KCtx& k, const double* q, double* F, const Box& E, int H, const int n[3], int bmask,
                        int rmask, DevCounters* cnt) {
  using C = FluxWalk<D, M, SYS>;
  auto kern = k_face_flux_walk<D, M, SYS, FLUX>;
  const size_t sm = C::smem_bytes();
  int dev = 0;
  cudaGetDevice(&dev);
  static int attr_dev_mask = 0;   // the attribute is per device
  if (!(attr_dev_mask & (1 << (dev & 31)))) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr_dev_mask |= 1 << (dev & 31);
  }
  const int ntx = (E.ext[0] + C::TX - 1) / C::TX;
  const int nty = (D == 3) ? (E.ext[1] + C::TY - 1) / C::TY : 1;
  const int ntiles = ntx * nty;
  int per_sm = 0, nsm = 148;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::WARPS * 32, sm);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (per_sm < 1) per_sm = 1;
  const int cap = per_sm * nsm;
  const int g = ntiles < cap ? ntiles : cap;
  if (k.launches) ++*k.launches;
  kern<<<g, C::WARPS * 32, sm, k.stream>>>(q, F, E, H, n[0], n[1], n[2], k.sy, k.sz, k.ncell, k.gamma, k.ch, bmask,
                                           rmask, cnt, ntx, nty, ntiles, k.tab);
}

template <int D, int M, int SYS>
void flux_tma_for(const KCtx& k, const double* q, double* F, const Box& E, int H, const int n[3], int bmask,
                  int rmask, DevCounters* cnt) {
  if constexpr (SYS == 0) {
    if (k.tab.flux == 1) {   // eqn.osher (Euler only, checked at ader_create)
      launch_flux_walk_t<D, M, SYS, 1>(k, q, F, E, H, n, bmask, rmask, cnt);
      return;
    }
  }
  launch_flux_walk_t<D, M, SYS, 0>(k, q, F, E, H, n, bmask, rmask, cnt);
}

}  // namespace

long long q_block_stride(int D, int M, int SYS) {
  long long nv = SYS == 1 ? 9 : D + 2, blk = nv;
  for (int i = 0; i < D + 1; ++i) blk *= M + 1;
  return blk + (blk & 1);
}

void launch_face_flux_tma(const KCtx& k, const double* q, double* F, const Box& ext, int H, const int n[3],
                          int bmask, int rmask, DevCounters* cnt) {
  if (ext.count() == 0) return;
#define ADER_FT(D_, M_, S_) \
  if (k.D == D_ && k.M == M_ && k.SYS == S_) { flux_tma_for<D_, M_, S_>(k, q, F, ext, H, n, bmask, rmask, cnt); return; }
  ADER_FT(2, 2, 0) ADER_FT(2, 3, 0) ADER_FT(3, 2, 0) ADER_FT(2, 2, 1) ADER_FT(2, 3, 1) ADER_FT(3, 2, 1)
#undef ADER_FT
}

}  // namespace ader
