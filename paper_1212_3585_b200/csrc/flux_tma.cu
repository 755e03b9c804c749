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

template <int D, int M, int SYS, int LX>
struct FluxTma {
  static constexpr int NV = Phys<SYS, D>::NV, N = M + 1, NS = ipow_c(N, D);
  static constexpr int BLK = NV * NS * N;           // doubles per cell block
  static constexpr int QS = BLK + (BLK & 1);        // block stride: 16-byte aligned blocks
  static constexpr int G = (NS <= 8) ? 8 : (NS <= 16 ? 16 : 32);
  static constexpr int CPW = 32 / G;                // lane groups per warp
  static constexpr int WARPS = LX * D / CPW;
  static_assert((LX * D) % CPW == 0 && LX % CPW == 0, "a warp's lane groups share one direction");
  static constexpr int SEG = (LX + 1) + (D - 1) * LX;   // blocks per stage
  static constexpr int STAGE = SEG * QS;                // doubles per stage
  static constexpr int RED = NV * (G + 1);              // reduction buffer per lane group
  static constexpr size_t smem_bytes() {
    return sizeof(double) * (2 * (size_t)STAGE + (size_t)WARPS * CPW * RED) + 2 * sizeof(unsigned long long);
  }
};

constexpr int kFluxYC = 16;

template <int D, int M, int SYS, int FLUX, int LX, int MINB>
__global__ void __launch_bounds__(FluxTma<D, M, SYS, LX>::WARPS * 32, MINB)
    k_face_flux_tma(const double* __restrict__ q, double* __restrict__ F, const Box E, const int H, const int n0,
                    const int n1, const int n2, const long long sy, const long long sz, const long long ncell,
                    const double gamma, const double ch, const int bmask, const int rmask,
                    DevCounters* __restrict__ cnt, const unsigned nrx, const unsigned nruns,
                    const __grid_constant__ DevTables T) {
  using C = FluxTma<D, M, SYS, LX>;
  constexpr int NV = C::NV, N = C::N, NS = C::NS, NT = NS / N, QS = C::QS, G = C::G, CPW = C::CPW;
  extern __shared__ __align__(128) double smem[];
  double* red = smem + 2 * C::STAGE;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(red + C::WARPS * CPW * C::RED);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // geometry of run `run`: first cell x0, row (cy, cz), valid cells nval
  auto run_geom = [&](unsigned run, int& x0, int& cy, int& cz, int& nval) -> bool {
    const unsigned xr = run % nrx;
    const unsigned t = run / nrx;
    const int yi = (int)(t % kFluxYC);
    const unsigned t2 = t / kFluxYC;
    const unsigned ez = (unsigned)E.ext[2];
    const int y = (int)(t2 / ez) * kFluxYC + yi;
    if (y >= E.ext[1]) return false;
    cz = E.lo[2] + (int)(t2 % ez);
    cy = E.lo[1] + y;
    x0 = E.lo[0] + (int)xr * LX;
    nval = min(LX, E.lo[0] + E.ext[0] - x0);
    return true;
  };
  // producer (one thread): copy the rows of `run` into stage s
  auto issue = [&](unsigned run, int s) {
    unsigned long long* bar = bars + s;
    int x0, cy, cz, nval;
    if (run >= nruns || !run_geom(run, x0, cy, cz, nval)) {
      mbar_arrive_expect_tx(bar, 0u);
      return;
    }
    const long long c0 = (long long)x0 + cy * sy + cz * sz;
    double* sb = smem + s * C::STAGE;
    const unsigned own = (unsigned)((nval + 1) * QS * sizeof(double));
    const unsigned oth = (unsigned)(nval * QS * sizeof(double));
    mbar_arrive_expect_tx(bar, own + (D - 1) * oth);
    bulk_g2s(sb, q + (c0 - 1) * QS, own, bar);
    bulk_g2s(sb + (LX + 1) * QS, q + (c0 - sy) * QS, oth, bar);
    if constexpr (D == 3) bulk_g2s(sb + (2 * LX + 1) * QS, q + (c0 - sz) * QS, oth, bar);
  };

  if (tid == 0) {
    mbar_init(bars + 0, 1);
    mbar_init(bars + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    issue(blockIdx.x, 0);
    issue(blockIdx.x + gridDim.x, 1);
  }

  const int dir = warp % D;                       // warp-uniform face direction
  const int slot = lane / G, p = lane & (G - 1);
  const int ci = (warp / D) * CPW + slot;         // cell of the run
  const bool pok = p < NS;
  const int ps = pok ? p : 0;
  const int s_ = ps / NT, tt = ps - (ps / NT) * NT;
  double wt = T.w[s_] * T.w[tt % N];
  if (D == 3) wt *= T.w[tt / N];
  double* rb = red + (warp * CPW + slot) * C::RED;   // [NV][G+1]
  const int zH = (D == 3) ? H : 0;
  bool good = true;

  for (unsigned k = 0;; ++k) {
    const unsigned run = blockIdx.x + k * gridDim.x;
    if (run >= nruns) break;
    const int s = (int)(k & 1u);
    mbar_wait_parity(bars + s, (k >> 1) & 1u);
    int x0, cy, cz, nval;
    if (run_geom(run, x0, cy, cz, nval)) {
      const int cx = x0 + ci;
      const bool ok = ci < nval;
      const long long cR = ok ? (long long)cx + cy * sy + cz * sz : 0;
      const bool inx = cx < H + n0, iny = cy < H + n1, inz = (D == 2) || cz < zH + n2;
      const double* sb = smem + s * C::STAGE;
      const double* qR = sb + (ci + 1) * QS;
      double v[NV];
      bool face_ok;
      if (dir == 0) {
        face_ok = ok && iny && inz;
        good &= point_flux_blocks<D, M, SYS, 0, FLUX, false>(
            sb + ci * QS, qR, ps, face_ok && pok, (bmask & 1) && cx == H, (bmask & 2) && cx == H + n0,
            (rmask & 1) && cx == H, (rmask & 2) && cx == H + n0, wt, gamma, ch, T, v);
      } else if (dir == 1) {
        face_ok = ok && inx && inz;
        good &= point_flux_blocks<D, M, SYS, 1, FLUX, false>(
            sb + (LX + 1 + ci) * QS, qR, ps, face_ok && pok, (bmask & 4) && cy == H, (bmask & 8) && cy == H + n1,
            (rmask & 4) && cy == H, (rmask & 8) && cy == H + n1, wt, gamma, ch, T, v);
      } else {
        face_ok = ok && inx && iny;
        if constexpr (D == 3)
          good &= point_flux_blocks<D, M, SYS, D - 1, FLUX, false>(
              sb + (2 * LX + 1 + ci) * QS, qR, ps, face_ok && pok, (bmask & 16) && cz == zH,
              (bmask & 32) && cz == zH + n2, (rmask & 16) && cz == zH, (rmask & 32) && cz == zH + n2, wt, gamma,
              ch, T, v);
      }
      if (!good) {
        record_error_flux(cnt, cR);
        good = true;
      }
      // point sums in point order (the order of k_face_flux_cells)
      if (pok) {
#pragma unroll
        for (int i = 0; i < NV; ++i) rb[i * (G + 1) + p] = v[i];
      }
      __syncwarp();
      if (p < NV && face_ok) {
        const double* row = rb + p * (G + 1);
        double acc = row[0];
#pragma unroll
        for (int j = 1; j < NS; ++j) acc += row[j];
        F[((long long)dir * ncell + cR) * NV + p] = acc;
      }
      __syncwarp();
    }
    __syncthreads();   // every warp is done with stage s
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(run + 2 * gridDim.x, s);
    }
  }
}

template <int D, int M, int SYS, int FLUX, int LX, int MINB>
void launch_flux_tma_t(const KCtx& k, const double* q, double* F, const Box& E, int H, const int n[3], int bmask,
                       int rmask, DevCounters* cnt) {
  using C = FluxTma<D, M, SYS, LX>;
  auto kern = k_face_flux_tma<D, M, SYS, FLUX, LX, MINB>;
  const size_t sm = C::smem_bytes();
  int dev = 0;
  cudaGetDevice(&dev);
  static int attr_dev_mask = 0;   // the attribute is per device
  if (!(attr_dev_mask & (1 << (dev & 31)))) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr_dev_mask |= 1 << (dev & 31);
  }
  const unsigned nrx = (unsigned)((E.ext[0] + LX - 1) / LX);
  const unsigned ych = (unsigned)((E.ext[1] + kFluxYC - 1) / kFluxYC);
  const unsigned long long nruns = (unsigned long long)nrx * ych * kFluxYC * E.ext[2];
  if (nruns == 0 || nruns >= (1ull << 32)) return;
  int per_sm = 0, nsm = 148;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::WARPS * 32, sm);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (per_sm < 1) per_sm = 1;
  const unsigned long long cap = (unsigned long long)per_sm * nsm;
  const unsigned g = (unsigned)(nruns < cap ? nruns : cap);
  if (k.launches) ++*k.launches;
  kern<<<g, C::WARPS * 32, sm, k.stream>>>(q, F, E, H, n[0], n[1], n[2], k.sy, k.sz, k.ncell, k.gamma, k.ch,
                                           bmask, rmask, cnt, nrx, (unsigned)nruns, k.tab);
}

template <int D, int M, int SYS>
void flux_tma_for(const KCtx& k, const double* q, double* F, const Box& E, int H, const int n[3], int bmask,
                  int rmask, DevCounters* cnt) {
  // LX cells per run; MINB CTAs per SM the register budget is sized for
  constexpr int LX = (D == 3) ? 4 : 8;
  constexpr int MINB = (SYS == 1) ? 1 : 2;
  if constexpr (SYS == 0) {
    if (k.tab.flux == 1) {   // eqn.osher (Euler only, checked at ader_create)
      launch_flux_tma_t<D, M, SYS, 1, LX, 1>(k, q, F, E, H, n, bmask, rmask, cnt);
      return;
    }
  }
  launch_flux_tma_t<D, M, SYS, 0, LX, MINB>(k, q, F, E, H, n, bmask, rmask, cnt);
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
