// flux_rot.cu — a3 space-time face flux of the uniform path (flux:F/G/H @
// P:158-172 with eqn.rusanov @ P:181-185 or eqn.osher @ P:186-196): the face
// traces formed from COALESCED block loads and warp-shuffle line sums.
//
// Why: a face point needs, per variable, the N-term contraction of a cell
// block along the face normal (q_h at xi = 0 or 1).  k_face_flux_cells gathers
// the N nodes of that line per lane; whatever the in-block layout, the lanes
// of one such load are spread over a variable's whole N^(d+1) slab for two of
// the three normals, so each 8-byte load costs ~6 L1 wavefronts and the kernel
// is bound by the L1 data pipe (540 wavefronts per 3D cell, 91 %
// of the pipe at 0.30 of HBM).  Here
//   * lane p of a cell's lane group is the SPATIAL node p = i + N j + N^2 k and
//     loads q[v][s][p] for every time level s: the 27 (16, 9) lanes read
//     consecutive doubles, 2-3 wavefronts per load;
//   * lane p takes the face point (tangential nodes of p, time level
//     s(p) = (i + j + k) mod N) on the faces of ALL d normals: along any grid
//     line of the node lattice s takes every value once (a Latin cube), so the
//     N lanes of a line hold the N time levels of the N face points the line
//     feeds, one each;
//   * the line sum is a rotation: in round r = 1..N-1 a lane reads, from the
//     lane r nodes further along the line (cyclically), that node's value at
//     the reader's time level, already multiplied by the provider's psi —
//     the provider sends coef * V[(s_provider - r) mod N], which depends only
//     on the provider and r, not on the direction, so the rotated copy of V is
//     built once per variable and block and serves every normal.
// Per 3D cell: 3 block loads (own, -y, -z; the -x trace is carried along an
// x run of RL cells, the own block yields xi = 0 and xi = 1 along x) = 45
// coalesced loads and 120 32-bit shuffles instead of 90 strided gathers.
//
// The point flux (point_flux_states) is that of k_face_flux_cells; the traces
// differ from it in the order of their N products (rotated by the lane's line
// index) and the point sums run in node order instead of point order, i.e.
// both kernels agree up to rounding.  Each block is loaded one phase before
// its use (the -y block during the x face, the -z block during the y face, the
// next cell's block during the last face).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "flux_point.cuh"
#include "launch.h"

namespace ader {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void record_error(DevCounters* c, int code, int stage, long long cell) {
  if (atomicCAS(&c->err_code, 0, code) == 0) {
    c->err_stage = stage;
    c->err_cell = (unsigned long long)cell;
  }
}

// P[r] = V[(s - r) mod N], r = 0..N-1, by selects (no local memory)
template <int N>
__device__ __forceinline__ void rotate_by(const double (&V)[N], int s, double (&P)[N]) {
#pragma unroll
  for (int r = 0; r < N; ++r) {
    double x = V[(N - r) % N];   // s = 0
#pragma unroll
    for (int t = 1; t < N; ++t) x = (s == t) ? V[(t - r + N) % N] : x;
    P[r] = x;
  }
}

// sum over the lanes of this lane's line of coef(lane) * value at the reader's time level
template <int N>
__device__ __forceinline__ double line_sum(const double (&P)[N], double coef, const int (&src)[N]) {
  double acc = coef * P[0];
#pragma unroll
  for (int r = 1; r < N; ++r) acc += __shfl_sync(kFull, coef * P[r], src[r]);
  return acc;
}

template <int D, int M, int SYS, int WARPS, int FLUX, int RL, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB)
k_face_flux_rot(const double* __restrict__ q, double* __restrict__ F, const Box E, const int H, const int n0,
                const int n1, const int n2, const long long sy, const long long sz, const long long ncell,
                const double gamma, const double ch, const int bmask, const int rmask,
                DevCounters* __restrict__ cnt, const long long QSB, const unsigned nrx, const unsigned YC,
                const __grid_constant__ DevTables T) {
  using PH = Phys<SYS, D>;
  constexpr int NV = PH::NV, N = M + 1, NS = ipow_c(N, D), NT = NS / N, NST = NS * N;
  constexpr int G = (NS <= 8) ? 8 : (NS <= 16 ? 16 : 32);
  constexpr int CPW = 32 / G;
  constexpr int K = D * NV;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = lane & (G - 1);
  const bool pok = p < NS;
  const int pn = pok ? p : 0;
  int idx[3];
  idx[0] = pn % N;
  idx[1] = (pn / N) % N;
  idx[2] = (D == 3) ? pn / (N * N) : 0;
  const int s = (idx[0] + idx[1] + idx[2]) % N;
  // source lanes of the rotation rounds, per normal
  int src[D][N];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    src[d][0] = lane;
#pragma unroll
    for (int r = 1; r < N; ++r) {
      const int nn = (idx[d] + r) % N;
      src[d][r] = pok ? lane + (nn - idx[d]) * ipow_c(N, d) : lane;
    }
  }
  // provider coefficients: psi(0) and psi(1) at the lane's node along each normal
  double c0[D], c1[D];
#pragma unroll
  for (int d = 0; d < D; ++d) { c0[d] = T.psi0[idx[d]]; c1[d] = T.psi1[idx[d]]; }
  // quadrature weight of this lane's face point on the face normal to d
  // (time level s, tangential nodes of p)
  double wt[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const int a0 = (d == 0) ? 1 : 0, a1 = (d == 2) ? 1 : 2;
    const int t1 = idx[a0], t2 = (D == 3) ? idx[a1] : 0;
    double w = T.w[s] * T.w[t1];
    if (D == 3) w *= T.w[t2];
    wt[d] = w;
  }
  // run of RL cells along x (32-bit index decomposition, the launcher
  // guarantees < 2^32 runs): x run fastest, then y inside chunks of YC rows,
  // then z, then the chunk (the -y / -z blocks were read a few MB earlier)
  const unsigned r = (blockIdx.x * WARPS + warp) * CPW + lane / G;
  const unsigned ez = (unsigned)E.ext[2];
  const unsigned t = r / nrx;
  const int x0 = (int)(r - t * nrx) * RL;
  const unsigned t2 = t / YC;
  const int yi = (int)(t - t2 * YC);
  const unsigned yb = t2 / ez;
  const int z = (int)(t2 - yb * ez);
  const int y = (int)(yb * YC + yi);
  const bool rowok = y < E.ext[1];
  const int cy = E.lo[1] + y, cz = E.lo[2] + z;
  const int zH = (D == 3) ? H : 0;
  const bool iny = cy < H + n1, inz = (D == 2) || cz < zH + n2;
  const long long BLK = QSB;

  __shared__ double red[WARPS * CPW][K][G + 1];
  double(*rb)[G + 1] = red[warp * CPW + lane / G];

  // a valid cell whose lower neighbours exist, read (and discarded) by lane groups without a cell
  const long long cS = E.lo[0] + E.lo[1] * sy + E.lo[2] * sz;
  auto cell_of = [&](int c) -> long long {
    const int x = x0 + c;
    return (rowok && x < E.ext[0]) ? (E.lo[0] + x) + cy * sy + cz * sz : cS;
  };
  auto load_block = [&](const double* qb, double (&V)[NV][N]) {
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int k = 0; k < N; ++k) V[v][k] = __ldg(qb + v * NST + k * NS + pn);
  };
  // xi = 1 trace along DIR of a loaded block (the lower cell's side of a face)
  auto upper_trace = [&](const double (&V)[NV][N], const int dir, double (&a)[NV]) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double P[N];
      rotate_by<N>(V[v], s, P);
      if (dir == 0) a[v] = line_sum<N>(P, c1[0], src[0]);
      else if (dir == 1) a[v] = line_sum<N>(P, c1[1], src[1]);
      else a[v] = line_sum<N>(P, c1[D - 1], src[D - 1]);
    }
  };
  auto put = [&](int row0, bool fok, const double (&val)[NV]) {
    if (pok) {
#pragma unroll
      for (int v = 0; v < NV; ++v) rb[row0 + v][p] = fok ? val[v] : 0.0;
    }
  };

  double ax[NV];        // xi = 1 trace along x of the previous cell of the run
  double Vn[NV][N];     // block in flight: loaded one phase before its use
  {
    const long long c0R = cell_of(0);
    load_block(q + (c0R - 1) * BLK, Vn);
    upper_trace(Vn, 0, ax);
    load_block(q + c0R * BLK, Vn);
  }

#pragma unroll 1
  for (int c = 0; c < RL; ++c) {
    const int x = x0 + c;
    const bool ok = rowok && x < E.ext[0];
    const int cx = E.lo[0] + x;
    const long long cR = ok ? cx + cy * sy + cz * sz : cS;
    const bool inx = cx < H + n0;
    // own block (in Vn): xi = 0 traces along every normal, xi = 1 along x for the next cell
    double b[D][NV], axn[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double P[N];
      rotate_by<N>(Vn[v], s, P);
#pragma unroll
      for (int d = 0; d < D; ++d) b[d][v] = line_sum<N>(P, c0[d], src[d]);
      axn[v] = line_sum<N>(P, c1[0], src[0]);
    }
    load_block(q + (cR - sy) * BLK, Vn);   // -y block, in flight during the x face
    bool good = true;
    double val[NV];
    {
      const bool fok = ok && iny && inz && pok;
      if (fok)
        good &= point_flux_states<D, SYS, 0, FLUX>(ax, b[0], (bmask & 1) && cx == H, (bmask & 2) && cx == H + n0,
                                                   (rmask & 1) && cx == H, (rmask & 2) && cx == H + n0, wt[0],
                                                   gamma, ch, T, val);
      put(0, fok, val);
#pragma unroll
      for (int v = 0; v < NV; ++v) ax[v] = axn[v];
    }
    {
      double a[NV];
      upper_trace(Vn, 1, a);
      if constexpr (D == 3) load_block(q + (cR - sz) * BLK, Vn);   // -z block, in flight during the y face
      else if (c + 1 < RL) load_block(q + cell_of(c + 1) * BLK, Vn);   // next own block
      const bool fok = ok && inx && inz && pok;
      if (fok)
        good &= point_flux_states<D, SYS, 1, FLUX>(a, b[1], (bmask & 4) && cy == H, (bmask & 8) && cy == H + n1,
                                                   (rmask & 4) && cy == H, (rmask & 8) && cy == H + n1, wt[1],
                                                   gamma, ch, T, val);
      put(NV, fok, val);
    }
    if constexpr (D == 3) {
      double a[NV];
      upper_trace(Vn, 2, a);
      if (c + 1 < RL) load_block(q + cell_of(c + 1) * BLK, Vn);   // next own block, in flight during the z face
      const bool fok = ok && inx && iny && pok;
      if (fok)
        good &= point_flux_states<D, SYS, 2, FLUX>(a, b[D - 1], (bmask & 16) && cz == zH,
                                                   (bmask & 32) && cz == zH + n2, (rmask & 16) && cz == zH,
                                                   (rmask & 32) && cz == zH + n2, wt[D - 1], gamma, ch, T, val);
      put(2 * NV, fok, val);
    }
    if (!good) record_error(cnt, 1, 2, cR);
    // point sums in a fixed (node) order: lane i sums row i
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

template <int D, int M, int SYS, int FLUX, int RL, int MINB>
void launch_rot(const KCtx& k, const double* q, double* F, const Box& E, int H, const int n[3], int bmask, int rmask,
                DevCounters* cnt, long long qs, int yc) {
  constexpr int WARPS = 4;
  constexpr int NS = ipow_c(M + 1, D);
  constexpr int CPW = 32 / ((NS <= 8) ? 8 : (NS <= 16 ? 16 : 32));
  const unsigned nrx = (unsigned)((E.ext[0] + RL - 1) / RL);
  if (k.launches) ++*k.launches;
  const long long ych = (E.ext[1] + yc - 1) / yc;
  const long long groups = (long long)nrx * ych * yc * E.ext[2];
  const unsigned g = (unsigned)((groups + WARPS * CPW - 1) / (WARPS * CPW));
  k_face_flux_rot<D, M, SYS, WARPS, FLUX, RL, MINB><<<g, WARPS * 32, 0, k.stream>>>(
      q, F, E, H, n[0], n[1], n[2], k.sy, k.sz, k.ncell, k.gamma, k.ch, bmask, rmask, cnt, qs, nrx, (unsigned)yc,
      k.tab);
}

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return (e && e[0]) ? std::atoi(e) : dflt;
}

template <int D, int M, int SYS, int FLUX>
void rot_variant(const KCtx& k, const double* q, double* F, const Box& E, int H, const int n[3], int bmask, int rmask,
                 DevCounters* cnt, long long qs) {
  // A/B knobs: rows per y chunk, CTAs per SM the register budget is set for (3: 168 registers,
  // no spills at D = 3; 4: 128 registers)
  static const int yc = env_int("ADER_FLUX_YC", 16) > 0 ? env_int("ADER_FLUX_YC", 16) : 16;
  static const int mb = env_int("ADER_FLUX_MINB", D == 3 ? 3 : 4);
  if (mb >= 4) launch_rot<D, M, SYS, FLUX, 8, 4>(k, q, F, E, H, n, bmask, rmask, cnt, qs, yc);
  else launch_rot<D, M, SYS, FLUX, 8, 3>(k, q, F, E, H, n, bmask, rmask, cnt, qs, yc);
}

}  // namespace

void launch_face_flux_rot(const KCtx& k, const double* q, double* F, const Box& ext, int H, const int n[3], int bmask,
                          int rmask, DevCounters* cnt, long long qs) {
  if (ext.count() == 0) return;
#define ADER_FR(D_, M_, S_)                                                                         \
  if (k.D == D_ && k.M == M_ && k.SYS == S_) {                                                      \
    if (S_ == 0 && k.tab.flux == 1) rot_variant<D_, M_, S_, (S_ == 0 ? 1 : 0)>(k, q, F, ext, H, n, bmask, rmask, cnt, qs); \
    else rot_variant<D_, M_, S_, 0>(k, q, F, ext, H, n, bmask, rmask, cnt, qs);                     \
    return;                                                                                         \
  }
  ADER_FR(2, 2, 0) ADER_FR(2, 3, 0) ADER_FR(3, 2, 0) ADER_FR(2, 2, 1) ADER_FR(2, 3, 1) ADER_FR(3, 2, 1)
#undef ADER_FR
}

}  // namespace ader
