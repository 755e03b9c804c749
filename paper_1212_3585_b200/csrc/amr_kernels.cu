// amr_kernels.cu — sm_100a kernels of the AMR / local-time-stepping path.
//   k_amr_average   averaging of virtual mothers (eqn.average @ P:743-753)
//   k_amr_project   projection of the mother's q_h into virtual children
//   k_amr_weno      dimension-by-dimension WENO of a listed active cell
//   k_predictor     (kernels.cu, list mode) space-time predictor
//   k_amr_flux_w + k_amr_update_w face fluxes incl. coarse-fine faces with flux memory, update
//                   (eqn.memory.sum) + one-step update (eq:finite_vol)
//   k_amr_indicator refinement indicator, reading R14 of eqn.indicator,
//                   evaluated without FMA contraction (bit-exact flags, H2)
// Citations: P:n = PAPER.md line n.
#include <cuda_runtime.h>

#include "amr.h"
#include "device.cuh"

namespace ader {

constexpr int ipow_a(int b, int e) { return e == 0 ? 1 : b * ipow_a(b, e - 1); }

// same-level cell at a (possibly out-of-domain) index: periodic wrap,
// transmissive clamp (R5) or reflective mirror (R22; bit k of *flip set: the
// caller negates the momentum along k)
__device__ __forceinline__ int amr_lookup_flip(const AmrDevView& V, int l, long long x, long long y, long long z,
                                               int* flip) {
  long long c[3] = {x, y, z};
  int fl = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (k >= V.D) { c[k] = 0; continue; }
    const long long n = V.n[l][k];
    if (c[k] < 0 || c[k] >= n) {
      const int side = c[k] < 0 ? 0 : 1;
      const int bc = V.bc[2 * k + side];
      if (bc == ADER_BC_PERIODIC) c[k] = ((c[k] % n) + n) % n;
      else if (bc == ADER_BC_REFLECTIVE) { c[k] = c[k] < 0 ? -1 - c[k] : 2 * n - 1 - c[k]; fl |= 1 << k; }
      else c[k] = c[k] < 0 ? 0 : n - 1;
    }
  }
  if (flip) *flip = fl;
  return V.map[l][(c[2] * V.n[l][1] + c[1]) * V.n[l][0] + c[0]];
}
__device__ __forceinline__ int amr_lookup(const AmrDevView& V, int l, long long x, long long y, long long z) {
  return amr_lookup_flip(V, l, x, y, z, nullptr);
}
// cell average component v seen through a (possibly reflecting) lookup
__device__ __forceinline__ double amr_u_at(const AmrDevView& V, int l, long long x, long long y, long long z, int v) {
  int fl = 0;
  const int id = amr_lookup_flip(V, l, x, y, z, &fl);
  const double a = V.u[(long long)id * V.NV + v];
  return (v >= 1 && v <= V.D && ((fl >> (v - 1)) & 1)) ? -a : a;
}

// row of a cell in w / q: its slot on a multi-rank context (R28), else its id
__device__ __forceinline__ long long wq_row(const AmrDevView& V, int id) { return V.slot ? (long long)V.slot[id] : id; }

__device__ __forceinline__ void amr_error(DevCounters* c, int code, int stage, long long cell) {
  if (atomicCAS(&c->err_code, 0, code) == 0) {
    c->err_stage = stage;
    c->err_cell = (unsigned long long)cell;
  }
}

// ---------------------------------------------------------------------------
__global__ void k_amr_average(AmrDevView V, const int* __restrict__ list, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * V.NV) return;
  const int m = list[i / V.NV], v = i % V.NV;
  const int ch = V.child[m];
  double s = 0.0;
  for (int q = 0; q < V.rd; ++q) s += V.u[(long long)(ch + q) * V.NV + v];
  V.u[(long long)m * V.NV + v] = s / (double)V.rd;
}

// sub-box average of the mother's polynomial (mode 0: WENO w, 1: q_h at tau)
template <int D, int M>
__device__ __forceinline__ double subbox(const AmrDevView& V, const SubTables& S, int cell, int mom, int v, int mode,
                                         const double* psi_tau) {
  constexpr int N = M + 1, NS = ipow_a(N, D), NST = NS * N;
  int off[3] = {0, 0, 0};
#pragma unroll
  for (int k = 0; k < D; ++k) off[k] = (int)(V.idx[(long long)cell * 3 + k] - V.idx[(long long)mom * 3 + k] * V.r);
  double acc = 0.0;
  if (mode == 0) {
    const double* w = V.w + (wq_row(V, mom) * V.NV + v) * NS;
#pragma unroll
    for (int p = 0; p < NS; ++p) {
      double c = S.Psub[off[0]][p % N] * S.Psub[off[1]][(p / N) % N];
      if (D == 3) c *= S.Psub[off[2]][p / (N * N)];
      acc += c * w[p];
    }
  } else {
    const double* q = V.q + (wq_row(V, mom) * V.NV + v) * NST;
    for (int p = 0; p < NST; ++p) {
      const int sp = p % NS, s = p / NS;
      double c = S.Psub[off[0]][sp % N] * S.Psub[off[1]][(sp / N) % N];
      if (D == 3) c *= S.Psub[off[2]][sp / (N * N)];
      acc += (c * psi_tau[s]) * q[p];
    }
  }
  return acc;
}

template <int D, int M>
__global__ void k_amr_project(AmrDevView V, const __grid_constant__ SubTables S, const int* __restrict__ list, int n,
                              double t0, double t1, double t2, double t3) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * V.NV) return;
  const int c = list[i / V.NV], v = i % V.NV;
  const double psi_tau[4] = {t0, t1, t2, t3};
  V.u[(long long)c * V.NV + v] = subbox<D, M>(V, S, c, V.mother[c], v, 1, psi_tau);
}

template <int D, int M>
__global__ void k_amr_init_pairs(AmrDevView V, const __grid_constant__ SubTables S, const int* __restrict__ pairs,
                                 int n, int mode, double t0, double t1, double t2, double t3) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * V.NV) return;
  const int k = i / V.NV, v = i % V.NV;
  const int c = pairs[2 * k], m = pairs[2 * k + 1];
  const double psi_tau[4] = {t0, t1, t2, t3};
  V.u[(long long)c * V.NV + v] = subbox<D, M>(V, S, c, m, v, mode, psi_tau);
}

// ---------------------------------------------------------------------------
// WENO of a listed active cell from its (2M+1)^D box, thread per (cell, var)
template <int D, int M, int NV>
__global__ void __launch_bounds__(128) k_amr_weno(AmrDevView V, const int* __restrict__ list, int n,
                                                  const __grid_constant__ DevTables T) {
  constexpr int N = M + 1, W = 2 * M + 1, NS = ipow_a(N, D);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * NV) return;
  const int c = list[i / NV], v = i % NV;
  const int l = V.level[c];
  const long long x0 = V.idx[(long long)c * 3], y0 = V.idx[(long long)c * 3 + 1], z0 = V.idx[(long long)c * 3 + 2];
  double* wo = V.w + (wq_row(V, c) * NV + v) * NS;
  if (D == 2) {
    double wx[W][N];
    for (int jy = 0; jy < W; ++jy) {
      double win[W];
#pragma unroll
      for (int o = 0; o < W; ++o) win[o] = amr_u_at(V, l, x0 + o - M, y0 + jy - M, 0, v);
      double out[N];
      weno1d<M>(T, win, out);
#pragma unroll
      for (int a = 0; a < N; ++a) wx[jy][a] = out[a];
    }
#pragma unroll
    for (int a = 0; a < N; ++a) {
      double win[W], out[N];
#pragma unroll
      for (int j = 0; j < W; ++j) win[j] = wx[j][a];
      weno1d<M>(T, win, out);
#pragma unroll
      for (int b = 0; b < N; ++b) wo[a + N * b] = out[b];
    }
  } else {
    double wxy[W][N][N];
    for (int jz = 0; jz < W; ++jz) {
      double wx[W][N];
      for (int jy = 0; jy < W; ++jy) {
        double win[W], out[N];
#pragma unroll
        for (int o = 0; o < W; ++o)
          win[o] = amr_u_at(V, l, x0 + o - M, y0 + jy - M, z0 + jz - M, v);
        weno1d<M>(T, win, out);
#pragma unroll
        for (int a = 0; a < N; ++a) wx[jy][a] = out[a];
      }
#pragma unroll
      for (int a = 0; a < N; ++a) {
        double win[W], out[N];
#pragma unroll
        for (int j = 0; j < W; ++j) win[j] = wx[j][a];
        weno1d<M>(T, win, out);
#pragma unroll
        for (int b = 0; b < N; ++b) wxy[jz][a][b] = out[b];
      }
    }
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int b = 0; b < N; ++b) {
        double win[W], out[N];
#pragma unroll
        for (int k = 0; k < W; ++k) win[k] = wxy[k][a][b];
        weno1d<M>(T, win, out);
#pragma unroll
        for (int cc = 0; cc < N; ++cc) wo[a + N * b + N * N * cc] = out[cc];
      }
  }
}

// ---------------------------------------------------------------------------
// WENO of the active children of one mother together (sibling patch): the
// R^D children's (2M+1)^D boxes overlap in a window of W = R + 2M cells per
// axis, so the dimension-by-dimension sweeps run once over the window in
// shared memory — NV * (R W^(D-1) + R^2 N W^(D-2) + R^3 N^2) 1D problems per
// patch, 21 per (cell, variable) at D = 3, R = 3, M = 2 against the 49 of the
// per-cell box.  Every 1D problem has the inputs of the corresponding problem
// of k_amr_weno, so w is bitwise the same.  One CTA per listed mother
// (level l - 1); children that are not active at level l, or have no w row on
// this rank, are skipped; window cells that do not exist (possible only
// beyond the box of every written child) read 0.  Variables in batches of VB
// so the three stage buffers fit 48 KB.
template <int D, int M, int NV, int R>
__global__ void __launch_bounds__(128) k_amr_weno_patch(AmrDevView V, const int* __restrict__ moms, int n, int l,
                                                        const __grid_constant__ DevTables T) {
  constexpr int N = M + 1, WW = 2 * M + 1, W = R + 2 * M, NS = ipow_a(N, D), RD = ipow_a(R, D);
  constexpr int VB = NV < 5 ? NV : 5;
  constexpr int NU = ipow_a(W, D);                                        // window cells
  constexpr int NX = ipow_a(W, D - 1) * R * N;                            // x-sweep outputs per variable
  constexpr int NY = (D == 3) ? W * R * R * N * N : 0;                    // y-sweep outputs per variable (3D)
  constexpr int SA = VB * (NU > NY ? NU : NY), SB = VB * NX;
  __shared__ double bufA[SA];   // window averages, then the y-sweep outputs
  __shared__ double bufB[SB];   // x-sweep outputs
  __shared__ int cid[RD];
  const int mom = moms[blockIdx.x];
  const int tid = threadIdx.x;
  const long long X0 = V.idx[(long long)mom * 3] * R, Y0 = V.idx[(long long)mom * 3 + 1] * R,
                  Z0 = (D == 3) ? V.idx[(long long)mom * 3 + 2] * R : 0;
  if (tid < RD) {
    const int cx = tid % R, cy = (tid / R) % R, cz = tid / (R * R);
    const int id = amr_lookup(V, l, X0 + cx, Y0 + cy, Z0 + cz);
    const bool wr = id >= 0 && V.status[id] == 0 && V.level[id] == l && (!V.slot || V.slot[id] != 0);
    cid[tid] = wr ? id : -1;
  }
  for (int v0 = 0; v0 < NV; v0 += VB) {
    const int nvb = (NV - v0 < VB) ? NV - v0 : VB;
    __syncthreads();
    // window averages U[v][z][y][x]
    for (int e = tid; e < nvb * NU; e += blockDim.x) {
      const int v = e / NU, c = e - v * NU;
      const int wx = c % W, wy = (c / W) % W, wz = c / (W * W);
      int fl = 0;
      const int id = amr_lookup_flip(V, l, X0 - M + wx, Y0 - M + wy, (D == 3) ? Z0 - M + wz : 0, &fl);
      double a = 0.0;
      if (id >= 0) {
        a = V.u[(long long)id * NV + v0 + v];
        const int gv = v0 + v;
        if (gv >= 1 && gv <= D && ((fl >> (gv - 1)) & 1)) a = -a;
      }
      bufA[v * NU + c] = a;
    }
    __syncthreads();
    // x sweep: (v, rest = (y[, z]) of the window, child column cx) -> B[v][rest][cx][a]
    constexpr int NR = ipow_a(W, D - 1);
    for (int e = tid; e < nvb * NR * R; e += blockDim.x) {
      const int v = e / (NR * R), t = e - v * (NR * R), rest = t / R, cx = t - rest * R;
      double win[WW], out[N];
#pragma unroll
      for (int o = 0; o < WW; ++o) win[o] = bufA[v * NU + rest * W + cx + o];
      weno1d<M>(T, win, out);
#pragma unroll
      for (int a = 0; a < N; ++a) bufB[v * NX + (rest * R + cx) * N + a] = out[a];
    }
    __syncthreads();
    if constexpr (D == 2) {
      // y sweep: (v, cy, cx, a) -> w[child][v][a + N b]
      for (int e = tid; e < nvb * R * R * N; e += blockDim.x) {
        const int v = e / (R * R * N), t = e - v * (R * R * N), cy = t / (R * N), t2 = t - cy * (R * N),
                  cx = t2 / N, a = t2 - cx * N;
        const int id = cid[cy * R + cx];
        if (id < 0) continue;
        double win[WW], out[N];
#pragma unroll
        for (int j = 0; j < WW; ++j) win[j] = bufB[v * NX + ((cy + j) * R + cx) * N + a];
        weno1d<M>(T, win, out);
        double* wo = V.w + (wq_row(V, id) * NV + v0 + v) * NS;
#pragma unroll
        for (int b = 0; b < N; ++b) wo[a + N * b] = out[b];
      }
    } else {
      // y sweep: (v, z of the window, cy, cx, a) -> A[v][z][cy][cx][a][b]
      for (int e = tid; e < nvb * W * R * R * N; e += blockDim.x) {
        const int v = e / (W * R * R * N), t = e - v * (W * R * R * N), wz = t / (R * R * N),
                  t2 = t - wz * (R * R * N), cy = t2 / (R * N), t3 = t2 - cy * (R * N), cx = t3 / N, a = t3 - cx * N;
        double win[WW], out[N];
#pragma unroll
        for (int j = 0; j < WW; ++j) win[j] = bufB[v * NX + (((wz * W) + cy + j) * R + cx) * N + a];
        weno1d<M>(T, win, out);
#pragma unroll
        for (int b = 0; b < N; ++b) bufA[v * NY + (((wz * R + cy) * R + cx) * N + a) * N + b] = out[b];
      }
      __syncthreads();
      // z sweep: (v, cz, cy, cx, a, b) -> w[child][v][a + N b + N^2 c]
      for (int e = tid; e < nvb * RD * N * N; e += blockDim.x) {
        const int v = e / (RD * N * N), t = e - v * (RD * N * N), ch = t / (N * N), ab = t - ch * (N * N);
        const int id = cid[ch];
        if (id < 0) continue;
        const int cx = ch % R, cy = (ch / R) % R, cz = ch / (R * R);
        const int a = ab / N, b = ab - a * N;
        double win[WW], out[N];
#pragma unroll
        for (int k = 0; k < WW; ++k) win[k] = bufA[v * NY + ((((cz + k) * R + cy) * R + cx) * N + a) * N + b];
        weno1d<M>(T, win, out);
        double* wo = V.w + (wq_row(V, id) * NV + v0 + v) * NS;
#pragma unroll
        for (int cc = 0; cc < N; ++cc) wo[a + N * b + N * N * cc] = out[cc];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// face flux / update.  Trace of a same-level cell X on its face (DIR, at_one)
// at tangential nodes (t1, t2) and time node s; coarse trace of K at the fine
// face points via the sub-interval tables.
template <int D, int M, int NV, int DIR>
__device__ __forceinline__ void trace_full(const double* __restrict__ qX, bool at_one, int t1, int t2, int s,
                                           const DevTables& T, double (&out)[NV]) {
  constexpr int N = M + 1, NS = ipow_a(N, D), NST = NS * N;
  constexpr int ax0 = (DIR == 0) ? 1 : 0, ax1 = (DIR == 2) ? 1 : 2;
  const int base = s * NS + t1 * ipow_a(N, ax0) + (D == 3 ? t2 * ipow_a(N, ax1) : 0);
  constexpr int sn = ipow_a(N, DIR);
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) a += (at_one ? T.psi1[k] : T.psi0[k]) * qX[v * NST + base + k * sn];
    out[v] = a;
  }
}

template <int D, int M, int NV, int DIR>
__device__ __forceinline__ void trace_coarse(const double* __restrict__ qK, bool at_one, int o1, int o2, int m, int t1,
                                             int t2, int s, const DevTables& T, const SubTables& S,
                                             double (&out)[NV]) {
  constexpr int N = M + 1, NS = ipow_a(N, D), NST = NS * N;
  constexpr int ax0 = (DIR == 0) ? 1 : 0, ax1 = (DIR == 2) ? 1 : 2;
  for (int v = 0; v < NV; ++v) out[v] = 0.0;
  for (int p = 0; p < NST; ++p) {
    int e[4];
    e[0] = p % N; e[1] = (p / N) % N; e[2] = (D == 3) ? (p / (N * N)) % N : 0;
    const int et = p / NS;
    double th = (at_one ? T.psi1[e[DIR]] : T.psi0[e[DIR]]) * S.Esub[o1][t1][e[ax0]];
    if (D == 3) th *= S.Esub[o2][t2][e[ax1]];
    th *= S.Esub[m][s][et];
#pragma unroll
    for (int v = 0; v < NV; ++v) out[v] += th * qK[v * NST + p];
  }
}

// two-point flux: eqn.rusanov or, for Euler with T.flux == 1,
// eqn.osher
template <int SYS, int D, int DIR>
__device__ __forceinline__ bool numflux_pt(const double (&um)[Phys<SYS, D>::NV], const double (&up)[Phys<SYS, D>::NV],
                                           double gamma, double ch, const DevTables& T,
                                           double (&f)[Phys<SYS, D>::NV]) {
  using PH = Phys<SYS, D>;
  constexpr int NV = PH::NV;
  double fL[NV], fR[NV], sL, sR;
  bool ok = PH::template flux_speed<DIR>(um, gamma, ch, fL, sL);
  ok &= PH::template flux_speed<DIR>(up, gamma, ch, fR, sR);
  if constexpr (SYS == 0) {
    if (T.flux == 1) {
      double dis[NV];
      ok &= osher_dissipation<D, DIR>(um, up, gamma, T, dis);
#pragma unroll
      for (int v = 0; v < NV; ++v) f[v] = 0.5 * (fL[v] + fR[v]) - 0.5 * dis[v];
      return ok;
    }
  }
  const double smax = fmax(sL, sR);
#pragma unroll
  for (int v = 0; v < NV; ++v) f[v] = 0.5 * (fL[v] + fR[v]) - 0.5 * smax * (up[v] - um[v]);
  return ok;
}

// ---------------------------------------------------------------------------
// a3 + a4 on the tree: face fluxes (same level, coarse-fine with flux memory,
// against virtual mothers, boundaries, walls) and the update of the active
// cells of one level.  A lane group of G >= N^D lanes per cell, a lane per
// space-time point of the face being processed (as in k_face_flux_cells), the
// point sums through shared memory in point order.
// face kinds: 0 same level (qL, qR full faces), 1 left boundary (qR only),
// 2 right boundary (qL only), 3 coarse left (qL = mother K), 4 coarse right
// (qR = K), 5 left wall (q^- = reflected q^+), 6 right wall, 7 memory of the
// cell's own virtual children (eqn.memory.sum @ P:693-709)
template <int D, int M, int SYS, int DIR>
__device__ __forceinline__ bool amr_face_point(int kind, const double* qL, const double* qR, int o1, int o2, int m,
                                               int s, int t1, int t2, double gamma, double ch, const DevTables& T,
                                               const SubTables& S, double (&ft)[Phys<SYS, D>::NV]) {
  constexpr int NV = Phys<SYS, D>::NV;
  double um[NV], up[NV];
  if (kind == 0 || kind == 2 || kind == 4 || kind == 6) trace_full<D, M, NV, DIR>(qL, true, t1, t2, s, T, um);
  if (kind == 0 || kind == 1 || kind == 3 || kind == 5) trace_full<D, M, NV, DIR>(qR, false, t1, t2, s, T, up);
  if (kind == 5) { for (int v = 0; v < NV; ++v) um[v] = up[v]; um[1 + DIR] = -up[1 + DIR]; }   // R22
  if (kind == 6) { for (int v = 0; v < NV; ++v) up[v] = um[v]; up[1 + DIR] = -um[1 + DIR]; }
  if (kind == 3) trace_coarse<D, M, NV, DIR>(qL, true, o1, o2, m, t1, t2, s, T, S, um);
  if (kind == 4) trace_coarse<D, M, NV, DIR>(qR, false, o1, o2, m, t1, t2, s, T, S, up);
  if (kind == 1) for (int v = 0; v < NV; ++v) um[v] = up[v];
  if (kind == 2) for (int v = 0; v < NV; ++v) up[v] = um[v];
  return numflux_pt<SYS, D, DIR>(um, up, gamma, ch, T, ft);
}

// What lies across face (dir, side) of cell c: the face kind (above; 8 = the
// active same-level neighbour computes it as its lower face; -1 error), the
// neighbour id, the cell's sub-face offsets inside a coarse neighbour and the
// w / q rows of the lower and upper side.  Evaluated by ONE lane per face
// (lane f of the cell's lane group takes face f = 2 dir + side) and broadcast,
// so the 2D chains of dependent loads (idx -> id map -> status -> mother ->
// row) of a cell run side by side instead of one after the other.
struct AmrFace {
  int kind, nb, o1, o2;
  long long rowL, rowR;
};
__device__ __forceinline__ AmrFace amr_face_info(const AmrDevView& V, int c, int dir, int side) {
  AmrFace f;
  const int l = V.level[c];
  long long ix[3] = {V.idx[(long long)c * 3], V.idx[(long long)c * 3 + 1], V.idx[(long long)c * 3 + 2]};
  const long long own[3] = {ix[0], ix[1], ix[2]};
  ix[dir] += side ? 1 : -1;
  const long long rowc = wq_row(V, c);
  const bool out = ix[dir] < 0 || ix[dir] >= V.n[l][dir];
  f.kind = -1; f.nb = -1; f.o1 = 0; f.o2 = 0; f.rowL = rowc; f.rowR = rowc;
  if (out && V.bc[2 * dir + side] == ADER_BC_TRANSMISSIVE) f.kind = side ? 2 : 1;
  else if (out && V.bc[2 * dir + side] == ADER_BC_REFLECTIVE) f.kind = side ? 6 : 5;
  else {
    f.nb = amr_lookup(V, l, ix[0], ix[1], ix[2]);
    const int st = f.nb >= 0 ? V.status[f.nb] : 9;
    if (st == 0 && side) {
      f.kind = 8;   // computed once, as the lower face of the neighbour (k_amr_update_w reads it there)
    } else if (st == 0) {
      f.kind = 0;
      f.rowL = wq_row(V, f.nb);
    } else if (st == 1) {
      // coarse-fine: the virtual neighbour scales its mother's q_h down
      const long long rowK = wq_row(V, V.mother[f.nb]);
      const int ax0 = (dir == 0) ? 1 : 0, ax1 = (dir == 2) ? 1 : 2;
      f.o1 = (int)(own[ax0] % V.r);
      f.o2 = (V.D == 3) ? (int)(own[ax1] % V.r) : 0;
      f.kind = side ? 4 : 3;
      if (side) f.rowR = rowK; else f.rowL = rowK;
    } else if (st == -1) {
      f.kind = V.child[c] >= 0 ? 7 : -1;
    }
  }
  return f;
}
__device__ __forceinline__ AmrFace amr_face_bcast(const AmrFace& f, int src) {
  AmrFace g;
  g.kind = __shfl_sync(0xffffffffu, f.kind, src);
  g.nb = __shfl_sync(0xffffffffu, f.nb, src);
  g.o1 = __shfl_sync(0xffffffffu, f.o1, src);
  g.o2 = __shfl_sync(0xffffffffu, f.o2, src);
  g.rowL = __shfl_sync(0xffffffffu, f.rowL, src);
  g.rowR = __shfl_sync(0xffffffffu, f.rowR, src);
  return g;
}

template <int D, int M, int SYS, int DIR, int G>
__device__ __forceinline__ bool amr_cell_face_w(const AmrDevView& V, int c, bool valid, int side, int m, int p,
                                                const AmrFace& fi, double gamma, double ch, const DevTables& T,
                                                const SubTables& S, double (*rb)[G + 1], double* Fout) {
  constexpr int NV = Phys<SYS, D>::NV, N = M + 1, NS = ipow_a(N, D), NST = NS * N, NT = NS / N;
  // Every lane group of the warp runs the same two __syncwarp()s whatever its
  // kind (2D: several cells per warp).
  const int kind = fi.kind, nb = fi.nb, o1 = fi.o1, o2 = fi.o2;
  const double *qL = V.q + fi.rowL * NV * NST, *qR = V.q + fi.rowR * NV * NST;
  bool ok = kind >= 0;
  if (valid && kind >= 0 && kind < 7 && p < NS) {
    const int s = p / NT, t = p - s * NT, t1 = t % N, t2 = t / N;
    double ft[NV];
    ok = amr_face_point<D, M, SYS, DIR>(kind, qL, qR, o1, o2, m, s, t1, t2, gamma, ch, T, S, ft);
    double wgt = T.w[s] * T.w[t1];
    if (D == 3) wgt *= T.w[t2];
#pragma unroll
    for (int v = 0; v < NV; ++v) rb[v][p] = wgt * ft[v];
  }
  __syncwarp();
  if (valid && p < NV) {
    if (kind == 7) {
      // virtual mother: the memory of our own virtual children on this face (eqn.memory.sum)
      const int ch0 = V.child[c];
      double acc = 0.0;
      for (int qd = 0; qd < V.rd; ++qd) {
        const int off[3] = {qd % V.r, (qd / V.r) % V.r, qd / (V.r * V.r)};
        if (off[DIR] != (side ? V.r - 1 : 0)) continue;
        double* mm = V.mem + ((long long)(ch0 + qd) * 6 + 2 * DIR + side) * NV;
        acc += mm[p];
        mm[p] = 0.0;
      }
      Fout[p] = acc / (double)V.rd;
    } else if (kind >= 0 && kind < 8) {
      double acc = rb[p][0];
#pragma unroll
      for (int j = 1; j < NS; ++j) acc += rb[p][j];
      Fout[p] = acc;
      if (kind == 3 || kind == 4) V.mem[((long long)nb * 6 + 2 * DIR + (side ? 0 : 1)) * NV + p] += acc;   // nb's face toward c
    }
  }
  __syncwarp();
  return ok;
}

// Face fluxes of the listed (active) cells: every lower face and the upper
// faces no active same-level neighbour computes (boundaries, walls,
// coarse-fine faces, faces against virtual mothers), each into the cell's own
// row of the flux-memory array (unused by active cells: memory lives on
// virtual children); a face between two active cells of a level is computed
// once, by its upper cell, with the same (lower, upper) traces either way.
template <int D, int M, int SYS, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_amr_flux_w(AmrDevView V, const __grid_constant__ SubTables S,
                                                            const int* __restrict__ list, int n, int m,
                                                            double gamma, double ch, DevCounters* cnt,
                                                            const __grid_constant__ DevTables T) {
  constexpr int NV = Phys<SYS, D>::NV, NS = ipow_a(M + 1, D);
  constexpr int G = (NS <= 8) ? 8 : (NS <= 16 ? 16 : 32);
  constexpr int CPW = 32 / G;
  __shared__ double red[WARPS * CPW][NV][G + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = lane & (G - 1), grp = warp * CPW + lane / G;
  const int i = (blockIdx.x * WARPS + warp) * CPW + lane / G;
  const bool valid = i < n;
  const int c = list[valid ? i : 0];
  double(*rb)[G + 1] = red[grp];
  double* F = V.mem + (long long)c * 6 * NV;
  // lane f < 2D of the lane group looks across face f; the others receive it
  AmrFace mine = amr_face_info(V, c, (p < 2 * D) ? (p >> 1) : 0, p & 1);
  const int base = lane & ~(G - 1);
  bool ok = true;
  ok &= amr_cell_face_w<D, M, SYS, 0, G>(V, c, valid, 0, m, p, amr_face_bcast(mine, base + 0), gamma, ch, T, S, rb, F + 0 * NV);
  ok &= amr_cell_face_w<D, M, SYS, 0, G>(V, c, valid, 1, m, p, amr_face_bcast(mine, base + 1), gamma, ch, T, S, rb, F + 1 * NV);
  ok &= amr_cell_face_w<D, M, SYS, 1, G>(V, c, valid, 0, m, p, amr_face_bcast(mine, base + 2), gamma, ch, T, S, rb, F + 2 * NV);
  ok &= amr_cell_face_w<D, M, SYS, 1, G>(V, c, valid, 1, m, p, amr_face_bcast(mine, base + 3), gamma, ch, T, S, rb, F + 3 * NV);
  if constexpr (D == 3) {
    ok &= amr_cell_face_w<D, M, SYS, 2, G>(V, c, valid, 0, m, p, amr_face_bcast(mine, base + 4), gamma, ch, T, S, rb, F + 4 * NV);
    ok &= amr_cell_face_w<D, M, SYS, 2, G>(V, c, valid, 1, m, p, amr_face_bcast(mine, base + 5), gamma, ch, T, S, rb, F + 5 * NV);
  }
  if (valid && !ok && (!V.own || V.own[c])) amr_error(cnt, 1, 2, c);   // multi-rank: band cells' errors do not count
}

// FV update (eq:finite_vol @ P:147-152) of the listed cells from the face
// fluxes k_amr_flux_w left in the flux-memory rows: the lower face of each
// direction from the cell's row, the upper face from the row of the active
// same-level neighbour (its lower face) or else from the cell's own row.
template <int D, int SYS>
__global__ void __launch_bounds__(256) k_amr_update_w(AmrDevView V, const int* __restrict__ list, int n,
                                                      double dtdx0, double dtdx1, double dtdx2) {
  constexpr int NV = Phys<SYS, D>::NV;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * NV) return;
  const int c = list[i / NV], p = i % NV;
  const int l = V.level[c];
  const double dtdx[3] = {dtdx0, dtdx1, dtdx2};
  double uu = V.u[(long long)c * NV + p];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    long long ix[3] = {V.idx[(long long)c * 3], V.idx[(long long)c * 3 + 1], V.idx[(long long)c * 3 + 2]};
    ix[d] += 1;
    const bool out = ix[d] >= V.n[l][d];
    long long hi = (long long)c * 6 + 2 * d + 1;
    if (!(out && (V.bc[2 * d + 1] == ADER_BC_TRANSMISSIVE || V.bc[2 * d + 1] == ADER_BC_REFLECTIVE))) {
      const int nb = amr_lookup(V, l, ix[0], ix[1], ix[2]);
      if (nb >= 0 && V.status[nb] == 0) hi = (long long)nb * 6 + 2 * d;
    }
    const double fhi = V.mem[hi * NV + p], flo = V.mem[((long long)c * 6 + 2 * d) * NV + p];
    uu = uu - dtdx[d] * (fhi - flo);
  }
  V.u[(long long)c * NV + p] = uu;
}

// ---------------------------------------------------------------------------
template <int D, int SYS>
__global__ void __launch_bounds__(256) k_amr_cfl(AmrDevView V, const int* __restrict__ list, int n, double i0,
                                                 double i1, double i2, double gamma, double ch,
                                                 DevCounters* __restrict__ cnt) {
  using PH = Phys<SYS, D>;
  constexpr int NV = PH::NV;
  __shared__ double sm[32];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0.0;
  if (i < n) {
    const int c = list[i];
    double uu[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) uu[v] = V.u[(long long)c * NV + v];
    const double inv[3] = {i0, i1, i2};
    if (!PH::cfl_speed(uu, gamma, ch, inv, s)) amr_error(cnt, 1, 4, c);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sm[warp] = s;
  __syncthreads();
  if (warp == 0) {
    s = (lane < (int)(blockDim.x >> 5)) ? sm[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
    if (lane == 0) atomicMax(&cnt->speed_bits, (unsigned long long)__double_as_longlong(s));
  }
}

// indicator, reading R14: every operation explicitly rounded (no FMA), in the
// oracle's order, so that chi and the refinement flags are bit-identical
__global__ void k_amr_indicator(AmrDevView V, const int* __restrict__ list, int n, double eps) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = list[i];
  const int l = V.level[c];
  const long long x0 = V.idx[(long long)c * 3], y0 = V.idx[(long long)c * 3 + 1], z0 = V.idx[(long long)c * 3 + 2];
  double phi[27];
  const int D = V.D;
  const int zl = D == 3 ? -1 : 0, zh = D == 3 ? 1 : 0;
  int b = 0;
  for (int dz = zl; dz <= zh; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx, ++b) {
        const int nb = amr_lookup(V, l, x0 + dx, y0 + dy, z0 + dz);
        phi[b] = V.u[(long long)(nb >= 0 ? nb : c) * V.NV];   // Phi = rho
      }
  const int st[3] = {1, 3, 9};
  int cc = 0;
  for (int k = 0; k < D; ++k) cc += st[k];
  double num = 0.0, den = 0.0;
  for (int k = 0; k < D; ++k)
    for (int q = 0; q < D; ++q) {
      double nn, e;
      if (k == q) {
        const double pp = phi[cc + st[k]], p0 = phi[cc], pm = phi[cc - st[k]];
        nn = __dadd_rn(__dsub_rn(pp, __dmul_rn(2.0, p0)), pm);
        e = __dadd_rn(__dadd_rn(fabs(__dsub_rn(pp, p0)), fabs(__dsub_rn(p0, pm))),
                      __dmul_rn(eps, __dadd_rn(__dadd_rn(fabs(pp), __dmul_rn(2.0, fabs(p0))), fabs(pm))));
      } else {
        const double a = phi[cc + st[k] + st[q]], bb = phi[cc + st[k] - st[q]];
        const double c2 = phi[cc - st[k] + st[q]], d2 = phi[cc - st[k] - st[q]];
        nn = __dmul_rn(0.25, __dadd_rn(__dsub_rn(__dsub_rn(a, bb), c2), d2));
        e = __dadd_rn(__dmul_rn(0.5, __dadd_rn(fabs(__dsub_rn(a, c2)), fabs(__dsub_rn(bb, d2)))),
                      __dmul_rn(__dmul_rn(0.25, eps),
                                __dadd_rn(__dadd_rn(__dadd_rn(fabs(a), fabs(bb)), fabs(c2)), fabs(d2))));
      }
      num = __dadd_rn(num, __dmul_rn(nn, nn));
      den = __dadd_rn(den, __dmul_rn(e, e));
    }
  V.chi[c] = (den == 0.0) ? 0.0 : __dsqrt_rn(__ddiv_rn(num, den));
}

template <int D, int SYS>
__global__ void k_amr_ic(AmrDevView V, const int* __restrict__ list, int n, const double* __restrict__ prim,
                         const double* __restrict__ wq, int nq, double gamma) {
  using PH = Phys<SYS, D>;
  constexpr int NV = PH::NV;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = 0.0;
  for (int g = 0; g < nq; ++g) {
    double uu[NV];
    PH::prim_to_cons(prim + ((long long)i * nq + g) * 9, gamma, uu);
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] += wq[g] * uu[v];
  }
  const int c = list[i];
#pragma unroll
  for (int v = 0; v < NV; ++v) V.u[(long long)c * NV + v] = acc[v];
}

// ---------------------------------------------------------------------------
// incremental topology updates (one launch each, instead of full re-uploads)
// meta[i] = {id, level, status, mother, child, idx0, idx1, idx2} (long long)
__global__ void k_amr_meta_scatter(AmrDevView V, const long long* __restrict__ meta, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long* m = meta + (long long)i * 8;
  const int id = (int)m[0];
  V.level[id] = (int)m[1];
  V.status[id] = (int)m[2];
  V.mother[id] = (int)m[3];
  V.child[id] = (int)m[4];
  V.idx[(long long)id * 3] = m[5];
  V.idx[(long long)id * 3 + 1] = m[6];
  V.idx[(long long)id * 3 + 2] = m[7];
}

// ch[i] = {level, linear index, value}
__global__ void k_amr_map_set(AmrDevView V, const long long* __restrict__ ch, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long* c = ch + (long long)i * 3;
  const_cast<int*>(V.map[c[0]])[c[1]] = (int)c[2];
}

__global__ void k_amr_zero_mem(AmrDevView V, const int* __restrict__ list, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * 6 * V.NV) return;
  const int c = list[i / (6 * V.NV)], j = i % (6 * V.NV);
  V.mem[(long long)c * 6 * V.NV + j] = 0.0;
}

// multi-rank exchange of cell averages: out[i][v] = u[ids[i]][v] / u[ids[i]][v] = in[i][v]
__global__ void k_amr_rows_gather(const double* __restrict__ u, const int* __restrict__ ids, int n, int nv,
                                  double* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)n * nv) return;
  out[i] = u[(long long)ids[i / nv] * nv + i % nv];
}
__global__ void k_amr_rows_scatter(double* __restrict__ u, const int* __restrict__ ids, int n, int nv,
                                   const double* __restrict__ in) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)n * nv) return;
  u[(long long)ids[i / nv] * nv + i % nv] = in[i];
}

// ===========================================================================
// launchers
// ===========================================================================
namespace {
inline unsigned gsz(long long n, int bs) { return (unsigned)((n + bs - 1) / bs); }
inline void cl(const KCtx& k) { if (k.launches) ++*k.launches; }
}  // namespace

#define AMR_DISPATCH(D_, M_, SYS_, ...)                                                         \
  do {                                                                                          \
    if (D_ == 2 && M_ == 2 && SYS_ == 0) { constexpr int D = 2, M = 2, SYS = 0; __VA_ARGS__; }  \
    else if (D_ == 2 && M_ == 3 && SYS_ == 0) { constexpr int D = 2, M = 3, SYS = 0; __VA_ARGS__; } \
    else if (D_ == 3 && M_ == 2 && SYS_ == 0) { constexpr int D = 3, M = 2, SYS = 0; __VA_ARGS__; } \
    else if (D_ == 2 && M_ == 2 && SYS_ == 1) { constexpr int D = 2, M = 2, SYS = 1; __VA_ARGS__; } \
    else if (D_ == 2 && M_ == 3 && SYS_ == 1) { constexpr int D = 2, M = 3, SYS = 1; __VA_ARGS__; } \
    else if (D_ == 3 && M_ == 2 && SYS_ == 1) { constexpr int D = 3, M = 2, SYS = 1; __VA_ARGS__; } \
  } while (0)

void amr_launch_meta_scatter(const KCtx& k, const AmrDevView& v, const long long* meta, int n) {
  if (n <= 0) return;
  cl(k);
  k_amr_meta_scatter<<<gsz(n, 256), 256, 0, k.stream>>>(v, meta, n);
}

void amr_launch_map_set(const KCtx& k, const AmrDevView& v, const long long* ch, int n) {
  if (n <= 0) return;
  cl(k);
  k_amr_map_set<<<gsz(n, 256), 256, 0, k.stream>>>(v, ch, n);
}

void amr_launch_rows_gather(const KCtx& k, const double* u, const int* ids, int n, int nv, double* out) {
  if (n <= 0) return;
  cl(k);
  k_amr_rows_gather<<<gsz((long long)n * nv, 256), 256, 0, k.stream>>>(u, ids, n, nv, out);
}

void amr_launch_rows_scatter(const KCtx& k, double* u, const int* ids, int n, int nv, const double* in) {
  if (n <= 0) return;
  cl(k);
  k_amr_rows_scatter<<<gsz((long long)n * nv, 256), 256, 0, k.stream>>>(u, ids, n, nv, in);
}

void amr_launch_zero_mem(const KCtx& k, const AmrDevView& v, const int* list, int n) {
  if (n <= 0) return;
  cl(k);
  k_amr_zero_mem<<<gsz((long long)n * 6 * v.NV, 256), 256, 0, k.stream>>>(v, list, n);
}

void amr_launch_average(const KCtx& k, const AmrDevView& v, const int* list, int n) {
  if (n <= 0) return;
  cl(k);
  k_amr_average<<<gsz((long long)n * v.NV, 256), 256, 0, k.stream>>>(v, list, n);
}

void amr_launch_project(const KCtx& k, const AmrDevView& v, const SubTables& st, const int* list, int n,
                        const double* pt) {
  if (n <= 0) return;
  cl(k);
  AMR_DISPATCH(k.D, k.M, k.SYS, (void)SYS;
               k_amr_project<D, M><<<gsz((long long)n * v.NV, 128), 128, 0, k.stream>>>(v, st, list, n, pt[0], pt[1],
                                                                                        pt[2], pt[3]));
}

void amr_launch_init_from_weno(const KCtx& k, const AmrDevView& v, const SubTables& st, const int* pairs, int n) {
  if (n <= 0) return;
  cl(k);
  AMR_DISPATCH(k.D, k.M, k.SYS, (void)SYS;
               k_amr_init_pairs<D, M><<<gsz((long long)n * v.NV, 128), 128, 0, k.stream>>>(v, st, pairs, n, 0, 0, 0,
                                                                                           0, 0));
}

void amr_launch_init_from_pred(const KCtx& k, const AmrDevView& v, const SubTables& st, const int* pairs, int n,
                               const double* pt) {
  if (n <= 0) return;
  cl(k);
  AMR_DISPATCH(k.D, k.M, k.SYS, (void)SYS;
               k_amr_init_pairs<D, M><<<gsz((long long)n * v.NV, 128), 128, 0, k.stream>>>(v, st, pairs, n, 1, pt[0],
                                                                                           pt[1], pt[2], pt[3]));
}

void amr_launch_weno(const KCtx& k, const AmrDevView& v, const int* list, int n) {
  if (n <= 0) return;
  cl(k);
  AMR_DISPATCH(k.D, k.M, k.SYS, {
    constexpr int NV = Phys<SYS, D>::NV;
    k_amr_weno<D, M, NV><<<gsz((long long)n * NV, 128), 128, 0, k.stream>>>(v, list, n, k.tab);
  });
}

void amr_launch_weno_patches(const KCtx& k, const AmrDevView& v, const int* moms, int n, int level) {
  if (n <= 0) return;
  cl(k);
  AMR_DISPATCH(k.D, k.M, k.SYS, {
    constexpr int NV = Phys<SYS, D>::NV;
    k_amr_weno_patch<D, M, NV, 3><<<n, 128, 0, k.stream>>>(v, moms, n, level, k.tab);
  });
}

void amr_launch_predictor(const KCtx& k, const AmrDevView& v, const int* list, int n, const double dtdx[3],
                          double tol, int max_sweeps, DevCounters* cnt) {
  if (n <= 0) return;
  Box none{{0, 0, 0}, {0, 0, 0}};
  launch_predictor_list(k, v.w, v.q, none, list, n, dtdx, tol, max_sweeps, cnt, v.own, nullptr, 0, false, nullptr,
                        0.0, v.slot);
}

void amr_launch_flux_update(const KCtx& k, const AmrDevView& v, const SubTables& st, const int* list, int n, int m,
                            const double dtdx[3], DevCounters* cnt) {
  if (n <= 0) return;
  cl(k);
  AMR_DISPATCH(k.D, k.M, k.SYS, {
    constexpr int NS = ipow_a(M + 1, D);
    constexpr int CPW = 32 / ((NS <= 8) ? 8 : (NS <= 16 ? 16 : 32));
    constexpr int WARPS = 4;
    k_amr_flux_w<D, M, SYS, WARPS><<<gsz(n, WARPS * CPW), WARPS * 32, 0, k.stream>>>(v, st, list, n, m, k.gamma,
                                                                                      k.ch, cnt, k.tab);
    cl(k);
    k_amr_update_w<D, SYS><<<gsz((long long)n * Phys<SYS, D>::NV, 256), 256, 0, k.stream>>>(v, list, n, dtdx[0],
                                                                                           dtdx[1], dtdx[2]);
  });
}

void amr_launch_cfl(const KCtx& k, const AmrDevView& v, const int* list, int n, const double inv_dx0[3],
                    DevCounters* cnt) {
  if (n <= 0) return;
  cl(k);
#define CFLK(D_, S_)                                                                                          \
  k_amr_cfl<D_, S_><<<gsz(n, 256), 256, 0, k.stream>>>(v, list, n, inv_dx0[0], inv_dx0[1], inv_dx0[2], k.gamma, \
                                                       k.ch, cnt)
  if (k.D == 2 && k.SYS == 0) CFLK(2, 0);
  else if (k.D == 3 && k.SYS == 0) CFLK(3, 0);
  else if (k.D == 2 && k.SYS == 1) CFLK(2, 1);
  else CFLK(3, 1);
#undef CFLK
}

void amr_launch_indicator(const KCtx& k, const AmrDevView& v, const int* list, int n, double eps) {
  if (n <= 0) return;
  cl(k);
  k_amr_indicator<<<gsz(n, 128), 128, 0, k.stream>>>(v, list, n, eps);
}

void amr_launch_ic(const KCtx& k, const AmrDevView& v, const int* list, int n, const double* prim, const double* wq,
                   int nq) {
  if (n <= 0) return;
  cl(k);
#define ICK(D_, S_) k_amr_ic<D_, S_><<<gsz(n, 128), 128, 0, k.stream>>>(v, list, n, prim, wq, nq, k.gamma)
  if (k.D == 2 && k.SYS == 0) ICK(2, 0);
  else if (k.D == 3 && k.SYS == 0) ICK(3, 0);
  else if (k.D == 2 && k.SYS == 1) ICK(2, 1);
  else ICK(3, 1);
#undef ICK
}

}  // namespace ader
