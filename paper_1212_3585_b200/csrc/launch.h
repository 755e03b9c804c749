// launch.h — host-side launchers of the sm_100a kernels (kernels.cu).
// All cell arrays are cell-major on the rank's padded grid (owned block plus a
// ghost layer of width H = M+1 on every axis of the d axes):
//   u  [cell][nu]              cell averages
//   wk [cell][nu][N^(k+1)]     dofs after WENO sweep k (x, then y, then z)
//   q  [cell][nu][N^(d+1)]     space-time predictor dofs, space fastest
//   F  [dir][cell][nu]         space-time averaged flux on the lower face of cell
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "tables.h"

namespace ader {

struct Box {
  int lo[3];     // padded coordinates of the first cell
  int ext[3];    // extent per axis (1 on unused axes)
  __host__ __device__ long long count() const { return (long long)ext[0] * ext[1] * ext[2]; }
};

struct DevCounters {              // device-resident, zeroed by the host
  unsigned long long sweeps;      // Picard sweeps summed over cells
  unsigned long long cells;       // predicted cells
  unsigned long long speed_bits;  // max CFL speed (bits of a non-negative double)
  unsigned long long err_cell;    // padded cell index of the first failure
  int sweeps_max;
  int err_code;                   // 0 ok, 1 inadmissible state, 2 predictor cap
  int err_stage;                  // 1 predictor, 2 flux, 3 update, 4 speed
  int pad;
  unsigned long long err_any;     // multi-rank: max over the ranks of err_code (set before every
                                  // host check, so all ranks stop at the same step)
  unsigned long long flat_cells;  // predicted cells flagged flat (no q block written)
};

// Device-resident step control of the uniform path: the time step is formed
// on the GPU from the reduced CFL speed, so K macro steps are enqueued without
// a host round trip per step (the host only reads this back every few steps).
struct StepState {
  double t, dt, last_dt;          // time reached, dt of the last step, last positive dt
  double dtdx[3];                 // dt / dx_dir of the last step (read by predictor / update)
  long long steps;                // steps with dt > 0
  double prev_dt;                 // dt of the step before the last (predictor guess, R25)
};

// Instrumentation hook (CUDA events around launches, set by ader_api.cpp).
struct ProfHook {
  void* ctx = nullptr;
  void (*begin)(void* ctx, int kind) = nullptr;
  void (*end)(void* ctx, int kind, double flops) = nullptr;
};

struct KCtx {
  ProfHook* hook;
  int D, M, SYS, NV;
  long long sy, sz;               // cell strides along y, z in the padded grid
  long long ncell;                // padded cells
  double gamma, ch;
  cudaStream_t stream;
  long long* launches;            // host counter of kernel launches (instrumentation)
  DevTables tab;
};

// returns false if (D, M, SYS) has no compiled instantiation
bool supported(int D, int M, int SYS);

// WENO sweep k along axis k (k = 0 x, 1 y, 2 z) on the cells of `region`.
void launch_weno_sweep(const KCtx& k, int sweep, const double* src, double* dst, const Box& region);
// Predictor on `region`: w -> q.  dtdx_dev (optional): read dt/dx from the
// device (StepState::dtdx) instead of dtdx.
// qs: stride of a cell's q block in doubles (0 = nu N^(d+1); the uniform path
// uses q_block_stride, the block size rounded up to even).
// qflat (optional, [padded cell], M = 2, no guess): cells whose nodes all carry the same w and
// that converge in the first sweep get qflat[cell] = 1 and NO q block (q_h = w - Tsum[s] G(node),
// rebuilt from w by launch_face_flux_cells); every other predicted cell gets 0 and its block.
// guess (reading R25): start the Picard iteration from the cell's previous q
// (read in place from q) extrapolated by r = dt_n / dt_{n-1}: r from gst
// (device StepState: dt / prev_dt) if given, else guess_r; r <= 0 = R3.
void launch_predictor(const KCtx& k, const double* w, double* q, const Box& region, const double dtdx[3],
                      double tol, int max_sweeps, DevCounters* cnt, const double* dtdx_dev = nullptr,
                      long long qs = 0, bool guess = false, const StepState* gst = nullptr, double guess_r = 0.0,
                      unsigned char* qflat = nullptr);
// Predictor on the cells of an id list (AMR levels): w, q indexed by id (or by
// slot[id] if given).  If emask is given only cells with emask[id] != 0 report
// solver errors.
void launch_predictor_list(const KCtx& k, const double* w, double* q, const Box& region, const int* list,
                           long long nlist, const double dtdx[3], double tol, int max_sweeps, DevCounters* cnt,
                           const unsigned char* emask = nullptr, const double* dtdx_dev = nullptr,
                           long long qs = 0, bool guess = false, const StepState* gst = nullptr,
                           double guess_r = 0.0, const int* slot = nullptr, unsigned char* qflat = nullptr);
// Face fluxes on the lower face of every cell of `ext` (owned block + 1 on each
// active axis), one lane group per cell computing all its lower faces
// (L2-friendly traversal).  bmask bit 2*dir (2*dir+1): the first (last) face
// along dir is a physical transmissive boundary and takes the interior trace
// on both sides; rmask, same bits: a reflective wall (R22), the exterior state
// is the interior trace with the normal momentum negated.
// qflat / w / dtdx (optional, D = 3, M = 2): the flags launch_predictor left, its w array and the
// dt/dx it used (dtdx_dev: read from the device instead) — flat cells' traces come from w.
void launch_face_flux_cells(const KCtx& k, const double* q, double* F, const Box& ext, int H, const int n[3],
                            int bmask, int rmask, DevCounters* cnt, long long qs,
                            const unsigned char* qflat = nullptr, const double* w = nullptr,
                            const double* dtdx = nullptr, const double* dtdx_dev = nullptr);
// The same fluxes (bitwise) with the q blocks streamed into shared memory by
// bulk copies (flux_tma.cu); q blocks at stride q_block_stride(D, M, SYS).
void launch_face_flux_tma(const KCtx& k, const double* q, double* F, const Box& ext, int H, const int n[3],
                          int bmask, int rmask, DevCounters* cnt);
// The same fluxes up to the rounding of the trace sums, from coalesced block
// loads and warp-shuffle line sums (flux_rot.cu); q blocks at stride qs.
void launch_face_flux_rot(const KCtx& k, const double* q, double* F, const Box& ext, int H, const int n[3],
                          int bmask, int rmask, DevCounters* cnt, long long qs);
// nu N^(d+1) rounded up to an even number of doubles (16-byte aligned blocks)
long long q_block_stride(int D, int M, int SYS);
// a1 + a2 fused (weno_pred.cu): WENO sweeps of the cell averages u and the
// predictor on `region`, q blocks at stride qs; bitwise the same q as
// launch_weno_sweep x3 + launch_predictor.
void launch_weno_predictor(const KCtx& k, const double* u, double* q, const Box& region, long long qs,
                           const double dtdx[3], double tol, int max_sweeps, DevCounters* cnt,
                           const double* dtdx_dev = nullptr);
// a2 + a3 fused (pred_flux.cu): the predictor on the cells of PR and the
// lower-face fluxes of the face box (owned + 1, as launch_face_flux_cells) in
// one tile walk with q kept in shared memory; faces between tiles go through
// the face-trace buffer bnd (pred_flux_buffer_doubles doubles).  Bitwise the
// same F as launch_predictor + launch_face_flux_cells.
void launch_pred_flux(const KCtx& k, const double* w, double* F, double* bnd, const Box& PR, int H, const int n[3],
                      int bmask, int rmask, double tol, int max_sweeps, DevCounters* cnt, const double dtdx[3],
                      const double* dtdx_dev = nullptr);
// size of that buffer (-1: unsupported (D, M, SYS))
long long pred_flux_buffer_doubles(int D, int M, int SYS, const Box& PR, int H, const int n[3]);
// FV update of `interior` in place + max CFL speed of the new state.
void launch_update(const KCtx& k, double* u, const double* F, const Box& interior, const double dtdx[3],
                   const double inv_dx[3], DevCounters* cnt, const double* dtdx_dev = nullptr);
// dt of the next step on the device (reading R1): dt = cfl / speed (speed from
// cnt->speed_bits, max over ranks), clipped to t_end, 0 once t >= t_end;
// updates st (t, dt, dtdx = dt / dx, steps).  Invalid dt -> err_code 3.
void launch_step_dt(const KCtx& k, DevCounters* cnt, StepState* st, double cfl, double t_end, const double dx[3]);
// set st to a host-chosen dt (loopback groups, debug dumps)
void launch_set_dt(const KCtx& k, StepState* st, double dt, const double dx[3]);
void launch_cfl_speed(const KCtx& k, const double* u, const Box& interior, const double inv_dx[3],
                      DevCounters* cnt);
// Ghost copy along one axis: for every cell of `region` (halo cells), copy the
// cell at map(coord[axis]) with the other coordinates unchanged.
//   mode 0: periodic wrap within [H, H+n), mode 1: clamp to [H, H+n-1],
//   mode 2: mirror about the wall with the normal momentum negated (R22)
void launch_fill_axis(const KCtx& k, double* u, const Box& region, int axis, int mode, int H, int n);
// Pack / unpack a box of u into / from a contiguous buffer [box cell][nu].
void launch_pack(const KCtx& k, const double* u, const Box& b, double* buf);
void launch_unpack(const KCtx& k, double* u, const Box& b, const double* buf);
// IC cell averages: prim[cell][nq][9] at the GL points of `ncells` consecutive
// owned cells starting at owned linear index first; weights wq[nq].
// IC cell averages of the box of extents n[] starting at the owned-block offset
// off[] (<= 0: into the ghost layer, inflow sides), cells x fastest.
void launch_ic_average(const KCtx& k, double* u, const double* prim, const double* wq, int nq,
                       long long first, long long ncells, const int n[3], int H, const int off[3]);
// Owned cells <-> compact [cell][stride] buffers (x fastest within the block).
void launch_gather(const KCtx& k, const double* src, int stride, const Box& b, double* out);
void launch_scatter(const KCtx& k, double* dst, int stride, const Box& b, const double* in);
// Block partial sums of u (times vol) over owned cells -> partial[block][nu]; returns #blocks.
int launch_cons_partials(const KCtx& k, const double* u, const Box& b, double vol, double* partial, int max_blocks);

}  // namespace ader
