// ader_api.cpp — C-ABI implementation (include/ader.h): validation, device
// memory, the host orchestrator of one macro step, ghost-layer exchange over
// NCCL, IC projection, debug dumps and kernel instrumentation.
//
// The host never computes cell data: every stage of the path runs in the
// kernels of kernels.cu; the host only schedules launches and reduces
// scalars (the CFL dt, report counters).
// Citations: P:n = PAPER.md line n.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/ader.h"
#include "launch.h"
#include "tables.h"
#include "amr.h"

using namespace ader;

// ---------------------------------------------------------------------------
// NCCL, loaded lazily (the soname already loaded by torch is reused)
// ---------------------------------------------------------------------------
namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool load(std::string& err) {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) { err = std::string("cannot load libnccl.so.2: ") + dlerror(); return false; }
#define SYM(x) x = reinterpret_cast<decltype(x)>(dlsym(h, "nccl" #x)); if (!x) { err = "missing nccl" #x; return false; }
    SYM(GetUniqueId) SYM(CommInitRank) SYM(CommDestroy) SYM(Send) SYM(Recv) SYM(GroupStart) SYM(GroupEnd)
    SYM(AllReduce) SYM(GetErrorString)
#undef SYM
    return true;
  }
};
NcclApi g_nccl;

// AmrComm hooks over the context's communicator (ctx = ncclComm_t)
ader_status amr_nccl_p2p(void* ctx, int n, const int* peers, double* const* sendp, const size_t* scount,
                         double* const* recvp, const size_t* rcount, cudaStream_t st) {
  ncclComm_t comm = (ncclComm_t)ctx;
  if (g_nccl.GroupStart() != ncclSuccess) return ADER_ERR_NCCL;
  bool ok = true;
  for (int i = 0; i < n; ++i) {
    if (scount[i]) ok &= g_nccl.Send(sendp[i], scount[i], ncclDouble, peers[i], comm, st) == ncclSuccess;
    if (rcount[i]) ok &= g_nccl.Recv(recvp[i], rcount[i], ncclDouble, peers[i], comm, st) == ncclSuccess;
  }
  ok &= g_nccl.GroupEnd() == ncclSuccess;
  return ok ? ADER_OK : ADER_ERR_NCCL;
}
ader_status amr_nccl_sum(void* ctx, double* buf, size_t n, cudaStream_t st) {
  return g_nccl.AllReduce(buf, buf, n, ncclDouble, ncclSum, (ncclComm_t)ctx, st) == ncclSuccess ? ADER_OK
                                                                                               : ADER_ERR_NCCL;
}
ader_status amr_nccl_max_u64(void* ctx, unsigned long long* buf, cudaStream_t st) {
  return g_nccl.AllReduce(buf, buf, 1, ncclUint64, ncclMax, (ncclComm_t)ctx, st) == ncclSuccess ? ADER_OK
                                                                                              : ADER_ERR_NCCL;
}

// Collectives through the caller's host callbacks (ader_create_host_comm): the
// device buffers are staged through one pinned buffer; the stream is
// synchronised around every call, so the caller's collective sees finished data.
struct HostComm {
  ader_host_comm u{};
  char* pin = nullptr;
  size_t cap = 0;
  bool grow(size_t bytes) {
    if (bytes <= cap) return true;
    if (pin) cudaFreeHost(pin);
    pin = nullptr;
    cap = 0;
    if (cudaMallocHost(&pin, bytes * 3 / 2 + 4096) != cudaSuccess) return false;
    cap = bytes * 3 / 2 + 4096;
    return true;
  }
  ~HostComm() { if (pin) cudaFreeHost(pin); }
};
ader_status host_p2p(void* ctx, int n, const int* peers, double* const* sendp, const size_t* scount,
                     double* const* recvp, const size_t* rcount, cudaStream_t st) {
  HostComm* h = (HostComm*)ctx;
  size_t tot = 0;
  for (int i = 0; i < n; ++i) tot += scount[i] + rcount[i];
  if (!h->grow(tot * sizeof(double))) return ADER_ERR_CUDA;
  std::vector<const double*> hs(n);
  std::vector<double*> hr(n);
  std::vector<int64_t> sc(n), rc(n);
  std::vector<int32_t> pe(n);
  double* b = (double*)h->pin;
  for (int i = 0; i < n; ++i) {
    hs[i] = b;
    if (scount[i] && cudaMemcpyAsync(b, sendp[i], scount[i] * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return ADER_ERR_CUDA;
    b += scount[i];
    hr[i] = b;
    b += rcount[i];
    sc[i] = (int64_t)scount[i];
    rc[i] = (int64_t)rcount[i];
    pe[i] = peers[i];
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) return ADER_ERR_CUDA;
  if (h->u.p2p(h->u.user, n, pe.data(), hs.data(), sc.data(), hr.data(), rc.data()) != 0) return ADER_ERR_NCCL;
  for (int i = 0; i < n; ++i)
    if (rcount[i] && cudaMemcpyAsync(recvp[i], hr[i], rcount[i] * sizeof(double), cudaMemcpyHostToDevice, st) != cudaSuccess)
      return ADER_ERR_CUDA;
  return cudaStreamSynchronize(st) == cudaSuccess ? ADER_OK : ADER_ERR_CUDA;
}
ader_status host_sum(void* ctx, double* buf, size_t n, cudaStream_t st) {
  HostComm* h = (HostComm*)ctx;
  if (!h->grow(n * sizeof(double))) return ADER_ERR_CUDA;
  if (cudaMemcpyAsync(h->pin, buf, n * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return ADER_ERR_CUDA;
  if (h->u.allreduce_sum(h->u.user, (double*)h->pin, (int64_t)n) != 0) return ADER_ERR_NCCL;
  if (cudaMemcpyAsync(buf, h->pin, n * sizeof(double), cudaMemcpyHostToDevice, st) != cudaSuccess) return ADER_ERR_CUDA;
  return cudaStreamSynchronize(st) == cudaSuccess ? ADER_OK : ADER_ERR_CUDA;
}
ader_status host_max_u64(void* ctx, unsigned long long* buf, cudaStream_t st) {
  HostComm* h = (HostComm*)ctx;
  if (!h->grow(sizeof(unsigned long long))) return ADER_ERR_CUDA;
  if (cudaMemcpyAsync(h->pin, buf, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return ADER_ERR_CUDA;
  if (h->u.allreduce_max_u64(h->u.user, (uint64_t*)h->pin, 1) != 0) return ADER_ERR_NCCL;
  if (cudaMemcpyAsync(buf, h->pin, sizeof(unsigned long long), cudaMemcpyHostToDevice, st) != cudaSuccess)
    return ADER_ERR_CUDA;
  return cudaStreamSynchronize(st) == cudaSuccess ? ADER_OK : ADER_ERR_CUDA;
}
}  // namespace

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
struct ProfRec { int kind; cudaEvent_t e0, e1; double flops; };

struct ader_ctx {
  ader_config cfg{};
  int d = 2, M = 2, N = 3, nv = 4, NS = 9, NST = 27, H = 3;
  long long qs = 27;                           // q block stride (nv NST rounded up to even, launch.h)
  double* pfb = nullptr;                       // face-trace buffer of the fused a2+a3 walk (pred_flux.cu)
  ader_partition_info part{};
  int n[3] = {1, 1, 1}, P[3] = {1, 1, 1};
  long long ncell = 0;
  double dx[3] = {1, 1, 1}, inv_dx[3] = {1, 1, 1};
  KCtx k{};
  cudaStream_t own_stream = nullptr;
  cudaStream_t io_stream = nullptr;            // ader_step_io: device-to-host copies of finished slabs
  cudaGraphExec_t step_graph = nullptr;        // one uniform macro step captured as a CUDA graph
  bool use_graphs = true;                      // ADER_NO_GRAPHS=1 at ader_create: direct launches (A/B)
  double graph_t_end = 0.0;                    // the t_end baked into it (k_step_dt's clip)
  long long graph_launches = 0;                // kernels per replay (launch accounting)
  std::vector<cudaEvent_t> io_ev;              // one per slab (created on first use)
  double *u = nullptr, *wx = nullptr, *wxy = nullptr, *w = nullptr, *q = nullptr, *F = nullptr;
  double *stage = nullptr;                     // compact staging buffer (set/get)
  double *sendb[6] = {}, *recvb[6] = {};       // halo buffers per side
  long long halo_cap = 0;
  DevCounters* cnt = nullptr;                  // device
  DevCounters* hcnt = nullptr;                 // pinned host mirror
  StepState* st = nullptr;                     // device step control (uniform path)
  StepState* hst = nullptr;                    // pinned host mirror
  double* cons_part = nullptr;                 // conserved-total block partials (device)
  double* cons_host = nullptr;                 // pinned host copy
  int cons_cap = 0;                            // blocks
  double t = 0.0;
  bool speed_valid = false;
  bool guess_ready = false;                    // R25: q holds the previous step's predictor of this state
  // flat cells (D = 3, M = 2): flags of the cells whose q block the predictor did not write
  // (q_h rebuilt from w by the face-flux kernel), valid while qflat_on; the dt/dx it used
  unsigned char* qflat = nullptr;
  bool qflat_on = false;
  unsigned long long flat0 = 0;                // flat_cells counter at the start of the call
  double pf_dtdx[3] = {0, 0, 0};
  const double* pf_dtdx_dev = nullptr;
  ader_ic_fn ic = nullptr;                     // the problem's IC (ADER_BC_EXACT sides, R26)
  void* ic_user = nullptr;
  bool has_exact = false;                      // a side of this rank is ADER_BC_EXACT
  double prev_dt_host = 0.0;                   // its dt (host-driven loopback steps)
  ncclComm_t comm = nullptr;
  HostComm* hostcomm = nullptr;                // collectives through host callbacks (ader_create_host_comm)
  AmrComm coll{};                              // the rank group's collectives (NCCL or host callbacks)
  bool loopback = false;                       // test-only rank group in one process (ader_debug_group_*)
  std::string err;
  // instrumentation
  bool prof = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> ev_pool;
  unsigned long long prof_sweeps0 = 0, prof_cells0 = 0;
  double kflops_sweep = 0.0;                   // predictor flops per cell per (full) sweep
  double kflops_first = 0.0;                   // the first sweep (time-constant guess: N^d flux evaluations)
  long long launches = 0;                      // kernels launched by this context
  AmrState* amr = nullptr;                     // lmax > 0: device-resident AMR
  ProfHook hook;
};

namespace {

ader_status fail(ader_ctx* c, ader_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return s;
}

#define CK(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) return fail(c, ADER_ERR_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
  } while (0)
#define NK(call)                                                                                   \
  do {                                                                                             \
    ncclResult_t r_ = (call);                                                                      \
    if (r_ != ncclSuccess) return fail(c, ADER_ERR_NCCL, "%s failed: %s", #call, g_nccl.GetErrorString(r_)); \
  } while (0)

int nvar_of(int system, int dim) { return system == ADER_MHD_GLM ? 9 : dim + 2; }

ader_status validate(const ader_config* cfg, std::string& why) {
  char b[256];
  auto bad = [&](const char* s) { why = s; return ADER_ERR_CONFIG; };
  if (cfg->abi_version != ADER_ABI_VERSION) return bad("abi_version mismatch");
  if (cfg->dim != 2 && cfg->dim != 3) return bad("dim must be 2 or 3");
  if (cfg->system != ADER_EULER && cfg->system != ADER_MHD_GLM) return bad("unknown system");
  if (cfg->degree < 2 || cfg->degree > 3) return bad("degree M must be 2 or 3");
  if (!supported(cfg->dim, cfg->degree, cfg->system)) return bad("(dim, degree, system) not compiled (3D needs M=2)");
  for (int k = 0; k < cfg->dim; ++k)
    if (cfg->n0[k] < 1) return bad("n0 must be >= 1 on every axis");
  if (cfg->dim == 2 && cfg->n0[2] != 1) return bad("n0[2] must be 1 in 2D");
  for (int k = 0; k < cfg->dim; ++k)
    if (!(cfg->hi[k] > cfg->lo[k])) return bad("hi must exceed lo");
  for (int k = 0; k < 2 * cfg->dim; ++k) {
    if (cfg->bc[k] != ADER_BC_PERIODIC && cfg->bc[k] != ADER_BC_TRANSMISSIVE && cfg->bc[k] != ADER_BC_REFLECTIVE &&
        cfg->bc[k] != ADER_BC_INFLOW && cfg->bc[k] != ADER_BC_EXACT)
      return bad("bad bc");
    if ((cfg->bc[k] == ADER_BC_INFLOW || cfg->bc[k] == ADER_BC_EXACT) && cfg->lmax > 0)
      return ADER_ERR_UNSUPPORTED;   // R23, R26: uniform grids
    if (cfg->bc[k] == ADER_BC_REFLECTIVE && cfg->system != ADER_EULER) return bad("reflective walls are Euler only");
    if (cfg->bc[k] == ADER_BC_REFLECTIVE && cfg->n0[k / 2] < cfg->degree + 1)
      return bad("a reflective axis needs at least M+1 cells");
  }
  for (int k = 0; k < cfg->dim; ++k)
    if ((cfg->bc[2 * k] == ADER_BC_PERIODIC) != (cfg->bc[2 * k + 1] == ADER_BC_PERIODIC))
      return bad("periodic bc must be set on both sides of an axis");
  if (cfg->lmax < 0 || cfg->lmax > 7) return bad("lmax out of range");
  if (cfg->lmax > 0 && cfg->refine_factor < cfg->degree) return bad("refine_factor r must be >= M (P:539-541)");
  if (cfg->lmax > 0 && cfg->refine_factor > 4) return bad("refine_factor must be <= 4");
  if (cfg->lmax > 0 && cfg->ic_quad > 4) return bad("AMR ic_quad must be <= 4");
  if (!(cfg->gamma > 1.0)) return bad("gamma must exceed 1");
  if (!(cfg->cfl > 0.0)) return bad("cfl must be positive");
  if (cfg->world_size < 1 || cfg->world_size > 8) return bad("world_size must be in 1..8");
  if (cfg->rank < 0 || cfg->rank >= cfg->world_size) return bad("rank out of range");
  if (cfg->ic_quad < 0 || cfg->ic_quad > 8) return bad("ic_quad must be in 0..8");
  if (cfg->pred_max_sweeps < 0 || cfg->pred_max_sweeps > 1000) return bad("pred_max_sweeps out of range");
  if (cfg->flux != ADER_FLUX_RUSANOV && cfg->flux != ADER_FLUX_OSHER) return bad("unknown flux");
  if (cfg->flux == ADER_FLUX_OSHER && cfg->system != ADER_EULER) return bad("the Osher flux is implemented for Euler only");
  if (cfg->flux_quad < 0 || cfg->flux_quad > 4) return bad("flux_quad must be in 0..4");
  if (cfg->load_balance < 0 || cfg->load_balance > 1) return bad("load_balance must be 0 or 1");
  if (cfg->pred_guess < 0 || cfg->pred_guess > 1) return bad("pred_guess must be 0 or 1");
  if (cfg->pred_guess == 1 && cfg->lmax > 0) return bad("pred_guess = 1 (reading R25) is for uniform grids");
  if (cfg->fuse_pred_flux < 0 || cfg->fuse_pred_flux > 1) return bad("fuse_pred_flux must be 0 or 1");
  (void)b;
  return ADER_OK;
}

// Process grid minimising the halo surface of the largest block.
void process_grid(const ader_config* cfg, int dims[3]) {
  const int ws = cfg->world_size;
  double best = 1e300;
  dims[0] = ws; dims[1] = 1; dims[2] = 1;
  for (int px = 1; px <= ws; ++px)
    for (int py = 1; px * py <= ws; ++py) {
      if (ws % (px * py)) continue;
      const int pz = ws / (px * py);
      if (cfg->dim == 2 && pz != 1) continue;
      const int p[3] = {px, py, pz};
      double e[3], surf = 0.0;
      bool ok = true;
      for (int k = 0; k < 3; ++k) {
        if (p[k] > cfg->n0[k]) ok = false;
        e[k] = std::ceil((double)cfg->n0[k] / p[k]);
      }
      if (!ok) continue;
      if (cfg->dim == 2) surf = e[0] + e[1];
      else surf = e[0] * e[1] + e[1] * e[2] + e[0] * e[2];
      if (surf < best - 1e-9) { best = surf; dims[0] = px; dims[1] = py; dims[2] = pz; }
    }
}

void partition(const ader_config* cfg, int rank, ader_partition_info* pi) {
  std::memset(pi, 0, sizeof(*pi));
  process_grid(cfg, pi->dims);
  int r = rank;
  pi->coord[0] = r % pi->dims[0]; r /= pi->dims[0];
  pi->coord[1] = r % pi->dims[1]; r /= pi->dims[1];
  pi->coord[2] = r;
  for (int k = 0; k < 3; ++k) {
    const long long n = cfg->n0[k];
    pi->lo[k] = (int)(n * pi->coord[k] / pi->dims[k]);
    pi->hi[k] = (int)(n * (pi->coord[k] + 1) / pi->dims[k]);
  }
  for (int k = 0; k < 3; ++k)
    for (int side = 0; side < 2; ++side) {
      int cc[3] = {pi->coord[0], pi->coord[1], pi->coord[2]};
      cc[k] += side ? 1 : -1;
      const bool periodic = k < cfg->dim && cfg->bc[2 * k] == ADER_BC_PERIODIC;
      if (k >= cfg->dim) { pi->nbr[2 * k + side] = -1; continue; }
      if (cc[k] < 0 || cc[k] >= pi->dims[k]) {
        if (!periodic) { pi->nbr[2 * k + side] = -1; continue; }
        cc[k] = (cc[k] + pi->dims[k]) % pi->dims[k];
      }
      pi->nbr[2 * k + side] = cc[0] + pi->dims[0] * (cc[1] + pi->dims[1] * cc[2]);
    }
  pi->halo = cfg->degree + 1;
}

Box make_box(int x0, int x1, int y0, int y1, int z0, int z1) {
  Box b;
  b.lo[0] = x0; b.lo[1] = y0; b.lo[2] = z0;
  b.ext[0] = std::max(0, x1 - x0); b.ext[1] = std::max(0, y1 - y0); b.ext[2] = std::max(0, z1 - z0);
  return b;
}

// owned block in padded coordinates
Box owned(const ader_ctx* c) {
  const int H = c->H, zH = c->d == 3 ? H : 0;
  return make_box(H, H + c->n[0], H, H + c->n[1], zH, zH + c->n[2]);
}
// block grown by g cells on every active axis
Box grown(const ader_ctx* c, int g) {
  const int H = c->H, zH = c->d == 3 ? H : 0, gz = c->d == 3 ? g : 0;
  return make_box(H - g, H + c->n[0] + g, H - g, H + c->n[1] + g, zH - gz, zH + c->n[2] + gz);
}

// ---- instrumentation -------------------------------------------------------
cudaEvent_t get_event(ader_ctx* c) {
  if (!c->ev_pool.empty()) { cudaEvent_t e = c->ev_pool.back(); c->ev_pool.pop_back(); return e; }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
struct Scope {
  ader_ctx* c; ProfRec r{};
  Scope(ader_ctx* c_, int kind, double flops) : c(c_) {
    if (!c->prof) return;
    r.kind = kind; r.flops = flops;
    r.e0 = get_event(c); r.e1 = get_event(c);
    cudaEventRecord(r.e0, c->k.stream);
  }
  ~Scope() {
    if (!c->prof) return;
    cudaEventRecord(r.e1, c->k.stream);
    c->recs.push_back(r);
  }
};

// hook used by the AMR orchestrator (amr.cpp): same records as Scope
void hook_begin(void* p, int kind) {
  ader_ctx* c = (ader_ctx*)p;
  if (!c->prof) return;
  ProfRec r{};
  r.kind = kind;
  r.e0 = get_event(c);
  r.e1 = nullptr;
  cudaEventRecord(r.e0, c->k.stream);
  c->recs.push_back(r);
}
void hook_end(void* p, int kind, double flops) {
  ader_ctx* c = (ader_ctx*)p;
  if (!c->prof || c->recs.empty() || c->recs.back().e1) return;
  ProfRec& r = c->recs.back();
  r.e1 = get_event(c);
  r.flops = flops;
  (void)kind;
  cudaEventRecord(r.e1, c->k.stream);
}

// Algorithmic FP64 flop model (FMA = 2, add/mul/div/sqrt = 1); see DESIGN.md.
double weno_problem_flops(int M) {
  const int N = M + 1, nS = (M % 2 == 0) ? 3 : 4;
  // per stencil: rec N*N FMA, sigma N*N FMA + N FMA, (sig+eps) 1 + 3 squarings + 1 div + 1 add
  // blend: 1 div, N*nS (mul + FMA)
  return nS * (2.0 * N * N + 2.0 * N * N + 2.0 * N + 6.0) + 1.0 + 3.0 * N * nS;
}
double flux_eval_flops(int sys, int d) {
  // pointwise physical fluxes in all d directions incl. the dt/dx scaling
  if (sys == ADER_EULER) return 1 + d + 2 * d + 4 + 1 + d * (d + 2) + d * (d + 2);
  return 40 + d * 30 + d * 9;
}
double pred_sweep_flops(const ader_ctx* c) {
  // NST flux evaluations + NV*NST*(2 d N [D contractions] + 2 N [T_tau] + 1 [dq])
  return c->NST * flux_eval_flops(c->cfg.system, c->d) + (double)c->nv * c->NST * (2.0 * c->d * c->N + 2.0 * c->N + 1.0);
}
double pred_first_sweep_flops(const ader_ctx* c) {
  // sweep 1 from the time-constant guess (kernels: predictor.cuh): N^d flux
  // evaluations, the D contractions on one time level (2 d N per dof), then
  // N time levels of w - Tsum_s G (2 flops) and the dq bookkeeping (1)
  return c->NS * flux_eval_flops(c->cfg.system, c->d) + (double)c->nv * c->NS * (2.0 * c->d * c->N + 3.0 * c->N);
}
double face_flops(const ader_ctx* c) {
  double two_point = (c->cfg.system == ADER_EULER) ? 2.0 * (12 + 2 * c->d) + 4.0 * c->nv : 2.0 * 90 + 4.0 * c->nv;
  if (c->cfg.flux == ADER_FLUX_OSHER) {
    // two physical fluxes, du, and per path point: the state (nv FMA) and
    // |A| du from the closed-form eigenvectors (~9 d + 50), then the blend
    const int nq = c->cfg.flux_quad > 0 ? c->cfg.flux_quad : 3;
    two_point = 2.0 * (10 + 2 * c->d) + c->nv + nq * (2.0 * c->nv + 9.0 * c->d + 50.0) + 3.0 * c->nv;
  }
  return c->NS * (4.0 * c->nv * c->N + two_point + 2.0 * c->nv + 2.0);
}

// ---- ghost layers ------------------------------------------------------------
// Ghost-layer plan of (axis, side) for a rank's block (ader_halo_desc, ader.h).
void halo_plan(int d, int H, const int n[3], const int P[3], const ader_partition_info& part, int rank,
               const int32_t* bc, int a, int side, ader_halo_desc* o) {
  std::memset(o, 0, sizeof(*o));
  o->peer = -1;
  if (a >= d) return;
  int lo[3], hi[3];
  for (int b = 0; b < 3; ++b) {
    if (b >= d) { lo[b] = 0; hi[b] = 1; continue; }
    if (b < a) { lo[b] = 0; hi[b] = P[b]; }      // processed axes: full padded extent
    else {                                       // unprocessed axes: owned extent, plus the
      lo[b] = H;                                 // inflow ghost layers (set at initialisation,
      hi[b] = H + n[b];                          // R23) so that their edges are filled too
      const bool dl = bc[2 * b] == ADER_BC_INFLOW || bc[2 * b] == ADER_BC_EXACT;
      const bool dh = bc[2 * b + 1] == ADER_BC_INFLOW || bc[2 * b + 1] == ADER_BC_EXACT;
      if (b != a && part.nbr[2 * b] < 0 && dl) lo[b] = 0;
      if (b != a && part.nbr[2 * b + 1] < 0 && dh) hi[b] = P[b];
    }
  }
  for (int b = 0; b < 3; ++b) { o->send_lo[b] = o->recv_lo[b] = lo[b]; o->send_hi[b] = o->recv_hi[b] = hi[b]; }
  if (side == 0) { o->recv_lo[a] = 0; o->recv_hi[a] = H; o->send_lo[a] = H; o->send_hi[a] = 2 * H; }
  else { o->recv_lo[a] = H + n[a]; o->recv_hi[a] = 2 * H + n[a]; o->send_lo[a] = n[a]; o->send_hi[a] = n[a] + H; }
  const int nb = part.nbr[2 * a + side];
  if (nb >= 0 && nb != rank) { o->kind = 1; o->peer = nb; }
  else if (nb >= 0 && bc[2 * a + side] == ADER_BC_PERIODIC) o->kind = 2;
  else o->kind = bc[2 * a + side] == ADER_BC_REFLECTIVE ? 4
               : (bc[2 * a + side] == ADER_BC_INFLOW ? 5 : (bc[2 * a + side] == ADER_BC_EXACT ? 6 : 3));
}

Box desc_box(const int32_t* lo, const int32_t* hi) { return make_box(lo[0], hi[0], lo[1], hi[1], lo[2], hi[2]); }

void axis_plans(const ader_ctx* c, int a, ader_halo_desc* dl, ader_halo_desc* dh) {
  halo_plan(c->d, c->H, c->n, c->P, c->part, c->cfg.rank, c->cfg.bc, a, 0, dl);
  halo_plan(c->d, c->H, c->n, c->P, c->part, c->cfg.rank, c->cfg.bc, a, 1, dh);
}

// Ghost layers of axis a in three phases: pack the slabs remote peers need,
// exchange them (NCCL, or the loopback copy of ader_debug_group_step), then
// unpack + fill the local sides.
void halo_pack(ader_ctx* c, double* u, int a) {
  ader_halo_desc dl, dh;
  axis_plans(c, a, &dl, &dh);
  if (dl.kind == 1) launch_pack(c->k, u, desc_box(dl.send_lo, dl.send_hi), c->sendb[2 * a]);
  if (dh.kind == 1) launch_pack(c->k, u, desc_box(dh.send_lo, dh.send_hi), c->sendb[2 * a + 1]);
}

ader_status halo_exchange_nccl(ader_ctx* c, int a) {
  ader_halo_desc dl, dh;
  axis_plans(c, a, &dl, &dh);
  const bool remote_lo = dl.kind == 1, remote_hi = dh.kind == 1;
  if (!remote_lo && !remote_hi) return ADER_OK;
  const size_t cnt = (size_t)desc_box(dl.recv_lo, dl.recv_hi).count() * c->nv;
  if (!c->coll.p2p) return fail(c, ADER_ERR_NCCL, "halo exchange without a communicator");
  // order on every rank: send low, recv high, send high, recv low (messages
  // between one pair of ranks then match in order, also when both neighbours
  // are the same rank)
  int peers[4];
  double* sp[4];
  double* rp[4];
  size_t sc[4], rc[4];
  int n = 0;
  auto add = [&](int peer, double* s_, size_t ns, double* r_, size_t nr) {
    peers[n] = peer; sp[n] = s_; sc[n] = ns; rp[n] = r_; rc[n] = nr; ++n;
  };
  if (remote_lo) add(dl.peer, c->sendb[2 * a], cnt, nullptr, 0);
  if (remote_hi) add(dh.peer, nullptr, 0, c->recvb[2 * a + 1], cnt);
  if (remote_hi) add(dh.peer, c->sendb[2 * a + 1], cnt, nullptr, 0);
  if (remote_lo) add(dl.peer, nullptr, 0, c->recvb[2 * a], cnt);
  const ader_status st = c->coll.p2p(c->coll.ctx, n, peers, sp, sc, rp, rc, c->k.stream);
  if (st != ADER_OK) return fail(c, st, "halo exchange (axis %d) failed", a);
  return ADER_OK;
}

void halo_unpack_local(ader_ctx* c, double* u, int a) {
  ader_halo_desc dl, dh;
  axis_plans(c, a, &dl, &dh);
  const Box rlo = desc_box(dl.recv_lo, dl.recv_hi), rhi = desc_box(dh.recv_lo, dh.recv_hi);
  if (dl.kind == 1) launch_unpack(c->k, u, rlo, c->recvb[2 * a]);
  if (dh.kind == 1) launch_unpack(c->k, u, rhi, c->recvb[2 * a + 1]);
  // local sides: periodic wrap onto ourselves, or transmissive copy (reading R5)
  auto mode = [](int kind) { return kind == 2 ? 0 : (kind == 4 ? 2 : 1); };
  // (kind 5, inflow: the ghost cells keep their initial values, R23; kind 6,
  // exact: set by refresh_exact before the step, R26)
  if (dl.kind != 1 && dl.kind != 5 && dl.kind != 6) launch_fill_axis(c->k, u, rlo, a, mode(dl.kind), c->H, c->n[a]);
  if (dh.kind != 1 && dh.kind != 5 && dh.kind != 6) launch_fill_axis(c->k, u, rhi, a, mode(dh.kind), c->H, c->n[a]);
}

ader_status fill_halo(ader_ctx* c, double* u) {
  Scope sc(c, ADER_K_HALO, 0.0);
  for (int a = 0; a < c->d; ++a) {
    halo_pack(c, u, a);
    ader_status st = halo_exchange_nccl(c, a);
    if (st != ADER_OK) return st;
    halo_unpack_local(c, u, a);
  }
  return ADER_OK;
}

// ---- one stage each ----------------------------------------------------------
void run_weno(ader_ctx* c) {
  // x sweep on the rows needed by the y (and z) sweeps, ..., last sweep on block+1
  const int H = c->H, M = c->M;
  const int zH = c->d == 3 ? H : 0;
  const int nx = c->n[0], ny = c->n[1], nz = c->n[2];
  double* dst_last = c->w;
  if (c->d == 2) {
    const Box rx = make_box(H - 1, H + nx + 1, H - 1 - M, H + ny + 1 + M, 0, 1);
    const Box ry = grown(c, 1);
    Scope s(c, ADER_K_WENO, weno_problem_flops(M) * (rx.count() * c->nv + ry.count() * c->nv * c->N));
    launch_weno_sweep(c->k, 0, c->u, c->wx, rx);
    launch_weno_sweep(c->k, 1, c->wx, dst_last, ry);
  } else {
    const Box rx = make_box(H - 1, H + nx + 1, H - 1 - M, H + ny + 1 + M, zH - 1 - M, zH + nz + 1 + M);
    const Box ry = make_box(H - 1, H + nx + 1, H - 1, H + ny + 1, zH - 1 - M, zH + nz + 1 + M);
    const Box rz = grown(c, 1);
    Scope s(c, ADER_K_WENO,
            weno_problem_flops(M) * (rx.count() * c->nv + ry.count() * c->nv * c->N + rz.count() * c->nv * c->N * c->N));
    launch_weno_sweep(c->k, 0, c->u, c->wx, rx);
    launch_weno_sweep(c->k, 1, c->wx, c->wxy, ry);
    launch_weno_sweep(c->k, 2, c->wxy, dst_last, rz);
  }
}

// Physical transmissive sides of this rank's block (bit 2a: low side of axis a).
int boundary_mask(const ader_ctx* c, int bc) {
  int m = 0;
  for (int a = 0; a < c->d; ++a) {
    if (c->part.nbr[2 * a] < 0 && c->cfg.bc[2 * a] == bc) m |= 1 << (2 * a);
    if (c->part.nbr[2 * a + 1] < 0 && c->cfg.bc[2 * a + 1] == bc) m |= 1 << (2 * a + 1);
  }
  return m;
}
int transmissive_mask(const ader_ctx* c) { return boundary_mask(c, ADER_BC_TRANSMISSIVE); }
int reflective_mask(const ader_ctx* c) { return boundary_mask(c, ADER_BC_REFLECTIVE); }

// ADER_PRED_FLAT_SKIP=1 (3D M = 2, opt-in): flat cells get a flag instead of their q block and the
// face-flux kernel rebuilds their q_h from w — bitwise the same F and state, but measured slower at
// C4 (the flux turns FP64-bound: 36 vs 29 ms), so every block is written by default
bool flat_skip_env() {
  static const bool on = (std::getenv("ADER_PRED_FLAT_SKIP") && std::getenv("ADER_PRED_FLAT_SKIP")[0] == '1') &&
                         !(std::getenv("ADER_PRED_FLAT") && std::getenv("ADER_PRED_FLAT")[0] == '0') &&
                         !(std::getenv("ADER_FLUX_TMA") && std::getenv("ADER_FLUX_TMA")[0] == '1') &&
                         !(std::getenv("ADER_FLUX_ROT") && std::getenv("ADER_FLUX_ROT")[0] == '1');
  return on;
}

void run_predictor(ader_ctx* c, double dt, const double* dtdx_dev = nullptr, bool guess = false,
                   bool allow_skip = true) {
  // owned block + the face-neighbour layer, except beyond transmissive sides (R5)
  Box r = grown(c, 1);
  const int tm = transmissive_mask(c) | reflective_mask(c);   // no predictor beyond walls either (R22)
  for (int a = 0; a < c->d; ++a) {
    if (tm & (1 << (2 * a))) { r.lo[a] += 1; r.ext[a] -= 1; }
    if (tm & (1 << (2 * a + 1))) r.ext[a] -= 1;
  }
  double dtdx[3] = {0, 0, 0};
  for (int k = 0; k < c->d; ++k) dtdx[k] = dt / c->dx[k];
  Scope s(c, ADER_K_PRED, 0.0);   // flops from the sweep counter (ader_kernel_stats)
  // reading R25: from the device step control (dt / prev_dt) in the device-driven
  // loop, else from the host's dt ratio (loopback groups)
  const bool g = guess && c->cfg.pred_guess == 1 && c->guess_ready;
  const double gr = (!dtdx_dev && c->prev_dt_host > 0.0 && dt > 0.0) ? dt / c->prev_dt_host : 0.0;
  // flat cells without a q block: not with the R25 guess (it reads the previous q blocks)
  const bool skip = allow_skip && c->qflat && c->cfg.pred_guess == 0 && flat_skip_env();
  launch_predictor(c->k, c->w, c->q, r, dtdx, c->cfg.pred_tol, c->cfg.pred_max_sweeps, c->cnt, dtdx_dev, c->qs, g,
                   dtdx_dev ? c->st : nullptr, gr, skip ? c->qflat : nullptr);
  c->qflat_on = skip;
  for (int k = 0; k < 3; ++k) c->pf_dtdx[k] = dtdx[k];
  c->pf_dtdx_dev = dtdx_dev;
  if (guess) { c->guess_ready = true; c->prev_dt_host = dt; }
}

// a1 + a2 fused (weno_pred.cu): the WENO sweeps and the predictor in one tile
// walk, w_x / w_xy / w kept on chip (ADER_WENO_PRED=0: separate kernels)
bool fused_weno_pred_env() {
  static const int on = [] {
    const char* e = std::getenv("ADER_WENO_PRED");
    return (e && e[0] == '1') ? 1 : 0;
  }();
  return on != 0;
}
// (the fused kernel has no R25 guess: pred_guess = 1 runs the separate kernels)
bool fused_weno_pred(const ader_ctx* c) { return fused_weno_pred_env() && c->cfg.pred_guess == 0; }

void run_weno_predictor(ader_ctx* c, double dt, const double* dtdx_dev = nullptr) {
  c->qflat_on = false;   // the fused walk writes every q block
  Box r = grown(c, 1);
  const int tm = transmissive_mask(c) | reflective_mask(c);   // as run_predictor (R5, R22)
  for (int a = 0; a < c->d; ++a) {
    if (tm & (1 << (2 * a))) { r.lo[a] += 1; r.ext[a] -= 1; }
    if (tm & (1 << (2 * a + 1))) r.ext[a] -= 1;
  }
  double dtdx[3] = {0, 0, 0};
  for (int k = 0; k < c->d; ++k) dtdx[k] = dt / c->dx[k];
  // algorithmic WENO flops: the problems of the three sweeps on the boxes the
  // unfused path needs (run_weno); predictor flops come from the sweep counter
  const int H = c->H, M = c->M, zH = c->d == 3 ? H : 0;
  const int nx = c->n[0], ny = c->n[1], nz = c->n[2];
  double wf;
  if (c->d == 2) {
    const Box rx = make_box(H - 1, H + nx + 1, H - 1 - M, H + ny + 1 + M, 0, 1);
    wf = weno_problem_flops(M) * (rx.count() * c->nv + r.count() * c->nv * c->N);
  } else {
    const Box rx = make_box(H - 1, H + nx + 1, H - 1 - M, H + ny + 1 + M, zH - 1 - M, zH + nz + 1 + M);
    const Box ry = make_box(H - 1, H + nx + 1, H - 1, H + ny + 1, zH - 1 - M, zH + nz + 1 + M);
    wf = weno_problem_flops(M) * (rx.count() * c->nv + ry.count() * c->nv * c->N + r.count() * c->nv * c->N * c->N);
  }
  Scope s(c, ADER_K_PRED, wf);
  launch_weno_predictor(c->k, c->u, c->q, r, c->qs, dtdx, c->cfg.pred_tol, c->cfg.pred_max_sweeps, c->cnt, dtdx_dev);
}

void face_boxes(const ader_ctx* c, Box fb[3]) {
  const int H = c->H, zH = c->d == 3 ? H : 0;
  for (int dir = 0; dir < 3; ++dir) {
    int e[3] = {c->n[0], c->n[1], c->n[2]};
    if (dir < c->d) e[dir] += 1;
    fb[dir] = make_box(H, H + e[0], H, H + e[1], zH, zH + e[2]);
    if (dir >= c->d) fb[dir] = make_box(0, 0, 0, 0, 0, 0);
  }
}

void run_flux(ader_ctx* c) {
  Box fb[3];
  face_boxes(c, fb);
  long long nf = 0;
  for (int k = 0; k < c->d; ++k) nf += fb[k].count();
  Scope s(c, ADER_K_FLUX, face_flops(c) * nf);
  const int H = c->H, zH = c->d == 3 ? H : 0;
  const Box ext = make_box(H, H + c->n[0] + 1, H, H + c->n[1] + 1, zH, zH + c->n[2] + (c->d == 3 ? 1 : 0));
  // ADER_FLUX_LEGACY=1: the round-1 kernel (direct global loads), for A/B checks
  static const bool legacy = !(std::getenv("ADER_FLUX_TMA") && std::getenv("ADER_FLUX_TMA")[0] == '1');
  // ADER_FLUX_ROT=1: coalesced block loads + warp-shuffle line sums (flux_rot.cu)
  static const bool rot = std::getenv("ADER_FLUX_ROT") && std::getenv("ADER_FLUX_ROT")[0] == '1';
  if (rot)
    launch_face_flux_rot(c->k, c->q, c->F, ext, H, c->n, transmissive_mask(c), reflective_mask(c), c->cnt, c->qs);
  else if (legacy)
    launch_face_flux_cells(c->k, c->q, c->F, ext, H, c->n, transmissive_mask(c), reflective_mask(c), c->cnt, c->qs,
                           c->qflat_on ? c->qflat : nullptr, c->w, c->pf_dtdx, c->pf_dtdx_dev);
  else
    launch_face_flux_tma(c->k, c->q, c->F, ext, H, c->n, transmissive_mask(c), reflective_mask(c), c->cnt);
}

// predictor region: the owned block + the face-neighbour layer, except beyond
// transmissive sides and walls (R5, R22)
Box predictor_region(const ader_ctx* c) {
  Box r = grown(c, 1);
  const int tm = transmissive_mask(c) | reflective_mask(c);
  for (int a = 0; a < c->d; ++a) {
    if (tm & (1 << (2 * a))) { r.lo[a] += 1; r.ext[a] -= 1; }
    if (tm & (1 << (2 * a + 1))) r.ext[a] -= 1;
  }
  return r;
}

// a2 + a3 in one tile walk (pred_flux.cu): q_h stays on chip (fuse_pred_flux = 1;
// pred_guess = 1 reads the previous q_h and keeps the separate kernels)
bool fused_pred_flux(const ader_ctx* c) {
  return c->pfb && c->cfg.fuse_pred_flux == 1 && c->cfg.pred_guess == 0 && !fused_weno_pred(c);
}

void run_pred_flux(ader_ctx* c, double dt, const double* dtdx_dev = nullptr) {
  const Box r = predictor_region(c);
  double dtdx[3] = {0, 0, 0};
  for (int k = 0; k < c->d; ++k) dtdx[k] = dt / c->dx[k];
  Box fb[3];
  face_boxes(c, fb);
  long long nf = 0;
  for (int k = 0; k < c->d; ++k) nf += fb[k].count();
  // flops: the faces' here, the Picard sweeps' from the device counters (ader_kernel_stats)
  Scope s(c, ADER_K_PRED_FLUX, face_flops(c) * nf);
  launch_pred_flux(c->k, c->w, c->F, c->pfb, r, c->H, c->n, transmissive_mask(c), reflective_mask(c),
                   c->cfg.pred_tol, c->cfg.pred_max_sweeps, c->cnt, dtdx, dtdx_dev);
  c->guess_ready = false;
}

void run_update(ader_ctx* c, double dt, const double* dtdx_dev = nullptr) {
  const Box r = owned(c);
  double dtdx[3] = {0, 0, 0};
  for (int k = 0; k < c->d; ++k) dtdx[k] = dt / c->dx[k];
  Scope s(c, ADER_K_UPDATE, (double)r.count() * c->nv * 3.0 * c->d);
  launch_update(c->k, c->u, c->F, r, dtdx, c->inv_dx, c->cnt, dtdx_dev);
}

ader_status check_errors(ader_ctx* c) {
  if (c->hcnt->err_code == 0 && c->hcnt->err_any != 0)
    return fail(c, ADER_ERR_SOLVER, "solver failure on another rank (code %llu) by t=%.17g", c->hcnt->err_any, c->t);
  if (c->hcnt->err_code == 0) return ADER_OK;
  const long long cell = (long long)c->hcnt->err_cell;
  const long long x = cell % c->P[0], y = (cell / c->P[0]) % c->P[1], z = cell / ((long long)c->P[0] * c->P[1]);
  const int zH = c->d == 3 ? c->H : 0;
  if (c->hcnt->err_code == 3)
    return fail(c, ADER_ERR_SOLVER, "invalid time step (CFL speed not positive and finite) at t=%.17g", c->t);
  const char* what = c->hcnt->err_code == 1 ? "inadmissible state (rho<=0 or p<=0)" : "predictor reached pred_max_sweeps";
  const char* stage[] = {"?", "predictor", "face flux", "update", "cfl"};
  return fail(c, ADER_ERR_SOLVER, "%s in %s at cell (%lld,%lld,%lld), level 0, t=%.17g", what,
              stage[std::min(4, std::max(0, c->hcnt->err_stage))], x - c->H + c->part.lo[0], y - c->H + c->part.lo[1],
              z - zH + c->part.lo[2], c->t);
}

// CFL speed of the current state, reduced over ranks; synchronises the stream.
ader_status global_speed(ader_ctx* c, double* speed) {
  if (!c->speed_valid) {
    CK(cudaMemsetAsync(&c->cnt->speed_bits, 0, sizeof(unsigned long long), c->k.stream));
    Scope s(c, ADER_K_OTHER, 0.0);
    launch_cfl_speed(c->k, c->u, owned(c), c->inv_dx, c->cnt);
  }
  if (c->coll.max_u64 && c->coll.max_u64(c->coll.ctx, &c->cnt->speed_bits, c->k.stream) != ADER_OK)
    return fail(c, ADER_ERR_NCCL, "allreduce(max) of the CFL speed failed");
  CK(cudaMemcpyAsync(c->hcnt, c->cnt, sizeof(DevCounters), cudaMemcpyDeviceToHost, c->k.stream));
  CK(cudaStreamSynchronize(c->k.stream));
  ader_status st = check_errors(c);
  if (st != ADER_OK) return st;
  unsigned long long b = c->hcnt->speed_bits;
  double s;
  std::memcpy(&s, &b, sizeof(s));
  *speed = s;
  c->speed_valid = true;
  return ADER_OK;
}

void free_ctx(ader_ctx* c) {
  if (!c) return;
  if (c->k.stream) cudaStreamSynchronize(c->k.stream);
  if (c->amr) amr_destroy(c->amr);
  double* bufs[] = {c->u, c->wx, c->wxy, c->w, c->q, c->F, c->stage, c->pfb};
  for (double* b : bufs)
    if (b) cudaFree(b);
  if (c->qflat) cudaFree(c->qflat);
  if (c->st) cudaFree(c->st);
  if (c->hst) cudaFreeHost(c->hst);
  if (c->cons_part) cudaFree(c->cons_part);
  if (c->cons_host) cudaFreeHost(c->cons_host);
  for (int i = 0; i < 6; ++i) {
    if (c->sendb[i]) cudaFree(c->sendb[i]);
    if (c->recvb[i]) cudaFree(c->recvb[i]);
  }
  if (c->cnt) cudaFree(c->cnt);
  if (c->hcnt) cudaFreeHost(c->hcnt);
  for (auto& r : c->recs) { if (r.e0) cudaEventDestroy(r.e0); if (r.e1) cudaEventDestroy(r.e1); }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->comm) g_nccl.CommDestroy(c->comm);
  delete c->hostcomm;
  if (c->step_graph) cudaGraphExecDestroy(c->step_graph);
  for (cudaEvent_t e : c->io_ev) cudaEventDestroy(e);
  if (c->io_stream) cudaStreamDestroy(c->io_stream);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  delete c;
}

// Gauss-Legendre rule on [0,1] for the IC averages (closed forms up to 4 points,
// Newton on the Legendre recurrence beyond).
void gl_rule(int Q, double* x, double* w) {
  if (Q == 1) { x[0] = 0.5; w[0] = 1.0; return; }
  if (Q == 2) { const double h = std::sqrt(3.0) / 6.0; x[0] = 0.5 - h; x[1] = 0.5 + h; w[0] = w[1] = 0.5; return; }
  if (Q == 3 || Q == 4) {
    DevTables t;
    build_tables(Q - 1, &t);
    for (int i = 0; i < Q; ++i) { x[i] = t.lam[i]; w[i] = t.w[i]; }
    return;
  }
  for (int i = 0; i < Q; ++i) {
    double z = -std::cos(M_PI * (i + 0.75) / (Q + 0.5)), dp = 1.0;
    for (int it = 0; it < 60; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= Q; ++k) { const double p2 = ((2 * k - 1) * z * p1 - (k - 1) * p0) / k; p0 = p1; p1 = p2; }
      dp = Q * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    x[i] = 0.5 * (1.0 + z);
    w[i] = 1.0 / ((1.0 - z * z) * dp * dp);
  }
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

static thread_local std::string g_create_err = "null context";
const char* ader_last_error(const ader_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

ader_status ader_partition(const ader_config* cfg, int32_t rank, ader_partition_info* out) {
  if (!cfg || !out) return ADER_ERR_ARG;
  std::string why;
  ader_config tmp = *cfg;
  tmp.rank = 0;
  ader_status st = validate(&tmp, why);
  if (st != ADER_OK) return st;
  if (rank < 0 || rank >= cfg->world_size) return ADER_ERR_ARG;
  partition(cfg, rank, out);
  return ADER_OK;
}

ader_status ader_rcb_partition(int32_t dim, const int32_t n0[3], const int64_t* weights, int32_t world,
                               int32_t* boxes) {
  if (!n0 || !weights || !boxes || dim < 1 || dim > 3 || world < 1 || world > 8) return ADER_ERR_ARG;
  long long n[3];
  for (int k = 0; k < 3; ++k) {
    n[k] = k < dim ? n0[k] : 1;
    if (n[k] < 1) return ADER_ERR_ARG;
  }
  const long long tot = n[0] * n[1] * n[2];
  std::vector<long long> w((size_t)tot);
  for (long long i = 0; i < tot; ++i) {
    if (weights[i] < 0) return ADER_ERR_ARG;
    w[(size_t)i] = weights[i];
  }
  int lo[8][3], hi[8][3];
  if (!rcb_partition(dim, n, w.data(), world, lo, hi)) return ADER_ERR_ARG;
  for (int p = 0; p < world; ++p)
    for (int k = 0; k < 3; ++k) { boxes[6 * p + k] = lo[p][k]; boxes[6 * p + 3 + k] = hi[p][k]; }
  return ADER_OK;
}

ader_status ader_halo_plan(const ader_config* cfg, int32_t rank, int32_t axis, int32_t side, ader_halo_desc* out) {
  if (!cfg || !out || axis < 0 || axis > 2 || side < 0 || side > 1) return ADER_ERR_ARG;
  ader_partition_info pi;
  ader_status st = ader_partition(cfg, rank, &pi);
  if (st != ADER_OK) return st;
  const int H = cfg->degree + 1;
  int n[3], P[3];
  for (int k = 0; k < 3; ++k) {
    n[k] = k < cfg->dim ? pi.hi[k] - pi.lo[k] : 1;
    P[k] = k < cfg->dim ? n[k] + 2 * H : 1;
  }
  halo_plan(cfg->dim, H, n, P, pi, rank, cfg->bc, axis, side, out);
  return ADER_OK;
}

ader_status ader_nccl_unique_id(uint8_t out[128]) {
  std::string err;
  if (!out) return ADER_ERR_ARG;
  if (!g_nccl.load(err)) return ADER_ERR_NCCL;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return ADER_ERR_NCCL;
  std::memcpy(out, &id, 128);
  return ADER_OK;
}

static ader_status create_impl(const ader_config* cfg, ader_ctx** out, bool loopback = false,
                               const ader_host_comm* hc = nullptr);

ader_status ader_create_host_comm(const ader_config* cfg, const ader_host_comm* comm, ader_ctx** out) {
  if (!cfg || !out || !comm || !comm->p2p || !comm->allreduce_sum || !comm->allreduce_max_u64) return ADER_ERR_ARG;
  *out = nullptr;
  std::string why;
  ader_status st = validate(cfg, why);
  if (st == ADER_OK && cfg->world_size < 2) { st = ADER_ERR_CONFIG; why = "ader_create_host_comm needs world_size >= 2"; }
  if (st != ADER_OK) {
    g_create_err = st == ADER_ERR_UNSUPPORTED ? "configuration not supported" : why;
    return st;
  }
  ader_ctx* c = nullptr;
  st = create_impl(cfg, &c, false, comm);
  if (st != ADER_OK) {
    g_create_err = c ? c->err : "allocation failed";
    free_ctx(c);
    return st;
  }
  *out = c;
  return ADER_OK;
}

ader_status ader_create(const ader_config* cfg, ader_ctx** out) {
  if (!cfg || !out) return ADER_ERR_ARG;
  *out = nullptr;
  std::string why;
  ader_status st = validate(cfg, why);
  if (st != ADER_OK) {
    g_create_err = st == ADER_ERR_UNSUPPORTED ? "configuration not supported (inflow boundaries need lmax = 0)" : why;
    return st;
  }
  ader_ctx* c = nullptr;
  st = create_impl(cfg, &c);
  if (st != ADER_OK) {
    g_create_err = c ? c->err : "allocation failed";
    free_ctx(c);
    return st;
  }
  *out = c;
  return ADER_OK;
}

static ader_status create_impl(const ader_config* cfg, ader_ctx** out, bool loopback, const ader_host_comm* hc) {
  ader_partition_info pi;
  partition(cfg, cfg->rank, &pi);
  const int H = cfg->degree + 1;
  for (int k = 0; k < cfg->dim; ++k) {
    const bool remote = (pi.nbr[2 * k] >= 0 && pi.nbr[2 * k] != cfg->rank) ||
                        (pi.nbr[2 * k + 1] >= 0 && pi.nbr[2 * k + 1] != cfg->rank);
    const bool wall = (pi.nbr[2 * k] < 0 && cfg->bc[2 * k] == ADER_BC_REFLECTIVE) ||
                      (pi.nbr[2 * k + 1] < 0 && cfg->bc[2 * k + 1] == ADER_BC_REFLECTIVE);
    if ((remote || wall) && pi.hi[k] - pi.lo[k] < H) {
      g_create_err = "rank block thinner than the ghost layer (M+1)";
      return ADER_ERR_CONFIG;
    }
  }
  ader_ctx* c = new ader_ctx();
  *out = c;
  c->cfg = *cfg;
  c->part = pi;
  for (int k = 0; k < 2 * c->d; ++k)
    if (pi.nbr[k] < 0 && cfg->bc[k] == ADER_BC_EXACT) c->has_exact = true;
  c->d = cfg->dim; c->M = cfg->degree; c->N = c->M + 1;
  c->nv = nvar_of(cfg->system, cfg->dim);
  c->NS = 1;
  for (int k = 0; k < c->d; ++k) c->NS *= c->N;
  c->NST = c->NS * c->N;
  c->H = H;
  if (c->cfg.pred_tol <= 0) c->cfg.pred_tol = 1e-13;
  if (c->cfg.pred_max_sweeps <= 0) c->cfg.pred_max_sweeps = 32;
  if (c->cfg.ic_quad <= 0) c->cfg.ic_quad = c->N;
  for (int k = 0; k < 3; ++k) {
    c->n[k] = (k < c->d) ? pi.hi[k] - pi.lo[k] : 1;
    c->P[k] = (k < c->d) ? c->n[k] + 2 * H : 1;
    c->dx[k] = (k < c->d) ? (cfg->hi[k] - cfg->lo[k]) / cfg->n0[k] : 1.0;
    c->inv_dx[k] = (k < c->d) ? 1.0 / c->dx[k] : 0.0;
  }
  c->ncell = (long long)c->P[0] * c->P[1] * c->P[2];
  if (cfg->lmax == 0 && (double)c->ncell * c->nv * std::pow((double)c->N, c->d - 1) >= 4294967040.0)
    return fail(c, ADER_ERR_CONFIG, "rank block of %lld padded cells exceeds the 32-bit kernel indexing; use more ranks",
                c->ncell);
  if (cfg->device >= 0) CK(cudaSetDevice(cfg->device));
  int dev = 0;
  CK(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10) {
    return fail(c, ADER_ERR_CUDA, "device %d is sm_%d%d; this library is built for sm_100a", dev, prop.major, prop.minor);
  }
  CK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
  if (!build_tables(c->M, &c->k.tab)) return fail(c, ADER_ERR_CONFIG, "no tables for M=%d", c->M);
  if (!build_osher_quadrature(cfg->flux_quad > 0 ? cfg->flux_quad : 3, &c->k.tab))
    return fail(c, ADER_ERR_CONFIG, "no path rule for flux_quad=%d", cfg->flux_quad);
  c->k.tab.flux = cfg->flux;

  c->k.D = c->d; c->k.M = c->M; c->k.SYS = cfg->system; c->k.NV = c->nv;
  c->k.sy = c->P[0]; c->k.sz = (long long)c->P[0] * c->P[1];
  c->k.ncell = c->ncell;
  c->k.gamma = cfg->gamma; c->k.ch = cfg->ch;
  c->k.stream = c->own_stream;
  c->k.launches = &c->launches;
  c->hook.ctx = c;
  c->hook.begin = hook_begin;
  c->hook.end = hook_end;
  c->k.hook = &c->hook;
  c->kflops_sweep = pred_sweep_flops(c);
  c->kflops_first = pred_first_sweep_flops(c);
  if (cfg->lmax > 0) {
    // device-resident cell-by-cell AMR (amr.cpp); uniform buffers are not used
    CK(cudaMalloc(&c->cnt, sizeof(DevCounters)));
    CK(cudaMemset(c->cnt, 0, sizeof(DevCounters)));
    CK(cudaMallocHost(&c->hcnt, sizeof(DevCounters)));
    std::memset(c->hcnt, 0, sizeof(DevCounters));
    AmrRanks ranks;
    ranks.rank = cfg->rank;
    ranks.world = cfg->world_size;
    for (int p = 0; p < cfg->world_size; ++p) {
      ader_partition_info pp;
      partition(cfg, p, &pp);
      for (int k = 0; k < 3; ++k) { ranks.lo[p][k] = pp.lo[k]; ranks.hi[p][k] = pp.hi[k]; }
    }
    AmrComm comm;
    if (cfg->world_size > 1 && !loopback && hc) {
      c->hostcomm = new HostComm();
      c->hostcomm->u = *hc;
      comm.ctx = c->hostcomm;
      comm.p2p = host_p2p;
      comm.sum = host_sum;
      comm.max_u64 = host_max_u64;
    } else if (cfg->world_size > 1 && !loopback) {
      std::string err;
      if (!g_nccl.load(err)) return fail(c, ADER_ERR_NCCL, "%s", err.c_str());
      ncclUniqueId id;
      std::memcpy(&id, cfg->nccl_id, sizeof(id));
      ncclResult_t r = g_nccl.CommInitRank(&c->comm, cfg->world_size, id, cfg->rank);
      if (r != ncclSuccess) {
        c->comm = nullptr;
        return fail(c, ADER_ERR_NCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r));
      }
      comm.ctx = c->comm;
      comm.p2p = amr_nccl_p2p;
      comm.sum = amr_nccl_sum;
      comm.max_u64 = amr_nccl_max_u64;
    }
    c->loopback = loopback;
    std::string err;
    c->amr = amr_create(cfg, &c->k, c->cnt, c->hcnt, ranks, comm, err);
    if (!c->amr) return fail(c, ADER_ERR_CUDA, "amr_create: %s", err.c_str());
    return ADER_OK;
  }
  const size_t nc = (size_t)c->ncell;
  auto alloc = [&](double** p, size_t n) { return cudaMalloc(p, n * sizeof(double)); };
  CK(alloc(&c->u, nc * c->nv));
  CK(alloc(&c->wx, nc * c->nv * c->N));
  if (c->d == 3) CK(alloc(&c->wxy, nc * c->nv * c->N * c->N));
  CK(alloc(&c->w, nc * c->nv * c->NS));
  c->qs = q_block_stride(c->d, c->M, c->cfg.system);
  CK(alloc(&c->q, nc * c->qs));
  CK(alloc(&c->F, nc * c->nv * c->d));
  if (c->d == 3 && c->M == 2 && flat_skip_env()) {   // flat-cell flags (cells outside the predictor's region stay 0)
    CK(cudaMalloc(&c->qflat, nc));
    CK(cudaMemset(c->qflat, 0, nc));
  }
  if (cfg->fuse_pred_flux == 1 && cfg->pred_guess == 0) {
    const long long nb = pred_flux_buffer_doubles(c->d, c->M, cfg->system, predictor_region(c), c->H, c->n);
    if (nb < 0) return fail(c, ADER_ERR_CUDA, "pred_flux: unsupported (d, M, system)");
    CK(alloc(&c->pfb, (size_t)std::max(1LL, nb)));
  }
  CK(alloc(&c->stage, (size_t)c->n[0] * c->n[1] * c->n[2] * std::max<size_t>(c->qs, (size_t)c->nv * c->d)));
  CK(cudaMemset(c->u, 0, nc * c->nv * sizeof(double)));
  CK(cudaMemset(c->F, 0, nc * c->nv * c->d * sizeof(double)));
  CK(cudaMalloc(&c->cnt, sizeof(DevCounters)));
  CK(cudaMemset(c->cnt, 0, sizeof(DevCounters)));
  CK(cudaMallocHost(&c->hcnt, sizeof(DevCounters)));
  std::memset(c->hcnt, 0, sizeof(DevCounters));
  CK(cudaMalloc(&c->st, sizeof(StepState)));
  CK(cudaMemset(c->st, 0, sizeof(StepState)));
  CK(cudaMallocHost(&c->hst, sizeof(StepState)));
  std::memset(c->hst, 0, sizeof(StepState));
  c->cons_cap = (int)((owned(c).count() + 255) / 256);
  CK(cudaMalloc(&c->cons_part, (size_t)c->cons_cap * c->nv * sizeof(double)));
  CK(cudaMallocHost(&c->cons_host, (size_t)c->cons_cap * c->nv * sizeof(double)));
  // halo buffers (largest slab over axes)
  long long cap = 0;
  for (int a = 0; a < c->d; ++a) {
    long long s = H;
    for (int b = 0; b < c->d; ++b)
      if (b != a) s *= c->P[b];
    cap = std::max(cap, s);
  }
  c->halo_cap = cap * c->nv;
  c->loopback = loopback;
  {
    const char* e = std::getenv("ADER_NO_GRAPHS");
    c->use_graphs = !(e && e[0] == '1');
  }
  if (cfg->world_size > 1) {
    for (int i = 0; i < 2 * c->d; ++i) {
      CK(alloc(&c->sendb[i], (size_t)c->halo_cap));
      CK(alloc(&c->recvb[i], (size_t)c->halo_cap));
    }
  }
  if (cfg->world_size > 1 && !loopback && hc) {
    c->hostcomm = new HostComm();
    c->hostcomm->u = *hc;
    c->coll.ctx = c->hostcomm;
    c->coll.p2p = host_p2p;
    c->coll.sum = host_sum;
    c->coll.max_u64 = host_max_u64;
  } else if (cfg->world_size > 1 && !loopback) {
    std::string err;
    if (!g_nccl.load(err)) return fail(c, ADER_ERR_NCCL, "%s", err.c_str());
    ncclUniqueId id;
    std::memcpy(&id, cfg->nccl_id, sizeof(id));
    ncclResult_t r = g_nccl.CommInitRank(&c->comm, cfg->world_size, id, cfg->rank);
    if (r != ncclSuccess) {
      c->comm = nullptr;
      return fail(c, ADER_ERR_NCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r));
    }
    c->coll.ctx = c->comm;
    c->coll.p2p = amr_nccl_p2p;
    c->coll.sum = amr_nccl_sum;
    c->coll.max_u64 = amr_nccl_max_u64;
  }
  c->kflops_sweep = pred_sweep_flops(c);
  c->kflops_first = pred_first_sweep_flops(c);
  return ADER_OK;
}

void ader_destroy(ader_ctx* c) { free_ctx(c); }

ader_status ader_set_stream(ader_ctx* c, void* s) {
  if (!c) return ADER_ERR_ARG;
  c->k.stream = s ? (cudaStream_t)s : c->own_stream;
  return ADER_OK;
}

double ader_time(const ader_ctx* c) { return c ? (c->amr ? amr_time(c->amr) : c->t) : 0.0; }

// Cell averages of ic(x - shift) on the box of extents ext[] at the owned-block
// offset off[] (<= 0: into the ghost layer): the host evaluates the callback
// at the ic_quad^d Gauss-Legendre points (reading R6), the GPU forms the averages.
static ader_status ic_box_average(ader_ctx* c, ader_ic_fn ic, void* user, const int off[3], const int ext[3],
                           const double shift[3]) {
  const int Q = c->cfg.ic_quad, d = c->d;
  double qx[16], qw[16];
  gl_rule(Q, qx, qw);
  int nq = 1;
  for (int k = 0; k < d; ++k) nq *= Q;
  std::vector<double> wq(nq);
  for (int g = 0; g < nq; ++g) {
    const int gi[3] = {g % Q, (g / Q) % Q, g / (Q * Q)};
    double wg = 1.0;
    for (int k = 0; k < d; ++k) wg *= qw[gi[k]];
    wq[g] = wg;
  }
  const long long ncells = (long long)ext[0] * ext[1] * ext[2];
  if (ncells == 0) return ADER_OK;
  const long long chunk = std::max<long long>(1, std::min<long long>(ncells, (1 << 22) / nq));
  std::vector<double> x((size_t)chunk * nq * 3), pr((size_t)chunk * nq * 9);
  double *dprim = nullptr, *dwq = nullptr;
  CK(cudaMalloc(&dprim, pr.size() * sizeof(double)));
  CK(cudaMalloc(&dwq, nq * sizeof(double)));
  CK(cudaMemcpy(dwq, wq.data(), nq * sizeof(double), cudaMemcpyHostToDevice));
  for (long long c0 = 0; c0 < ncells; c0 += chunk) {
    const long long ncur = std::min(chunk, ncells - c0);
    for (long long i = 0; i < ncur; ++i) {
      const long long lin = c0 + i;
      const long long ii[3] = {lin % ext[0] + off[0] + c->part.lo[0], (lin / ext[0]) % ext[1] + off[1] + c->part.lo[1],
                               lin / ((long long)ext[0] * ext[1]) + off[2] + c->part.lo[2]};
      for (int g = 0; g < nq; ++g) {
        const int gi[3] = {g % Q, (g / Q) % Q, g / (Q * Q)};
        double* xp = &x[(i * nq + g) * 3];
        for (int k = 0; k < 3; ++k)
          xp[k] = (k < d) ? (c->cfg.lo[k] + ((double)ii[k] + qx[gi[k]]) * c->dx[k]) - shift[k] : 0.0;
      }
    }
    std::fill(pr.begin(), pr.begin() + ncur * nq * 9, 0.0);
    ic(x.data(), ncur * nq, pr.data(), user);
    CK(cudaMemcpyAsync(dprim, pr.data(), (size_t)ncur * nq * 9 * sizeof(double), cudaMemcpyHostToDevice, c->k.stream));
    launch_ic_average(c->k, c->u, dprim, dwq, nq, c0, ncur, ext, c->H, off);
    CK(cudaStreamSynchronize(c->k.stream));
  }
  cudaFree(dprim);
  cudaFree(dwq);
  return ADER_OK;
}

// Reading R26: the ghost layer of every ADER_BC_EXACT side of this rank, over
// the full padded extent of the other axes, takes the averages of the exact
// solution ic(x - t exact_vel) at the step's start time t = c->t.
static ader_status refresh_exact(ader_ctx* c) {
  if (!c->has_exact || !c->ic) return ADER_OK;
  const double shift[3] = {c->t * c->cfg.exact_vel[0], c->t * c->cfg.exact_vel[1], c->t * c->cfg.exact_vel[2]};
  for (int a = 0; a < c->d; ++a)
    for (int side = 0; side < 2; ++side) {
      if (c->part.nbr[2 * a + side] >= 0 || c->cfg.bc[2 * a + side] != ADER_BC_EXACT) continue;
      int off[3] = {0, 0, 0}, ext[3] = {1, 1, 1};
      for (int k = 0; k < c->d; ++k) { off[k] = -c->H; ext[k] = c->n[k] + 2 * c->H; }
      off[a] = side ? c->n[a] : -c->H;
      ext[a] = c->H;
      ader_status st = ic_box_average(c, c->ic, c->ic_user, off, ext, shift);
      if (st != ADER_OK) return st;
    }
  return ADER_OK;
}

ader_status ader_set_initial(ader_ctx* c, ader_ic_fn ic, void* user) {
  if (!c || !ic) return ADER_ERR_ARG;
  if (c->amr && c->loopback && c->cfg.world_size > 1)
    return fail(c, ADER_ERR_ARG, "AMR group contexts are initialised through ader_debug_group_set_initial");
  if (c->amr) {
    std::string e;
    ader_status s = amr_set_initial(c->amr, ic, user, e);
    if (s != ADER_OK) c->err = e;
    return s;
  }
  c->ic = ic;
  c->ic_user = user;
  // IC box: the owned block, grown into the ghost layer on inflow and exact sides (R23, R26)
  int off[3] = {0, 0, 0}, ext[3] = {c->n[0], c->n[1], c->n[2]};
  for (int k = 0; k < c->d; ++k) {
    const bool dl = c->cfg.bc[2 * k] == ADER_BC_INFLOW || c->cfg.bc[2 * k] == ADER_BC_EXACT;
    const bool dh = c->cfg.bc[2 * k + 1] == ADER_BC_INFLOW || c->cfg.bc[2 * k + 1] == ADER_BC_EXACT;
    if (c->part.nbr[2 * k] < 0 && dl) { off[k] = -c->H; ext[k] += c->H; }
    if (c->part.nbr[2 * k + 1] < 0 && dh) ext[k] += c->H;
  }
  const double zero[3] = {0, 0, 0};
  ader_status ist = ic_box_average(c, ic, user, off, ext, zero);
  if (ist != ADER_OK) return ist;
  {
    StepState s0{};   // time restarts at 0
    CK(cudaMemcpy(c->st, &s0, sizeof(StepState), cudaMemcpyHostToDevice));
  }
  c->t = 0.0;
  c->speed_valid = false;
  c->guess_ready = false;
  return ADER_OK;
}

ader_status ader_set_cells(ader_ctx* c, const double* u_host, int64_t n_cells) {
  if (!c || !u_host) return ADER_ERR_ARG;
  if (c->amr) return fail(c, ADER_ERR_UNSUPPORTED, "ader_set_cells: uniform grids only (use ader_set_initial)");
  const Box b = owned(c);
  if (n_cells != b.count()) return fail(c, ADER_ERR_ARG, "n_cells %lld != owned %lld", (long long)n_cells, b.count());
  CK(cudaMemcpyAsync(c->stage, u_host, (size_t)n_cells * c->nv * sizeof(double), cudaMemcpyHostToDevice, c->k.stream));
  launch_scatter(c->k, c->u, c->nv, b, c->stage);
  CK(cudaStreamSynchronize(c->k.stream));
  c->speed_valid = false;
  c->guess_ready = false;   // R25: a new state has no previous step
  return ADER_OK;
}

ader_status ader_get_state(const ader_ctx* cc, double* u_host, int64_t capacity) {
  ader_ctx* c = const_cast<ader_ctx*>(cc);
  if (!c || !u_host) return ADER_ERR_ARG;
  if (c->amr) return fail(c, ADER_ERR_UNSUPPORTED, "ader_get_state: uniform grids only (use ader_get_cells)");
  const Box b = owned(c);
  if (capacity < b.count()) return fail(c, ADER_ERR_ARG, "capacity too small");
  launch_gather(c->k, c->u, c->nv, b, c->stage);
  CK(cudaMemcpyAsync(u_host, c->stage, (size_t)b.count() * c->nv * sizeof(double), cudaMemcpyDeviceToHost, c->k.stream));
  CK(cudaStreamSynchronize(c->k.stream));
  return ADER_OK;
}

ader_status ader_get_cells(const ader_ctx* cc, ader_cell* out, int64_t capacity, int64_t* n) {
  ader_ctx* c = const_cast<ader_ctx*>(cc);
  if (!c || !n) return ADER_ERR_ARG;
  if (c->amr) {
    std::string e;
    ader_status s = amr_get_cells(c->amr, out, capacity, n, e);
    if (s != ADER_OK) c->err = e;
    return s;
  }
  const Box b = owned(c);
  *n = b.count();
  if (!out) return ADER_OK;
  if (capacity < b.count()) return fail(c, ADER_ERR_ARG, "capacity too small");
  std::vector<double> u((size_t)b.count() * c->nv);
  ader_status st = ader_get_state(c, u.data(), b.count());
  if (st != ADER_OK) return st;
  long long i = 0;
  for (int z = 0; z < c->n[2]; ++z)
    for (int y = 0; y < c->n[1]; ++y)
      for (int x = 0; x < c->n[0]; ++x, ++i) {
        ader_cell& e = out[i];
        std::memset(&e, 0, sizeof(e));
        e.level = 0; e.status = 0;
        e.idx[0] = x + c->part.lo[0]; e.idx[1] = y + c->part.lo[1]; e.idx[2] = z + c->part.lo[2];
        for (int v = 0; v < c->nv; ++v) e.u[v] = u[i * c->nv + v];
      }
  return ADER_OK;
}

namespace {
// second half of a uniform macro step, after the ghost fill + WENO: predictor,
// face fluxes, update (fused with the next CFL speed)
void advance_dt(ader_ctx* c, double dt, const double* dtdx_dev = nullptr) {
  if (fused_pred_flux(c)) run_pred_flux(c, dt, dtdx_dev);
  else {
    if (fused_weno_pred(c)) run_weno_predictor(c, dt, dtdx_dev);
    else run_predictor(c, dt, dtdx_dev, true);
    run_flux(c);
  }
  cudaMemsetAsync(&c->cnt->speed_bits, 0, sizeof(unsigned long long), c->k.stream);
  run_update(c, dt, dtdx_dev);
  c->speed_valid = true;   // computed by the update of the new state
  c->t += dt;
}

// Tail of a macro step for ader_step_io: face fluxes and the update in K slabs
// along the last axis, each finished slab of the owned state gathered and
// copied to the host on a second stream while the next slabs' fluxes run.
// The update of slab i needs the lower faces of slab i+1's first level, so
// the order is flux(0), flux(1), update(0), copy(0), flux(2), update(1), ...
// Same kernels and arithmetic as run_flux + run_update: bitwise the same state.
ader_status tail_to_host(ader_ctx* c, const double* dtdx_dev, double* out_host) {
  const int W = c->d - 1, H = c->H, zH = c->d == 3 ? H : 0;
  const int lo = (W == 2) ? zH : H, nW = c->n[W];
  const int K = std::max(1, std::min(8, nW / 8));
  if (!c->io_stream) CK(cudaStreamCreateWithFlags(&c->io_stream, cudaStreamNonBlocking));
  while ((int)c->io_ev.size() < K + 1) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->io_ev.push_back(e);
  }
  auto cut = [&](int i) { return lo + (int)((long long)nW * i / K); };
  Box fb[3];
  face_boxes(c, fb);
  long long nf = 0;
  for (int k = 0; k < c->d; ++k) nf += fb[k].count();
  const double fl_per_face = face_flops(c);
  const long long plane = (long long)c->n[0] * (c->d == 3 ? c->n[1] : 1);   // owned cells per level of W
  auto flux = [&](int i) {
    Box e = make_box(H, H + c->n[0] + 1, H, H + c->n[1] + 1, zH, zH + c->n[2] + (c->d == 3 ? 1 : 0));
    e.lo[W] = cut(i);
    e.ext[W] = cut(i + 1) - cut(i) + (i + 1 == K ? 1 : 0);
    Scope s(c, ADER_K_FLUX, fl_per_face * (double)nf * e.ext[W] / (nW + 1));
    launch_face_flux_cells(c->k, c->q, c->F, e, H, c->n, transmissive_mask(c), reflective_mask(c), c->cnt, c->qs,
                           c->qflat_on ? c->qflat : nullptr, c->w, c->pf_dtdx, c->pf_dtdx_dev);
  };
  auto update_copy = [&](int i) -> ader_status {
    Box r = owned(c);
    r.lo[W] = cut(i);
    r.ext[W] = cut(i + 1) - cut(i);
    {
      Scope s(c, ADER_K_UPDATE, (double)r.count() * c->nv * 3.0 * c->d);
      double dtdx[3] = {0, 0, 0};
      launch_update(c->k, c->u, c->F, r, dtdx, c->inv_dx, c->cnt, dtdx_dev);
    }
    const long long off = (long long)(cut(i) - lo) * plane * c->nv;
    launch_gather(c->k, c->u, c->nv, r, c->stage + off);
    CK(cudaEventRecord(c->io_ev[i], c->k.stream));
    CK(cudaStreamWaitEvent(c->io_stream, c->io_ev[i], 0));
    CK(cudaMemcpyAsync(out_host + off, c->stage + off, (size_t)r.count() * c->nv * sizeof(double),
                       cudaMemcpyDeviceToHost, c->io_stream));
    return ADER_OK;
  };
  flux(0);
  for (int i = 0; i < K; ++i) {
    if (i + 1 < K) flux(i + 1);
    ader_status st = update_copy(i);
    if (st != ADER_OK) return st;
  }
  // later work on the compute stream (and its syncs) also covers the copies
  CK(cudaEventRecord(c->io_ev[K], c->io_stream));
  CK(cudaStreamWaitEvent(c->k.stream, c->io_ev[K], 0));
  c->speed_valid = true;
  return ADER_OK;
}

// One macro step enqueued without a host round trip: ghost layers, WENO, the
// CFL speed (from the previous update, or a CFL kernel), NCCL max over ranks,
// dt on the device (k_step_dt), predictor, fluxes, update.
ader_status enqueue_step(ader_ctx* c, double t_end, double* out_host = nullptr, bool head_done = false) {
  const bool fused = fused_weno_pred(c);
  if (!head_done) {
    ader_status st = fill_halo(c, c->u);
    if (st != ADER_OK) return st;
    if (!fused) run_weno(c);
  }
  {
    Scope sc(c, ADER_K_OTHER, 0.0);
    if (!c->speed_valid) {
      CK(cudaMemsetAsync(&c->cnt->speed_bits, 0, sizeof(unsigned long long), c->k.stream));
      launch_cfl_speed(c->k, c->u, owned(c), c->inv_dx, c->cnt);
    }
    if (c->coll.max_u64 && c->coll.max_u64(c->coll.ctx, &c->cnt->speed_bits, c->k.stream) != ADER_OK)
      return fail(c, ADER_ERR_NCCL, "allreduce(max) of the CFL speed failed");
    launch_step_dt(c->k, c->cnt, c->st, c->cfg.cfl, t_end, c->dx);
  }
  const bool chunked = out_host && !fused_pred_flux(c);
  if (fused_pred_flux(c)) run_pred_flux(c, 0.0, c->st->dtdx);
  else {
    if (fused) run_weno_predictor(c, 0.0, c->st->dtdx);
    else run_predictor(c, 0.0, c->st->dtdx, true);
    if (!chunked) run_flux(c);
  }
  CK(cudaMemsetAsync(&c->cnt->speed_bits, 0, sizeof(unsigned long long), c->k.stream));
  if (chunked) return tail_to_host(c, c->st->dtdx, out_host);
  run_update(c, 0.0, c->st->dtdx);
  c->speed_valid = true;
  if (out_host) {   // fused walk: the whole state after the update
    const Box b = owned(c);
    launch_gather(c->k, c->u, c->nv, b, c->stage);
    CK(cudaMemcpyAsync(out_host, c->stage, (size_t)b.count() * c->nv * sizeof(double), cudaMemcpyDeviceToHost,
                       c->k.stream));
  }
  return ADER_OK;
}

// host mirror of the step control (synchronises the stream).  With several
// ranks the error code is max-reduced first (err_any), so a solver failure on
// one rank stops every rank at the same chunk boundary instead of leaving the
// others blocked in the next step's collectives.
ader_status read_state(ader_ctx* c) {
  if (c->coll.max_u64) {
    CK(cudaMemsetAsync(&c->cnt->err_any, 0, sizeof(unsigned long long), c->k.stream));
    CK(cudaMemcpyAsync(&c->cnt->err_any, &c->cnt->err_code, sizeof(int), cudaMemcpyDeviceToDevice, c->k.stream));
    if (c->coll.max_u64(c->coll.ctx, &c->cnt->err_any, c->k.stream) != ADER_OK)
      return fail(c, ADER_ERR_NCCL, "allreduce(max) of the error code failed");
  }
  CK(cudaMemcpyAsync(c->hst, c->st, sizeof(StepState), cudaMemcpyDeviceToHost, c->k.stream));
  CK(cudaMemcpyAsync(c->hcnt, c->cnt, sizeof(DevCounters), cudaMemcpyDeviceToHost, c->k.stream));
  CK(cudaStreamSynchronize(c->k.stream));
  c->t = c->hst->t;
  return ADER_OK;
}


ader_status step_begin(ader_ctx* c, unsigned long long* sw0, unsigned long long* pc0) {
  CK(cudaMemcpyAsync(c->hcnt, c->cnt, sizeof(DevCounters), cudaMemcpyDeviceToHost, c->k.stream));
  CK(cudaStreamSynchronize(c->k.stream));
  *sw0 = c->hcnt->sweeps;
  *pc0 = c->hcnt->cells;
  c->flat0 = c->hcnt->flat_cells;
  return ADER_OK;
}

ader_status step_finish(ader_ctx* c, ader_status st, ader_step_report* r, unsigned long long sw0,
                        unsigned long long pc0) {
  CK(cudaMemcpyAsync(c->hcnt, c->cnt, sizeof(DevCounters), cudaMemcpyDeviceToHost, c->k.stream));
  CK(cudaStreamSynchronize(c->k.stream));
  if (st == ADER_OK) st = check_errors(c);
  r->t = c->t;
  r->cell_updates = r->macro_steps * owned(c).count();
  r->updates_per_level[0] = r->cell_updates;
  r->pred_sweeps_total = (int64_t)(c->hcnt->sweeps - sw0);
  r->pred_cells = (int64_t)(c->hcnt->cells - pc0);
  r->pred_flat_cells = (int64_t)(c->hcnt->flat_cells - c->flat0);
  r->pred_sweeps_max = c->hcnt->sweeps_max;
  // conserved totals (diagnostic): block partials on device, summed in order here
  const Box b = owned(c);
  double vol = 1.0;
  for (int k = 0; k < c->d; ++k) vol *= c->dx[k];
  // (buffers allocated at ader_create: a cudaMalloc / cudaFree here stalled the
  // stream for hundreds of ms on some boxes)
  const int maxb = (int)((b.count() + 255) / 256);
  if (c->cons_part && maxb <= c->cons_cap) {
    const int nb = launch_cons_partials(c->k, c->u, b, vol, c->cons_part, maxb);
    CK(cudaMemcpyAsync(c->cons_host, c->cons_part, (size_t)nb * c->nv * sizeof(double), cudaMemcpyDeviceToHost,
                       c->k.stream));
    CK(cudaStreamSynchronize(c->k.stream));
    for (int i = 0; i < nb; ++i)
      for (int v = 0; v < c->nv; ++v) r->cons_total[v] += c->cons_host[(size_t)i * c->nv + v];
  }
  return st;
}

// Reading R1: dt = CFL / speed, clipped to t_end.
ader_status dt_from_speed(ader_ctx* c, double speed, double t_end, double* dt) {
  double v = c->cfg.cfl / speed;
  if (!(v > 0.0) || !std::isfinite(v)) return fail(c, ADER_ERR_SOLVER, "invalid dt %g at t=%.17g", v, c->t);
  if (c->t + v > t_end) v = t_end - c->t;
  *dt = v;
  return ADER_OK;
}
}  // namespace

// One uniform macro step as a CUDA graph (the steady state: CFL speed from the
// previous update, no host work between steps), replayed for every step of a
// chunk: the ~20 kernels of a step (ghost fills, WENO sweeps, dt, predictor,
// fluxes, update) launch as one graph, which removes the per-launch host cost
// that bounds small grids.  Used when nothing needs the host per step: one
// rank, no exact-solution sides, profiling off, not the fused WENO+predictor
// experiment.  Re-captured when t_end changes (k_step_dt clips against it).
bool graphs_ok(const ader_ctx* c) {
  return c->use_graphs && !c->prof && c->cfg.world_size == 1 && !c->loopback && !c->has_exact && !fused_weno_pred(c) &&
         c->cfg.pred_guess == 0 && c->speed_valid;
}

ader_status enqueue_step_graph(ader_ctx* c, double t_end) {
  if (c->step_graph && c->graph_t_end != t_end) {
    cudaGraphExecDestroy(c->step_graph);
    c->step_graph = nullptr;
  }
  if (!c->step_graph) {
    const long long l0 = c->launches;
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(c->k.stream, cudaStreamCaptureModeThreadLocal));
    ader_status st = enqueue_step(c, t_end);
    cudaError_t e = cudaStreamEndCapture(c->k.stream, &g);
    if (st != ADER_OK) { if (g) cudaGraphDestroy(g); return st; }
    CK(e);
    e = cudaGraphInstantiate(&c->step_graph, g, 0);
    cudaGraphDestroy(g);
    CK(e);
    c->graph_t_end = t_end;
    c->graph_launches = c->launches - l0;
    c->launches = l0;
  }
  CK(cudaGraphLaunch(c->step_graph, c->k.stream));
  c->launches += c->graph_launches;
  return ADER_OK;
}

// Head of an ader_step_io step with a new host state (one rank, periodic /
// transmissive / reflective sides): the state arrives in K slabs along the last
// axis W on the copy stream, and as each slab lands the compute stream
// scatters it, fills its ghost cells along the other axes, runs the WENO
// sweeps along those axes on its levels and takes its CFL speed; after the
// last slab the ghost levels along W are filled, swept, and the sweep along W
// runs on all levels.  The same kernels on the same cells as fill_halo +
// run_weno + the CFL kernel, so the step is bitwise unchanged; the copy-in
// overlaps all but the last slab's sweeps.
bool pipelined_head_ok(const ader_ctx* c) {
  if (c->cfg.world_size > 1 || fused_weno_pred(c) || c->has_exact) return false;
  for (int k = 0; k < 2 * c->d; ++k)
    if (c->cfg.bc[k] == ADER_BC_INFLOW || c->cfg.bc[k] == ADER_BC_EXACT) return false;
  // worth it for states the copy takes milliseconds on (the slab launches cost ~0.1 ms)
  // (ADER_STEP_IO_PIPELINE=1 forces it for small states: tests)
  const char* e = std::getenv("ADER_STEP_IO_PIPELINE");
  return c->n[c->d - 1] >= 16 && (owned(c).count() * c->nv * 8 >= (64LL << 20) || (e && e[0] == '1'));
}

ader_status head_from_host(ader_ctx* c, const double* in_host) {
  const int d = c->d, W = d - 1, H = c->H, M = c->M, zH = d == 3 ? H : 0;
  const int lo = (W == 2) ? zH : H, nW = c->n[W];
  const int K = std::max(1, std::min(8, nW / 8));
  if (!c->io_stream) CK(cudaStreamCreateWithFlags(&c->io_stream, cudaStreamNonBlocking));
  while ((int)c->io_ev.size() < 2 * K + 2) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->io_ev.push_back(e);
  }
  auto cut = [&](int i) { return lo + (int)((long long)nW * i / K); };
  const long long plane = (long long)c->n[0] * (d == 3 ? c->n[1] : 1);
  const int nx = c->n[0], ny = c->n[1], nz = c->n[2];
  // the sweeps' boxes (run_weno); per slab restricted to its owned levels of W
  Box rx, ry;
  if (d == 2) rx = make_box(H - 1, H + nx + 1, H - 1 - M, H + ny + 1 + M, 0, 1);
  else {
    rx = make_box(H - 1, H + nx + 1, H - 1 - M, H + ny + 1 + M, zH - 1 - M, zH + nz + 1 + M);
    ry = make_box(H - 1, H + nx + 1, H - 1, H + ny + 1, zH - 1 - M, zH + nz + 1 + M);
  }
  auto restrict_w = [&](Box b, int a, int e) { b.lo[W] = a; b.ext[W] = e - a; return b; };
  const double pf = weno_problem_flops(M) * c->nv;
  // the ordering of run_weno's sweeps is kept per level: x before y on a level
  // (3D); the copy-in of slab i+1 overlaps the work on slab i
  auto enqueue_copy = [&](int i) -> ader_status {
    Box r = owned(c);
    r.lo[W] = cut(i);
    r.ext[W] = cut(i + 1) - cut(i);
    const long long off = (long long)(cut(i) - lo) * plane * c->nv;
    if (i == 0) CK(cudaEventRecord(c->io_ev[2 * K], c->k.stream));   // stage free (previous users done)
    CK(cudaStreamWaitEvent(c->io_stream, c->io_ev[2 * K], 0));
    CK(cudaMemcpyAsync(c->stage + off, in_host + off, (size_t)r.count() * c->nv * sizeof(double),
                       cudaMemcpyHostToDevice, c->io_stream));
    CK(cudaEventRecord(c->io_ev[i], c->io_stream));
    return ADER_OK;
  };
  for (int i = 0; i < K; ++i) {
    ader_status st = enqueue_copy(i);
    if (st != ADER_OK) return st;
  }
  CK(cudaMemsetAsync(&c->cnt->speed_bits, 0, sizeof(unsigned long long), c->k.stream));
  int wdone = lo + M;   // levels [lo + M, wdone) of the sweep along W are done
  for (int i = 0; i < K; ++i) {
    Box r = owned(c);
    r.lo[W] = cut(i);
    r.ext[W] = cut(i + 1) - cut(i);
    const long long off = (long long)(cut(i) - lo) * plane * c->nv;
    CK(cudaStreamWaitEvent(c->k.stream, c->io_ev[i], 0));
    launch_scatter(c->k, c->u, c->nv, r, c->stage + off);
    {
      Scope s(c, ADER_K_HALO, 0.0);
      for (int a = 0; a < W; ++a) {   // local ghost fills of the other axes on these levels
        ader_halo_desc dl, dh;
        axis_plans(c, a, &dl, &dh);
        auto mode = [](int kind) { return kind == 2 ? 0 : (kind == 4 ? 2 : 1); };
        Box rl = restrict_w(desc_box(dl.recv_lo, dl.recv_hi), cut(i), cut(i + 1));
        Box rh = restrict_w(desc_box(dh.recv_lo, dh.recv_hi), cut(i), cut(i + 1));
        launch_fill_axis(c->k, c->u, rl, a, mode(dl.kind), H, c->n[a]);
        launch_fill_axis(c->k, c->u, rh, a, mode(dh.kind), H, c->n[a]);
      }
    }
    {
      const Box bx = restrict_w(rx, cut(i), cut(i + 1));
      Scope s(c, ADER_K_WENO, pf * (bx.count() + (d == 3 ? (double)restrict_w(ry, cut(i), cut(i + 1)).count() * c->N : 0.0)));
      launch_weno_sweep(c->k, 0, c->u, c->wx, bx);
      if (d == 3) launch_weno_sweep(c->k, 1, c->wx, c->wxy, restrict_w(ry, cut(i), cut(i + 1)));
    }
    {
      Scope s(c, ADER_K_OTHER, 0.0);
      launch_cfl_speed(c->k, c->u, r, c->inv_dx, c->cnt);
    }
    // the sweep along W on the levels whose 2M+1 window is in (no ghost levels)
    const int wb = cut(i + 1) - M;
    if (wb > wdone) {
      const Box bz = restrict_w(grown(c, 1), wdone, wb);
      Scope s(c, ADER_K_WENO, pf * bz.count() * (d == 3 ? c->N * c->N : c->N));
      launch_weno_sweep(c->k, W, d == 3 ? c->wxy : c->wx, c->w, bz);
      wdone = wb;
    }
  }
  c->speed_valid = true;
  // ghost levels along W, their sweeps, then the sweep along W on all levels
  {
    Scope s(c, ADER_K_HALO, 0.0);
    ader_halo_desc dl, dh;
    axis_plans(c, W, &dl, &dh);
    auto mode = [](int kind) { return kind == 2 ? 0 : (kind == 4 ? 2 : 1); };
    launch_fill_axis(c->k, c->u, desc_box(dl.recv_lo, dl.recv_hi), W, mode(dl.kind), H, c->n[W]);
    launch_fill_axis(c->k, c->u, desc_box(dh.recv_lo, dh.recv_hi), W, mode(dh.kind), H, c->n[W]);
  }
  {
    const int glo = (d == 3 ? zH : H) - 1 - M, ghi = lo + nW + 1 + M;
    const Box b0 = restrict_w(rx, glo, lo), b1 = restrict_w(rx, lo + nW, ghi);
    // the sweep along W on the levels left: [lo - 1, lo + M) and [wdone, lo + nW + 1)
    const Box z0 = restrict_w(grown(c, 1), lo - 1, lo + M), z1 = restrict_w(grown(c, 1), wdone, lo + nW + 1);
    const double per = d == 3 ? c->N * c->N : c->N;
    double fl = pf * (b0.count() + b1.count()) + pf * per * (z0.count() + z1.count());
    if (d == 3) fl += pf * c->N * (restrict_w(ry, glo, lo).count() + restrict_w(ry, lo + nW, ghi).count());
    Scope s(c, ADER_K_WENO, fl);
    launch_weno_sweep(c->k, 0, c->u, c->wx, b0);
    launch_weno_sweep(c->k, 0, c->u, c->wx, b1);
    if (d == 3) {
      launch_weno_sweep(c->k, 1, c->wx, c->wxy, restrict_w(ry, glo, lo));
      launch_weno_sweep(c->k, 1, c->wx, c->wxy, restrict_w(ry, lo + nW, ghi));
    }
    launch_weno_sweep(c->k, W, d == 3 ? c->wxy : c->wx, c->w, z0);
    launch_weno_sweep(c->k, W, d == 3 ? c->wxy : c->wx, c->w, z1);
  }
  c->guess_ready = false;
  return ADER_OK;
}

ader_status ader_step_io(ader_ctx* c, const double* in_host, double* out_host, double t_end, ader_step_report* rep) {
  if (!c || !out_host) return ADER_ERR_ARG;
  const auto w0 = std::chrono::steady_clock::now();
  if (c->loopback) return fail(c, ADER_ERR_ARG, "group contexts step through ader_debug_group_step");
  if (c->amr) return fail(c, ADER_ERR_UNSUPPORTED, "ader_step_io: uniform grids only (use ader_step + ader_get_cells)");
  const Box b = owned(c);
  const bool pipe = in_host && pipelined_head_ok(c);
  if (in_host && !pipe) {
    CK(cudaMemcpyAsync(c->stage, in_host, (size_t)b.count() * c->nv * sizeof(double), cudaMemcpyHostToDevice,
                       c->k.stream));
    launch_scatter(c->k, c->u, c->nv, b, c->stage);
    c->speed_valid = false;
    c->guess_ready = false;
  }
  ader_step_report r;
  std::memset(&r, 0, sizeof(r));
  unsigned long long sw0 = 0, pc0 = 0;
  ader_status st = step_begin(c, &sw0, &pc0);
  if (st != ADER_OK) return st;
  st = read_state(c);
  if (st != ADER_OK) return st;
  const long long steps0 = c->hst->steps;
  if (pipe) {   // the copy-in overlaps the ghost fill and sweeps of the slabs already in
    st = head_from_host(c, in_host);
    if (st == ADER_OK && c->t < t_end) st = enqueue_step(c, t_end, out_host, true);
    else if (st == ADER_OK) {
      launch_gather(c->k, c->u, c->nv, b, c->stage);
      CK(cudaMemcpyAsync(out_host, c->stage, (size_t)b.count() * c->nv * sizeof(double), cudaMemcpyDeviceToHost,
                         c->k.stream));
    }
  } else if (c->t < t_end) {
    if (c->has_exact) st = refresh_exact(c);
    if (st == ADER_OK) st = enqueue_step(c, t_end, out_host);
  } else {
    launch_gather(c->k, c->u, c->nv, b, c->stage);
    CK(cudaMemcpyAsync(out_host, c->stage, (size_t)b.count() * c->nv * sizeof(double), cudaMemcpyDeviceToHost,
                       c->k.stream));
  }
  if (st == ADER_OK) st = read_state(c);
  r.macro_steps = c->hst->steps - steps0;
  r.dt0 = c->hst->last_dt;
  r.min_threshold_margin = 1e300;
  st = step_finish(c, st, &r, sw0, pc0);
  r.wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
  if (rep) *rep = r;
  return st;
}

ader_status ader_step(ader_ctx* c, double t_end, int64_t max_macro_steps, ader_step_report* rep) {
  if (!c) return ADER_ERR_ARG;
  const auto w0 = std::chrono::steady_clock::now();
  if (c->loopback) return fail(c, ADER_ERR_ARG, "group contexts step through ader_debug_group_step");
  if (c->amr) {
    std::string e;
    ader_status s = amr_step(c->amr, t_end, max_macro_steps, rep, e);
    if (s != ADER_OK) c->err = e;
    if (rep) rep->wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
    return s;
  }
  ader_step_report r;
  std::memset(&r, 0, sizeof(r));
  unsigned long long sw0 = 0, pc0 = 0;
  ader_status st = step_begin(c, &sw0, &pc0);
  if (st != ADER_OK) return st;
  st = read_state(c);
  if (st != ADER_OK) return st;
  const long long steps0 = c->hst->steps;
  // enqueue the steps in chunks; dt lives on the device, the host only checks
  // time / errors between chunks (steps past t_end are no-ops, dt = 0)
  // (exact boundaries, R26: one step per chunk, the host refreshes their ghost
  // layers at each step's start time)
  const int64_t chunk = c->has_exact ? 1 : 16;
  int64_t enq = 0;
  while (enq < max_macro_steps && c->t < t_end) {
    const int64_t nstep = std::min<int64_t>(chunk, max_macro_steps - enq);
    const auto h0 = std::chrono::steady_clock::now();
    if (c->has_exact) st = refresh_exact(c);
    for (int64_t i = 0; i < nstep && st == ADER_OK; ++i)
      st = graphs_ok(c) ? enqueue_step_graph(c, t_end) : enqueue_step(c, t_end);
    if (st != ADER_OK) break;
    enq += nstep;
    const auto h1 = std::chrono::steady_clock::now();
    st = read_state(c);
    if (std::getenv("ADER_GAP_TRACE"))
      std::fprintf(stderr, "step chunk: %lld steps enqueued in %.3f ms, read-back after %.3f ms\n", (long long)nstep,
                   std::chrono::duration<double, std::milli>(h1 - h0).count(),
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h1).count());
    if (st != ADER_OK) break;
    if (c->hcnt->err_code || c->hcnt->err_any) break;
  }
  if (st == ADER_OK) st = read_state(c);
  r.macro_steps = c->hst->steps - steps0;
  r.dt0 = c->hst->last_dt;
  r.min_threshold_margin = 1e300;   // uniform grid: no adapt
  st = step_finish(c, st, &r, sw0, pc0);
  r.wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
  if (rep) *rep = r;
  return st;
}

// Test-only rank group in one process (ader.h): the ranks of a partition share
// one GPU and step in lockstep; the halo slabs that NCCL would carry are copied
// device to device between the contexts, the CFL max is taken on the host.
ader_status ader_debug_group_create(const ader_config* cfg, int32_t n, ader_ctx** out) {
  if (!cfg || !out || n < 1 || n > 8) return ADER_ERR_ARG;
  for (int i = 0; i < n; ++i) out[i] = nullptr;
  for (int i = 0; i < n; ++i) {
    ader_config ci = *cfg;
    ci.rank = i;
    ci.world_size = n;
    std::string why;
    ader_status st = validate(&ci, why);
    if (st == ADER_OK) st = create_impl(&ci, &out[i], true);
    if (st != ADER_OK) {
      g_create_err = out[i] ? out[i]->err : why;
      for (int j = 0; j <= i; ++j) { free_ctx(out[j]); out[j] = nullptr; }
      return st;
    }
  }
  return ADER_OK;
}

ader_status ader_debug_group_set_initial(ader_ctx** cs, int32_t n, ader_ic_fn ic, void* user) {
  if (!cs || n < 1 || !ic) return ADER_ERR_ARG;
  for (int i = 0; i < n; ++i)
    if (!cs[i] || !cs[i]->loopback || cs[i]->cfg.world_size != n || cs[i]->cfg.rank != i ||
        (cs[i]->amr != nullptr) != (cs[0]->amr != nullptr))
      return ADER_ERR_ARG;
  if (!cs[0]->amr) {
    for (int i = 0; i < n; ++i) {
      ader_status s = ader_set_initial(cs[i], ic, user);
      if (s != ADER_OK) return s;
    }
    return ADER_OK;
  }
  std::vector<AmrState*> g(n);
  for (int i = 0; i < n; ++i) g[i] = cs[i]->amr;
  std::string e;
  ader_status s = amr_group_set_initial(g.data(), n, ic, user, e);
  if (s != ADER_OK) cs[0]->err = e;
  return s;
}

ader_status ader_debug_group_step(ader_ctx** cs, int32_t n, double t_end, int64_t max_macro_steps,
                                  ader_step_report* reps) {
  if (!cs || n < 1) return ADER_ERR_ARG;
  for (int i = 0; i < n; ++i)
    if (!cs[i] || !cs[i]->loopback || cs[i]->cfg.world_size != n || cs[i]->cfg.rank != i) return ADER_ERR_ARG;
  ader_ctx* c = cs[0];
  if (c->amr) {
    std::vector<AmrState*> g(n);
    for (int i = 0; i < n; ++i) {
      if (!cs[i]->amr) return ADER_ERR_ARG;
      g[i] = cs[i]->amr;
    }
    std::string e;
    ader_status s = amr_group_step(g.data(), n, t_end, max_macro_steps, reps, e);
    if (s != ADER_OK) c->err = e;
    return s;
  }
  const int d = c->d;
  std::vector<ader_step_report> r(n);
  std::vector<unsigned long long> sw0(n), pc0(n);
  ader_status st = ADER_OK;
  for (int i = 0; i < n && st == ADER_OK; ++i) {
    std::memset(&r[i], 0, sizeof(r[i]));
    st = step_begin(cs[i], &sw0[i], &pc0[i]);
  }
  auto sync_all = [&]() {
    for (int i = 0; i < n; ++i) cudaStreamSynchronize(cs[i]->k.stream);
  };
  int64_t steps = 0;
  while (st == ADER_OK && steps < max_macro_steps && c->t < t_end) {
    for (int i = 0; i < n && st == ADER_OK; ++i) st = refresh_exact(cs[i]);   // R26
    if (st != ADER_OK) break;
    for (int a = 0; a < d; ++a) {
      for (int i = 0; i < n; ++i) halo_pack(cs[i], cs[i]->u, a);
      sync_all();
      for (int i = 0; i < n; ++i) {
        ader_halo_desc dl, dh;
        axis_plans(cs[i], a, &dl, &dh);
        const size_t bytes = (size_t)desc_box(dl.recv_lo, dl.recv_hi).count() * cs[i]->nv * sizeof(double);
        // my low ghosts = the low neighbour's high slab, my high ghosts = the high neighbour's low slab
        if (dl.kind == 1)
          cudaMemcpyAsync(cs[i]->recvb[2 * a], cs[dl.peer]->sendb[2 * a + 1], bytes, cudaMemcpyDeviceToDevice,
                          cs[i]->k.stream);
        if (dh.kind == 1)
          cudaMemcpyAsync(cs[i]->recvb[2 * a + 1], cs[dh.peer]->sendb[2 * a], bytes, cudaMemcpyDeviceToDevice,
                          cs[i]->k.stream);
      }
      sync_all();
      for (int i = 0; i < n; ++i) halo_unpack_local(cs[i], cs[i]->u, a);
    }
    double speed = 0.0;
    for (int i = 0; i < n && st == ADER_OK; ++i) {
      if (!fused_weno_pred(cs[i])) run_weno(cs[i]);
      double s = 0.0;
      st = global_speed(cs[i], &s);   // no communicator: this rank's max
      speed = std::max(speed, s);
    }
    if (st != ADER_OK) break;
    double dt = 0.0;
    st = dt_from_speed(c, speed, t_end, &dt);
    if (st != ADER_OK) break;
    for (int i = 0; i < n; ++i) {
      advance_dt(cs[i], dt);
      r[i].dt0 = dt;
      r[i].macro_steps++;
    }
    ++steps;
  }
  for (int i = 0; i < n; ++i) {
    ader_status s2 = step_finish(cs[i], st, &r[i], sw0[i], pc0[i]);
    if (st == ADER_OK && s2 != ADER_OK) { st = s2; if (i) c->err = cs[i]->err; }
    if (reps) reps[i] = r[i];
  }
  return st;
}

ader_status ader_refine(ader_ctx* c, ader_step_report* rep) {
  if (!c) return ADER_ERR_ARG;
  if (rep) { std::memset(rep, 0, sizeof(*rep)); rep->min_threshold_margin = 1e300; }
  if (c->loopback && c->cfg.world_size > 1) return fail(c, ADER_ERR_ARG, "group contexts adapt inside ader_debug_group_step");
  if (c->amr) {
    std::string e;
    ader_status s = amr_adapt(c->amr, rep, e);
    if (s != ADER_OK) c->err = e;
    return s;
  }
  return ADER_OK;   // uniform grid: nothing to adapt
}

ader_status ader_set_profiling(ader_ctx* c, int32_t on) {
  if (!c) return ADER_ERR_ARG;
  CK(cudaStreamSynchronize(c->k.stream));
  for (auto& r : c->recs) { if (r.e0) c->ev_pool.push_back(r.e0); if (r.e1) c->ev_pool.push_back(r.e1); }
  c->recs.clear();
  c->prof = on != 0;
  CK(cudaMemcpy(c->hcnt, c->cnt, sizeof(DevCounters), cudaMemcpyDeviceToHost));
  c->prof_sweeps0 = c->hcnt->sweeps;
  c->prof_cells0 = c->hcnt->cells;
  return ADER_OK;
}

ader_status ader_kernel_stats(ader_ctx* c, double ms[ADER_K_COUNT], int64_t launches[ADER_K_COUNT],
                              double flops[ADER_K_COUNT]) {
  if (!c) return ADER_ERR_ARG;
  CK(cudaStreamSynchronize(c->k.stream));
  for (int i = 0; i < ADER_K_COUNT; ++i) {
    if (ms) ms[i] = 0.0;
    if (launches) launches[i] = 0;
    if (flops) flops[i] = 0.0;
  }
  for (auto& r : c->recs) {
    float t = 0.f;
    if (!r.e1) continue;
    CK(cudaEventElapsedTime(&t, r.e0, r.e1));
    if (ms) ms[r.kind] += t;
    if (launches) launches[r.kind] += 1;
    if (flops) flops[r.kind] += r.flops;
  }
  CK(cudaMemcpy(c->hcnt, c->cnt, sizeof(DevCounters), cudaMemcpyDeviceToHost));
  // predictor flops from the device counters: every predicted cell's first
  // sweep at its real cost, the later sweeps as full sweeps (plus, for the fused
  // WENO + predictor kernel, the WENO flops its scopes carry)
  // (fused a2 + a3 walk: its scopes carry the face flops, the sweeps are added here)
  if (flops) {
    const double cells = (double)(c->hcnt->cells - c->prof_cells0);
    const double sweeps = (double)(c->hcnt->sweeps - c->prof_sweeps0);
    int np = 0, npf = 0;
    for (auto& r : c->recs) {
      if (!r.e1) continue;
      np += r.kind == ADER_K_PRED;
      npf += r.kind == ADER_K_PRED_FLUX;
    }
    flops[(np == 0 && npf > 0) ? ADER_K_PRED_FLUX : ADER_K_PRED] +=
        cells * c->kflops_first + (sweeps - cells) * c->kflops_sweep;
  }
  if (std::getenv("ADER_GAP_TRACE") && c->recs.size() > 1) {
    // diagnostics: idle gaps of the stream between consecutive timed scopes
    std::vector<std::pair<float, int>> gaps;
    double tot = 0.0;
    for (size_t i = 1; i < c->recs.size(); ++i) {
      if (!c->recs[i - 1].e1 || !c->recs[i].e0) continue;
      float g = 0.f;
      if (cudaEventElapsedTime(&g, c->recs[i - 1].e1, c->recs[i].e0) != cudaSuccess) continue;
      tot += g;
      gaps.push_back({g, (int)i});
    }
    std::sort(gaps.begin(), gaps.end(), [](auto& a, auto& b) { return a.first > b.first; });
    std::fprintf(stderr, "gap trace: %zu scopes, idle between scopes %.3f ms; largest:", c->recs.size(), tot);
    for (size_t j = 0; j < gaps.size() && j < 6; ++j)
      std::fprintf(stderr, " %.3f ms before scope %d (kind %d)", gaps[j].first, gaps[j].second,
                   c->recs[gaps[j].second].kind);
    std::fprintf(stderr, "\n");
  }
  return ADER_OK;
}

ader_status ader_launch_count(const ader_ctx* c, int64_t* n) {
  if (!c || !n) return ADER_ERR_ARG;
  *n = c->launches;
  return ADER_OK;
}

int64_t ader_sizeof(int32_t what) {
  switch (what) {
    case 0: return (int64_t)sizeof(ader_config);
    case 1: return (int64_t)sizeof(ader_step_report);
    case 2: return (int64_t)sizeof(ader_cell);
    case 3: return (int64_t)sizeof(ader_partition_info);
    case 4: return (int64_t)sizeof(ader_halo_desc);
    default: return -1;
  }
}

ader_status ader_debug_dump(ader_ctx* c, int32_t what, double dt, double* out, int64_t capacity) {
  if (!c || !out) return ADER_ERR_ARG;
  if (c->amr) return fail(c, ADER_ERR_UNSUPPORTED, "ader_debug_dump: uniform grids only");
  if (c->loopback) return fail(c, ADER_ERR_ARG, "ader_debug_dump: not on a loopback group context");
  const Box b = owned(c);
  ader_status st = fill_halo(c, c->u);
  if (st != ADER_OK) return st;
  run_weno(c);
  if (what == 0) {
    if (capacity < b.count() * c->nv * c->NS) return fail(c, ADER_ERR_ARG, "capacity too small");
    launch_gather(c->k, c->w, c->nv * c->NS, b, c->stage);
    CK(cudaMemcpyAsync(out, c->stage, (size_t)b.count() * c->nv * c->NS * sizeof(double), cudaMemcpyDeviceToHost, c->k.stream));
    CK(cudaStreamSynchronize(c->k.stream));
    return ADER_OK;
  }
  // FLUX stage of the fused a2 + a3 walk: the fluxes come from the walk (q_h is
  // never stored there); the PRED stage always runs the separate predictor
  const bool walk = what == 2 && fused_pred_flux(c);
  if (walk) {
    CK(cudaMemsetAsync(c->F, 0, (size_t)c->ncell * c->nv * c->d * sizeof(double), c->k.stream));
    run_pred_flux(c, dt);
  } else if (fused_weno_pred(c)) run_weno_predictor(c, dt);
  else run_predictor(c, dt, nullptr, false, what != 1);   // the PRED dump needs every q block
  c->guess_ready = false;   // q no longer holds the last step's predictor
  if (what == 1) {
    if (capacity < b.count() * c->nv * c->NST) return fail(c, ADER_ERR_ARG, "capacity too small");
    launch_gather(c->k, c->q, (int)c->qs, b, c->stage);
    const size_t row = (size_t)c->nv * c->NST * sizeof(double);
    CK(cudaMemcpy2DAsync(out, row, c->stage, (size_t)c->qs * sizeof(double), row, (size_t)b.count(),
                         cudaMemcpyDeviceToHost, c->k.stream));
    CK(cudaStreamSynchronize(c->k.stream));
    CK(cudaMemcpy(c->hcnt, c->cnt, sizeof(DevCounters), cudaMemcpyDeviceToHost));
    return check_errors(c);
  }
  if (what == 2) {
    if (!walk) {
      CK(cudaMemsetAsync(c->F, 0, (size_t)c->ncell * c->nv * c->d * sizeof(double), c->k.stream));
      run_flux(c);
    }
    const int zH = c->d == 3 ? c->H : 0;
    const Box e = make_box(c->H, c->H + c->n[0] + 1, c->H, c->H + c->n[1] + 1, zH, zH + c->n[2] + (c->d == 3 ? 1 : 0));
    if (capacity < e.count() * c->nv * c->d) return fail(c, ADER_ERR_ARG, "capacity too small");
    double* tmp = nullptr;
    CK(cudaMalloc(&tmp, (size_t)e.count() * c->nv * sizeof(double)));
    for (int dir = 0; dir < c->d; ++dir) {
      launch_gather(c->k, c->F + (size_t)dir * c->ncell * c->nv, c->nv, e, tmp);
      CK(cudaMemcpyAsync(out + (size_t)dir * e.count() * c->nv, tmp, (size_t)e.count() * c->nv * sizeof(double),
                         cudaMemcpyDeviceToHost, c->k.stream));
    }
    CK(cudaStreamSynchronize(c->k.stream));
    cudaFree(tmp);
    CK(cudaMemcpy(c->hcnt, c->cnt, sizeof(DevCounters), cudaMemcpyDeviceToHost));
    return check_errors(c);
  }
  return ADER_ERR_ARG;
}

}  // extern "C"
