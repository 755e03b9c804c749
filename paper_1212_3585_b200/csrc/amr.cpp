// amr.cpp — host orchestration of the device-resident AMR (see amr.h).
//
// The tree topology (status, links) is mirrored here because the adapt rules
// are integer logic on a few hundred thousand cells once per macro step; all
// floating-point work runs on the GPU.  The adapt follows the same readings
// as DESIGN.md R14-R20 (order-independent closure, simultaneous recoarsening
// that the closure may revert, GC), written independently of oracle/.
// Citations: P:n = PAPER.md line n.
#include "amr.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace ader {

namespace {
struct HCell {
  int level = 0, status = 0, mother = -1, child = -1;
  long long idx[3] = {0, 0, 0};
  bool alive = false, isnew = false;
};

// one pending device initialisation of a cell's average
struct Init { int cell, mother, mode; };   // mode 0: WENO sub-box, 1: q_h at tau=1, 2: IC
}  // namespace

struct AmrState {
  ader_config cfg{};
  KCtx* k = nullptr;
  DevCounters* cnt = nullptr;
  DevCounters* hcnt = nullptr;
  int d = 2, M = 2, N = 3, nv = 4, NS = 9, NST = 27, r = 3, rd = 9, lmax = 1;
  long long n[kAmrMaxLevels][3]{};
  double dx[kAmrMaxLevels][3]{};
  std::vector<HCell> cells;
  std::vector<int> free_blocks;                       // first ids of freed r^d blocks
  std::vector<std::vector<int>> hmap;                 // dense id maps per level
  int cap = 0;
  AmrDevView V{};
  int* dmap[kAmrMaxLevels]{};
  int* dlist = nullptr;
  long long dlist_cap = 0;
  // lists (host) and their offsets inside dlist
  // (dlist: the active lists of all levels first, so that their concatenation
  // is the all-levels active list at oall = 0; one rank: owned = active)
  std::vector<int> lact[kAmrMaxLevels], lvch[kAmrMaxLevels], lvmo[kAmrMaxLevels];
  long long oact[kAmrMaxLevels]{}, ovch[kAmrMaxLevels]{}, ovmo[kAmrMaxLevels]{}, oall = 0, nall = 0;
  // reconstruction work lists: the active cells of a level split into sibling patches (mother ids,
  // amr_launch_weno_patches) and the cells reconstructed from their own box (amr_launch_weno)
  std::vector<int> lwc[kAmrMaxLevels], lwp[kAmrMaxLevels];
  long long owc[kAmrMaxLevels]{}, owp[kAmrMaxLevels]{};
  SubTables st{};
  double t = 0.0;
  ader_ic_fn ic = nullptr;
  void* user = nullptr;
  std::vector<Init> inits;
  std::vector<int> chi_ids;
  std::vector<double> chi;
  long long updates[kAmrMaxLevels]{};
  std::string err;
  // incremental uploads: the tree as the device last saw it, staging buffers
  std::vector<HCell> mirror;
  char* dscratch = nullptr;
  size_t dscratch_cap = 0;
  char* hstage = nullptr;
  size_t hstage_cap = 0;
  // multi-rank (amr.h): ownership, compute set, owned active lists, exchange plans
  AmrRanks ranks;
  AmrComm comm;
  int band = 0;                                       // compute-set margin in level-0 cells
  bool band_sets = false;                             // ADER_AMR_BAND=1: the uniform band instead of R28 sets
  std::vector<int> lpres[kAmrMaxLevels];              // active cells whose averages this rank holds (multi-rank)
  // multi-rank: rows of w / q only for the cells this rank computes (R28);
  // a cell keeps its row while it stays computed, rows of cells that leave
  // are released one list rebuild later (the adapt's new-cell initialisation
  // still reads the refined mothers' w / q); row 0 is scratch for the rest
  std::vector<int> slot_of, slot_defer, free_slots;
  int nslots = 1, slot_cap = 0;
  std::vector<char> own, comp;                        // per id
  long long nlev[kAmrMaxLevels]{};                    // alive cells per level (whole tree)
  std::vector<int> lown[kAmrMaxLevels];               // owned active cells (multi-rank)
  long long nown[kAmrMaxLevels]{}, oownall = 0, nownall = 0;
  struct XPlan {                                      // per level, ids ascending per peer
    std::vector<int> sids, rids;
    std::vector<long long> soff, roff;                // [world + 1] offsets into sids / rids
    long long dso = 0, dro = 0;                       // their offsets inside dlist
  } xp[kAmrMaxLevels];
  double margin = 1e300;      // min threshold margin of the adapts since the last reset (report)
  double* rb_buf = nullptr;   // dynamic load balancing: per-id averages and gather scratch,
  double* rb_tmp = nullptr;   // kept across rebalances and grown 2x when the id space grows
  size_t rb_cap = 0;          // (doubles)
  double* xsend = nullptr;
  double* xrecv = nullptr;
  size_t xcap = 0;                                    // doubles
  // ids whose record changed since the last upload (upload_topology then
  // compares only those with the device mirror)
  std::vector<int> dirty;
  std::vector<char> isdirty;
  bool all_dirty = true;
  // undo journal of the tentative recoarsening (instead of copying the tree)
  bool jon = false;
  std::vector<std::pair<int, HCell>> jcells;          // (id, previous value)
  std::vector<std::pair<std::pair<int, long long>, int>> jmap;   // ((level, linear index), previous id)
  // host-side phase timers (seconds), printed at destroy if ADER_AMR_TIMING is set
  double tm_speed = 0, tm_advance = 0, tm_check = 0, tm_ind = 0, tm_apply = 0, tm_exch = 0;
  double tm_a[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // adapt_apply sub-phases
  double tm_u[4] = {0, 0, 0, 0};                // upload_topology: capacity, host scans, staging
  long long tm_steps = 0;
  int nrebal = 0;                               // dynamic load-balancing repartitions (R24)
};

namespace {

#define ACK(call)                                                                        \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) { err = std::string(#call) + ": " + cudaGetErrorString(e_); return ADER_ERR_CUDA; } \
  } while (0)

double now_s() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

// Persistent host worker threads for the O(cells) scans of the tree mirror
// (spawning std::threads per scan cost more than the scans below 256k ids).
class HostPool {
 public:
  static HostPool& get() {
    static HostPool p;
    return p;
  }
  int size() const { return (int)workers_.size() + 1; }
  // fn(t) for t in [0, T), t = 0 on the calling thread; returns when all are done
  void run(int T, const std::function<void(int)>& fn) {
    T = std::max(1, std::min(T, size()));
    if (T == 1) { fn(0); return; }
    {
      std::lock_guard<std::mutex> g(m_);
      job_ = &fn;
      njob_ = T;
      pending_ = T - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> g(m_);
    done_.wait(g, [&] { return pending_ == 0; });
    job_ = nullptr;
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

 private:
  HostPool() {
    const unsigned hc = std::thread::hardware_concurrency();
    const int n = (int)std::max(1u, std::min(8u, hc ? hc : 1u)) - 1;
    for (int w = 0; w < n; ++w) workers_.emplace_back([this, w] { loop(w + 1); });
  }
  void loop(int id) {
    long seen = 0;
    for (;;) {
      const std::function<void(int)>* job;
      int nj;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        job = job_;
        nj = njob_;
      }
      if (job && id < nj) {
        (*job)(id);
        std::lock_guard<std::mutex> g(m_);
        if (--pending_ == 0) done_.notify_all();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int njob_ = 0, pending_ = 0;
  long gen_ = 0;
  bool stop_ = false;
};

// host threads for a scan of n ids (one below 16k ids; ADER_HOST_THREADS caps it, A/B)
int host_threads(int n) {
  static const int cap = [] {
    const char* e = std::getenv("ADER_HOST_THREADS");
    return e ? std::max(1, std::atoi(e)) : 64;
  }();
  if (n < (1 << 14) || cap == 1) return 1;
  return std::min(cap, HostPool::get().size());
}

// fn(t, i0, i1) on T contiguous chunks of [0, n), chunk 0 on the calling thread
template <class F>
void parallel_chunks(int n, int T, F fn) {
  if (T <= 1) { fn(0, 0, n); return; }
  HostPool::get().run(T, [&](int t) { fn(t, (int)((long long)n * t / T), (int)((long long)n * (t + 1) / T)); });
}

double lagrange(const DevTables& T, int N, int p, double x) {
  double v = 1.0;
  for (int k = 0; k < N; ++k)
    if (k != p) v *= (x - T.lam[k]) / (T.lam[p] - T.lam[k]);
  return v;
}

void build_sub(const DevTables& T, int N, int r, SubTables* S) {
  std::memset(S, 0, sizeof(*S));
  S->r = r;
  for (int c = 0; c < r; ++c) {
    for (int p = 0; p < N; ++p) {
      // r * int_{c/r}^{(c+1)/r} psi_p = sum_k w_k psi_p((c + lam_k)/r)  (exact, degree M)
      double acc = 0.0;
      for (int k = 0; k < N; ++k) acc += T.w[k] * lagrange(T, N, p, (c + T.lam[k]) / r);
      S->Psub[c][p] = acc;
    }
    for (int k = 0; k < N; ++k)
      for (int p = 0; p < N; ++p) S->Esub[c][k][p] = lagrange(T, N, p, (c + T.lam[k]) / r);
  }
}

// CUDA-event scope through the context's instrumentation hook
struct AScope {
  const AmrState* A; int kind; double fl;
  AScope(const AmrState* a, int k, double f) : A(a), kind(k), fl(f) {
    if (A->k->hook && A->k->hook->begin) A->k->hook->begin(A->k->hook->ctx, kind);
  }
  ~AScope() {
    if (A->k->hook && A->k->hook->end) A->k->hook->end(A->k->hook->ctx, kind, fl);
  }
};

long long lin(const AmrState* A, int l, const long long* ix) { return (ix[2] * A->n[l][1] + ix[1]) * A->n[l][0] + ix[0]; }

// level-0 ancestor index of a cell
void ancestor0(const AmrState* A, const HCell& C, long long a[3]) {
  long long f = 1;
  for (int l = 0; l < C.level; ++l) f *= A->r;
  for (int k = 0; k < 3; ++k) a[k] = k < A->d ? C.idx[k] / f : 0;
}

int owner_of(const AmrState* A, const long long a[3]) {
  for (int p = 0; p < A->ranks.world; ++p) {
    bool in = true;
    for (int k = 0; k < A->d && in; ++k) in = a[k] >= A->ranks.lo[p][k] && a[k] < A->ranks.hi[p][k];
    if (in) return p;
  }
  return -1;
}

// is level-0 cell a within `band` cells (per axis, periodic wrap) of rank p's block?
bool in_comp(const AmrState* A, int p, const long long a[3]) {
  for (int k = 0; k < A->d; ++k) {
    const long long lo = A->ranks.lo[p][k], hi = A->ranks.hi[p][k] - 1, n0 = A->n[0][k];
    const bool per = A->cfg.bc[2 * k] == ADER_BC_PERIODIC;
    long long best = -1;
    for (int sh = per ? -1 : 0; sh <= (per ? 1 : 0); ++sh) {
      const long long x = a[k] + sh * n0;
      const long long dd = x < lo ? lo - x : (x > hi ? x - hi : 0);
      if (best < 0 || dd < best) best = dd;
    }
    if (best > A->band) return false;
  }
  return true;
}

int hlookup(const AmrState* A, int l, const long long* ix0, bool skip_outside) {
  long long ix[3] = {ix0[0], ix0[1], ix0[2]};
  for (int k = 0; k < A->d; ++k) {
    const long long nn = A->n[l][k];
    if (ix[k] < 0 || ix[k] >= nn) {
      const int side = ix[k] < 0 ? 0 : 1;
      if (A->cfg.bc[2 * k + side] == ADER_BC_PERIODIC) ix[k] = ((ix[k] % nn) + nn) % nn;
      else {
        if (skip_outside) return -1;
        ix[k] = ix[k] < 0 ? 0 : nn - 1;
      }
    }
  }
  if (A->d == 2) ix[2] = 0;
  return A->hmap[l][lin(A, l, ix)];
}

int voronoi(const AmrState* A, int id, int* out) {
  const HCell& C = A->cells[id];
  int cnt = 0;
  const int zl = A->d == 3 ? -1 : 0, zh = A->d == 3 ? 1 : 0;
  for (int dz = zl; dz <= zh; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        if (!dx && !dy && !dz) continue;
        const long long ix[3] = {C.idx[0] + dx, C.idx[1] + dy, C.idx[2] + dz};
        out[cnt++] = hlookup(A, C.level, ix, true);
      }
  return cnt;
}

// ---- multi-rank compute sets from the dependencies of the owned updates ------
// (reading R28; replaces the uniform 2(M+1) level-0 band).  Bit p of the masks
// = rank p.  With an exchange of the owners' active averages after every level
// update, a rank must itself compute (WENO + predictor + flux/update):
//   P  its owned active cells; the active face neighbours of owned cells and the
//      active mothers of virtual-child face neighbours (their q_h enter the
//      owned faces); the active fine cells across the faces of the virtual
//      children of owned cells (they deposit the flux memory the owned update
//      consumes, eqn.memory.sum); the active mothers of virtual children inside
//      the WENO box of any P cell (projection), recursively;
// and must hold current averages of
//   R  the active cells in the (2M+1)^d WENO boxes of P cells and below the
//      virtual mothers in them (received from their owners after each update);
//   V  the virtual cells in those boxes (projected / averaged locally, R16).
// Every rank evaluates the masks of all ranks on its copy of the tree (the
// result is the same everywhere), so both sides of an exchange agree.
// Cells whose neighbourhood lies inside their owner's block only carry their
// owner's bit; work is done near block boundaries (dist0) and for cells that
// received foreign bits.
struct RankSets {
  std::vector<unsigned char> P, R, V;
  std::vector<signed char> owner;     // per id, -1 for dead ids
};

void rank_sets(const AmrState* A, RankSets& S) {
  const int nu = (int)A->cells.size(), d = A->d, M = A->M, W = A->ranks.world;
  S.P.assign(nu, 0); S.R.assign(nu, 0); S.V.assign(nu, 0); S.owner.assign(nu, -1);
  // owner of every level-0 cell, and its Chebyshev distance (capped) to the
  // nearest level-0 cell of another owner (periodic wrap)
  const long long n0x = A->n[0][0], n0y = A->n[0][1], n0z = A->n[0][2], n0 = n0x * n0y * n0z;
  std::vector<signed char> own0(n0);
  for (long long z = 0; z < n0z; ++z)
    for (long long y = 0; y < n0y; ++y)
      for (long long x = 0; x < n0x; ++x) {
        const long long a[3] = {x, y, z};
        own0[(z * n0y + y) * n0x + x] = (signed char)owner_of(A, a);
      }
  auto wrap0 = [&](long long c, int k, bool& ok) -> long long {
    const long long nn = A->n[0][k];
    if (c >= 0 && c < nn) return c;
    if (A->cfg.bc[2 * k + (c < 0 ? 0 : 1)] != ADER_BC_PERIODIC) { ok = false; return 0; }
    return ((c % nn) + nn) % nn;
  };
  // does the box of level-0 ancestors [alo, ahi] (per axis, wrapped) hold a cell not owned by o?
  auto foreign_in = [&](const long long* alo, const long long* ahi, int o) {
    for (long long z = alo[2]; z <= ahi[2]; ++z)
      for (long long y = alo[1]; y <= ahi[1]; ++y)
        for (long long x = alo[0]; x <= ahi[0]; ++x) {
          bool ok = true;
          const long long xx = wrap0(x, 0, ok), yy = d > 1 ? wrap0(y, 1, ok) : 0, zz = d > 2 ? wrap0(z, 2, ok) : 0;
          if (ok && own0[(zz * n0y + yy) * n0x + xx] != o) return true;
        }
    return false;
  };
  // cells whose level-l box of radius rad may reach a foreign level-0 cell
  auto near_foreign = [&](const HCell& C, int rad, int o) {
    long long f = 1;
    for (int l = 0; l < C.level; ++l) f *= A->r;
    long long alo[3] = {0, 0, 0}, ahi[3] = {0, 0, 0};
    for (int k = 0; k < d; ++k) {
      const long long lo = C.idx[k] - rad, hi = C.idx[k] + rad;
      alo[k] = lo >= 0 ? lo / f : -((-lo + f - 1) / f);
      ahi[k] = hi >= 0 ? hi / f : -((-hi + f - 1) / f);
    }
    return foreign_in(alo, ahi, o);
  };
  for (int i = 0; i < nu; ++i) {
    const HCell& C = A->cells[i];
    if (!C.alive) continue;
    long long a0[3];
    ancestor0(A, C, a0);
    S.owner[i] = own0[(a0[2] * n0y + a0[1]) * n0x + a0[0]];
    const unsigned char ob = (unsigned char)(1u << S.owner[i]);
    if (C.status == 0) S.P[i] = ob;
    else S.V[i] = ob;
  }
  (void)W;
  std::vector<int> work;
  auto addP = [&](int c, unsigned char m) {
    if ((S.P[c] | m) != S.P[c]) { S.P[c] |= m; work.push_back(c); }
  };
  // face neighbours of owned cells near a foreign block
  for (int i = 0; i < nu; ++i) {
    const HCell& C = A->cells[i];
    if (!C.alive || C.status != 0 || !near_foreign(C, 1, S.owner[i])) continue;
    const unsigned char ob = (unsigned char)(1u << S.owner[i]);
    for (int dir = 0; dir < d; ++dir)
      for (int side = 0; side < 2; ++side) {
        long long ix[3] = {C.idx[0], C.idx[1], C.idx[2]};
        ix[dir] += side ? 1 : -1;
        const int nb = hlookup(A, C.level, ix, true);
        if (nb < 0 || S.owner[nb] == S.owner[i]) continue;
        const HCell& Nb = A->cells[nb];
        if (Nb.status == 0) addP(nb, ob);
        else if (Nb.status == 1) addP(Nb.mother, ob);
        else if (C.child >= 0) {
          // the fine cells across this face from our virtual children deposit our flux memory
          for (int q = 0; q < A->rd; ++q) {
            const HCell& K = A->cells[C.child + q];
            const long long off = K.idx[dir] - C.idx[dir] * A->r;
            if (off != (side ? A->r - 1 : 0)) continue;
            long long jx[3] = {K.idx[0], K.idx[1], K.idx[2]};
            jx[dir] += side ? 1 : -1;
            const int f = hlookup(A, K.level, jx, true);
            if (f >= 0 && A->cells[f].status == 0) addP(f, ob);
          }
        }
      }
  }
  // WENO boxes: owner-only P cells whose box may reach a foreign block, and
  // every cell that received foreign bits
  for (int i = 0; i < nu; ++i) {
    const HCell& C = A->cells[i];
    if (C.alive && C.status == 0 && S.P[i] == (unsigned char)(1u << S.owner[i]) && near_foreign(C, M, S.owner[i]))
      work.push_back(i);
  }
  std::vector<int> stack;
  while (!work.empty()) {
    const int p = work.back();
    work.pop_back();
    const unsigned char m = S.P[p];
    const HCell& C = A->cells[p];
    const int zr = d == 3 ? M : 0, yr = d >= 2 ? M : 0;
    for (int dz = -zr; dz <= zr; ++dz)
      for (int dy = -yr; dy <= yr; ++dy)
        for (int dx = -M; dx <= M; ++dx) {
          const long long ix[3] = {C.idx[0] + dx, C.idx[1] + dy, C.idx[2] + dz};
          const int b = hlookup(A, C.level, ix, false);
          if (b < 0) continue;
          const HCell& B = A->cells[b];
          if (B.status == 0) { S.R[b] |= m; continue; }
          S.V[b] |= m;
          if (B.status == 1) { addP(B.mother, m); continue; }
          // virtual mother: everything below it is averaged into it
          stack.push_back(b);
          while (!stack.empty()) {
            const int v = stack.back();
            stack.pop_back();
            const int ch = A->cells[v].child;
            if (ch < 0) continue;
            for (int q = 0; q < A->rd; ++q) {
              const HCell& K = A->cells[ch + q];
              if (K.status == 0) S.R[ch + q] |= m;
              else if (K.status == -1) { S.V[ch + q] |= m; stack.push_back(ch + q); }
            }
          }
        }
  }
}

// writable cell / map entry; records the previous value while journaling
HCell& wcell(AmrState* A, int i) {
  if (A->jon) A->jcells.push_back({i, A->cells[i]});
  if (!A->all_dirty) {
    if ((size_t)i >= A->isdirty.size()) A->isdirty.resize(std::max<size_t>(A->cells.size(), (size_t)i + 1), 0);
    if (!A->isdirty[i]) { A->isdirty[i] = 1; A->dirty.push_back(i); }
  }
  return A->cells[i];
}
void set_map(AmrState* A, int l, long long k, int v) {
  if (A->jon) A->jmap.push_back({{l, k}, A->hmap[l][k]});
  A->hmap[l][k] = v;
}

int alloc_block(AmrState* A) {
  if (!A->free_blocks.empty()) {
    const int id = A->free_blocks.back();
    A->free_blocks.pop_back();
    return id;
  }
  const int id = (int)A->cells.size();
  A->cells.resize(A->cells.size() + A->rd);
  return id;
}

int make_children(AmrState* A, int m, int status) {
  const int id = alloc_block(A);
  wcell(A, m).child = id;
  const int l = A->cells[m].level + 1;
  for (int q = 0; q < A->rd; ++q) {
    HCell& C = wcell(A, id + q);
    C = HCell();
    C.alive = true;
    C.level = l;
    C.status = status;
    C.mother = m;
    const int off[3] = {q % A->r, (q / A->r) % A->r, A->d == 3 ? q / (A->r * A->r) : 0};
    for (int k = 0; k < 3; ++k) C.idx[k] = k < A->d ? A->cells[m].idx[k] * A->r + off[k] : 0;
    set_map(A, l, lin(A, l, C.idx), id + q);
  }
  return id;
}

void destroy_children(AmrState* A, int m, std::vector<int>* freed) {
  const int ch = A->cells[m].child;
  if (ch < 0) return;
  for (int q = 0; q < A->rd; ++q) {
    if (A->cells[ch + q].child >= 0) destroy_children(A, ch + q, freed);
    const HCell& C = A->cells[ch + q];
    set_map(A, C.level, lin(A, C.level, C.idx), -1);
    wcell(A, ch + q) = HCell();
  }
  freed->push_back(ch);
  wcell(A, m).child = -1;
}

void refine_cell(AmrState* A, int c, bool t0) {
  if (A->cells[c].child < 0) make_children(A, c, 0);
  else
    for (int q = 0; q < A->rd; ++q) wcell(A, A->cells[c].child + q).status = 0;
  wcell(A, c).status = -1;
  const int ch = A->cells[c].child;
  for (int q = 0; q < A->rd; ++q) {
    wcell(A, ch + q).isnew = true;
    A->inits.push_back({ch + q, c, t0 ? 2 : 0});
  }
}

void virtually_refine(AmrState* A, int v, bool t0) {
  const int ch = make_children(A, v, 1);
  for (int q = 0; q < A->rd; ++q) A->inits.push_back({ch + q, v, t0 ? 2 : 1});
}

void closure(AmrState* A, bool t0) {
  // the virtual mothers (found by a threaded scan in id order; the ones the
  // closure creates are appended and visited in the same pass): rules 4-5 act
  // only around them.  Passes repeat until none acts (least fixed point, R17).
  int nb[26];
  const int nu = (int)A->cells.size(), T = host_threads(nu);
  std::vector<std::vector<int>> part(T);
  parallel_chunks(nu, T, [&](int t, int i0, int i1) {
    for (int i = i0; i < i1; ++i)
      if (A->cells[i].alive && A->cells[i].status == -1) part[t].push_back(i);
  });
  std::vector<int> vm;
  for (const auto& P : part) vm.insert(vm.end(), P.begin(), P.end());
  bool changed = true;
  while (changed) {
    changed = false;
    for (size_t j = 0; j < vm.size(); ++j) {
      const int i = vm[j];
      if (!A->cells[i].alive || A->cells[i].status != -1) continue;
      const int k = voronoi(A, i, nb);
      for (int q = 0; q < k; ++q) {
        const int v = nb[q];
        if (v < 0 || A->cells[v].child >= 0) continue;
        if (A->cells[v].status == 0) { virtually_refine(A, v, t0); changed = true; }
        else if (A->cells[v].status == 1) {
          const int m = A->cells[v].mother;
          refine_cell(A, m, t0);
          vm.push_back(m);
          changed = true;
        }
      }
    }
  }
}

void garbage_collect(AmrState* A, std::vector<int>* freed) {
  int nb[26];
  // candidates (active cells with children) found by a threaded scan; no
  // candidate descends from another (an active cell has no active
  // descendant), so visiting them in id order afterwards equals the serial scan
  const int nu = (int)A->cells.size(), T = host_threads(nu);
  std::vector<std::vector<int>> part(T);
  parallel_chunks(nu, T, [&](int t, int i0, int i1) {
    for (int i = i0; i < i1; ++i) {
      const HCell& C = A->cells[i];
      if (C.alive && C.status == 0 && C.child >= 0) part[t].push_back(i);
    }
  });
  for (const auto& P : part)
  for (const int i : P) {
    HCell& C = A->cells[i];
    if (!C.alive || C.status != 0 || C.child < 0) continue;
    const int k = voronoi(A, i, nb);
    bool need = false;
    for (int j = 0; j < k && !need; ++j) need = nb[j] >= 0 && A->cells[nb[j]].status == -1;
    if (!need) destroy_children(A, i, freed);
  }
}

// ---- device mirrors ---------------------------------------------------------
ader_status ensure_capacity(AmrState* A, std::string& err) {
  const int need = (int)A->cells.size();
  if (need <= A->cap) return ADER_OK;
  // grow geometrically from a reserve of (1 + r^d lmax) level-0 cells: every
  // reallocation copies all per-id arrays and synchronises the stream
  const long long n0 = A->n[0][0] * A->n[0][1] * A->n[0][2];
  const int nc = (int)std::min<long long>(std::max<long long>({2LL * need, n0 * (1 + A->rd * std::max(1, A->lmax)), 1024}),
                                          2000000000LL);
  auto grow = [&](void** p, size_t elem) -> cudaError_t {
    void* np = nullptr;
    cudaError_t e = cudaMalloc(&np, (size_t)nc * elem);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(np, 0, (size_t)nc * elem, A->k->stream);
    if (*p) {
      cudaMemcpyAsync(np, *p, (size_t)A->cap * elem, cudaMemcpyDeviceToDevice, A->k->stream);
      cudaStreamSynchronize(A->k->stream);
      cudaFree(*p);
    }
    *p = np;
    return cudaSuccess;
  };
  AmrDevView& V = A->V;
  ACK(grow((void**)&V.u, sizeof(double) * A->nv));
  ACK(grow((void**)&V.mem, sizeof(double) * 6 * A->nv));
  if (A->ranks.world == 1) {
    ACK(grow((void**)&V.w, sizeof(double) * A->nv * A->NS));
    ACK(grow((void**)&V.q, sizeof(double) * A->nv * A->NST));
  } else {
    ACK(grow((void**)&V.slot, sizeof(int)));
  }
  ACK(grow((void**)&V.chi, sizeof(double)));
  ACK(grow((void**)&V.level, sizeof(int)));
  ACK(grow((void**)&V.status, sizeof(int)));
  ACK(grow((void**)&V.mother, sizeof(int)));
  ACK(grow((void**)&V.child, sizeof(int)));
  ACK(grow((void**)&V.idx, sizeof(long long) * 3));
  if (A->ranks.world > 1) ACK(grow((void**)&V.own, 1));
  A->cap = nc;
  return ADER_OK;
}

// Stage host data through one pinned buffer into one device scratch buffer
// (bump allocation per upload batch); returns device pointers.
struct Uploader {
  AmrState* A;
  std::vector<std::pair<const void*, size_t>> parts;
  size_t add(const void* p, size_t bytes) {
    size_t off = 0;
    for (auto& q : parts) off += (q.second + 255) / 256 * 256;
    parts.push_back({p, bytes});
    return off;
  }
  ader_status run(std::string& err) {
    size_t tot = 0;
    for (auto& q : parts) tot += (q.second + 255) / 256 * 256;
    if (tot == 0) return ADER_OK;
    cudaStream_t sm = A->k->stream;
    if (tot > A->dscratch_cap) {
      if (A->dscratch) { cudaStreamSynchronize(sm); cudaFree(A->dscratch); }
      A->dscratch_cap = tot * 2 + (1 << 20);   // geometric: pinned / device reallocations are slow
      ACK(cudaMalloc(&A->dscratch, A->dscratch_cap));
    }
    if (tot > A->hstage_cap) {
      if (A->hstage) { cudaStreamSynchronize(sm); cudaFreeHost(A->hstage); }
      A->hstage_cap = tot * 2 + (1 << 20);
      ACK(cudaMallocHost(&A->hstage, A->hstage_cap));
    }
    ACK(cudaStreamSynchronize(sm));   // previous use of the staging buffer finished
    size_t off = 0;
    for (auto& q : parts) {
      if (q.second) std::memcpy(A->hstage + off, q.first, q.second);
      off += (q.second + 255) / 256 * 256;
    }
    ACK(cudaMemcpyAsync(A->dscratch, A->hstage, tot, cudaMemcpyHostToDevice, sm));
    return ADER_OK;
  }
};

// Multi-rank rows of w / q (see slot_of): release the rows deferred at the
// previous rebuild whose cells are still not computed, defer the rows of cells
// that left the compute lists, give new computed cells a row, grow w / q
// (rows kept) and return the per-id row array for the device (0 = scratch).
ader_status assign_slots(AmrState* A, std::vector<int>& dev_slot, std::string& err) {
  const int nu = (int)A->cells.size();
  if ((int)A->slot_of.size() < nu) A->slot_of.resize(nu, -1);
  std::vector<char> need(nu, 0);
  for (int l = 0; l <= A->lmax; ++l)
    for (int i : A->lact[l]) need[i] = 1;
  for (int i : A->slot_defer)
    if (i < nu && A->slot_of[i] >= 0 && !need[i]) { A->free_slots.push_back(A->slot_of[i]); A->slot_of[i] = -1; }
  A->slot_defer.clear();
  for (int i = 0; i < nu; ++i) {
    if (A->slot_of[i] >= 0 && !need[i]) A->slot_defer.push_back(i);
    if (need[i] && A->slot_of[i] < 0) {
      if (!A->free_slots.empty()) { A->slot_of[i] = A->free_slots.back(); A->free_slots.pop_back(); }
      else A->slot_of[i] = A->nslots++;
    }
  }
  if (A->nslots > A->slot_cap) {
    const int nc = std::max(A->nslots + A->nslots / 2, 1024);
    AmrDevView& V = A->V;
    auto grow = [&](double** p, size_t row) -> cudaError_t {
      double* np = nullptr;
      cudaError_t e = cudaMalloc(&np, (size_t)nc * row * sizeof(double));
      if (e != cudaSuccess) return e;
      if (*p) {
        cudaMemcpyAsync(np, *p, (size_t)A->slot_cap * row * sizeof(double), cudaMemcpyDeviceToDevice, A->k->stream);
        cudaStreamSynchronize(A->k->stream);
        cudaFree(*p);
      }
      *p = np;
      return cudaSuccess;
    };
    ACK(grow(&V.w, (size_t)A->nv * A->NS));
    ACK(grow(&V.q, (size_t)A->nv * A->NST));
    A->slot_cap = nc;
  }
  dev_slot.resize(nu);
  for (int i = 0; i < nu; ++i) dev_slot[i] = A->slot_of[i] >= 0 ? A->slot_of[i] : 0;
  return ADER_OK;
}

// Push the host tree to the device: only the ids whose links or status changed
// since the last upload (plus the map entries they occupy), and the per-level
// id lists.
ader_status upload_topology(AmrState* A, std::string& err) {
  double w0 = now_s();
  ader_status s = ensure_capacity(A, err);
  if (s != ADER_OK) return s;
  A->tm_u[0] += now_s() - w0; w0 = now_s();
  const int nu = (int)A->cells.size();
  if ((int)A->mirror.size() < nu) A->mirror.resize(nu);
  std::vector<long long> meta, clears, sets;
  // candidates: every id on the first upload, else the ids written since
  std::vector<int> cand;
  const bool full = A->all_dirty || A->dirty.size() * 4 > (size_t)nu;
  if (!full) {
    // the written ids in id order: a scan of the byte flags is cheaper than
    // sorting the (up to nu / 4) ids
    cand.reserve(A->dirty.size());
    const size_t lim = std::min(A->isdirty.size(), (size_t)nu);
    for (size_t i = 0; i < lim; ++i)
      if (A->isdirty[i]) cand.push_back((int)i);
  }
  for (int i : A->dirty)
    if ((size_t)i < A->isdirty.size()) A->isdirty[i] = 0;
  A->dirty.clear();
  A->all_dirty = false;
  const int ncand = full ? nu : (int)cand.size();
  // compare the candidates with the device mirror (threaded; per-chunk records
  // concatenated in chunk order = the serial order)
  struct Diff { std::vector<long long> meta, clears, sets; };
  const int TD = host_threads(ncand);
  std::vector<Diff> dp(TD);
  parallel_chunks(ncand, TD, [&](int t, int c0, int c1) {
    Diff& D = dp[t];
    for (int ci = c0; ci < c1; ++ci) {
      const int i = full ? ci : cand[ci];
      if (i >= nu) continue;
      const HCell& C = A->cells[i];
      HCell& P = A->mirror[i];
      const bool same_pos = C.alive == P.alive && C.level == P.level && C.idx[0] == P.idx[0] &&
                            C.idx[1] == P.idx[1] && C.idx[2] == P.idx[2];
      const bool same = same_pos && C.status == P.status && C.mother == P.mother && C.child == P.child;
      if (same && (C.alive || !P.alive)) continue;
      const long long m[8] = {i, C.level, C.alive ? C.status : 9, C.mother, C.child, C.idx[0], C.idx[1], C.idx[2]};
      D.meta.insert(D.meta.end(), m, m + 8);
      if (P.alive && (!C.alive || !same_pos)) {
        D.clears.push_back(P.level); D.clears.push_back(lin(A, P.level, P.idx)); D.clears.push_back(-1);
      }
      if (C.alive && (!P.alive || !same_pos)) {
        D.sets.push_back(C.level); D.sets.push_back(lin(A, C.level, C.idx)); D.sets.push_back(i);
      }
      P = C;
    }
  });
  for (const Diff& D : dp) {
    meta.insert(meta.end(), D.meta.begin(), D.meta.end());
    clears.insert(clears.end(), D.clears.begin(), D.clears.end());
    sets.insert(sets.end(), D.sets.begin(), D.sets.end());
  }
  A->tm_u[3] += now_s() - w0;
  for (int l = 0; l <= A->lmax; ++l) {
    A->lact[l].clear(); A->lvch[l].clear(); A->lvmo[l].clear(); A->lown[l].clear(); A->lpres[l].clear();
    A->xp[l] = AmrState::XPlan();
  }
  const int W = A->ranks.world, me = A->ranks.rank;
  A->own.assign(nu, W > 1 ? 0 : 1);
  A->comp.assign(nu, W > 1 ? 0 : 1);
  std::vector<int> owner(W > 1 ? nu : 0, -1);
  std::vector<std::vector<int>> send_to(W > 1 ? (size_t)(A->lmax + 1) * W : 0);
  for (int l = 0; l < kAmrMaxLevels; ++l) A->nlev[l] = 0;
  if (W == 1) {
    // one rank: every alive cell is owned and computed; lists in id order
    // (contiguous id chunks scanned by host threads, appended in chunk order)
    struct Part {
      std::vector<int> l[3][kAmrMaxLevels];
      long long n[kAmrMaxLevels]{};
    };
    const int T = host_threads(nu);
    std::vector<Part> parts(T);
    parallel_chunks(nu, T, [&](int t, int i0, int i1) {
      Part& P = parts[t];
      for (int i = i0; i < i1; ++i) {
        const HCell& C = A->cells[i];
        if (!C.alive) continue;
        P.n[C.level]++;
        P.l[C.status == 0 ? 0 : (C.status == 1 ? 1 : 2)][C.level].push_back(i);
      }
    });
    for (int l = 0; l <= A->lmax; ++l) {
      size_t na = 0, nc = 0, nm = 0;
      for (const Part& P : parts) { na += P.l[0][l].size(); nc += P.l[1][l].size(); nm += P.l[2][l].size(); }
      A->lact[l].reserve(na); A->lvch[l].reserve(nc); A->lvmo[l].reserve(nm);
      for (const Part& P : parts) {
        A->nlev[l] += P.n[l];
        A->lact[l].insert(A->lact[l].end(), P.l[0][l].begin(), P.l[0][l].end());
        A->lvch[l].insert(A->lvch[l].end(), P.l[1][l].begin(), P.l[1][l].end());
        A->lvmo[l].insert(A->lvmo[l].end(), P.l[2][l].begin(), P.l[2][l].end());
      }
    }
  }
  RankSets RS;
  const bool dep = W > 1 && !A->band_sets;
  if (dep) rank_sets(A, RS);
  const unsigned char mb = (unsigned char)(1u << me);
  for (int i = 0; i < (W > 1 ? nu : 0); ++i) {
    const HCell& C = A->cells[i];
    if (!C.alive) continue;
    A->nlev[C.level]++;
    bool compute;   // this rank runs WENO + predictor + flux/update (active) or the ghost fill (virtual)
    if (dep) {
      owner[i] = RS.owner[i];
      A->own[i] = owner[i] == me;
      if (C.status == 0) {
        compute = RS.P[i] & mb;
        A->comp[i] = A->own[i] || ((RS.P[i] | RS.R[i]) & mb);
        if (A->own[i])
          for (int p = 0; p < W; ++p)
            if (p != me && ((RS.P[i] | RS.R[i]) >> p & 1)) send_to[(size_t)C.level * W + p].push_back(i);
      } else {
        // virtual children of cells this rank computes also get their flux memory
        // cleared / projected (R16); virtual cells in the boxes (V)
        compute = (RS.V[i] & mb) || (C.status == 1 && (RS.P[C.mother] & mb));
        A->comp[i] = compute;
      }
    } else {
      long long a0[3];
      ancestor0(A, C, a0);
      owner[i] = owner_of(A, a0);
      A->own[i] = owner[i] == me;
      A->comp[i] = A->own[i] || in_comp(A, me, a0);
      compute = A->comp[i];
      if (A->own[i] && C.status == 0)
        for (int p = 0; p < W; ++p)
          if (p != me && in_comp(A, p, a0)) send_to[(size_t)C.level * W + p].push_back(i);
    }
    if (C.status == 0) {
      if (compute) A->lact[C.level].push_back(i);
      if (A->comp[i]) A->lpres[C.level].push_back(i);
    } else if (compute) {
      if (C.status == 1) A->lvch[C.level].push_back(i);
      else A->lvmo[C.level].push_back(i);
    }
    if (A->own[i] && C.status == 0) A->lown[C.level].push_back(i);
  }
  size_t xneed = 0;
  if (W > 1)
    for (int l = 0; l <= A->lmax; ++l) {
      AmrState::XPlan& X = A->xp[l];
      X.soff.assign(W + 1, 0);
      X.roff.assign(W + 1, 0);
      for (int p = 0; p < W; ++p) {
        X.soff[p] = (long long)X.sids.size();
        if (p != me) X.sids.insert(X.sids.end(), send_to[(size_t)l * W + p].begin(), send_to[(size_t)l * W + p].end());
        X.roff[p] = (long long)X.rids.size();
        if (p != me)
          for (int i : A->lpres[l])
            if (owner[i] == p) X.rids.push_back(i);
      }
      X.soff[W] = (long long)X.sids.size();
      X.roff[W] = (long long)X.rids.size();
      xneed = std::max(xneed, std::max(X.sids.size(), X.rids.size()) * (size_t)A->nv);
    }
  // reconstruction lists: a mother with at least `thr` listed active children is reconstructed as
  // one sibling patch (thr: where the patch's 1D problems undercut the per-cell boxes'), the other
  // cells from their own box; ADER_AMR_WENO_PATCH=0 keeps every cell on its own box
  {
    static const bool patch_on = !(std::getenv("ADER_AMR_WENO_PATCH") && std::getenv("ADER_AMR_WENO_PATCH")[0] == '0');
    const int N = A->N, WW = 2 * A->M + 1, Wp = A->r + 2 * A->M, R = A->r;
    const double pc = A->d == 2 ? WW + N : WW * WW + WW * N + N * N;
    const double pp = A->d == 2 ? R * Wp + R * R * N : R * Wp * Wp + R * R * N * Wp + R * R * R * N * N;
    const int thr = (int)std::ceil(pp / pc);
    for (int l = 0; l <= A->lmax; ++l) { A->lwc[l].clear(); A->lwp[l].clear(); }
    A->lwc[0] = A->lact[0];
    if (patch_on && A->r == 3 && A->lmax >= 1) {
      // siblings occupy one block of r^d consecutive ids and the lists are in id order, so the
      // listed children of a mother are adjacent: one pass per level, chunked over host threads
      // (a chunk starts at the first group that begins inside it and finishes its last group)
      for (int l = 1; l <= A->lmax; ++l) {
        const std::vector<int>& L = A->lact[l];
        const int nl = (int)L.size(), T = host_threads(nl);
        std::vector<std::vector<int>> pc_(T), pp_(T);
        parallel_chunks(nl, T, [&](int t, int i0, int i1) {
          int j = i0;
          if (j > 0)
            while (j < i1 && A->cells[L[j]].mother == A->cells[L[j - 1]].mother) ++j;
          while (j < i1) {
            const int mo = A->cells[L[j]].mother;
            int e = j + 1;
            while (e < nl && A->cells[L[e]].mother == mo) ++e;
            if (e - j >= thr) pp_[t].push_back(mo);
            else pc_[t].insert(pc_[t].end(), L.begin() + j, L.begin() + e);
            j = e;
          }
        });
        for (int t = 0; t < T; ++t) {
          A->lwc[l].insert(A->lwc[l].end(), pc_[t].begin(), pc_[t].end());
          A->lwp[l].insert(A->lwp[l].end(), pp_[t].begin(), pp_[t].end());
        }
      }
    } else {
      for (int l = 1; l <= A->lmax; ++l) A->lwc[l] = A->lact[l];
    }
  }
  size_t tot = 0;
  for (int l = 0; l <= A->lmax; ++l) tot += A->lwc[l].size() + A->lwp[l].size();
  for (int l = 0; l <= A->lmax; ++l)
    tot += A->lact[l].size() + A->lvch[l].size() + A->lvmo[l].size() + A->lown[l].size() + A->xp[l].sids.size() +
           A->xp[l].rids.size();
  std::vector<int> all;
  all.reserve(tot);
  A->oall = 0;
  for (int l = 0; l <= A->lmax; ++l) {
    A->oact[l] = (long long)all.size(); all.insert(all.end(), A->lact[l].begin(), A->lact[l].end());
  }
  A->nall = (long long)all.size();
  if (W > 1) {
    A->oownall = (long long)all.size();
    for (int l = 0; l <= A->lmax; ++l) {
      A->nown[l] = (long long)A->lown[l].size();
      all.insert(all.end(), A->lown[l].begin(), A->lown[l].end());
    }
    A->nownall = (long long)all.size() - A->oownall;
  } else {
    for (int l = 0; l <= A->lmax; ++l) A->nown[l] = (long long)A->lact[l].size();
    A->oownall = A->oall;
    A->nownall = A->nall;
  }
  for (int l = 0; l <= A->lmax; ++l) {
    A->ovch[l] = (long long)all.size(); all.insert(all.end(), A->lvch[l].begin(), A->lvch[l].end());
    A->ovmo[l] = (long long)all.size(); all.insert(all.end(), A->lvmo[l].begin(), A->lvmo[l].end());
    A->xp[l].dso = (long long)all.size(); all.insert(all.end(), A->xp[l].sids.begin(), A->xp[l].sids.end());
    A->xp[l].dro = (long long)all.size(); all.insert(all.end(), A->xp[l].rids.begin(), A->xp[l].rids.end());
    A->owc[l] = (long long)all.size(); all.insert(all.end(), A->lwc[l].begin(), A->lwc[l].end());
    A->owp[l] = (long long)all.size(); all.insert(all.end(), A->lwp[l].begin(), A->lwp[l].end());
  }
  if (xneed > A->xcap) {
    if (A->xsend) { cudaStreamSynchronize(A->k->stream); cudaFree(A->xsend); cudaFree(A->xrecv); }
    A->xcap = xneed * 3 / 2 + 1024;
    ACK(cudaMalloc(&A->xsend, sizeof(double) * A->xcap));
    ACK(cudaMalloc(&A->xrecv, sizeof(double) * A->xcap));
  }
  cudaStream_t sm = A->k->stream;
  if ((long long)all.size() > A->dlist_cap) {
    if (A->dlist) { cudaStreamSynchronize(sm); cudaFree(A->dlist); }
    A->dlist_cap = (long long)all.size() * 3 / 2 + 1024;
    ACK(cudaMalloc(&A->dlist, sizeof(int) * A->dlist_cap));
  }
  Uploader up{A, {}};
  A->tm_u[1] += now_s() - w0; w0 = now_s();
  const size_t om = up.add(meta.data(), meta.size() * sizeof(long long));
  const size_t oc = up.add(clears.data(), clears.size() * sizeof(long long));
  const size_t os = up.add(sets.data(), sets.size() * sizeof(long long));
  const size_t ol = up.add(all.data(), all.size() * sizeof(int));
  const size_t oo = W > 1 ? up.add(A->own.data(), A->own.size()) : 0;
  std::vector<int> dslot;
  if (W > 1) {
    s = assign_slots(A, dslot, err);
    if (s != ADER_OK) return s;
  }
  const size_t osl = W > 1 ? up.add(dslot.data(), sizeof(int) * dslot.size()) : 0;
  s = up.run(err);
  if (s != ADER_OK) return s;
  if (W > 1) ACK(cudaMemcpyAsync(A->V.own, A->dscratch + oo, A->own.size(), cudaMemcpyDeviceToDevice, sm));
  if (W > 1)
    ACK(cudaMemcpyAsync(A->V.slot, A->dscratch + osl, sizeof(int) * dslot.size(), cudaMemcpyDeviceToDevice, sm));
  A->tm_u[2] += now_s() - w0; w0 = now_s();
  amr_launch_meta_scatter(*A->k, A->V, (const long long*)(A->dscratch + om), (int)(meta.size() / 8));
  amr_launch_map_set(*A->k, A->V, (const long long*)(A->dscratch + oc), (int)(clears.size() / 3));
  amr_launch_map_set(*A->k, A->V, (const long long*)(A->dscratch + os), (int)(sets.size() / 3));
  ACK(cudaMemcpyAsync(A->dlist, A->dscratch + ol, sizeof(int) * all.size(), cudaMemcpyDeviceToDevice, sm));
  return ADER_OK;
}

const int* L_act(const AmrState* A, int l) { return A->dlist + A->oact[l]; }
const int* L_vch(const AmrState* A, int l) { return A->dlist + A->ovch[l]; }
const int* L_vmo(const AmrState* A, int l) { return A->dlist + A->ovmo[l]; }
// WENO of the listed active cells of level l: sibling patches + the remaining cells' own boxes
void launch_weno_level(AmrState* A, int l) {
  amr_launch_weno(*A->k, A->V, A->dlist + A->owc[l], (int)A->lwc[l].size());
  amr_launch_weno_patches(*A->k, A->V, A->dlist + A->owp[l], (int)A->lwp[l].size(), l);
}

void psi_at(const AmrState* A, double tau, double out[4]) {
  for (int s = 0; s < 4; ++s) out[s] = s < A->N ? lagrange(A->k->tab, A->N, s, tau) : 0.0;
}

// IC cell averages of the listed cells (Q^d GL points, host callback, device sum)
ader_status ic_cells(AmrState* A, const std::vector<int>& ids, std::string& err) {
  if (ids.empty()) return ADER_OK;
  const int Q = A->cfg.ic_quad, d = A->d;
  // Gauss-Legendre rule on [0,1] from the context tables when Q == N, else closed forms
  double qx[8], qw[8];
  DevTables tq;
  if (Q == 3 || Q == 4) { build_tables(Q - 1, &tq); for (int i = 0; i < Q; ++i) { qx[i] = tq.lam[i]; qw[i] = tq.w[i]; } }
  else if (Q == 2) { const double h = std::sqrt(3.0) / 6.0; qx[0] = 0.5 - h; qx[1] = 0.5 + h; qw[0] = qw[1] = 0.5; }
  else { qx[0] = 0.5; qw[0] = 1.0; }
  int nq = 1;
  for (int k = 0; k < d; ++k) nq *= Q;
  std::vector<double> wq(nq);
  for (int g = 0; g < nq; ++g) {
    const int gi[3] = {g % Q, (g / Q) % Q, g / (Q * Q)};
    double wg = 1.0;
    for (int k = 0; k < d; ++k) wg *= qw[gi[k]];
    wq[g] = wg;
  }
  const size_t nc = ids.size();
  std::vector<double> x(nc * nq * 3), pr(nc * nq * 9, 0.0);
  for (size_t i = 0; i < nc; ++i) {
    const HCell& C = A->cells[ids[i]];
    for (int g = 0; g < nq; ++g) {
      const int gi[3] = {g % Q, (g / Q) % Q, g / (Q * Q)};
      for (int k = 0; k < 3; ++k)
        x[(i * nq + g) * 3 + k] = k < d ? A->cfg.lo[k] + ((double)C.idx[k] + qx[gi[k]]) * A->dx[C.level][k] : 0.0;
    }
  }
  A->ic(x.data(), (int64_t)(nc * nq), pr.data(), A->user);
  double *dpr = nullptr, *dwq = nullptr;
  int* dids = nullptr;
  ACK(cudaMalloc(&dpr, sizeof(double) * pr.size()));
  ACK(cudaMalloc(&dwq, sizeof(double) * nq));
  ACK(cudaMalloc(&dids, sizeof(int) * nc));
  cudaStream_t sm = A->k->stream;
  ACK(cudaMemcpyAsync(dpr, pr.data(), sizeof(double) * pr.size(), cudaMemcpyHostToDevice, sm));
  ACK(cudaMemcpyAsync(dwq, wq.data(), sizeof(double) * nq, cudaMemcpyHostToDevice, sm));
  ACK(cudaMemcpyAsync(dids, ids.data(), sizeof(int) * nc, cudaMemcpyHostToDevice, sm));
  amr_launch_ic(*A->k, A->V, dids, (int)nc, dpr, dwq, nq);
  ACK(cudaStreamSynchronize(sm));
  cudaFree(dpr); cudaFree(dwq); cudaFree(dids);
  return ADER_OK;
}

// apply the pending initialisations (after the topology is on the device)
ader_status run_inits(AmrState* A, std::string& err) {
  // keep only the last init per live cell (a cell may be re-initialised in a cascade)
  std::vector<int> last(A->cells.size(), -1);
  for (size_t i = 0; i < A->inits.size(); ++i)
    if (A->inits[i].cell < (int)A->cells.size()) last[A->inits[i].cell] = (int)i;
  std::vector<int> pw, pp, ic;
  for (size_t i = 0; i < A->inits.size(); ++i) {
    const Init& z = A->inits[i];
    if (last[z.cell] != (int)i || !A->cells[z.cell].alive) continue;
    if (z.mode == 0) { pw.push_back(z.cell); pw.push_back(z.mother); }
    else if (z.mode == 1) { pp.push_back(z.cell); pp.push_back(z.mother); }
    else ic.push_back(z.cell);
  }
  A->inits.clear();
  Uploader up{A, {}};
  const size_t ow = up.add(pw.data(), pw.size() * sizeof(int));
  const size_t op = up.add(pp.data(), pp.size() * sizeof(int));
  ader_status s = up.run(err);
  if (s != ADER_OK) return s;
  amr_launch_init_from_weno(*A->k, A->V, A->st, (const int*)(A->dscratch + ow), (int)(pw.size() / 2));
  double pt[4];
  psi_at(A, 1.0, pt);
  amr_launch_init_from_pred(*A->k, A->V, A->st, (const int*)(A->dscratch + op), (int)(pp.size() / 2), pt);
  std::sort(ic.begin(), ic.end());
  return ic_cells(A, ic, err);
}

using Group = std::vector<AmrState*>;

// CFL speed (reading R1) over the owned active cells, maximised over the ranks
ader_status fetch_speed(const Group& G, double* speed, std::string& err) {
  double best = 0.0;
  for (AmrState* A : G) {
    cudaStream_t sm = A->k->stream;
    ACK(cudaMemsetAsync(&A->cnt->speed_bits, 0, sizeof(unsigned long long), sm));
    double inv[3] = {0, 0, 0};
    for (int k = 0; k < A->d; ++k) inv[k] = 1.0 / A->dx[0][k];
    amr_launch_cfl(*A->k, A->V, A->dlist + A->oownall, (int)A->nownall, inv, A->cnt);
    if (G.size() == 1 && A->ranks.world > 1) {
      ader_status s = A->comm.max_u64(A->comm.ctx, &A->cnt->speed_bits, sm);
      if (s != ADER_OK) { err = "allreduce(max) of the CFL speed failed"; return s; }
    }
    ACK(cudaMemcpyAsync(A->hcnt, A->cnt, sizeof(DevCounters), cudaMemcpyDeviceToHost, sm));
    ACK(cudaStreamSynchronize(sm));
    unsigned long long b = A->hcnt->speed_bits;
    double v;
    std::memcpy(&v, &b, sizeof(double));
    best = std::max(best, v);
  }
  *speed = best;
  return ADER_OK;
}

// Owners' new averages of the active cells of level l overwrite the other
// ranks' copies (compute-set band); NCCL through the hooks for one context per
// rank, device copies inside a loopback group.
ader_status exchange(const Group& G, int l, std::string& err) {
  if (G[0]->ranks.world <= 1) return ADER_OK;
  for (AmrState* A : G) {
    const AmrState::XPlan& X = A->xp[l];
    amr_launch_rows_gather(*A->k, A->V.u, A->dlist + X.dso, (int)X.sids.size(), A->nv, A->xsend);
  }
  const int W = G[0]->ranks.world;
  if (G.size() > 1) {
    for (AmrState* A : G) ACK(cudaStreamSynchronize(A->k->stream));
    for (AmrState* A : G) {
      const int me = A->ranks.rank;
      for (int p = 0; p < W; ++p) {
        if (p == me) continue;
        const AmrState* P = G[p];
        const long long n = A->xp[l].roff[p + 1] - A->xp[l].roff[p];
        if (n != P->xp[l].soff[me + 1] - P->xp[l].soff[me]) { err = "exchange plans disagree"; return ADER_ERR_SOLVER; }
        if (n)
          ACK(cudaMemcpyAsync(A->xrecv + A->xp[l].roff[p] * A->nv, P->xsend + P->xp[l].soff[me] * A->nv,
                              sizeof(double) * n * A->nv, cudaMemcpyDeviceToDevice, A->k->stream));
      }
    }
    // the peers' send buffers are reused by their next exchange
    for (AmrState* A : G) ACK(cudaStreamSynchronize(A->k->stream));
  } else {
    AmrState* A = G[0];
    const AmrState::XPlan& X = A->xp[l];
    std::vector<int> peers;
    std::vector<double*> sp, rp;
    std::vector<size_t> sc, rc;
    for (int p = 0; p < W; ++p) {
      const size_t ns = (size_t)(X.soff[p + 1] - X.soff[p]), nr = (size_t)(X.roff[p + 1] - X.roff[p]);
      if (p == A->ranks.rank || (!ns && !nr)) continue;
      peers.push_back(p);
      sp.push_back(A->xsend + X.soff[p] * A->nv); sc.push_back(ns * A->nv);
      rp.push_back(A->xrecv + X.roff[p] * A->nv); rc.push_back(nr * A->nv);
    }
    if (!peers.empty()) {
      ader_status s = A->comm.p2p(A->comm.ctx, (int)peers.size(), peers.data(), sp.data(), sc.data(), rp.data(),
                                  rc.data(), A->k->stream);
      if (s != ADER_OK) { err = "halo exchange of the AMR averages failed"; return s; }
    }
  }
  for (AmrState* A : G) {
    const AmrState::XPlan& X = A->xp[l];
    amr_launch_rows_scatter(*A->k, A->V.u, A->dlist + X.dro, (int)X.rids.size(), A->nv, A->xrecv);
  }
  return ADER_OK;
}

// solver errors of this rank; with one context per rank the error code is
// max-reduced over the ranks first (err_any), so every rank leaves the step
// loop at the same point instead of the others blocking in the next exchange
ader_status check_err(AmrState* A, std::string& err, bool reduce) {
  cudaStream_t sm = A->k->stream;
  if (reduce && A->ranks.world > 1) {
    ACK(cudaMemsetAsync(&A->cnt->err_any, 0, sizeof(unsigned long long), sm));
    ACK(cudaMemcpyAsync(&A->cnt->err_any, &A->cnt->err_code, sizeof(int), cudaMemcpyDeviceToDevice, sm));
    ader_status s = A->comm.max_u64(A->comm.ctx, &A->cnt->err_any, sm);
    if (s != ADER_OK) { err = "allreduce(max) of the error code failed"; return s; }
  }
  ACK(cudaMemcpyAsync(A->hcnt, A->cnt, sizeof(DevCounters), cudaMemcpyDeviceToHost, sm));
  ACK(cudaStreamSynchronize(sm));
  if (reduce && A->ranks.world > 1 && !A->hcnt->err_code && A->hcnt->err_any) {
    char b[160];
    snprintf(b, sizeof(b), "solver failure on another rank (code %llu), t=%.17g", A->hcnt->err_any, A->t);
    err = b;
    return ADER_ERR_SOLVER;
  }
  if (A->hcnt->err_code) {
    const long long id = (long long)A->hcnt->err_cell;
    char b[512];
    const HCell& C = A->cells[(size_t)id < A->cells.size() ? id : 0];
    snprintf(b, sizeof(b), "%s at level %d cell (%lld,%lld,%lld), t=%.17g",
             A->hcnt->err_code == 1 ? "inadmissible state (rho<=0 or p<=0)" : "predictor reached pred_max_sweeps",
             C.level, C.idx[0], C.idx[1], C.idx[2], A->t);
    err = b;
    return ADER_ERR_SOLVER;
  }
  return ADER_OK;
}

// ---- local time stepping (recursive form of eqn.update.criterion, R15) -------
ader_status advance(const Group& G, int l, int m, double dt0, std::string& err) {
  AmrState* A0 = G[0];
  double dt = dt0;
  for (int k = 0; k < l; ++k) dt /= A0->r;
  double dtdx[3] = {0, 0, 0};
  for (int k = 0; k < A0->d; ++k) dtdx[k] = dt / A0->dx[l][k];
  for (AmrState* A : G) {
    // ghost refresh (R16): averaging of virtual mothers on levels >= l, finest first
    {
      AScope sc(A, ADER_K_HALO, 0.0);
      for (int lv = A->lmax - 1; lv >= l; --lv) amr_launch_average(*A->k, A->V, L_vmo(A, lv), (int)A->lvmo[lv].size());
      if (l >= 1) {
        double pt[4];
        psi_at(A, (double)m / A->r, pt);
        amr_launch_project(*A->k, A->V, A->st, L_vch(A, l), (int)A->lvch[l].size(), pt);
      }
    }
    const int na = (int)A->lact[l].size();
    const int W = 2 * A->M + 1;
    double wfl = 0.0;   // 1D WENO problems of the per-cell box reconstruction
    {
      double per = 0.0, rows = 1.0;
      for (int k = 0; k < A->d; ++k) { per += rows * (A->d - k == 1 ? 1.0 : std::pow((double)W, A->d - 1 - k)); rows *= A->N; }
      const int N = A->N, nS = (A->M % 2 == 0) ? 3 : 4;
      wfl = (double)na * A->nv * per * (nS * (4.0 * N * N + 2.0 * N + 6.0) + 1.0 + 3.0 * N * nS);
    }
    { AScope sc(A, ADER_K_WENO, wfl); launch_weno_level(A, l); }
    { AScope sc(A, ADER_K_PRED, 0.0);
      amr_launch_predictor(*A->k, A->V, L_act(A, l), na, dtdx, A->cfg.pred_tol, A->cfg.pred_max_sweeps, A->cnt); }
  }
  if (l < A0->lmax && A0->nlev[l + 1] > 0)
    for (int k = 0; k < A0->r; ++k) {
      ader_status s = advance(G, l + 1, k, dt0, err);
      if (s != ADER_OK) return s;
    }
  for (AmrState* A : G) {
    const int na = (int)A->lact[l].size();
    { AScope sc(A, ADER_K_FLUX, 0.0); amr_launch_flux_update(*A->k, A->V, A->st, L_act(A, l), na, m, dtdx, A->cnt); }
    A->updates[l] += A->nown[l];
  }
  AScope sc(A0, ADER_K_HALO, 0.0);
  return exchange(G, l, err);
}

// ---- adapt (rules 1-7) --------------------------------------------------------
// phase 1: ghost refresh at t^{n+1}, indicator and WENO polynomials of the
// compute-set active cells (device); the local chi array comes back to the host
ader_status adapt_indicator(AmrState* A, bool t0, std::vector<double>& chi, std::string& err) {
  cudaStream_t sm = A->k->stream;
  if (!t0) {
    // ghost refresh at t^{n+1}: averages (finest first), projections at tau = 1
    for (int lv = A->lmax - 1; lv >= 0; --lv) amr_launch_average(*A->k, A->V, L_vmo(A, lv), (int)A->lvmo[lv].size());
    double pt[4];
    psi_at(A, 1.0, pt);
    for (int l = 1; l <= A->lmax; ++l) amr_launch_project(*A->k, A->V, A->st, L_vch(A, l), (int)A->lvch[l].size(), pt);
  }
  // indicator on all active cells (device), WENO polynomials of all active cells (R18)
  const int na = (int)A->nall;
  amr_launch_indicator(*A->k, A->V, A->dlist + A->oall, na, A->cfg.chi_eps);
  if (!t0)
    for (int l = 0; l <= A->lmax; ++l) launch_weno_level(A, l);
  chi.assign(A->cells.size(), 0.0);
  ACK(cudaMemcpyAsync(chi.data(), A->V.chi, sizeof(double) * A->cells.size(), cudaMemcpyDeviceToHost, sm));
  ACK(cudaStreamSynchronize(sm));
  // only the owner's chi is authoritative (its 3^d box lies inside the band)
  for (size_t i = 0; i < chi.size(); ++i)
    if (i >= A->own.size() || !A->own[i]) chi[i] = 0.0;
  return ADER_OK;
}

// phase 2 (same on every rank, on the global chi): marks, closure, simultaneous
// recoarsening, GC, device topology, new-cell initialisation
ader_status adapt_apply(AmrState* A, bool t0, const std::vector<double>& chi, std::string& err) {
  cudaStream_t sm = A->k->stream;
  int nb[26];
  double w0 = now_s();
  for (auto& c : A->cells) c.isnew = false;
  const int nu = (int)A->cells.size();
  std::vector<char> mark(nu, 0);
  // refinement marks, and how close any strict comparison of P:622-624 came to
  // flipping: min over the active cells of the relative distance of chi to
  // chi_ref and chi_rec (ader_step_report.min_threshold_margin; the oracle
  // computes the same; a min is exact in any order)
  const int TM = host_threads(nu);
  std::vector<double> mpart(TM, 1e300);
  parallel_chunks(nu, TM, [&](int t, int i0, int i1) {
    double mm = 1e300;
    for (int i = i0; i < i1; ++i) {
      const HCell& C = A->cells[i];
      if (!C.alive || C.status != 0) continue;
      mark[i] = C.level < A->lmax && chi[i] > A->cfg.chi_ref;
      const double m1 = std::fabs(chi[i] - A->cfg.chi_ref) / A->cfg.chi_ref;
      const double m2 = std::fabs(chi[i] - A->cfg.chi_rec) / A->cfg.chi_rec;
      mm = std::min(mm, std::min(m1, m2));
    }
    mpart[t] = mm;
  });
  for (double m : mpart) A->margin = std::min(A->margin, m);
  for (int i = 0; i < nu; ++i)
    if (mark[i]) refine_cell(A, i, t0);
  A->tm_a[0] += now_s() - w0; w0 = now_s();
  closure(A, t0);
  A->tm_a[1] += now_s() - w0; w0 = now_s();
  std::vector<int> freed;
  std::vector<int> coarsened;
  if (!t0) {
    const int nu2 = (int)A->cells.size();
    std::vector<char> cand(nu2, 0);
    parallel_chunks(nu2, host_threads(nu2), [&](int, int i0, int i1) {
      for (int i = i0; i < i1; ++i) {
        const HCell& C = A->cells[i];
        if (!C.alive || C.status != -1) continue;
        bool ok = true;
        for (int q = 0; q < A->rd && ok; ++q) {
          const int kid = C.child + q;
          const HCell& K = A->cells[kid];
          if (K.status != 0 || K.child >= 0 || K.isnew || !(kid < nu && chi[kid] < A->cfg.chi_rec) ||
              (kid < nu && mark[kid]))
            ok = false;
        }
        cand[i] = ok;
      }
    });
    std::vector<int> cl;   // candidate ids, ascending
    for (int i = 0; i < nu2; ++i)
      if (cand[i]) cl.push_back(i);
    bool any_cand = !cl.empty();
    while (any_cand) {
      // tentative simultaneous rule 7, then closure; reverted candidates retry
      // (the changes are journaled and undone in reverse order on a revert)
      const size_t snap_size = A->cells.size();
      const std::vector<int> snap_free = A->free_blocks;
      const size_t snap_inits = A->inits.size();
      A->jon = true;
      A->jcells.clear();
      A->jmap.clear();
      std::vector<char> destroy(cl.size(), 0);
      for (size_t j = 0; j < cl.size(); ++j) {
        const int k = voronoi(A, cl[j], nb);
        bool busy = false;
        for (int q = 0; q < k && !busy; ++q) busy = nb[q] >= 0 && A->cells[nb[q]].status == -1;
        destroy[j] = !busy;
      }
      std::vector<int> fr;
      for (size_t j = 0; j < cl.size(); ++j) {
        const int i = cl[j];
        if (destroy[j]) destroy_children(A, i, &fr);
        else
          for (int q = 0; q < A->rd; ++q) wcell(A, A->cells[i].child + q).status = 1;
        wcell(A, i).status = 0;
      }
      closure(A, false);
      A->jon = false;
      bool reverted = false;
      std::vector<int> kept;
      for (int i : cl) {
        if (A->cells[i].status == -1) { cand[i] = 0; reverted = true; }
        else kept.push_back(i);
      }
      if (!reverted) {
        freed.insert(freed.end(), fr.begin(), fr.end());
        coarsened.insert(coarsened.end(), cl.begin(), cl.end());
        break;
      }
      for (size_t j = A->jmap.size(); j-- > 0;) A->hmap[A->jmap[j].first.first][A->jmap[j].first.second] = A->jmap[j].second;
      for (size_t j = A->jcells.size(); j-- > 0;)
        if ((size_t)A->jcells[j].first < snap_size) A->cells[A->jcells[j].first] = A->jcells[j].second;
      A->cells.resize(snap_size);
      A->free_blocks = snap_free;
      A->inits.resize(snap_inits);
      cl.swap(kept);   // reverted candidates retry no more
    }
  }
  A->tm_a[2] += now_s() - w0; w0 = now_s();
  garbage_collect(A, &freed);
  A->tm_a[3] += now_s() - w0; w0 = now_s();
  // device: averages of coarsened mothers from their (old) children first
  if (!coarsened.empty()) {
    // children ids are still valid on the device (freed blocks are reused only later)
    Uploader up{A, {}};
    const size_t oc = up.add(coarsened.data(), sizeof(int) * coarsened.size());
    ader_status s0 = up.run(err);
    if (s0 != ADER_OK) return s0;
    // the device child links of these mothers are the pre-adapt ones
    amr_launch_average(*A->k, A->V, (const int*)(A->dscratch + oc), (int)coarsened.size());
  }
  A->tm_a[4] += now_s() - w0; w0 = now_s();
  ader_status s = upload_topology(A, err);
  if (s != ADER_OK) return s;
  A->tm_a[5] += now_s() - w0; w0 = now_s();
  s = run_inits(A, err);
  if (s != ADER_OK) return s;
  // clear the flux memory of every virtual child (synchronized time: all consumed)
  for (int l = 1; l <= A->lmax; ++l) amr_launch_zero_mem(*A->k, A->V, L_vch(A, l), (int)A->lvch[l].size());
  for (int b : freed) A->free_blocks.push_back(b);
  for (auto& c : A->cells) c.isnew = false;
  ACK(cudaStreamSynchronize(sm));
  A->tm_a[6] += now_s() - w0;
  return ADER_OK;
}

// ---- dynamic load balancing (reading R24) ----------
// cost of a level-0 cell: local steps per macro step of its active subtree
// cells (sum of r^level); identical on every rank (the tree is replicated)
std::vector<long long> level0_weights(const AmrState* A) {
  std::vector<long long> w((size_t)(A->n[0][0] * A->n[0][1] * A->n[0][2]), 0);
  long long rl[kAmrMaxLevels];
  rl[0] = 1;
  for (int l = 1; l < kAmrMaxLevels; ++l) rl[l] = rl[l - 1] * A->r;
  for (const HCell& C : A->cells) {
    if (!C.alive || C.status != 0) continue;
    long long a0[3];
    ancestor0(A, C, a0);
    w[(size_t)lin(A, 0, a0)] += rl[C.level];
  }
  return w;
}

// max over ranks of the rank's cost, over the mean
double imbalance(const AmrState* A, const AmrRanks& R, const std::vector<long long>& w) {
  long long tot = 0, mx = 0;
  for (int p = 0; p < R.world; ++p) {
    long long s = 0;
    for (long long z = R.lo[p][2]; z < R.hi[p][2]; ++z)
      for (long long y = R.lo[p][1]; y < R.hi[p][1]; ++y)
        for (long long x = R.lo[p][0]; x < R.hi[p][0]; ++x) s += w[(size_t)((z * A->n[0][1] + y) * A->n[0][0] + x)];
    tot += s;
    mx = std::max(mx, s);
  }
  return tot > 0 ? (double)mx * R.world / (double)tot : 1.0;
}

// Re-cut the level-0 blocks when that lowers the imbalance by more than 2 %
// (and the current one exceeds 5 %).  At synchronized time the only state of
// a cell is its average (the flux memory is cleared, WENO / predictor dofs are
// recomputed every step), so the move is: every rank contributes the averages
// of the cells it owns under the old blocks to a zeroed per-id array, one sum
// over the ranks (exact: a single non-zero term per entry) gives every rank
// all averages, the ownership / compute sets / exchange plans are rebuilt for
// the new blocks and each rank copies the rows of its new compute set.
ader_status rebalance(const Group& G, std::string& err) {
  AmrState* A0 = G[0];
  const int W = A0->ranks.world;
  if (W <= 1 || A0->cfg.load_balance != 1) return ADER_OK;
  const std::vector<long long> w = level0_weights(A0);
  AmrRanks nr = A0->ranks;
  if (!rcb_partition(A0->d, A0->n[0], w.data(), W, nr.lo, nr.hi)) return ADER_OK;
  const double cur = imbalance(A0, A0->ranks, w), nxt = imbalance(A0, nr, w);
  if (!(cur > 1.05 && nxt * 1.02 < cur)) return ADER_OK;
  // The cells whose level-0 ancestor changes owner move from the old to the
  // new owner (one grouped point-to-point of their averages, ids ascending
  // on both sides); then every rank's new compute and present sets are built
  // and one exchange of every level brings the present copies up to date.  At
  // synchronized time a cell's only state is its average (the flux memory is
  // cleared, the WENO / predictor dofs are recomputed every step).
  const size_t nu = A0->cells.size(), nv = (size_t)A0->nv;
  ader_status s = ADER_OK;
  auto owner_in = [&](const AmrState* A, const AmrRanks& R, const HCell& C) {
    long long a[3];
    ancestor0(A, C, a);
    for (int p = 0; p < R.world; ++p) {
      bool in = true;
      for (int k = 0; k < A->d && in; ++k) in = a[k] >= R.lo[p][k] && a[k] < R.hi[p][k];
      if (in) return p;
    }
    return -1;
  };
  struct Move { std::vector<int> sids, rids; std::vector<long long> soff, roff; };
  std::vector<Move> mv(G.size());
  for (size_t g = 0; g < G.size() && s == ADER_OK; ++g) {
    AmrState* A = G[g];
    const int me = A->ranks.rank;
    std::vector<std::vector<int>> snd(W), rcv(W);
    for (size_t i = 0; i < nu; ++i) {
      const HCell& C = A->cells[i];
      if (!C.alive) continue;   // virtual cells too: the new owner exports them (ader_get_cells)
      const int po = owner_in(A, A->ranks, C), pn = owner_in(A, nr, C);
      if (po == pn) continue;
      if (po == me) snd[pn].push_back((int)i);
      if (pn == me) rcv[po].push_back((int)i);
    }
    Move& M = mv[g];
    M.soff.assign(W + 1, 0);
    M.roff.assign(W + 1, 0);
    for (int p = 0; p < W; ++p) {
      M.soff[p] = (long long)M.sids.size();
      M.sids.insert(M.sids.end(), snd[p].begin(), snd[p].end());
      M.roff[p] = (long long)M.rids.size();
      M.rids.insert(M.rids.end(), rcv[p].begin(), rcv[p].end());
    }
    M.soff[W] = (long long)M.sids.size();
    M.roff[W] = (long long)M.rids.size();
    const size_t need = std::max(M.sids.size(), M.rids.size()) * nv + 1;
    if (A->rb_cap < need) {   // persistent, grown 2x
      const size_t cap = std::max(need, 2 * A->rb_cap);
      cudaStreamSynchronize(A->k->stream);
      if (A->rb_buf) cudaFree(A->rb_buf);
      if (A->rb_tmp) cudaFree(A->rb_tmp);
      A->rb_buf = A->rb_tmp = nullptr;
      A->rb_cap = 0;
      if (cudaMalloc(&A->rb_buf, sizeof(double) * cap) != cudaSuccess ||
          cudaMalloc(&A->rb_tmp, sizeof(double) * cap) != cudaSuccess) { err = "cudaMalloc (rebalance)"; s = ADER_ERR_CUDA; break; }
      A->rb_cap = cap;
    }
  }
  // device id lists of the moves (one upload per rank), then gather the sent rows
  std::vector<const int*> dsids(G.size(), nullptr), drids(G.size(), nullptr);
  for (size_t g = 0; g < G.size() && s == ADER_OK; ++g) {
    AmrState* A = G[g];
    Uploader up{A, {}};
    const size_t os = up.add(mv[g].sids.data(), sizeof(int) * mv[g].sids.size());
    const size_t orr = up.add(mv[g].rids.data(), sizeof(int) * mv[g].rids.size());
    s = up.run(err);
    if (s != ADER_OK) break;
    dsids[g] = (const int*)(A->dscratch + os);
    drids[g] = (const int*)(A->dscratch + orr);
    amr_launch_rows_gather(*A->k, A->V.u, dsids[g], (int)mv[g].sids.size(), A->nv, A->rb_buf);
  }
  if (s == ADER_OK && G.size() > 1) {
    for (AmrState* A : G) cudaStreamSynchronize(A->k->stream);
    for (size_t g = 0; g < G.size() && s == ADER_OK; ++g) {
      AmrState* A = G[g];
      const int me = A->ranks.rank;
      for (int p = 0; p < W; ++p) {
        if (p == me) continue;
        const long long n = mv[g].roff[p + 1] - mv[g].roff[p];
        if (n != mv[p].soff[me + 1] - mv[p].soff[me]) { err = "rebalance plans disagree"; s = ADER_ERR_SOLVER; break; }
        if (n && cudaMemcpyAsync(A->rb_tmp + mv[g].roff[p] * nv, G[p]->rb_buf + mv[p].soff[me] * nv,
                                 sizeof(double) * n * nv, cudaMemcpyDeviceToDevice, A->k->stream) != cudaSuccess) {
          err = "rebalance copy"; s = ADER_ERR_CUDA; break;
        }
      }
    }
    for (AmrState* A : G) cudaStreamSynchronize(A->k->stream);
  } else if (s == ADER_OK) {
    const Move& M = mv[0];
    std::vector<int> peers;
    std::vector<double*> sp, rp;
    std::vector<size_t> sc, rc;
    for (int p = 0; p < W; ++p) {
      const size_t ns = (size_t)(M.soff[p + 1] - M.soff[p]), nr2 = (size_t)(M.roff[p + 1] - M.roff[p]);
      if (p == A0->ranks.rank || (!ns && !nr2)) continue;
      peers.push_back(p);
      sp.push_back(A0->rb_buf + M.soff[p] * nv); sc.push_back(ns * nv);
      rp.push_back(A0->rb_tmp + M.roff[p] * nv); rc.push_back(nr2 * nv);
    }
    if (!peers.empty()) {
      s = A0->comm.p2p(A0->comm.ctx, (int)peers.size(), peers.data(), sp.data(), sc.data(), rp.data(), rc.data(),
                       A0->k->stream);
      if (s != ADER_OK) err = "rebalance point-to-point failed";
    }
  }
  for (size_t g = 0; g < G.size() && s == ADER_OK; ++g) {
    AmrState* A = G[g];
    amr_launch_rows_scatter(*A->k, A->V.u, drids[g], (int)mv[g].rids.size(), A->nv, A->rb_tmp);
    cudaStreamSynchronize(A->k->stream);   // the id lists live in the upload scratch
  }
  // new blocks: ownership, compute / present sets, lists, exchange plans
  for (size_t g = 0; g < G.size() && s == ADER_OK; ++g) {
    AmrState* A = G[g];
    for (int p = 0; p < W; ++p)
      for (int k = 0; k < 3; ++k) { A->ranks.lo[p][k] = nr.lo[p][k]; A->ranks.hi[p][k] = nr.hi[p][k]; }
    s = upload_topology(A, err);
    if (s != ADER_OK) break;
    // virtual children that entered this rank's lists: no flux memory from before
    for (int l = 1; l <= A->lmax; ++l) amr_launch_zero_mem(*A->k, A->V, L_vch(A, l), (int)A->lvch[l].size());
    A->nrebal++;
  }
  // the owners' averages to every rank's new present copies
  for (int l = 0; l <= A0->lmax && s == ADER_OK; ++l) s = exchange(G, l, err);
  auto cleanup = [&]() {
    for (AmrState* A : G) cudaStreamSynchronize(A->k->stream);
  };
  cleanup();
  return s;
}

// One adapt pass of every rank of the group on the global indicator.
ader_status adapt(const Group& G, bool t0, std::string& err) {
  std::vector<double> chi, mine;
  double w0 = now_s();
  for (AmrState* A : G) {
    ader_status s = adapt_indicator(A, t0, mine, err);
    if (s != ADER_OK) return s;
    if (chi.size() < mine.size()) chi.resize(mine.size(), 0.0);
    for (size_t i = 0; i < mine.size(); ++i) chi[i] += mine[i];   // one owner per cell: exact
  }
  G[0]->tm_ind += now_s() - w0;
  w0 = now_s();
  AmrState* A0 = G[0];
  if (G.size() == 1 && A0->ranks.world > 1 && !chi.empty()) {
    cudaStream_t sm = A0->k->stream;
    ACK(cudaMemcpyAsync(A0->V.chi, chi.data(), sizeof(double) * chi.size(), cudaMemcpyHostToDevice, sm));
    ader_status s = A0->comm.sum(A0->comm.ctx, A0->V.chi, chi.size(), sm);
    if (s != ADER_OK) { err = "allreduce(sum) of the indicator failed"; return s; }
    ACK(cudaMemcpyAsync(chi.data(), A0->V.chi, sizeof(double) * chi.size(), cudaMemcpyDeviceToHost, sm));
    ACK(cudaStreamSynchronize(sm));
  }
  for (AmrState* A : G) {
    ader_status s = adapt_apply(A, t0, chi, err);
    if (s != ADER_OK) return s;
  }
  A0->tm_apply += now_s() - w0;
  w0 = now_s();
  // the band copies of new / re-initialised active cells come from their owners
  for (int l = 0; l <= A0->lmax; ++l) {
    ader_status s = exchange(G, l, err);
    if (s != ADER_OK) return s;
  }
  for (AmrState* A : G) ACK(cudaStreamSynchronize(A->k->stream));
  A0->tm_exch += now_s() - w0;
  return rebalance(G, err);
}

}  // namespace

// ===========================================================================
namespace {
bool rcb_box(int d, const long long n0[3], const long long* w, const int blo[3], const int bhi[3], int p0, int np,
             int lo[][3], int hi[][3]) {
  if (np == 1) {
    for (int k = 0; k < 3; ++k) { lo[p0][k] = blo[k]; hi[p0][k] = bhi[k]; }
    return true;
  }
  int ax = 0;
  for (int k = 1; k < d; ++k)
    if (bhi[k] - blo[k] > bhi[ax] - blo[ax]) ax = k;
  const int n1 = np / 2, n2 = np - n1, ext = bhi[ax] - blo[ax];
  if (ext < np) return false;
  std::vector<long long> plane((size_t)ext, 0);
  long long tot = 0;
  for (long long z = blo[2]; z < bhi[2]; ++z)
    for (long long y = blo[1]; y < bhi[1]; ++y)
      for (long long x = blo[0]; x < bhi[0]; ++x) {
        const long long c[3] = {x, y, z};
        const long long v = w[(size_t)((z * n0[1] + y) * n0[0] + x)];
        plane[(size_t)(c[ax] - blo[ax])] += v;
        tot += v;
      }
  int cut = -1;
  long long best = 0, acc = 0;
  for (int c = blo[ax] + 1; c < bhi[ax]; ++c) {
    acc += plane[(size_t)(c - 1 - blo[ax])];
    if (c - blo[ax] < n1 || bhi[ax] - c < n2) continue;
    const long long dev = std::llabs(acc * np - tot * n1);
    if (cut < 0 || dev < best) { cut = c; best = dev; }
  }
  int lhi[3] = {bhi[0], bhi[1], bhi[2]}, ulo[3] = {blo[0], blo[1], blo[2]};
  lhi[ax] = cut;
  ulo[ax] = cut;
  return rcb_box(d, n0, w, blo, lhi, p0, n1, lo, hi) && rcb_box(d, n0, w, ulo, bhi, p0 + n1, n2, lo, hi);
}
}  // namespace

bool rcb_partition(int d, const long long n0[3], const long long* w, int world, int lo[][3], int hi[][3]) {
  const int blo[3] = {0, 0, 0};
  const int bhi[3] = {(int)n0[0], d >= 2 ? (int)n0[1] : 1, d >= 3 ? (int)n0[2] : 1};
  return world >= 1 && rcb_box(d, n0, w, blo, bhi, 0, world, lo, hi);
}

int amr_rebalances(const AmrState* A) { return A->nrebal; }

AmrState* amr_create(const ader_config* cfg, KCtx* k, DevCounters* cnt, DevCounters* hcnt, const AmrRanks& ranks,
                     const AmrComm& comm, std::string& err) {
  AmrState* A = new AmrState();
  A->cfg = *cfg;
  A->k = k; A->cnt = cnt; A->hcnt = hcnt;
  A->ranks = ranks;
  A->comm = comm;
  // compute-set margin: the dependency chain of an owned update (face
  // neighbours' predictors, their WENO boxes, the coarser mothers projected into
  // virtual children, finer cells depositing flux memory) stays within
  // (M+1) sum_l r^-l < 2 (M+1) level-0 cells of the owned block for r >= M
  A->band = 2 * (cfg->degree + 1);
  {
    const char* e = std::getenv("ADER_AMR_BAND");   // A/B: the round-1 uniform band
    A->band_sets = e && e[0] == '1';
  }
  A->d = cfg->dim; A->M = cfg->degree; A->N = A->M + 1;
  A->nv = cfg->system == ADER_MHD_GLM ? 9 : cfg->dim + 2;
  A->NS = 1;
  for (int i = 0; i < A->d; ++i) A->NS *= A->N;
  A->NST = A->NS * A->N;
  A->r = cfg->refine_factor; A->lmax = cfg->lmax;
  A->rd = 1;
  for (int i = 0; i < A->d; ++i) A->rd *= A->r;
  if (A->cfg.ic_quad <= 0) A->cfg.ic_quad = A->N;
  if (A->cfg.pred_tol <= 0) A->cfg.pred_tol = 1e-13;
  if (A->cfg.pred_max_sweeps <= 0) A->cfg.pred_max_sweeps = 32;
  build_sub(k->tab, A->N, A->r, &A->st);
  A->hmap.resize(A->lmax + 1);
  for (int l = 0; l <= A->lmax; ++l) {
    long long s = 1, f = 1;
    for (int q = 0; q < l; ++q) f *= A->r;
    for (int i = 0; i < 3; ++i) {
      A->n[l][i] = i < A->d ? cfg->n0[i] * f : 1;
      A->dx[l][i] = i < A->d ? (cfg->hi[i] - cfg->lo[i]) / (double)A->n[l][i] : 1.0;
      s *= A->n[l][i];
    }
    A->hmap[l].assign((size_t)s, -1);
    if (cudaMalloc(&A->dmap[l], sizeof(int) * s) != cudaSuccess) { err = "cudaMalloc map"; delete A; return nullptr; }
    cudaMemset(A->dmap[l], 0xff, sizeof(int) * s);   // -1 everywhere
    A->V.map[l] = A->dmap[l];
    for (int i = 0; i < 3; ++i) A->V.n[l][i] = A->n[l][i];
  }
  for (int i = 0; i < 6; ++i) A->V.bc[i] = cfg->bc[i];
  A->V.D = A->d; A->V.NV = A->nv; A->V.r = A->r; A->V.rd = A->rd;
  const long long n0 = A->n[0][0] * A->n[0][1] * A->n[0][2];
  A->cells.resize(n0);
  for (long long i = 0; i < n0; ++i) {
    HCell& C = A->cells[i];
    C.alive = true;
    C.idx[0] = i % A->n[0][0]; C.idx[1] = (i / A->n[0][0]) % A->n[0][1]; C.idx[2] = i / (A->n[0][0] * A->n[0][1]);
    A->hmap[0][i] = (int)i;
  }
  if (upload_topology(A, err) != ADER_OK) { amr_destroy(A); return nullptr; }
  return A;
}

void amr_destroy(AmrState* A) {
  if (!A) return;
  if (std::getenv("ADER_AMR_TIMING") && A->tm_steps)
    std::fprintf(stderr,
                 "amr host phases over %lld macro steps (ms/step): speed+sync %.3f, advance enqueue %.3f, "
                 "check/sync %.3f, adapt: indicator+sync %.3f, apply (host tree, uploads, inits) %.3f, "
                 "exchange+sync %.3f; cells %zu\n",
                 A->tm_steps, 1e3 * A->tm_speed / A->tm_steps, 1e3 * A->tm_advance / A->tm_steps,
                 1e3 * A->tm_check / A->tm_steps, 1e3 * A->tm_ind / A->tm_steps, 1e3 * A->tm_apply / A->tm_steps,
                 1e3 * A->tm_exch / A->tm_steps, A->cells.size());
  if (std::getenv("ADER_AMR_TIMING") && A->tm_steps)
    std::fprintf(stderr, "  apply (ms/step): marks+refine %.3f, closure %.3f, recoarsening %.3f, GC %.3f, "
                         "coarsened averages %.3f, upload topology %.3f, inits+sync %.3f\n",
                 1e3 * A->tm_a[0] / A->tm_steps, 1e3 * A->tm_a[1] / A->tm_steps, 1e3 * A->tm_a[2] / A->tm_steps,
                 1e3 * A->tm_a[3] / A->tm_steps, 1e3 * A->tm_a[4] / A->tm_steps, 1e3 * A->tm_a[5] / A->tm_steps,
                 1e3 * A->tm_a[6] / A->tm_steps);
  if (std::getenv("ADER_AMR_TIMING") && A->tm_steps)
    std::fprintf(stderr, "  upload (ms/step): capacity %.3f, host scans/lists %.3f (of which mirror diff %.3f), staging+H2D %.3f\n",
                 1e3 * A->tm_u[0] / A->tm_steps, 1e3 * A->tm_u[1] / A->tm_steps, 1e3 * A->tm_u[3] / A->tm_steps,
                 1e3 * A->tm_u[2] / A->tm_steps);
  cudaStreamSynchronize(A->k->stream);
  if (std::getenv("ADER_AMR_MEM"))
    std::fprintf(stderr, "amr memory rank %d/%d: ids %zu (capacity %d), w/q rows %d (capacity %d): w/q %.3f GB, "
                         "per-id w/q would be %.3f GB\n", A->ranks.rank, A->ranks.world, A->cells.size(), A->cap,
                 A->ranks.world > 1 ? A->nslots : (int)A->cells.size(), A->ranks.world > 1 ? A->slot_cap : A->cap,
                 8e-9 * A->nv * (A->NS + A->NST) * (A->ranks.world > 1 ? A->slot_cap : A->cap),
                 8e-9 * A->nv * (A->NS + A->NST) * A->cap);
  void* ps[] = {A->V.u, A->V.mem, A->V.w, A->V.q, A->V.chi, A->V.level, A->V.status, A->V.mother, A->V.child, A->V.idx, A->V.slot,
                A->V.own, A->dlist, A->xsend, A->xrecv, A->rb_buf, A->rb_tmp};
  for (void* p : ps)
    if (p) cudaFree(p);
  for (int l = 0; l < kAmrMaxLevels; ++l)
    if (A->dmap[l]) cudaFree(A->dmap[l]);
  if (A->dscratch) cudaFree(A->dscratch);
  if (A->hstage) cudaFreeHost(A->hstage);
  delete A;
}

double amr_time(const AmrState* A) { return A->t; }

int64_t amr_num_active(const AmrState* A) { return (int64_t)A->nall; }

namespace {
ader_status set_initial(const Group& G, ader_ic_fn ic, void* user, std::string& err) {
  for (AmrState* A : G) {
    A->ic = ic; A->user = user;
    std::vector<int> ids;
    for (int i = 0; i < (int)A->cells.size(); ++i)
      if (A->cells[i].alive) ids.push_back(i);
    ader_status s = ic_cells(A, ids, err);
    if (s != ADER_OK) return s;
  }
  for (int l = 0; l < G[0]->lmax; ++l) {     // initial hierarchy (R20)
    ader_status s = adapt(G, true, err);
    if (s != ADER_OK) return s;
  }
  for (AmrState* A : G) A->t = 0.0;
  return ADER_OK;
}

ader_status step(const Group& G, double t_end, int64_t max_steps, ader_step_report* reps, std::string& err) {
  const size_t n = G.size();
  std::vector<ader_step_report> R(n);
  std::vector<unsigned long long> sw0(n), pc0(n);
  std::vector<int> rb0(n);
  for (size_t i = 0; i < n; ++i) {
    AmrState* A = G[i];
    std::memset(&R[i], 0, sizeof(R[i]));
    A->margin = 1e300;
    for (int l = 0; l < kAmrMaxLevels; ++l) A->updates[l] = 0;
    ACK(cudaMemcpyAsync(A->hcnt, A->cnt, sizeof(DevCounters), cudaMemcpyDeviceToHost, A->k->stream));
    ACK(cudaStreamSynchronize(A->k->stream));
    sw0[i] = A->hcnt->sweeps; pc0[i] = A->hcnt->cells;
    rb0[i] = A->nrebal;
  }
  ader_status s = ADER_OK;
  AmrState* A0 = G[0];
  int64_t steps = 0;
  while (steps < max_steps && A0->t < t_end) {
    double speed = 0.0;
    double w0 = now_s();
    s = fetch_speed(G, &speed, err);
    for (size_t i = 0; i < n && s == ADER_OK; ++i) s = check_err(G[i], err, G.size() == 1);
    A0->tm_speed += now_s() - w0;
    if (s != ADER_OK) break;
    double dt = A0->cfg.cfl / speed;
    if (!(dt > 0.0) || !std::isfinite(dt)) { err = "invalid dt"; s = ADER_ERR_SOLVER; break; }
    if (A0->t + dt > t_end) dt = t_end - A0->t;
    w0 = now_s();
    s = advance(G, 0, 0, dt, err);
    A0->tm_advance += now_s() - w0;
    w0 = now_s();
    for (size_t i = 0; i < n && s == ADER_OK; ++i) s = check_err(G[i], err, G.size() == 1);
    A0->tm_check += now_s() - w0;
    A0->tm_steps++;
    if (s != ADER_OK) break;
    for (size_t i = 0; i < n; ++i) { G[i]->t += dt; R[i].dt0 = dt; R[i].macro_steps++; }
    ++steps;
    if (A0->cfg.adapt_every > 0 && steps % A0->cfg.adapt_every == 0) {
      s = adapt(G, false, err);
      if (s != ADER_OK) break;
    }
  }
  for (size_t i = 0; i < n; ++i) {
    AmrState* A = G[i];
    ACK(cudaMemcpyAsync(A->hcnt, A->cnt, sizeof(DevCounters), cudaMemcpyDeviceToHost, A->k->stream));
    ACK(cudaStreamSynchronize(A->k->stream));
    R[i].t = A->t;
    for (int l = 0; l < kAmrMaxLevels && l <= A->lmax; ++l) {
      R[i].updates_per_level[l] = A->updates[l];
      R[i].cell_updates += A->updates[l];
    }
    R[i].pred_sweeps_total = (int64_t)(A->hcnt->sweeps - sw0[i]);
    R[i].pred_cells = (int64_t)(A->hcnt->cells - pc0[i]);
    R[i].pred_sweeps_max = A->hcnt->sweeps_max;
    R[i].rebalances = A->nrebal - rb0[i];
    R[i].min_threshold_margin = A->margin;
    if (reps) reps[i] = R[i];
  }
  return s;
}
}  // namespace

ader_status amr_set_initial(AmrState* A, ader_ic_fn ic, void* user, std::string& err) {
  return set_initial(Group{A}, ic, user, err);
}

ader_status amr_adapt(AmrState* A, ader_step_report* rep, std::string& err) {
  A->margin = 1e300;
  ader_status s = adapt(Group{A}, false, err);
  if (rep) rep->min_threshold_margin = A->margin;
  return s;
}

ader_status amr_step(AmrState* A, double t_end, int64_t max_steps, ader_step_report* rep, std::string& err) {
  return step(Group{A}, t_end, max_steps, rep, err);
}

ader_status amr_group_set_initial(AmrState* const* g, int n, ader_ic_fn ic, void* user, std::string& err) {
  return set_initial(Group(g, g + n), ic, user, err);
}

ader_status amr_group_step(AmrState* const* g, int n, double t_end, int64_t max_steps, ader_step_report* reps,
                           std::string& err) {
  return step(Group(g, g + n), t_end, max_steps, reps, err);
}

ader_status amr_get_cells(AmrState* A, ader_cell* out, int64_t cap, int64_t* n, std::string& err) {
  // this rank's cells per level; in (level, z, y, x) order either by a scan of
  // the level's dense map or, when the map is much larger than the level's
  // cell count (deep, sparse levels), by sorting the ids on their map index
  std::vector<std::vector<int>> per(A->lmax + 1);
  for (int i = 0; i < (int)A->cells.size(); ++i)
    if (A->cells[i].alive && A->own[i]) per[A->cells[i].level].push_back(i);
  int64_t cnt = 0;
  for (const auto& v : per) cnt += (int64_t)v.size();
  *n = cnt;
  if (!out) return ADER_OK;
  if (cap < cnt) { err = "capacity too small"; return ADER_ERR_ARG; }
  std::vector<double> u(A->cells.size() * A->nv);
  ACK(cudaMemcpyAsync(u.data(), A->V.u, sizeof(double) * u.size(), cudaMemcpyDeviceToHost, A->k->stream));
  ACK(cudaStreamSynchronize(A->k->stream));
  for (int l = 0; l <= A->lmax; ++l) {
    std::vector<int>& ids = per[l];
    if (A->hmap[l].size() > 32 * ids.size()) {
      std::vector<std::pair<long long, int>> key(ids.size());
      for (size_t j = 0; j < ids.size(); ++j) key[j] = {lin(A, l, A->cells[ids[j]].idx), ids[j]};
      std::sort(key.begin(), key.end());
      for (size_t j = 0; j < ids.size(); ++j) ids[j] = key[j].second;
    } else {
      ids.clear();
      for (int id : A->hmap[l])
        if (id >= 0 && A->own[id]) ids.push_back(id);
    }
  }
  int64_t i = 0;
  for (int l = 0; l <= A->lmax; ++l)
    for (int id : per[l]) {
      ader_cell& e = out[i++];
      std::memset(&e, 0, sizeof(e));
      const HCell& C = A->cells[id];
      e.level = C.level; e.status = C.status;
      for (int k = 0; k < 3; ++k) e.idx[k] = C.idx[k];
      for (int v = 0; v < A->nv; ++v) e.u[v] = u[(size_t)id * A->nv + v];
    }
  return ADER_OK;
}

}  // namespace ader
