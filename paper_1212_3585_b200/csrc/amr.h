// amr.h — device-resident cell-by-cell AMR with local time stepping.
//
// Storage: every cell (any level, any status) has an id; per-id SoA arrays on
// the device hold the cell average, the flux memory of virtual children, the
// WENO and predictor dofs, and the tree links.  Each level has a dense id map
// over its full index range (n0 * r^l per axis) for O(1) neighbour lookup,
// and per-level id lists of active cells, virtual children and virtual
// mothers.  The tree topology is mirrored on the host, where the integer
// adapt logic (rules 1-7) runs; every floating-point step (reconstruction,
// predictor, fluxes, update, projection, averaging, indicator, new-child
// initialisation, CFL) runs in the kernels of amr_kernels.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/ader.h"
#include "launch.h"
#include "tables.h"

namespace ader {

constexpr int kAmrMaxLevels = 8;

// Sub-interval tables for refinement factor r (host-built, kernel parameter):
//   Psub[c][p]    = r * int_{c/r}^{(c+1)/r} psi_p          (projection / sub-box averages)
//   Esub[c][k][p] = psi_p((c + lambda_k) / r)              (coarse traces at fine points)
struct SubTables {
  int r;
  double Psub[4][kMaxN];
  double Esub[4][kMaxN][kMaxN];
};

struct AmrDevView {            // raw device pointers handed to kernels
  double* u;                   // [cap][NV]
  double* mem;                 // [cap][6][NV]
  double* w;                   // [cap][NV][NS]
  double* q;                   // [cap][NV][NST]
  double* chi;                 // [cap]
  int* level; int* status; int* mother; int* child;
  long long* idx;              // [cap][3]
  unsigned char* own;          // [cap] multi-rank: 1 = this rank's cell (errors count); nullptr for one rank
  int* slot;                   // [cap] multi-rank: row of the cell in w / q (rows only for the cells this
                               // rank computes, R28; row 0 is scratch); nullptr for one rank (row = id)
  const int* map[kAmrMaxLevels];
  long long n[kAmrMaxLevels][3];
  int bc[6];
  int D, NV, r, rd;
};

struct AmrState;

// Multi-rank AMR: every rank mirrors the whole tree (the adapt is
// deterministic integer logic on the global indicator), owns the subtrees of
// its level-0 block and computes the cells whose level-0 ancestor lies within
// `band` level-0 cells of that block; after every level update the owners'
// new averages overwrite the other ranks' copies.  With one context per rank
// the collectives go through these hooks (NCCL, ader_api.cpp); a loopback
// group (several contexts in one process) exchanges by device copies.
struct AmrComm {
  void* ctx = nullptr;
  // grouped point-to-point: to peers[i] send scount[i] doubles from sendp[i],
  // from peers[i] receive rcount[i] doubles into recvp[i]
  ader_status (*p2p)(void* ctx, int n, const int* peers, double* const* sendp, const size_t* scount,
                     double* const* recvp, const size_t* rcount, cudaStream_t s) = nullptr;
  ader_status (*sum)(void* ctx, double* buf, size_t n, cudaStream_t s) = nullptr;            // in place
  ader_status (*max_u64)(void* ctx, unsigned long long* buf, cudaStream_t s) = nullptr;      // in place
};

struct AmrRanks {
  int rank = 0, world = 1;
  int lo[8][3]{}, hi[8][3]{};   // level-0 block [lo, hi) of every rank
};

// Recursive coordinate bisection of the level-0 cells (reading R24, the
// algorithm of ader_rcb_partition in ader.h): w[n0 x * y * z] >= 0, boxes into
// lo/hi[world].  False if some box cannot give each of its ranks a plane.
bool rcb_partition(int d, const long long n0[3], const long long* w, int world, int lo[][3], int hi[][3]);

AmrState* amr_create(const ader_config* cfg, KCtx* k, DevCounters* cnt, DevCounters* hcnt, const AmrRanks& ranks,
                     const AmrComm& comm, std::string& err);
void amr_destroy(AmrState* a);
ader_status amr_set_initial(AmrState* a, ader_ic_fn ic, void* user, std::string& err);
ader_status amr_step(AmrState* a, double t_end, int64_t max_steps, ader_step_report* rep, std::string& err);
ader_status amr_adapt(AmrState* a, ader_step_report* rep, std::string& err);
int amr_rebalances(const AmrState* a);   // repartitions so far (dynamic load balancing)
// lockstep variants over the ranks of a loopback group (one process, one GPU)
ader_status amr_group_set_initial(AmrState* const* g, int n, ader_ic_fn ic, void* user, std::string& err);
ader_status amr_group_step(AmrState* const* g, int n, double t_end, int64_t max_steps, ader_step_report* reps,
                           std::string& err);
// cells of this rank's subtrees (all cells for one rank)
ader_status amr_get_cells(AmrState* a, ader_cell* out, int64_t cap, int64_t* n, std::string& err);
double amr_time(const AmrState* a);
int64_t amr_num_active(const AmrState* a);

// --- kernels (amr_kernels.cu) ------------------------------------------------
void amr_launch_meta_scatter(const KCtx& k, const AmrDevView& v, const long long* meta, int n);
void amr_launch_map_set(const KCtx& k, const AmrDevView& v, const long long* ch, int n);
void amr_launch_zero_mem(const KCtx& k, const AmrDevView& v, const int* list, int n);
void amr_launch_rows_gather(const KCtx& k, const double* u, const int* ids, int n, int nv, double* out);
void amr_launch_rows_scatter(const KCtx& k, double* u, const int* ids, int n, int nv, const double* in);
void amr_launch_average(const KCtx& k, const AmrDevView& v, const int* list, int n);
void amr_launch_project(const KCtx& k, const AmrDevView& v, const SubTables& st, const int* list, int n,
                        const double* psi_tau);
void amr_launch_weno(const KCtx& k, const AmrDevView& v, const int* list, int n);
// WENO of the active children (level `level`, refinement factor 3) of the listed mothers, one
// sibling patch per CTA; bitwise the w of amr_launch_weno on those children
void amr_launch_weno_patches(const KCtx& k, const AmrDevView& v, const int* moms, int n, int level);
void amr_launch_predictor(const KCtx& k, const AmrDevView& v, const int* list, int n, const double dtdx[3],
                          double tol, int max_sweeps, DevCounters* cnt);
void amr_launch_flux_update(const KCtx& k, const AmrDevView& v, const SubTables& st, const int* list, int n,
                            int m, const double dtdx[3], DevCounters* cnt);
void amr_launch_cfl(const KCtx& k, const AmrDevView& v, const int* list, int n, const double inv_dx0[3],
                    DevCounters* cnt);
void amr_launch_indicator(const KCtx& k, const AmrDevView& v, const int* list, int n, double eps);
// children of mother ids (pairs child, mother): ū = sub-box average of the mother's WENO polynomial
void amr_launch_init_from_weno(const KCtx& k, const AmrDevView& v, const SubTables& st, const int* pairs, int n);
// (child, mother) pairs: ū = sub-box average of the mother's q_h at tau (psi_tau[N])
void amr_launch_init_from_pred(const KCtx& k, const AmrDevView& v, const SubTables& st, const int* pairs, int n,
                               const double* psi_tau);
// ū of listed cells from point values prim[cell][nq][9] and weights
void amr_launch_ic(const KCtx& k, const AmrDevView& v, const int* list, int n, const double* prim,
                   const double* wq, int nq);

}  // namespace ader
