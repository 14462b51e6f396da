// Host driver and C ABI of hjb200 (include/hjb200.h).
//
// hjb_solve replaces the reference's parallel_jacobi (pkg/src/hjacobi/
// parallel.py:255-309), F variants by default and B variants with
// HJB_FLAG_VARIANT_B.  The P ring workers become the items of one batched
// launch per phase; the ring exchange of the reference (parallel.py:212-221)
// is an index remap on one GPU (every block keeps its column position in the
// device copy of G) and an NCCL send/recv of the blocks that cross a GPU
// boundary with several GPUs.  Per sweep:
//   F pre-pass: Gram(diag) -> factor -> Jacobi -> W -> update  (parallel.py:138-148)
//   steps:      Gram(pair) -> factor (structured; B: dense pair) -> Jacobi
//               (F: to convergence; B: one cycle) -> W = R0^-1 R_final -> update
//                                                              (parallel.py:185-210)
//               [-> NCCL block exchange]                       (parallel.py:212-221)
//   one host read of the per-item counters, all-reduced over GPUs
//                                                              (parallel.py:239-244)
// Pivots of order <= 64 use the single cluster pivot kernel of round 1
// (pivot.cu) instead of factor / Jacobi / factor (inner_v1).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hjb200.h"
#include "kernels.h"
#include "schedule.h"

using namespace hjb;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      return fail(HJB_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));          \
  } while (0)
#define NK(x)                                                                           \
  do {                                                                                  \
    ncclResult_t r_ = (x);                                                              \
    if (r_ != ncclSuccess)                                                              \
      return fail(HJB_ENCCL, std::string(#x) + ": " + ncclGetErrorString(r_));          \
  } while (0)

// grow-only device buffer
struct DBuf {
  void *p = nullptr;
  size_t n = 0;
  int dev = -1;
  cudaError_t reserve(size_t bytes) {
    if (bytes <= n && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(bytes, 256));
    if (e == cudaSuccess) n = std::max<size_t>(bytes, 256);
    return e;
  }
};

struct HBuf {
  void *p = nullptr;
  size_t n = 0;
  cudaError_t reserve(size_t bytes) {
    if (bytes <= n && p) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMallocHost(&p, std::max<size_t>(bytes, 256));
    if (e == cudaSuccess) n = std::max<size_t>(bytes, 256);
    return e;
  }
};

struct Workspace {
  DBuf G, items, gitems, A, D, W, U, Gc, R0, Dc, Gp, stats, signs, red, lam, flag;
  HBuf stats_h, red_h;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;  // tail split of the Jacobi launch (run_phase)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::vector<cudaEvent_t> events;
};

std::mutex g_mu;
Workspace g_ws[64];

struct Comm {
  ncclComm_t nccl = nullptr;
  int world = 1, rank = 0, device = 0;
};

size_t esz(int dtype) { return dtype == HJB_C128 ? 16 : 8; }

constexpr int RED_N = 9;  // int64 DiagInfo counters all-reduced at the end of a multi-GPU solve

struct Partition {
  std::vector<int> off, width;  // per block (0-based block index)
  int bmax = 0;
};

Partition uniform_partition(int64_t n, int nbl) {  // blocking.py:63-68
  Partition P;
  const int64_t q = n / nbl, r = n % nbl;
  int64_t o = 0;
  for (int b = 0; b < nbl; ++b) {
    const int w = int(q + (b < r ? 1 : 0));
    P.off.push_back(int(o));
    P.width.push_back(w);
    P.bmax = std::max(P.bmax, w);
    o += w;
  }
  return P;
}

// Inner level: the factor prologue, the ring-of-rings Jacobi kernel and the
// factor epilogue (three launches), or the single cluster pivot kernel of
// round 1 (one launch).  Measured (profiles/r2_inner_v1_ab.jsonl): the three
// kernels win for pivots of order 128 and 256 (cfg2 396 vs 433 ms, cfg3 629
// vs 674 ms), the single launch for order <= 64 (cfg1 54.6 vs 61.6 ms), where
// a pivot is too small to amortise two more launches.  HJB_PIVOT_V1=1 / =0
// forces one or the other (A/B runs).
bool inner_v1(int nmax) {
  static const int forced = [] {
    const char *e = std::getenv("HJB_PIVOT_V1");
    return e ? (std::atoi(e) != 0 ? 1 : 0) : -1;
  }();
  return forced >= 0 ? forced == 1 : nmax <= 64;
}

// round-1 prologue / epilogue inside the cluster pivot kernel (HJB_FACTOR_V1=1, A/B only)
bool factor_v1() {
  static const bool v1 = [] {
    const char *e = std::getenv("HJB_FACTOR_V1");
    return e && std::atoi(e) != 0;
  }();
  return v1;
}

JacobiArgs jacobi_args(const PivotArgs &pa, int jac_mode) {
  JacobiArgs j{};
  j.items = pa.items;
  j.count = pa.count;
  j.nmax = pa.nmax;
  j.ld = pa.nmax;
  j.R0 = pa.R0g;
  j.Rout = pa.W;
  j.signs = pa.signs;
  j.orth_tol = pa.orth_tol;
  j.quad_tol = pa.quad_tol;
  j.max_sweeps = pa.max_sweeps;
  j.stats = pa.stats;
  j.prof = pa.prof;  // phase clocks are the Jacobi kernel's
  static const bool nocheck = [] {  // A/B only: run the final zero-rotation sweep instead of the Gram check
    const char *e = std::getenv("HJB_JAC_NOCHECK");
    return e && std::atoi(e) != 0;
  }();
  j.dscr = nocheck ? nullptr : static_cast<double *>(pa.dscr);
  j.mode = jac_mode;
  return j;
}

// the pivot-phase launches of one batch: factor prologue, Jacobi, factor
// epilogue (or the single v1 launch)
cudaError_t launch_inner(bool cx, PivotArgs pa, int cluster_req, cudaStream_t st, int *cluster_used, int *launches,
                         int jac_mode = JAC_CONVERGE) {
  const bool vb = pa.fp_input == FP_DENSE_PAIR;  // B variants: always the round-2 kernels
  if (inner_v1(pa.nmax) && !vb) {
    pa.mode = PV_FULL;
    ++*launches;
    return launch_pivot(cx, pa, cluster_req, st, cluster_used);
  }
  const JacobiArgs j = jacobi_args(pa, jac_mode);
  pa.prof = nullptr;
  pa.mode = PV_PROLOGUE;
  cudaError_t e = (factor_v1() && !vb) ? launch_pivot(cx, pa, 0, st, nullptr) : launch_factor_prologue(cx, pa, st);
  if (e != cudaSuccess) return e;
  JacShape sh = jacobi_default_shape(cx, pa.nmax, pa.count);
  if (cluster_req > 0 && cluster_req != sh.c && !jacobi_shape_for(pa.nmax, cluster_req, &sh))
    return cudaErrorInvalidConfiguration;  // no instantiated shape with that cluster size
  if (cluster_used) *cluster_used = sh.c;
  e = launch_jacobi(cx, j, sh, st);
  if (e != cudaSuccess) return e;
  pa.mode = PV_EPILOGUE;
  *launches += 3;
  return (factor_v1() && !vb) ? launch_pivot(cx, pa, 0, st, nullptr) : launch_factor_epilogue(cx, pa, st);
}

// items [off, off + cnt) of a batch: every per-item array advanced by off
PivotArgs sub_batch(const PivotArgs &pa, bool cx, int off, int cnt) {
  const size_t w = cx ? 16 : 8;
  PivotArgs s = pa;
  s.items = pa.items + off;
  s.count = cnt;
  s.A = static_cast<char *>(pa.A) + size_t(off) * pa.bmax * pa.bmax * w;
  s.D = pa.D + size_t(off) * 2 * pa.bmax;
  s.W = static_cast<char *>(pa.W) + size_t(off) * pa.nmax * pa.nmax * w;
  s.R0g = static_cast<char *>(pa.R0g) + size_t(off) * pa.nmax * pa.nmax * w;
  s.stats = pa.stats + size_t(off) * ST_N;
  s.dscr = pa.dscr ? static_cast<char *>(pa.dscr) + size_t(off) * pa.nmax * sizeof(double) : nullptr;
  return s;
}

// Tail split of the Jacobi launch (HJB_TAIL_SPLIT=0 disables; A/B).  A batch
// of `count` pivots on a GPU that holds `cap` of them at once runs
// ceil(count / cap) waves; when the last wave is mostly empty (cfg5r: 128
// pivots, 37 resident: 17 pivots on 68 of 148 SMs) those pivots go to a
// second stream, and the epilogue and update of the full waves -- which only
// need their own pivots -- run beside them on the idle SMs.
bool tail_split_enabled() {
  static const bool on = [] {
    const char *e = std::getenv("HJB_TAIL_SPLIT");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

struct PhaseCtx {
  bool cx;
  int64_t m, ld;
  void *G;
  int bmax, nmax, cluster, cluster_req;
  const int8_t *signs;
  double otol, qtol;
  int max_sweeps;
  Workspace *ws;
  cudaStream_t st;
  int splits_used = 0;
  int launches = 0;  // kernels launched by this solve
  bool tail_split = true;
  int tail_splits = 0;  // steps whose Jacobi launch was split
};

// Gram -> pivot -> update for one batch of items (device item table).
// gram_items_d != null: B variants -- three Gram items per pair (A_ii, A_jj,
// A_ij) feed the dense pair factor, and the Jacobi kernel runs one cycle
// (jac_mode) instead of sweeping to convergence (parallel.py:160-174, 199-200)
int run_phase(PhaseCtx &c, const Item *items_d, int count, int64_t *stats_d, void *Rout,
              cudaEvent_t *ev, const Item *gram_items_d = nullptr, int jac_mode = JAC_CONVERGE) {
  if (count == 0) return HJB_OK;
  GramArgs g{};
  g.G = c.G;
  g.ldg = c.ld;
  g.m = c.m;
  g.items = gram_items_d ? gram_items_d : items_d;
  g.count = gram_items_d ? 3 * count : count;
  g.bmax = c.bmax;
  g.A = c.ws->A.p;
  g.D = static_cast<double *>(c.ws->D.p);
  g.Apart = c.ws->Gp.p;
  g.part_bytes = c.ws->Gp.n;
  if (ev) CK(cudaEventRecord(ev[0], c.st));
  int splits = 1;
  CK(launch_gram(c.cx, g, c.st, &splits));
  c.splits_used = splits;
  c.launches += splits > 1 ? 2 : 1;
  if (ev) CK(cudaEventRecord(ev[1], c.st));
  PivotArgs pa{};
  pa.G = c.G;
  pa.ldg = c.ld;
  pa.m = c.m;
  pa.items = items_d;
  pa.count = count;
  pa.bmax = c.bmax;
  pa.A = c.ws->A.p;
  pa.D = static_cast<double *>(c.ws->D.p);
  pa.signs = c.signs;
  pa.orth_tol = c.otol;
  pa.quad_tol = c.qtol;
  pa.max_sweeps = c.max_sweeps;
  pa.W = c.ws->W.p;
  pa.stats = stats_d;
  pa.Rout = Rout;
  pa.nmax = c.nmax;
  pa.uscr = c.ws->U.p;
  pa.gchk = c.ws->Gc.p;
  pa.R0g = c.ws->R0.p;
  pa.dscr = c.ws->Dc.p;
  pa.fp_input = gram_items_d ? FP_DENSE_PAIR : FP_STRUCTURED;
  UpdateArgs u{};
  u.G = c.G;
  u.ldg = c.ld;
  u.m = c.m;
  u.items = items_d;
  u.count = count;
  u.nmax = c.nmax;
  u.W = c.ws->W.p;
  u.stats = stats_d;
  // ---- tail split (see tail_split_enabled) ----
  int n1 = count;
  JacShape sh = jacobi_default_shape(c.cx, c.nmax, count);
  if (tail_split_enabled() && c.tail_split && !gram_items_d && !inner_v1(c.nmax) && !factor_v1() && c.cluster_req == 0 && !Rout &&
      c.ws->stream2 && jac_mode == JAC_CONVERGE) {
    const int cap = jacobi_wave_capacity(c.cx, c.nmax, sh);
    if (cap > 0 && count > cap) {
      const int tail = count % cap;
      if (tail > 0 && 10 * tail <= 7 * cap) n1 = count - tail;  // last wave at most 70 % full
    }
  }
  if (n1 < count) {
    cudaStream_t s2 = c.ws->stream2;
    CK(launch_factor_prologue(c.cx, pa, c.st));
    CK(cudaEventRecord(c.ws->ev_fork, c.st));
    CK(cudaStreamWaitEvent(s2, c.ws->ev_fork, 0));
    const PivotArgs pa1 = sub_batch(pa, c.cx, 0, n1), pa2 = sub_batch(pa, c.cx, n1, count - n1);
    CK(launch_jacobi(c.cx, jacobi_args(pa1, jac_mode), sh, c.st));
    CK(launch_jacobi(c.cx, jacobi_args(pa2, jac_mode), sh, s2));
    CK(launch_factor_epilogue(c.cx, pa1, c.st));
    if (ev) CK(cudaEventRecord(ev[2], c.st));
    UpdateArgs u1 = u, u2 = u;
    u1.count = n1;
    u2.items = items_d + n1;
    u2.count = count - n1;
    u2.W = static_cast<char *>(c.ws->W.p) + size_t(n1) * c.nmax * c.nmax * (c.cx ? 16 : 8);
    u2.stats = stats_d + size_t(n1) * ST_N;
    CK(launch_update(c.cx, u1, c.st));
    CK(launch_factor_epilogue(c.cx, pa2, s2));
    CK(launch_update(c.cx, u2, s2));
    CK(cudaEventRecord(c.ws->ev_join, s2));
    CK(cudaStreamWaitEvent(c.st, c.ws->ev_join, 0));
    c.cluster = sh.c;
    c.launches += 7;
    ++c.tail_splits;
    if (ev) CK(cudaEventRecord(ev[3], c.st));
    return HJB_OK;
  }
  int used = 0;
  CK(launch_inner(c.cx, pa, c.cluster_req, c.st, &used, &c.launches, jac_mode));
  c.cluster = used;
  if (ev) CK(cudaEventRecord(ev[2], c.st));
  CK(launch_update(c.cx, u, c.st));
  ++c.launches;
  if (ev) CK(cudaEventRecord(ev[3], c.st));
  return HJB_OK;
}

int reserve_phase_buffers(Workspace &ws, bool cx, int bmax, int nmax, int max_count, int64_t m,
                          int gram_items = 0) {
  const size_t w = cx ? 16 : 8;
  (void)m;
  const int gcount = std::max(max_count, gram_items);  // B variants: three Gram items per pair
  CK(ws.A.reserve(size_t(gcount) * bmax * bmax * w));
  CK(ws.D.reserve(size_t(gcount) * 2 * bmax * 8));
  CK(ws.W.reserve(size_t(max_count) * nmax * nmax * w));
  CK(ws.U.reserve(size_t(max_count) * (nmax / 2) * (nmax / 2 + 1) * w));  // pivot factor U (L2 scratch)
  CK(ws.Gc.reserve(size_t(max_count) * pivot_check_elems(nmax) * w));    // final-sweep Gram check
  CK(ws.R0.reserve(size_t(max_count) * nmax * nmax * w));                 // R0 between prologue and Jacobi
  CK(ws.Dc.reserve(size_t(max_count) * nmax * sizeof(double)));          // Jacobi final-sweep check norms
  CK(ws.Gp.reserve(std::min<size_t>(gram_scratch_bytes(cx, gcount, bmax), size_t(768) << 20)));  // Gram split-K partials
  return HJB_OK;
}

}  // namespace

extern "C" {

int hjb_version(void) { return HJB_ABI_VERSION; }
const char *hjb_last_error(void) { return g_err.c_str(); }
int hjb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int hjb_steps_per_sweep(int32_t strategy, int32_t p) {
  if (p < 1 || (strategy != HJB_MODULUS && strategy != HJB_ROUND_ROBIN)) return -1;
  return strategy == HJB_MODULUS ? 2 * p : 2 * p - 1;
}

int hjb_schedule(int32_t strategy, int32_t p, int32_t sweeps, int32_t *layouts, int32_t *plans) {
  if (p < 1 || sweeps < 0 || (strategy != HJB_MODULUS && strategy != HJB_ROUND_ROBIN) || !layouts)
    return fail(HJB_EINVAL, "hjb_schedule: invalid argument");
  try {
    RingSchedule rs(strategy, p);
    int64_t step = 0;
    for (int sw = 1; sw <= sweeps; ++sw) {
      for (int s = 0; s < rs.steps_per_sweep(); ++s, ++step) {
        for (int q = 0; q < p; ++q) {
          layouts[(step * p + q) * 2 + 0] = rs.i_blk(q);
          layouts[(step * p + q) * 2 + 1] = rs.j_blk(q);
        }
        std::vector<StepPlan> pl = rs.advance(sw);
        if (plans)
          for (int q = 0; q < p; ++q) {
            int32_t *o = plans + (step * p + q) * 4;
            o[0] = pl[q].snd_rnk;
            o[1] = pl[q].snd_blk;
            o[2] = pl[q].rcv_rnk;
            o[3] = pl[q].rcv_blk;
          }
      }
    }
  } catch (const std::exception &e) {
    return fail(HJB_EINVAL, e.what());
  }
  return HJB_OK;
}

int hjb_exchange_plan(int32_t strategy, int32_t p, int32_t world, int32_t rank, int32_t sweeps,
                      int32_t max_xfers, int32_t *out, int32_t *counts) {
  if (p < 1 || world < 1 || rank < 0 || rank >= world || p < world || sweeps < 0 || max_xfers < 1 || !out || !counts)
    return fail(HJB_EINVAL, "hjb_exchange_plan: invalid argument");
  try {
    RingSchedule rs(strategy, p);
    int64_t step = 0;
    for (int sw = 1; sw <= sweeps; ++sw)
      for (int s = 0; s < rs.steps_per_sweep(); ++s, ++step) {
        std::vector<Xfer> xf;
        step_transfers(rs.advance(sw), p, world, rank, xf);
        if (int(xf.size()) > max_xfers) return fail(HJB_EINVAL, "hjb_exchange_plan: max_xfers too small");
        counts[step] = int32_t(xf.size());
        for (size_t t = 0; t < xf.size(); ++t) {
          int32_t *o = out + (step * max_xfers + int64_t(t)) * 3;
          o[0] = xf[t].blk;
          o[1] = xf[t].peer;
          o[2] = xf[t].send ? 1 : 0;
        }
      }
  } catch (const std::exception &e) {
    return fail(HJB_EINVAL, e.what());
  }
  return HJB_OK;
}

int hjb_partition(int64_t n, int32_t nbl, int64_t *offsets) {
  if (nbl < 1 || n < nbl || !offsets) return fail(HJB_EINVAL, "hjb_partition: need 1 <= nbl <= n");
  const Partition P = uniform_partition(n, nbl);
  for (int b = 0; b < nbl; ++b) offsets[b] = P.off[b];
  offsets[nbl] = n;
  return HJB_OK;
}

int hjb_block_owners(int32_t strategy, int32_t p, int32_t world, int32_t sweeps, int32_t *owner) {
  if (p < 1 || world < 1 || p < world || sweeps < 0 || !owner ||
      (strategy != HJB_MODULUS && strategy != HJB_ROUND_ROBIN))
    return fail(HJB_EINVAL, "hjb_block_owners: invalid argument");
  try {
    const std::vector<int> o = final_block_owners(strategy, p, world, sweeps);
    for (int b = 0; b < 2 * p; ++b) owner[b] = o[b];
  } catch (const std::exception &e) {
    return fail(HJB_EINVAL, e.what());
  }
  return HJB_OK;
}

int hjb_comm_unique_id(char out[128]) {
  ncclUniqueId id;
  NK(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "nccl unique id size");
  std::memcpy(out, &id, 128);
  return HJB_OK;
}

int hjb_comm_init(const char id[128], int32_t world, int32_t rank, int32_t device, void **comm) {
  if (!comm || world < 1 || rank < 0 || rank >= world) return fail(HJB_EINVAL, "hjb_comm_init: bad rank/world");
  CK(cudaSetDevice(device));
  Comm *c = new Comm();
  c->world = world;
  c->rank = rank;
  c->device = device;
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  ncclResult_t r = ncclCommInitRank(&c->nccl, world, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(HJB_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  *comm = c;
  return HJB_OK;
}

int hjb_comm_destroy(void *comm) {
  if (!comm) return HJB_OK;
  Comm *c = static_cast<Comm *>(comm);
  if (c->nccl) ncclCommDestroy(c->nccl);
  delete c;
  return HJB_OK;
}

int hjb_pivot_ld(int32_t bmax) { return pivot_nmax(bmax); }

static long long *g_pivot_prof = nullptr;
// Debug: per-CTA phase clocks of subsequent hjb_pivot launches (device
// buffer of [count*cluster][8] int64, or NULL to disable).
int hjb_pivot_set_profile(void *prof) {
  g_pivot_prof = static_cast<long long *>(prof);
  return HJB_OK;
}

int hjb_pivot_order(int32_t dtype, int32_t bmax, int32_t count, int32_t cluster, int32_t *nmax,
                    int32_t *warps) {
  const bool cx = dtype == HJB_C128;
  const int nm = pivot_nmax(bmax);
  if (nm < 0 || count < 1) return HJB_EINVAL;
  const int c = cluster > 0 ? cluster : pivot_choose_cluster(cx, nm, count);
  *nmax = nm;
  *warps = pivot_choose_threads(cx, nm, c) / 32;
  return HJB_OK;
}

int hjb_inner_order(int32_t dtype, int32_t bmax, int32_t count, int32_t cluster, int32_t *desc) {
  const bool cx = dtype == HJB_C128;
  const int nm = pivot_nmax(bmax);
  if (nm < 0 || count < 1 || !desc) return fail(HJB_EINVAL, "hjb_inner_order: bad arguments");
  if (inner_v1(nm)) {
    const int c = cluster > 0 ? cluster : pivot_choose_cluster(cx, nm, count);
    desc[0] = 1;
    desc[1] = nm;
    desc[2] = pivot_choose_threads(cx, nm, c) / 32;
    desc[3] = desc[4] = 0;
    return HJB_OK;
  }
  JacShape sh = jacobi_default_shape(cx, nm, count);
  if (cluster > 0 && cluster != sh.c && !jacobi_shape_for(nm, cluster, &sh))
    return fail(HJB_EINVAL, "hjb_inner_order: no Jacobi shape with that cluster size");
  desc[0] = 2;
  desc[1] = nm;
  desc[2] = sh.c;
  desc[3] = sh.w;
  desc[4] = sh.spw;
  return HJB_OK;
}

int hjb_pivot_occupancy(int32_t dtype, int32_t bmax, int32_t cluster, int32_t threads) {
  return pivot_max_active_clusters(dtype == HJB_C128, pivot_nmax(bmax), cluster, threads);
}

int hjb_tune(int32_t pivot_threads, int32_t pivot_cluster) {
  pivot_tune(pivot_threads, pivot_cluster);
  return HJB_OK;
}

int hjb_solve(const hjb_problem *pr, hjb_result *res) {
  if (!pr || !res) return fail(HJB_EINVAL, "null problem/result");
  std::memset(res, 0, sizeof(*res));
  res->fail_rank = res->fail_r = res->fail_s = -1;
  const bool cx = pr->dtype == HJB_C128;
  if (pr->dtype != HJB_F64 && pr->dtype != HJB_C128) return fail(HJB_EINVAL, "dtype must be float64 or complex128");
  const int64_t m = pr->m, n = pr->n;
  if (m < 1 || n < 1 || pr->ldg < m) return fail(HJB_EINVAL, "bad shape / leading dimension");
  if (pr->p < 1) return fail(HJB_EINVAL, "p must be >= 1");
  const int P = pr->p, nbl = 2 * P;
  if (nbl > n) return fail(HJB_EINVAL, "need at least " + std::to_string(nbl) + " columns for p=" + std::to_string(P) + " workers");
  if (pr->strategy != HJB_MODULUS && pr->strategy != HJB_ROUND_ROBIN) return fail(HJB_EINVAL, "unknown strategy");
  if (pr->max_sweeps < 1) return fail(HJB_EINVAL, "max_sweeps must be >= 1");
  if (!pr->signs || !pr->G_in || !pr->G_out) return fail(HJB_EINVAL, "null G/signs pointer");
  for (int64_t k = 0; k < n; ++k)
    if (pr->signs[k] != 1 && pr->signs[k] != -1) return fail(HJB_EINVAL, "sign vector entries must be -1 or +1");
  const Partition part = uniform_partition(n, nbl);
  const int bmax = part.bmax;
  const int nmax = pivot_nmax(bmax);
  if (nmax < 0) return fail(HJB_EINVAL, "block width " + std::to_string(bmax) + " > 128 is not supported (raise p)");
  Comm *comm = static_cast<Comm *>(pr->comm);
  const int world = comm ? comm->world : 1, grank = comm ? comm->rank : 0;
  if (P < world) return fail(HJB_EINVAL, "p must be >= the number of GPUs");

  std::lock_guard<std::mutex> lock(g_mu);
  if (pr->device < 0 || pr->device >= 64) return fail(HJB_EINVAL, "bad device");
  CK(cudaSetDevice(pr->device));
  Workspace &ws = g_ws[pr->device];
  if (!ws.stream) CK(cudaStreamCreateWithFlags(&ws.stream, cudaStreamNonBlocking));
  if (!ws.stream2) {
    CK(cudaStreamCreateWithFlags(&ws.stream2, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ws.ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ws.ev_join, cudaEventDisableTiming));
  }
  cudaStream_t st = pr->stream ? static_cast<cudaStream_t>(pr->stream) : ws.stream;
  const size_t w = esz(pr->dtype);

  // ---- working copy of G (column positions never change) ----
  void *Gd = nullptr;
  int64_t ld = pr->ldg;
  const bool dev_io = pr->memspace == HJB_DEVICE;
  if (dev_io) {
    Gd = pr->G_out;
    if (pr->G_out != pr->G_in)
      CK(cudaMemcpy2DAsync(pr->G_out, ld * w, pr->G_in, ld * w, m * w, n, cudaMemcpyDeviceToDevice, st));
  } else {
    ld = cx ? m : m + (m & 1);  // even ld keeps 16-byte cp.async alignment
    CK(ws.G.reserve(size_t(ld) * n * w));
    Gd = ws.G.p;
    CK(cudaMemcpy2DAsync(Gd, ld * w, pr->G_in, pr->ldg * w, m * w, n, cudaMemcpyHostToDevice, st));
  }
  CK(ws.signs.reserve(n));
  CK(cudaMemcpyAsync(ws.signs.p, pr->signs, n, cudaMemcpyHostToDevice, st));

  // ---- sweep range: [s0, s1] (a resumed solve starts at sweep s0 from the
  // state G_in had after sweep s0 - 1; the ring layout is data-independent) ----
  const int s0 = std::max(1, pr->first_sweep);
  if (s0 > pr->max_sweeps) return fail(HJB_EINVAL, "first_sweep > max_sweeps");
  if (pr->sweep_count < 0) return fail(HJB_EINVAL, "sweep_count must be >= 0");
  const int s1 = pr->sweep_count > 0 ? std::min(pr->max_sweeps, s0 + pr->sweep_count - 1) : pr->max_sweeps;
  const int nsw = s1 - s0 + 1;

  // ---- schedule -> per-sweep item tables of this GPU's workers ----
  RingSchedule ring(pr->strategy, P);
  const int steps = ring.steps_per_sweep();
  try {
    for (int sw = 1; sw < s0; ++sw)
      for (int s = 0; s < steps; ++s) ring.advance(sw);
  } catch (const std::exception &e) {
    return fail(HJB_EINVAL, e.what());
  }
  const int q_lo = workers_lo(P, world, grank), q_hi = workers_lo(P, world, grank + 1), nloc = q_hi - q_lo;
  // B variants (2B / 3B, parallel.py:160-174): no F pre-pass, the dense pair
  // factor, one Jacobi cycle per step
  const bool vb = pr->flags & HJB_FLAG_VARIANT_B;
  // layouts for sweeps s0..s1: [sweep - s0][1 + steps][nloc or 2*nloc]
  const int per_sweep_items = 2 * nloc + steps * nloc;
  std::vector<Item> items(size_t(nsw) * per_sweep_items);
  std::vector<Item> gitems(vb ? size_t(nsw) * steps * 3 * nloc : 0);  // Gram items of the B variants
  std::vector<std::vector<Xfer>> xfers(size_t(nsw) * steps);
  try {
    for (int sw = s0; sw <= s1; ++sw) {
      Item *base = items.data() + size_t(sw - s0) * per_sweep_items;
      for (int q = q_lo; q < q_hi; ++q) {  // pre-pass: the two blocks each worker holds
        const int bi = ring.i_blk(q) - 1, bj = ring.j_blk(q) - 1;
        base[2 * (q - q_lo) + 0] = Item{part.off[bi], part.width[bi], 0, 0};
        base[2 * (q - q_lo) + 1] = Item{part.off[bj], part.width[bj], 0, 0};
      }
      for (int s = 0; s < steps; ++s) {
        Item *row = base + 2 * nloc + s * nloc;
        for (int q = q_lo; q < q_hi; ++q) {
          const int bi = ring.i_blk(q) - 1, bj = ring.j_blk(q) - 1;
          row[q - q_lo] = Item{part.off[bi], part.width[bi], part.off[bj], part.width[bj]};
          if (vb) {
            Item *g3 = gitems.data() + ((size_t(sw - s0) * steps + s) * nloc + (q - q_lo)) * 3;
            g3[0] = Item{part.off[bi], part.width[bi], 0, 0};
            g3[1] = Item{part.off[bj], part.width[bj], 0, 0};
            g3[2] = row[q - q_lo];
          }
        }
        std::vector<StepPlan> pl = ring.advance(sw);
        step_transfers(pl, P, world, grank, xfers[size_t(sw - s0) * steps + s]);
      }
    }
  } catch (const std::exception &e) {
    return fail(HJB_EINVAL, e.what());
  }
  CK(ws.items.reserve(items.size() * sizeof(Item)));
  CK(cudaMemcpyAsync(ws.items.p, items.data(), items.size() * sizeof(Item), cudaMemcpyHostToDevice, st));
  if (vb) {
    CK(ws.gitems.reserve(std::max<size_t>(gitems.size(), 1) * sizeof(Item)));
    CK(cudaMemcpyAsync(ws.gitems.p, gitems.data(), gitems.size() * sizeof(Item), cudaMemcpyHostToDevice, st));
  }
  const int max_count = std::max(2 * nloc, 1);
  if (int rc = reserve_phase_buffers(ws, cx, bmax, nmax, max_count, m, vb ? 3 * nloc : 0)) return rc;
  const size_t stats_per_sweep = size_t(per_sweep_items) * ST_N;
  CK(ws.stats.reserve(2 * stats_per_sweep * sizeof(int64_t)));
  CK(ws.stats_h.reserve(stats_per_sweep * sizeof(int64_t)));
  CK(ws.red.reserve((RED_N + 1) * sizeof(int64_t)));
  CK(ws.red_h.reserve((RED_N + 1) * sizeof(int64_t)));

  const bool phase_times = pr->flags & HJB_FLAG_PHASE_TIMES;
  const int nev = phase_times ? 4 * (1 + steps) + 2 * steps : 0;
  while (int(ws.events.size()) < nev + 2) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    ws.events.push_back(e);
  }
  cudaEvent_t ev_start = ws.events[0], ev_stop = ws.events[1];
  CK(cudaEventRecord(ev_start, st));

  PhaseCtx ctx{};
  ctx.cx = cx;
  ctx.m = m;
  ctx.ld = ld;
  ctx.G = Gd;
  ctx.bmax = bmax;
  ctx.nmax = nmax;
  ctx.cluster = 0;
  ctx.cluster_req = 0;
  ctx.signs = static_cast<const int8_t *>(ws.signs.p);
  ctx.otol = pr->orth_tol;
  ctx.qtol = pr->quad_tol;
  ctx.max_sweeps = pr->max_sweeps;
  ctx.ws = &ws;
  ctx.st = st;
  ctx.tail_split = !(pr->flags & HJB_FLAG_NO_TAIL_SPLIT);
  std::vector<int64_t> hstats(stats_per_sweep);
  double tg = 0, tp = 0, tu = 0, tx = 0;

  for (int sw = s0; sw <= s1; ++sw) {
    const Item *it_d = static_cast<const Item *>(ws.items.p) + size_t(sw - s0) * per_sweep_items;
    int64_t *stats_d = static_cast<int64_t *>(ws.stats.p) + size_t((sw - 1) & 1) * stats_per_sweep;
    cudaEvent_t *ev = phase_times ? &ws.events[2] : nullptr;
    if (!vb)
      if (int rc = run_phase(ctx, it_d, 2 * nloc, stats_d, nullptr, ev)) return rc;
    for (int s = 0; s < steps; ++s) {
      cudaEvent_t *evs = phase_times ? &ws.events[2 + 4 * (1 + s)] : nullptr;
      const Item *git = vb ? static_cast<const Item *>(ws.gitems.p) + (size_t(sw - s0) * steps + s) * nloc * 3 : nullptr;
      // first step of a sweep: one cycle over all pairs of the pivot; later
      // steps: the cross pairs only (parallel.py:162-174)
      if (int rc = run_phase(ctx, it_d + 2 * nloc + s * nloc, nloc,
                             stats_d + size_t(2 * nloc + s * nloc) * ST_N, nullptr, evs, git,
                             !vb ? JAC_CONVERGE : (s == 0 ? JAC_ONE_CYCLE : JAC_CROSS)))
        return rc;
      const auto &xf = xfers[size_t(sw - s0) * steps + s];
      if (!xf.empty()) {
        if (phase_times) CK(cudaEventRecord(ws.events[2 + 4 * (1 + steps) + 2 * s], st));
        NK(ncclGroupStart());
        for (const Xfer &x : xf) {
          char *ptr = static_cast<char *>(Gd) + size_t(part.off[x.blk]) * ld * w;
          const size_t bytes = size_t(part.width[x.blk]) * ld * w;
          if (x.send) {
            NK(ncclSend(ptr, bytes, ncclChar, x.peer, comm->nccl, st));
            res->exchange_bytes += int64_t(bytes);
          } else {
            NK(ncclRecv(ptr, bytes, ncclChar, x.peer, comm->nccl, st));
          }
        }
        NK(ncclGroupEnd());
        if (phase_times) CK(cudaEventRecord(ws.events[2 + 4 * (1 + steps) + 2 * s + 1], st));
      }
    }
    // ---- per-sweep counters (parallel.py:239-244) ----
    CK(cudaMemcpyAsync(ws.stats_h.p, stats_d, stats_per_sweep * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::memcpy(hstats.data(), ws.stats_h.p, stats_per_sweep * sizeof(int64_t));
    int64_t rot = 0;
    int err = HJB_OK;
    for (int t = vb ? 2 * nloc : 0; t < per_sweep_items; ++t) {
      const int64_t *sv = hstats.data() + size_t(t) * ST_N;
      const bool pre = t < 2 * nloc;
      const Item &itm = items[size_t(sw - s0) * per_sweep_items + t];
      const int64_t Nq = itm.ni + itm.nj;
      res->inner_sweeps += sv[ST_SWEEPS];
      res->inner_pair_visits += sv[ST_SWEEPS] * (Nq * (Nq - 1) / 2);
      rot += sv[ST_NROT];
      res->rotations += sv[ST_NROT];
      res->big_rotations += sv[ST_NBIG];
      double mt;
      std::memcpy(&mt, &sv[ST_MAXT], 8);
      res->max_abs_t = std::max(res->max_abs_t, mt);
      if (!vb) res->fallbacks += sv[ST_FALLBACK];
      if (pre) {
        res->prepass_visited += 1;
        res->prepass_updated += sv[ST_NROT] > 0;
      } else {
        res->pairs_visited += 1;
        res->pairs_updated += sv[ST_NROT] > 0;
      }
      if (sv[ST_STATUS] != PV_OK && err == HJB_OK) {
        const int q = q_lo + (pre ? t / 2 : (t - 2 * nloc) % std::max(nloc, 1));
        res->fail_rank = q;
        if (sv[ST_STATUS] == PV_INDEFINITE) {
          err = HJB_PIVOT_INDEFINITE;
          res->fail_r = int32_t(sv[ST_FR]);
          res->fail_s = int32_t(sv[ST_FS]);
        } else {
          err = HJB_CHOL_FAIL;
        }
      }
    }
    if (phase_times) {
      float ms = 0;
      for (int s = vb ? 1 : 0; s < 1 + steps; ++s) {
        cudaEvent_t *e = &ws.events[2 + 4 * s];
        if (s > 0 && nloc == 0) continue;
        CK(cudaEventElapsedTime(&ms, e[0], e[1])); tg += ms;
        CK(cudaEventElapsedTime(&ms, e[1], e[2])); tp += ms;
        CK(cudaEventElapsedTime(&ms, e[2], e[3])); tu += ms;
      }
      for (int s = 0; s < steps; ++s)
        if (!xfers[size_t(sw - s0) * steps + s].empty()) {
          CK(cudaEventElapsedTime(&ms, ws.events[2 + 4 * (1 + steps) + 2 * s],
                                  ws.events[2 + 4 * (1 + steps) + 2 * s + 1]));
          tx += ms;
        }
    }
    if (comm) {  // all-reduce of the sweep's rotation count and error (parallel.py:99-118)
      int64_t *rh = static_cast<int64_t *>(ws.red_h.p);
      rh[0] = rot;
      rh[1] = err != HJB_OK ? 1 : 0;
      CK(cudaMemcpyAsync(ws.red.p, rh, 2 * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      NK(ncclAllReduce(ws.red.p, ws.red.p, 2, ncclInt64, ncclSum, comm->nccl, st));
      CK(cudaMemcpyAsync(rh, ws.red.p, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      rot = rh[0];
      if (rh[1] && err == HJB_OK) err = HJB_CHOL_FAIL;  // another GPU failed
    }
    res->sweeps = sw;
    if (err != HJB_OK) {
      res->cluster_size = ctx.cluster;
      return fail(err, err == HJB_PIVOT_INDEFINITE
                           ? "worker " + std::to_string(res->fail_rank) + ": pivot (" + std::to_string(res->fail_r) +
                                 ", " + std::to_string(res->fail_s) + ") is not positive definite"
                           : "worker " + std::to_string(res->fail_rank) + ": matrix is not positive definite");
    }
    if (rot == 0) {
      res->converged = 1;
      break;
    }
  }

  // ---- DiagInfo over all GPUs (parallel.py:302-308: sums over workers,
  // max of max |t|) ----
  if (comm) {
    int64_t *rh = static_cast<int64_t *>(ws.red_h.p);
    const int64_t mine[RED_N] = {res->rotations,       res->big_rotations,  res->pairs_visited,
                                 res->pairs_updated,   res->prepass_visited, res->prepass_updated,
                                 res->fallbacks,       res->inner_sweeps,   res->inner_pair_visits};
    std::memcpy(rh, mine, sizeof(mine));
    CK(cudaMemcpyAsync(ws.red.p, rh, sizeof(mine), cudaMemcpyHostToDevice, st));
    NK(ncclAllReduce(ws.red.p, ws.red.p, RED_N, ncclInt64, ncclSum, comm->nccl, st));
    double *mt = reinterpret_cast<double *>(static_cast<int64_t *>(ws.red.p) + RED_N);
    CK(cudaMemcpyAsync(mt, &res->max_abs_t, sizeof(double), cudaMemcpyHostToDevice, st));
    NK(ncclAllReduce(mt, mt, 1, ncclFloat64, ncclMax, comm->nccl, st));
    CK(cudaMemcpyAsync(rh, ws.red.p, RED_N * sizeof(int64_t) + sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    int64_t *dst[RED_N] = {&res->rotations,       &res->big_rotations,   &res->pairs_visited,
                           &res->pairs_updated,   &res->prepass_visited, &res->prepass_updated,
                           &res->fallbacks,       &res->inner_sweeps,    &res->inner_pair_visits};
    for (int k = 0; k < RED_N; ++k) *dst[k] = rh[k];
    std::memcpy(&res->max_abs_t, rh + RED_N, sizeof(double));
  }

  // ---- gather: every block from the GPU whose worker holds it after the
  // sweeps actually run (parallel.py:299-301) ----
  if (comm) {
    std::vector<int> owner;
    try {
      owner = final_block_owners(pr->strategy, P, world, res->sweeps);
    } catch (const std::exception &e) {
      return fail(HJB_EINVAL, e.what());
    }
    const bool to_root = pr->flags & HJB_FLAG_GATHER_ROOT;
    NK(ncclGroupStart());
    for (int b = 0; b < nbl; ++b) {
      char *ptr = static_cast<char *>(Gd) + size_t(part.off[b]) * ld * w;
      const size_t bytes = size_t(part.width[b]) * ld * w;
      if (!to_root) {
        NK(ncclBroadcast(ptr, ptr, bytes, ncclChar, owner[b], comm->nccl, st));
      } else if (owner[b] != 0) {  // rank 0 receives every block it does not hold
        if (grank == owner[b]) NK(ncclSend(ptr, bytes, ncclChar, 0, comm->nccl, st));
        if (grank == 0) NK(ncclRecv(ptr, bytes, ncclChar, owner[b], comm->nccl, st));
      }
    }
    NK(ncclGroupEnd());
  }
  CK(cudaEventRecord(ev_stop, st));
  if (!dev_io)
    CK(cudaMemcpy2DAsync(pr->G_out, pr->ldg * w, Gd, ld * w, m * w, n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  float tot = 0;
  CK(cudaEventElapsedTime(&tot, ev_start, ev_stop));
  res->t_total_ms = tot;
  res->t_gram_ms = tg;
  res->t_pivot_ms = tp;
  res->t_update_ms = tu;
  res->t_exchange_ms = tx;
  res->cluster_size = ctx.cluster;
  res->gram_splits = ctx.splits_used;
  res->kernel_launches = ctx.launches;
  res->tail_splits = ctx.tail_splits;
  return HJB_OK;
}

// ---------------------------------------------------------------- kernel-level entry points

int hjb_plane_rotations(int32_t dtype, int32_t count, const double *a_rr, const double *a_ss, const void *a_rs,
                        const int8_t *j_rr, const int8_t *j_ss, double *out) {
  if (count < 0 || (count > 0 && (!a_rr || !a_ss || !a_rs || !j_rr || !j_ss || !out)))
    return fail(HJB_EINVAL, "hjb_plane_rotations: bad arguments");
  if (count == 0) return HJB_OK;
  const bool cx = dtype == HJB_C128;
  const size_t w = cx ? 16 : 8;
  std::vector<int8_t> same(count);
  for (int k = 0; k < count; ++k) same[k] = j_rr[k] == j_ss[k];
  int dev = 0;
  CK(cudaGetDevice(&dev));
  char *buf = nullptr;
  const size_t bytes = size_t(count) * (8 + 8 + w + 1 + 64) + 64;
  CK(cudaMalloc(&buf, bytes));
  double *darr = reinterpret_cast<double *>(buf);
  double *dass = darr + count;
  char *dars = reinterpret_cast<char *>(dass + count);
  double *dout = reinterpret_cast<double *>(dars + size_t(count) * w);
  int8_t *dsame = reinterpret_cast<int8_t *>(dout + size_t(count) * 8);
  cudaError_t e = cudaMemcpy(darr, a_rr, count * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dass, a_ss, count * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dars, a_rs, count * w, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dsame, same.data(), count, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = launch_plane_rotations(cx, count, darr, dass, dars, dsame, dout, nullptr);
  if (e == cudaSuccess) e = cudaMemcpy(out, dout, size_t(count) * 64, cudaMemcpyDeviceToHost);
  cudaFree(buf);
  CK(e);
  return HJB_OK;
}

static int upload_items(Workspace &ws, const int32_t *items_host, int count, cudaStream_t st) {
  CK(ws.items.reserve(size_t(count) * sizeof(Item)));
  CK(cudaMemcpyAsync(ws.items.p, items_host, size_t(count) * sizeof(Item), cudaMemcpyHostToDevice, st));
  return HJB_OK;
}

int hjb_gram(int32_t dtype, int64_t m, const void *G, int64_t ldg, const int32_t *items_host, int32_t count,
             int32_t bmax, void *A, double *D, void *stream) {
  if (count < 1 || bmax < 1 || m < 1 || !G || !A || !D) return fail(HJB_EINVAL, "hjb_gram: bad arguments");
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_mu);
  Workspace &ws = g_ws[dev];
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = upload_items(ws, items_host, count, st)) return rc;
  const bool cx = dtype == HJB_C128;
  if (int rc = reserve_phase_buffers(ws, cx, bmax, std::max(64, pivot_nmax(bmax)), count, m)) return rc;
  GramArgs g{};
  g.G = G;
  g.ldg = ldg;
  g.m = m;
  g.items = static_cast<const Item *>(ws.items.p);
  g.count = count;
  g.bmax = bmax;
  g.A = A;
  g.D = D;
  g.Apart = ws.Gp.p;
  g.part_bytes = ws.Gp.n;
  CK(launch_gram(cx, g, st));
  CK(cudaStreamSynchronize(st));
  return HJB_OK;
}

int hjb_pivot(int32_t dtype, int64_t m, const void *G, int64_t ldg, const int32_t *items_host, int32_t count,
              int32_t bmax, const void *A, const double *D, const int8_t *signs_dev, double orth_tol,
              double quad_tol, int32_t max_sweeps, void *W, int64_t *stats, void *R_out, int32_t cluster,
              void *stream) {
  if (count < 1 || bmax < 1 || !A || !D || !W || !stats || !signs_dev || max_sweeps < 1)
    return fail(HJB_EINVAL, "hjb_pivot: bad arguments");
  const int nmax = pivot_nmax(bmax);
  if (nmax < 0) return fail(HJB_EINVAL, "hjb_pivot: block width too large");
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_mu);
  Workspace &ws = g_ws[dev];
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = upload_items(ws, items_host, count, st)) return rc;
  PivotArgs pa{};
  pa.G = G;
  pa.ldg = ldg;
  pa.m = m;
  pa.items = static_cast<const Item *>(ws.items.p);
  pa.count = count;
  pa.bmax = bmax;
  pa.A = const_cast<void *>(A);
  pa.D = D;
  pa.signs = signs_dev;
  pa.orth_tol = orth_tol;
  pa.quad_tol = quad_tol;
  pa.max_sweeps = max_sweeps;
  pa.W = W;
  pa.stats = stats;
  pa.Rout = R_out;
  pa.nmax = nmax;
  pa.prof = g_pivot_prof;
  CK(ws.U.reserve(size_t(count) * (nmax / 2) * (nmax / 2 + 1) * (dtype == HJB_C128 ? 16 : 8)));
  pa.uscr = ws.U.p;
  CK(ws.Gc.reserve(size_t(count) * pivot_check_elems(nmax) * (dtype == HJB_C128 ? 16 : 8)));
  pa.gchk = ws.Gc.p;
  CK(ws.R0.reserve(size_t(count) * nmax * nmax * (dtype == HJB_C128 ? 16 : 8)));
  pa.R0g = ws.R0.p;
  CK(ws.Dc.reserve(size_t(count) * nmax * sizeof(double)));
  pa.dscr = ws.Dc.p;
  int launches = 0;
  cudaError_t e = launch_inner(dtype == HJB_C128, pa, cluster, st, nullptr, &launches);
  if (e == cudaErrorInvalidConfiguration) return fail(HJB_EINVAL, "hjb_pivot: unsupported cluster size");
  CK(e);
  CK(cudaStreamSynchronize(st));
  return HJB_OK;
}

int hjb_jacobi(int32_t dtype, const int32_t *items_host, int32_t count, int32_t bmax, const void *R0, void *R_out,
               const int8_t *signs_dev, double orth_tol, double quad_tol, int32_t max_sweeps, int64_t *stats,
               int32_t cluster, void *stream) {
  if (count < 1 || bmax < 1 || !R0 || !R_out || !stats || !signs_dev || max_sweeps < 1)
    return fail(HJB_EINVAL, "hjb_jacobi: bad arguments");
  const int nmax = pivot_nmax(bmax);
  if (nmax < 0) return fail(HJB_EINVAL, "hjb_jacobi: block width too large");
  const bool cx = dtype == HJB_C128;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_mu);
  Workspace &ws = g_ws[dev];
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = upload_items(ws, items_host, count, st)) return rc;
  CK(cudaMemsetAsync(stats, 0, size_t(count) * ST_N * sizeof(int64_t), st));
  JacobiArgs j{};
  j.items = static_cast<const Item *>(ws.items.p);
  j.count = count;
  j.nmax = nmax;
  j.ld = nmax;
  j.R0 = R0;
  j.Rout = R_out;
  j.signs = signs_dev;
  j.orth_tol = orth_tol;
  j.quad_tol = quad_tol;
  j.max_sweeps = max_sweeps;
  j.stats = stats;
  j.prof = g_pivot_prof;
  CK(ws.Dc.reserve(size_t(count) * nmax * sizeof(double)));
  j.dscr = static_cast<double *>(ws.Dc.p);
  JacShape sh = jacobi_default_shape(cx, nmax, count);
  if (cluster > 0 && cluster != sh.c && !jacobi_shape_for(nmax, cluster, &sh))
    return fail(HJB_EINVAL, "hjb_jacobi: no Jacobi shape with that cluster size");
  CK(launch_jacobi(cx, j, sh, st));
  CK(cudaStreamSynchronize(st));
  return HJB_OK;
}

int hjb_update(int32_t dtype, int64_t m, void *G, int64_t ldg, const int32_t *items_host, int32_t count,
               int32_t bmax, const void *W, const int64_t *stats, void *stream) {
  if (count < 1 || bmax < 1 || !G || !W || !stats) return fail(HJB_EINVAL, "hjb_update: bad arguments");
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_mu);
  Workspace &ws = g_ws[dev];
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = upload_items(ws, items_host, count, st)) return rc;
  UpdateArgs u{};
  u.G = G;
  u.ldg = ldg;
  u.m = m;
  u.items = static_cast<const Item *>(ws.items.p);
  u.count = count;
  u.nmax = pivot_nmax(bmax);
  u.W = W;
  u.stats = stats;
  CK(launch_update(dtype == HJB_C128, u, st));
  CK(cudaStreamSynchronize(st));
  return HJB_OK;
}

int hjb_extract(int32_t dtype, int64_t m, int64_t n, const void *G, int64_t ldg, const int8_t *signs_dev,
                double *lam, void *U, int64_t ldu, const int64_t *perm, void *stream) {
  if (m < 1 || n < 0 || !G || !lam || !U || !signs_dev) return fail(HJB_EINVAL, "hjb_extract: bad arguments");
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_mu);
  Workspace &ws = g_ws[dev];
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CK(ws.flag.reserve(sizeof(int)));
  CK(cudaMemsetAsync(ws.flag.p, 0, sizeof(int), st));
  CK(launch_extract(dtype == HJB_C128, m, n, G, ldg, signs_dev, lam, U, ldu, perm,
                    static_cast<int *>(ws.flag.p), st));
  int zf = 0;
  CK(cudaMemcpyAsync(&zf, ws.flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (zf) return fail(HJB_CHOL_FAIL, "zero-norm column: factor is rank deficient");
  return HJB_OK;
}

int hjb_orthogonality(int32_t dtype, int64_t m, int64_t n, const void *U, int64_t ldu, double *out,
                      void *stream) {
  if (m < 1 || n < 0 || !U || !out || ldu < m) return fail(HJB_EINVAL, "hjb_orthogonality: bad arguments");
  if (dtype != HJB_C128 && (ldu & 1)) return fail(HJB_EINVAL, "hjb_orthogonality: ldu must be even for float64");
  *out = 0.0;
  if (n == 0) return HJB_OK;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_mu);
  Workspace &ws = g_ws[dev];
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool cx = dtype == HJB_C128;
  // column blocks of width 64; every block pair (i <= j) is one Gram item
  const int bw = 64;
  const int nbl = int((n + bw - 1) / bw);
  std::vector<Item> all;
  all.reserve(size_t(nbl) * (nbl + 1) / 2);
  for (int i = 0; i < nbl; ++i)
    for (int j = i; j < nbl; ++j) {
      const int oi = i * bw, oj = j * bw;
      all.push_back(Item{oi, int(std::min<int64_t>(bw, n - oi)), oj, int(std::min<int64_t>(bw, n - oj))});
    }
  const int chunk = int(std::min<size_t>(all.size(), 4096));
  if (int rc = reserve_phase_buffers(ws, cx, bw, 64, chunk, m)) return rc;
  CK(ws.items.reserve(all.size() * sizeof(Item)));
  CK(cudaMemcpyAsync(ws.items.p, all.data(), all.size() * sizeof(Item), cudaMemcpyHostToDevice, st));
  CK(ws.red.reserve(sizeof(unsigned long long)));
  unsigned long long *acc = static_cast<unsigned long long *>(ws.red.p);
  CK(cudaMemsetAsync(acc, 0, sizeof(unsigned long long), st));
  for (size_t s0 = 0; s0 < all.size(); s0 += chunk) {
    const int count = int(std::min<size_t>(chunk, all.size() - s0));
    const Item *items_d = static_cast<const Item *>(ws.items.p) + s0;
    GramArgs g{};
    g.G = U;
    g.ldg = ldu;
    g.m = m;
    g.items = items_d;
    g.count = count;
    g.bmax = bw;
    g.A = ws.A.p;
    g.D = static_cast<double *>(ws.D.p);
    g.Apart = ws.Gp.p;
    g.part_bytes = ws.Gp.n;
    CK(launch_gram(cx, g, st));
    CK(launch_orth_max(cx, items_d, count, bw, ws.A.p, acc, st));
  }
  unsigned long long bits = 0;
  CK(cudaMemcpyAsync(&bits, acc, sizeof(bits), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::memcpy(out, &bits, sizeof(double));
  return HJB_OK;
}

}  // extern "C"
