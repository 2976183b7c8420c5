// api.cpp -- the C ABI of include/edit_sync.h: validation, NCCL communicators of the
// M x N mesh (Alg. 1 l.400), workspace carving and the per-unit
// enqueue sequence of Sync() (Alg. 2).
//
// Per unit, N > 1, peer path with the device scalar exchange (the default):
//   K1 pg_norm(local, anchor -> ||Delta_shard||^2) + [last CTA: K-scalar exchange of the
//      partials over NVLink mailboxes + K2 decide (z-test, EMA, Eq. 2 weights,
//      rollback)]
//   RS  Dbar slice = sum_j w_j (anchor - local_j) pulled from the sync row (Eq. 3, l.452)
//      + [last CTA: K-scalar exchange of the ||Dbar slice||^2 partials (Eq. 4)]
//   AG  every Dbar slice pulled from its owner + beta + Nesterov + write-back (l.454-455)
// = 3 dependent launches per unit.  N == 1: K1 (+K2 in its last CTA) then K4, which
// recomputes Delta from local and anchor: two HBM passes.  EDIT_XCHG=nccl / EDIT_ALGO_NCCL
// keep the NCCL baselines (ncclAllGather of the scalars; ncclAllReduce with PreMulSum).
#include <cuda_runtime.h>
#include <nccl.h>

typedef int CUresult_t;  // CUresult (driver API) without including cuda.h
#include <stdio.h>
#include <stdlib.h>
#include <dlfcn.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3 (ranges for nsys; no-ops without a tool)

#include "handle.h"

using namespace edit;

namespace {
// EDIT_NVTX=1: one NVTX range per enqueued unit sync and per round (host-side enqueue spans;
// nsys correlates the CUDA launches inside them).  Scoped: popped on every return path.
struct NvtxRange {
  bool on;
  NvtxRange(bool enable, const char* fmt, int arg) : on(enable) {
    if (!on) return;
    char name[64];
    snprintf(name, sizeof name, fmt, arg);
    nvtxRangePushA(name);
  }
  ~NvtxRange() {
    if (on) nvtxRangePop();
  }
};

thread_local std::string g_last_error;

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Layout {
  size_t scratch_off, ema_off, rec_off, parts_off, total;
  std::vector<size_t> part1, part2;  // per unit: offsets (bytes, from parts_off) of the per-CTA partials
};

Layout layout_of(const edit_sync_config_t& c) {
  Layout L{};
  size_t off = 0;
  const bool nccl = c.sync_dim > 1 && c.algo == EDIT_ALGO_NCCL;
  L.scratch_off = off;
  off += align_up(sizeof(LayerScratch) * (size_t)c.num_layers, 256);
  L.ema_off = off;
  off += align_up(sizeof(edit_ema_t) * (size_t)c.num_layers * c.sync_dim, 256);
  L.rec_off = off;
  off += align_up(sizeof(edit_layer_stats_t) * (size_t)c.num_layers, 256);
  // per-CTA fp64 partials of K1 and K3, one region per unit (so units on different
  // streams never share slots): grid_of(numel, kVecReduce) each
  L.parts_off = off;
  size_t p = 0;
  for (int i = 0; i < c.num_layers; ++i) {
    const size_t g = (size_t)grid_of(c.layer_numel[i], kVecReduce);
    L.part1.push_back(p);
    p += align_up(g * sizeof(double), 256);
    L.part2.push_back(p);
    if (c.sync_dim > 1) {
      const size_t g2 = nccl ? g : (size_t)rs_partial_slots(c.layer_numel[i], c.sync_dim);
      p += align_up(g2 * sizeof(double), 256);
    }
  }
  off += p;
  L.total = off;
  return L;
}

edit_status_t validate(const edit_sync_config_t* c) {
  if (!c) return fail(EDIT_ERR_INVALID_ARG, "null config");
  if (c->shard_dim < 1 || c->shard_dim > EDIT_MAX_SHARD)
    return fail(EDIT_ERR_INVALID_ARG, "shard_dim (M) must be in [1, 8]");
  if (c->sync_dim < 1 || c->sync_dim > EDIT_MAX_SYNC)
    return fail(EDIT_ERR_INVALID_ARG, "sync_dim (N) must be in [1, 8]");
  if (c->rank < 0 || c->rank >= c->shard_dim * c->sync_dim)
    return fail(EDIT_ERR_INVALID_ARG, "rank must be in [0, M*N)");
  if (c->num_layers < 1) return fail(EDIT_ERR_INVALID_ARG, "num_layers must be >= 1");
  if (!c->layer_numel) return fail(EDIT_ERR_INVALID_ARG, "null layer_numel");
  for (int i = 0; i < c->num_layers; ++i)
    if (c->layer_numel[i] < 0) return fail(EDIT_ERR_INVALID_ARG, "negative layer_numel");
  if (c->param_dtype != EDIT_BF16 && c->param_dtype != EDIT_F32)
    return fail(EDIT_ERR_INVALID_ARG, "param_dtype must be EDIT_BF16 or EDIT_F32");
  if (!(c->outer_lr > 0.f)) return fail(EDIT_ERR_INVALID_ARG, "outer_lr (nu) must be > 0");
  if (!(c->outer_momentum >= 0.f && c->outer_momentum < 1.f))
    return fail(EDIT_ERR_INVALID_ARG, "outer_momentum (mu) must be in [0, 1)");
  if (!(c->clip_threshold > 0.f)) return fail(EDIT_ERR_INVALID_ARG, "clip_threshold (phi) must be > 0");
  if (!(c->clip_eps > 0.f)) return fail(EDIT_ERR_INVALID_ARG, "clip_eps must be > 0");
  if (!(c->ema_alpha > 0.f && c->ema_alpha <= 1.f))
    return fail(EDIT_ERR_INVALID_ARG, "ema_alpha must be in (0, 1]");
  if (!(c->anomaly_threshold > 0.f)) return fail(EDIT_ERR_INVALID_ARG, "anomaly_threshold (delta) must be > 0");
  if (c->ema_warmup_rounds < 0) return fail(EDIT_ERR_INVALID_ARG, "ema_warmup_rounds must be >= 0");
  if (c->flags & ~(EDIT_NO_AE | EDIT_NO_WA | EDIT_NO_GC)) return fail(EDIT_ERR_INVALID_ARG, "unknown flags");
  if (c->algo != EDIT_ALGO_PEER && c->algo != EDIT_ALGO_NCCL)
    return fail(EDIT_ERR_INVALID_ARG, "algo must be EDIT_ALGO_PEER or EDIT_ALGO_NCCL");
  return EDIT_OK;
}

#define CUDA_TRY(h, expr)                                                                   \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      if (h) (h)->poisoned = true;                                                          \
      return fail(EDIT_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_));         \
    }                                                                                       \
  } while (0)

#define NCCL_TRY(h, expr)                                                                   \
  do {                                                                                      \
    ncclResult_t r_ = (expr);                                                               \
    if (r_ != ncclSuccess) {                                                                \
      if (h) (h)->poisoned = true;                                                          \
      return fail(EDIT_ERR_NCCL, std::string(#expr ": ") + ncclGetErrorString(r_));         \
    }                                                                                       \
  } while (0)

#define TRY(expr)                              \
  do {                                         \
    edit_status_t s_ = (expr);                 \
    if (s_ != EDIT_OK) return s_;              \
  } while (0)

// cudaEventRecord that stays a real (external) event record when `st` is being captured into
// a CUDA graph (EDIT_GRAPH=1): the round's done / profiling events are read by the host later.
cudaError_t record_event(cudaEvent_t ev, cudaStream_t st) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  const cudaError_t e = cudaStreamIsCapturing(st, &cap);
  if (e != cudaSuccess) return e;
  return cap == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal)
                                              : cudaEventRecord(ev, st);
}

// the peer kernels' variant: LDG full grids for full-speed rounds (EDIT_PEER_KERNELS), the
// persistent TMA pipelines whenever the grid is capped (partition / co-resident modes)
int full_speed(edit_sync_t h, const Mode& m) { return (m.part == 0 && m.cap == 0 && m.smem_kb == 0) ? h->peer_ldg : 0; }

bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusActive;
}

// The mailbox exchange arguments of lane `ln` for `phase`; takes the lane's next host-side
// sequence number (graph mode: the device counter is used instead).
XchgArgs xchg_args(edit_sync_t h, Lane& ln, int phase) {
  XchgArgs x{};
  x.mp = ln.mp;
  x.K = h->K;
  x.me = h->cfg.rank;
  x.phase = phase;
  x.seq = ++ln.seq[phase];
  x.dseq = ln.dseq;
  x.err = h->err_dev;
  x.err_host = h->err_host_dev;
  x.timeout_ns = h->timeout_ns;
  return x;
}

edit_status_t check_unit_args(edit_sync_t h, int32_t layer, const void* local, const void* anchor,
                              const void* momentum) {
  if (!h) return fail(EDIT_ERR_INVALID_ARG, "null handle");
  TRY(check_err(h));
  if (layer < 0 || layer >= h->cfg.num_layers) return fail(EDIT_ERR_INVALID_ARG, "layer out of range");
  if (h->numel[layer] > 0 && (!local || !anchor || !momentum)) return fail(EDIT_ERR_INVALID_ARG, "null buffer");
  if ((((uintptr_t)local) | ((uintptr_t)anchor) | ((uintptr_t)momentum)) & 15u)
    return fail(EDIT_ERR_INVALID_ARG, "buffers must be 16-byte aligned");
  return EDIT_OK;
}

void clear_graphs(edit_sync_t h) {
  for (RoundGraph& g : h->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  h->graphs.clear();
}

}  // namespace

namespace edit {

edit_status_t fail(edit_status_t st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

edit_status_t check_err(edit_sync_t h) {
  if (!h->poisoned && h->err_host && *reinterpret_cast<volatile int*>(h->err_host) != 0) h->poisoned = true;
  if (h->poisoned)
    return fail(EDIT_ERR_STATE, h->err_host && *reinterpret_cast<volatile int*>(h->err_host)
                                    ? "device scalar exchange timed out (a peer rank stopped syncing); handle poisoned"
                                    : "handle poisoned by an earlier CUDA/NCCL error");
  return EDIT_OK;
}

edit_status_t create_local(const edit_sync_config_t* cfg, void* workspace, size_t workspace_bytes,
                           edit_sync_t* out) {
  TRY(validate(cfg));
  if (!out) return fail(EDIT_ERR_INVALID_ARG, "null out");
  *out = nullptr;
  const Layout L = layout_of(*cfg);
  if (!workspace) return fail(EDIT_ERR_INVALID_ARG, "null workspace");
  if (((uintptr_t)workspace & 255u) != 0) return fail(EDIT_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  if (workspace_bytes < L.total) return fail(EDIT_ERR_NO_MEMORY, "workspace too small");

  edit_sync* h = new (std::nothrow) edit_sync();
  if (!h) return fail(EDIT_ERR_NO_MEMORY, "host allocation");
  h->cfg = *cfg;
  h->numel.assign(cfg->layer_numel, cfg->layer_numel + cfg->num_layers);
  h->cfg.layer_numel = h->numel.data();
  h->M = cfg->shard_dim;
  h->N = cfg->sync_dim;
  h->K = h->M * h->N;
  h->sync_idx = cfg->rank / h->M;   // row index n (R20)
  h->shard_idx = cfg->rank % h->M;  // column index m
  *out = h;  // (on failure the caller destroys it)

#define LCUDA(expr)                                                                         \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess) return fail(EDIT_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
  } while (0)

  LCUDA(cudaSetDevice(cfg->device));
  LCUDA(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, cfg->device));
  h->peer_ctas = h->num_sms;
  if (const char* e = getenv("EDIT_XCHG")) h->dev_xchg = strcmp(e, "nccl") != 0;
  if (const char* e = getenv("EDIT_GRAPH")) h->graph = atoi(e) != 0;
  if (const char* e = getenv("EDIT_PEER_KERNELS"))
    h->peer_ldg = !strcmp(e, "tma") ? 0 : !strcmp(e, "ldg2") ? 3 : !strcmp(e, "ldgall") ? 5 : 1;
  if (const char* e = getenv("EDIT_NVTX")) h->nvtx = atoi(e) != 0;
  if (const char* e = getenv("EDIT_GROUP_NUMEL")) {
    const long long v = atoll(e);
    if (v >= 0 && v < (1ll << 31)) h->group_numel = v;
  }
  if (const char* e = getenv("EDIT_PEER_TILE")) {
    const int v = atoi(e);
    if (v >= 32 && v <= 4096 && (v & 31) == 0) h->peer_tile = v;
  }
  // mailbox wait bound: a peer that stops syncing for longer poisons the handle on every rank
  // (default 600 s, like torch's NCCL watchdog; 0 = wait forever as NCCL itself does)
  double tmo = 600.0;
  if (const char* e = getenv("EDIT_XCHG_TIMEOUT_S")) tmo = atof(e);
  h->timeout_ns = tmo > 0 ? (unsigned long long)(tmo * 1e9) : 0ull;
  if (const char* e = getenv("EDIT_SCHED_CTAS")) {  // 0 = full grids also in scheduler rounds
    const int v = atoi(e);
    if (v >= 0) h->sched_ctas = std::min(v, kMaxPeerCtas);
  }
  if (const char* e = getenv("EDIT_SCHED_SMEM_KB")) {
    const int v = atoi(e);
    if (v > 0) h->sched_smem_kb = v;
  }
  if (const char* e = getenv("EDIT_PEER_CTAS")) {
    const int v = atoi(e);
    if (v > 0) h->peer_ctas = std::min(v, kMaxPeerCtas);
  }

  h->ws = static_cast<char*>(workspace);
  h->scratch = reinterpret_cast<LayerScratch*>(h->ws + L.scratch_off);
  h->ema = reinterpret_cast<edit_ema_t*>(h->ws + L.ema_off);
  h->rec = reinterpret_cast<edit_layer_stats_t*>(h->ws + L.rec_off);
  for (int i = 0; i < cfg->num_layers; ++i) {
    h->part1.push_back(reinterpret_cast<double*>(h->ws + L.parts_off + L.part1[i]));
    h->part2.push_back(reinterpret_cast<double*>(h->ws + L.parts_off + L.part2[i]));
  }
  // zero scratch (ticket counters), EMA (mu = sigma = 0, count = 0: R8) and records
  LCUDA(cudaMemset(h->ws + L.scratch_off, 0, L.total - L.scratch_off));
  // sticky exchange error flag: device word + mapped host mirror
  LCUDA(cudaMalloc(reinterpret_cast<void**>(&h->err_dev), sizeof(int)));
  LCUDA(cudaMemset(h->err_dev, 0, sizeof(int)));
  LCUDA(cudaHostAlloc(reinterpret_cast<void**>(&h->err_host), sizeof(int), cudaHostAllocMapped));
  *h->err_host = 0;
  LCUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->err_host_dev), h->err_host, 0));

  h->done.assign(cfg->num_layers, nullptr);
  for (auto& e : h->done) LCUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  h->gate_ev.assign(cfg->num_layers, nullptr);
  for (auto& e : h->gate_ev) LCUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  h->pre_ev.assign(cfg->num_layers, nullptr);
  for (auto& e : h->pre_ev) LCUDA(cudaEventCreate(&e));
  h->post_ev.assign(cfg->num_layers, nullptr);
  for (auto& e : h->post_ev) LCUDA(cudaEventCreate(&e));
  LCUDA(cudaEventCreate(&h->end_ev));
  LCUDA(cudaEventCreate(&h->rnd_ev0));
  LCUDA(cudaEventCreate(&h->rnd_ev1));
  h->tune_ms.assign(kTuneCands, {});
  h->fwd_ms.assign(cfg->num_layers, 0.0);
  h->sched_sms.assign(cfg->num_layers, 0);
  if (const char* e = getenv("EDIT_SM_GBPS")) {
    const double v = atof(e);
    if (v > 0) h->sm_gbps = v;
  }
  if (const char* e = getenv("EDIT_SCHED_GATE")) h->sched_gate = atoi(e) != 0;
  LCUDA(cudaEventCreateWithFlags(&h->fork, cudaEventDisableTiming));

  // EDIT_LANES (1..8) -- must be equal on every rank.  Lanes hide the latency of the scalar
  // chain of the exchange: N > 1 -> 4 (measured 350M 1x2 3.27 -> 2.78 ms, 1B 7.90 -> 7.21 ms,
  // 7B 43.0 -> 42.5 ms vs 2 lanes, profiles/r1_lanes_2gpu.txt); N == 1 -> 2 (no exchange;
  // 7B 1x1 27.0 ms with 2 or 4 lanes)
  int nlanes = h->N > 1 ? 4 : 2;
  if (const char* e = getenv("EDIT_LANES")) {
    const int v = atoi(e);
    if (v >= 1 && v <= 8) nlanes = v;
  }
  int prio_lo = 0, prio_hi = 0;
  LCUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  // lane-stream priority (EDIT_SCHED_PRIORITY=high|normal|low).  Default high: the
  // scheduler's default auto-partition mode wants each SM a forward CTA releases to go to a
  // sync CTA first (edit_sched_set_partition(h, 0, .) -- full grids -- switches to low: then a
  // concurrent forward's GEMM CTAs are placed first and the sync fills the gaps)
  int prio = prio_hi;
  if (const char* e = getenv("EDIT_SCHED_PRIORITY")) {
    if (!strcmp(e, "low")) prio = prio_lo;
    else if (!strcmp(e, "normal")) prio = 0;
  }
  h->lane_prio = prio;
  h->lanes.resize(nlanes);
  h->peer = h->N > 1 && cfg->algo == EDIT_ALGO_PEER;
  int64_t max_numel = 0;
  for (int64_t x : h->numel) max_numel = std::max(max_numel, x);
  const size_t esz = cfg->param_dtype == EDIT_BF16 ? 2 : 4;
  for (int li = 0; li < nlanes; ++li) {
    Lane& ln = h->lanes[li];
    LCUDA(cudaStreamCreateWithPriority(&ln.stream, cudaStreamNonBlocking, prio));
    LCUDA(cudaEventCreateWithFlags(&ln.tail, cudaEventDisableTiming));
    LCUDA(cudaEventCreateWithFlags(&ln.last, cudaEventDisableTiming));
    if (h->K == 1) continue;
    LCUDA(cudaMalloc(reinterpret_cast<void**>(&ln.bar), sizeof(double) * (1 + kMaxRanks)));
    LCUDA(cudaMemset(ln.bar, 0, sizeof(double) * (1 + kMaxRanks)));
    if (h->dev_xchg) {
      LCUDA(cudaMalloc(reinterpret_cast<void**>(&ln.mailbox), align_up(mailbox_bytes(h->K), 256)));
      LCUDA(cudaMemset(ln.mailbox, 0, align_up(mailbox_bytes(h->K), 256)));
      if (h->graph) {
        LCUDA(cudaMalloc(reinterpret_cast<void**>(&ln.dseq), sizeof(unsigned long long) * kXchgPhases));
        LCUDA(cudaMemset(ln.dseq, 0, sizeof(unsigned long long) * kXchgPhases));
      }
    }
    if (h->peer) {
      const Slicing sl = slicing_of(max_numel, h->N, 0, h->peer_tile);
      LCUDA(cudaMalloc(&ln.Lown, align_up((size_t)std::max<int64_t>(max_numel, 8) * esz, 256)));
      LCUDA(cudaMalloc(reinterpret_cast<void**>(&ln.Down), align_up((size_t)sl.slice * 8 * sizeof(float), 256)));
      ln.pp.L[h->sync_idx] = ln.Lown;
      ln.pp.D[h->sync_idx] = ln.Down;
    } else if (h->N > 1) {
      LCUDA(cudaMalloc(reinterpret_cast<void**>(&ln.S), align_up((size_t)std::max<int64_t>(max_numel, 8) * 4, 256)));
    }
  }
  LCUDA(cudaDeviceSynchronize());
#undef LCUDA
  return EDIT_OK;
}

// ------------------------------------------------------------------------------ one unit
edit_status_t plan_unit(edit_sync_t h, Lane& ln, int32_t layer, void* local, float* anchor, float* momentum,
                        cudaStream_t st, const Mode& mode, UnitPlan& p) {
  p = UnitPlan{};
  p.ln = &ln;
  p.layer = layer;
  p.local = local;
  p.anchor = anchor;
  p.momentum = momentum;
  p.st = st;
  p.mode = mode;
  const int N = h->N;
  LayerScratch* scr = &h->scratch[layer];
  p.S = (N > 1 && !h->peer) ? ln.S : nullptr;
  // peer path: read the members' registered locals directly, else stage a copy of ours
  p.direct = h->peer && !h->reg_local.empty() && h->reg_local[layer] == local;
  p.pp = ln.pp;
  if (p.direct)
    for (int j = 0; j < N; ++j) p.pp.L[j] = h->reg_peer[layer][j];
  p.ev = h->profiling ? &h->prof[(size_t)layer * (EDIT_NUM_PHASES + 1)] : nullptr;
  // K2's arguments: module norms of every replica on every rank from one K-scalar gather
  // (R6)
  DecideArgs& d = p.d;
  d.parts = h->K > 1 ? scr->recv1 : &scr->send1;
  d.M = h->M;
  d.N = N;
  d.my_n = h->sync_idx;
  d.ema = h->ema + (size_t)layer * N;
  d.rec = h->rec + layer;
  d.w_out = &scr->w;
  d.w_all_out = scr->w_all;
  d.rollback_out = &scr->rollback;
  d.gsq_out = &scr->gsq;
  d.alpha = h->cfg.ema_alpha;
  d.delta = h->cfg.anomaly_threshold;
  d.warmup = h->cfg.ema_warmup_rounds;
  d.flags = h->cfg.flags;
  UpdateArgs& u = p.u;
  u.local = local;
  u.anchor = anchor;
  u.momentum = momentum;
  u.n = h->numel[layer];
  u.rollback = &scr->rollback;
  u.nu = h->cfg.outer_lr;
  u.mu = h->cfg.outer_momentum;
  u.phi = h->cfg.clip_threshold;
  u.eps = h->cfg.clip_eps;
  u.flags = h->cfg.flags;
  u.rec = h->rec + layer;
  p.gathered = !h->reg_gather.empty() && h->numel[layer] > 0;
  if (p.gathered) {
    u.gather_M = h->M;
    u.gather_off = (int64_t)h->shard_idx * h->numel[layer];
    for (int q = 0; q < h->M; ++q) u.gather[q] = h->reg_gather[layer][q];
  }
  if (h->peer) {
    p.sl = slicing_of(h->numel[layer], N, h->sync_idx, h->peer_tile);
    u.gparts = scr->recv2;  // every slice of every shard, rank order
    u.n_gparts = h->K;
  } else if (N > 1) {
    u.dbar = p.S;
    u.gparts = h->M > 1 ? scr->recv2 : &scr->send2;
    u.n_gparts = h->M > 1 ? h->M : 1;
  } else {
    u.dbar = nullptr;  // Dbar = Delta, G_bar = G (module level)
    u.gparts = &scr->gsq;
    u.n_gparts = 1;
  }
  return EDIT_OK;
}

edit_status_t enqueue_step(edit_sync_t h, UnitPlan& p, int step) {
  Lane& ln = *p.ln;
  const int32_t layer = p.layer;
  const int64_t n = h->numel[layer];
  const int dt = h->cfg.param_dtype;
  LayerScratch* scr = &h->scratch[layer];
  const int N = h->N, M = h->M;
  cudaStream_t st = p.st;
  cudaEvent_t* ev = p.ev;
  // fold: the scalar exchanges run in the last CTA of the producing kernel (mailboxes), and
  // K2 in K1's last CTA; off only for the NCCL scalar-gather baseline (EDIT_XCHG=nccl)
  const bool fold = h->K == 1 || h->dev_xchg;
  int launched = 0;
  switch (step) {
    case kStepBegin:
      if (!capturing(st)) {
        // this lane's buffers and this unit's scratch may have been used last on another
        // stream (edit_layer_sync on any caller stream, rounds, the scheduler): order after it
        CUDA_TRY(h, cudaStreamWaitEvent(st, ln.last, 0));
        CUDA_TRY(h, cudaStreamWaitEvent(st, h->done[layer], 0));
      }
      if (ev) CUDA_TRY(h, record_event(ev[0], st));
      break;
    case kStepNorm: {  // K1: Delta and its shard norm (Alg. 2 l.442-443) [+ exchange + K2]
      FoldArgs f{};
      f.on = fold ? 1 : 0;
      if (fold) {
        if (h->K > 1) f.x = xchg_args(h, ln, 0);
        else f.x.K = 1;
        f.dec = p.d;
      }
      if (p.mode.part > 0 && !p.S && (!h->peer || p.direct))
        launched += launch_pg_norm_tma(dt, p.local, p.anchor, n, scr, h->part1[layer], p.mode.part, f, st);
      else if (h->peer && !p.direct)
        launched += launch_pg_norm_copy(dt, p.local, p.anchor, ln.Lown, n, scr, h->part1[layer], p.mode.cap, f, st);
      else
        launched += launch_pg_norm(dt, p.local, p.anchor, p.S, n, scr, h->part1[layer], p.mode.cap, f, st);
      CUDA_TRY(h, cudaGetLastError());
      if (ev) CUDA_TRY(h, record_event(ev[1], st));
      break;
    }
    case kStepDecide:
      if (!fold) {  // NCCL baseline: gather the K partials, then K2
        NCCL_TRY(h, ncclAllGather(&scr->send1, scr->recv1, 1, ncclFloat64, ln.global, st));
        launched += launch_decide(p.d, st);
        CUDA_TRY(h, cudaGetLastError());
      }
      if (ev) CUDA_TRY(h, record_event(ev[2], st));
      break;
    case kStepExchange:
      if (h->peer) {
        // Eq. 3 as a reduce-scatter over NVLink peer memory: this rank's slice of Dbar; its
        // last CTA exchanges the slice norms (also the barrier after which every member's D
        // slice is complete)
        FoldArgs f{};
        f.on = h->dev_xchg ? 1 : 0;
        if (h->dev_xchg) f.x = xchg_args(h, ln, 1);
        launched += launch_rs(dt, p.pp, p.sl, p.anchor, ln.Down, scr, h->part2[layer], p.mode.peer_ctas,
                              p.mode.smem_kb, full_speed(h, p.mode), f, st);
        CUDA_TRY(h, cudaGetLastError());
        if (ev) CUDA_TRY(h, record_event(ev[3], st));
      } else if (N > 1) {
        // Eq. 3: Dbar = sum_n w_n Delta_n, the weight applied inside NCCL (PreMulSum)
        NCCL_TRY(h, ncclAllReduce(p.S, p.S, (size_t)n, ncclFloat32, ln.ops[layer], ln.sync, st));
        if (ev) CUDA_TRY(h, record_event(ev[3], st));
        launched += launch_sumsq(p.S, n, scr, h->part2[layer], p.mode.cap, st);
        CUDA_TRY(h, cudaGetLastError());
      }
      break;
    case kStepDbarNorm:
      if (h->peer) {
        if (!h->dev_xchg) NCCL_TRY(h, ncclAllGather(&scr->send2, scr->recv2, 1, ncclFloat64, ln.global, st));
        if (ev) CUDA_TRY(h, record_event(ev[4], st));
      } else if (N > 1) {
        if (M > 1) NCCL_TRY(h, ncclAllGather(&scr->send2, scr->recv2, 1, ncclFloat64, ln.shard, st));
        if (ev) CUDA_TRY(h, record_event(ev[4], st));
      }
      break;
    case kStepUpdate:
      if (h->peer) {
        launched += launch_ag_update(dt, p.u, p.pp, p.sl, p.mode.peer_ctas, p.mode.smem_kb, full_speed(h, p.mode), st);
      } else if (p.mode.part > 0 && !p.u.dbar && !p.gathered) {
        launched += launch_update_tma(dt, p.u, p.mode.part, st);
      } else {
        launched += launch_update(dt, p.u, p.mode.cap, st);
      }
      CUDA_TRY(h, cudaGetLastError());
      break;
    case kStepGather:
      if (p.gathered) {
        // every member of the shard group has stored its shard into every gathered module
        // once this barrier completes (their update kernels precede their contributions)
        if (h->dev_xchg) {
          launched += launch_xchg(xchg_args(h, ln, 2), ln.bar, ln.bar + 1, nullptr, st);
          CUDA_TRY(h, cudaGetLastError());
        } else {
          double* gd = h->gather_dev + (size_t)layer * (h->M + 1);
          NCCL_TRY(h, ncclAllGather(gd, gd + 1, 1, ncclFloat64, ln.shard, st));
        }
      }
      break;
    case kStepEnd:
      if (ev) {
        CUDA_TRY(h, record_event(ev[5], st));
        h->pending.push_back(layer);
      }
      CUDA_TRY(h, record_event(h->done[layer], st));  // read by edit_sync_stats / acquire
      CUDA_TRY(h, record_event(ln.last, st));
      break;
    default:
      return fail(EDIT_ERR_INVALID_ARG, "bad step");
  }
  h->launches += launched;
  return EDIT_OK;
}

// ------------------------------------------------------------------------------ unit groups
// Capacity of a lane's staging (elements) and D (vectors) buffers, as create_local sized them.
static void lane_capacity(edit_sync_t h, int64_t* elems, int64_t* dvecs) {
  int64_t max_numel = 0;
  for (int64_t x : h->numel) max_numel = std::max(max_numel, x);
  *elems = std::max<int64_t>(max_numel, 8);
  *dvecs = slicing_of(max_numel, h->N, 0, h->peer_tile).slice;
}

std::vector<std::vector<int32_t>> form_groups(edit_sync_t h, const int32_t* layers, int nunits) {
  std::vector<std::vector<int32_t>> out;
  const bool on = h->peer && h->dev_xchg && h->K > 1 && h->group_numel > 0 && h->reg_gather.empty();
  if (!on) {
    for (int i = 0; i < nunits; ++i) out.push_back({layers[i]});
    return out;
  }
  int64_t cap_e = 0, cap_d = 0;
  lane_capacity(h, &cap_e, &cap_d);
  cap_e = std::min<int64_t>(cap_e, h->group_numel);
  std::vector<int32_t> cur;
  int64_t used_e = 0, used_d = 0;
  auto flush = [&] {
    if (!cur.empty()) out.push_back(cur);
    cur.clear();
    used_e = used_d = 0;
  };
  for (int i = 0; i < nunits; ++i) {
    const int32_t u = layers[i];
    const int64_t n = h->numel[u];
    const int64_t ne = (n + 7) / 8 * 8;                            // staging offsets stay 16-B aligned
    const int64_t nd = slicing_of(n, h->N, 0, h->peer_tile).slice;  // D region (vectors)
    if (n <= 0 || ne > cap_e || nd > cap_d) {  // alone (empty or large units)
      flush();
      out.push_back({u});
      continue;
    }
    if ((int)cur.size() == kMaxGroup || used_e + ne > cap_e || used_d + nd > cap_d) flush();
    cur.push_back(u);
    used_e += ne;
    used_d += nd;
  }
  flush();
  return out;
}

edit_status_t plan_group(edit_sync_t h, Lane& ln, const std::vector<int32_t>& layers, void* const* locals,
                         float* const* anchors, float* const* momenta, cudaStream_t st, GroupPlan& gp) {
  gp.ln = &ln;
  gp.st = st;
  gp.units.assign(layers.size(), UnitPlan{});
  GroupArgs& g = gp.g;
  g = GroupArgs{};
  g.B = (int32_t)layers.size();
  g.M = h->M;
  g.N = h->N;
  g.my_n = h->sync_idx;
  g.K = h->K;
  g.alpha = h->cfg.ema_alpha;
  g.delta = h->cfg.anomaly_threshold;
  g.warmup = h->cfg.ema_warmup_rounds;
  g.nu = h->cfg.outer_lr;
  g.mu = h->cfg.outer_momentum;
  g.phi = h->cfg.clip_threshold;
  g.eps = h->cfg.clip_eps;
  g.flags = h->cfg.flags;
  const size_t esz = h->cfg.param_dtype == EDIT_BF16 ? 2 : 4;
  int64_t off_e = 0, off_d = 0;
  int32_t c1 = 0, c2 = 0, c3 = 0;
  for (int s = 0; s < g.B; ++s) {
    const int32_t u = layers[s];
    Mode mode{};
    mode.peer_ctas = h->peer_ctas;
    TRY(plan_unit(h, ln, u, locals[s], anchors[s], momenta[s], st, mode, gp.units[s]));
    const UnitPlan& p = gp.units[s];
    GroupSeg& q = g.seg[s];
    const int64_t n = h->numel[u];
    q.local = locals[s];
    q.anchor = anchors[s];
    q.momentum = momenta[s];
    q.n = n;
    q.slice = p.sl.slice;
    for (int j = 0; j < h->N; ++j) {
      // registered locals are read in place; otherwise every member's staging copy, at the
      // same offset on every member
      q.L[j] = p.direct ? p.pp.L[j] : static_cast<const char*>(ln.pp.L[j]) + off_e * esz;
      q.D[j] = ln.pp.D[j] + off_d * 8;
    }
    q.Lcopy = p.direct ? nullptr : static_cast<char*>(ln.Lown) + off_e * esz;
    q.Dmine = ln.Down + off_d * 8;
    q.scr = &h->scratch[u];
    q.parts1 = h->part1[u];
    q.parts2 = h->part2[u];
    q.ema = h->ema + (size_t)u * h->N;
    q.rec = h->rec + u;
    q.c1 = c1;
    q.c2 = c2;
    q.c3 = c3;
    const int64_t n8 = n >> 3, s0 = (int64_t)h->sync_idx * q.slice;
    const int64_t cnt = std::max<int64_t>(0, std::min(s0 + q.slice, n8) - s0);
    c1 += (int32_t)group_k1_ctas(n);
    c2 += (int32_t)rs_ldg_grid(cnt);
    c3 += (int32_t)group_ag_ctas(q.slice, h->N);
    off_e += (n + 7) / 8 * 8;
    off_d += q.slice;
  }
  g.c1_end = c1;
  g.c2_end = c2;
  g.c3_end = c3;
  return EDIT_OK;
}

edit_status_t enqueue_group_step(edit_sync_t h, GroupPlan& gp, int step) {
  Lane& ln = *gp.ln;
  cudaStream_t st = gp.st;
  const int dt = h->cfg.param_dtype;
  int launched = 0;
  auto mark = [&](int k) -> edit_status_t {  // profiling event k of every unit of the group
    for (UnitPlan& p : gp.units)
      if (p.ev) CUDA_TRY(h, record_event(p.ev[k], st));
    return EDIT_OK;
  };
  switch (step) {
    case kStepBegin:
      if (!capturing(st)) {
        CUDA_TRY(h, cudaStreamWaitEvent(st, ln.last, 0));
        for (UnitPlan& p : gp.units) CUDA_TRY(h, cudaStreamWaitEvent(st, h->done[p.layer], 0));
      }
      TRY(mark(0));
      break;
    case kStepNorm:  // K1 of every unit + one exchange of the group's norms + K2 per unit
      gp.g.x = xchg_args(h, ln, 0);
      launched += launch_group_norm(dt, gp.g, st);
      CUDA_TRY(h, cudaGetLastError());
      TRY(mark(1));
      break;
    case kStepDecide:
      TRY(mark(2));
      break;
    case kStepExchange:  // Eq. 3 RS of every unit + one exchange of the Dbar-norm partials
      gp.g.x = xchg_args(h, ln, 1);
      launched += launch_group_rs(dt, gp.g, st);
      CUDA_TRY(h, cudaGetLastError());
      TRY(mark(3));
      break;
    case kStepDbarNorm:
      TRY(mark(4));
      break;
    case kStepUpdate:
      launched += launch_group_ag(dt, gp.g, st);
      CUDA_TRY(h, cudaGetLastError());
      break;
    case kStepGather:
      break;  // (groups are not formed when the fused shard all-gather is registered)
    case kStepEnd:
      TRY(mark(5));
      for (UnitPlan& p : gp.units) {
        if (p.ev) h->pending.push_back(p.layer);
        CUDA_TRY(h, record_event(h->done[p.layer], st));
      }
      CUDA_TRY(h, record_event(ln.last, st));
      break;
    default:
      return fail(EDIT_ERR_INVALID_ARG, "bad step");
  }
  h->launches += launched;
  return EDIT_OK;
}

edit_status_t enqueue_units(edit_sync_t const* hs, int nh, int nunits, const int32_t* layers,
                            void* const* locals, float* const* anchors, float* const* momenta,
                            const cudaStream_t* streams, bool use_lanes) {
  for (int k = 0; k < nh; ++k) TRY(check_err(hs[k]));
  if (use_lanes)
    for (int k = 0; k < nh; ++k) {
      edit_sync_t h = hs[k];
      CUDA_TRY(h, cudaSetDevice(h->cfg.device));
      CUDA_TRY(h, cudaEventRecord(h->fork, streams[k]));
      for (Lane& ln : h->lanes) CUDA_TRY(h, cudaStreamWaitEvent(ln.stream, h->fork, 0));
    }
  // edit_sync_round: runs of small units as groups (the same partition on every handle and
  // rank); item i on lane i % lanes
  std::vector<std::vector<int32_t>> groups;
  if (use_lanes) groups = form_groups(hs[0], layers, nunits);
  else
    for (int i = 0; i < nunits; ++i) groups.push_back({layers[i]});
  std::vector<int> first(groups.size());  // index into locals/anchors/momenta of each item
  for (size_t gi = 0, at = 0; gi < groups.size(); at += groups[gi].size(), ++gi) first[gi] = (int)at;
  std::vector<UnitPlan> plans(nh);
  std::vector<GroupPlan> gplans(nh);
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    if (groups[gi].size() > 1) {
      const int i0 = first[gi];
      for (int k = 0; k < nh; ++k) {
        edit_sync_t h = hs[k];
        Lane& ln = h->lanes[gi % h->lanes.size()];
        const size_t at = (size_t)k * nunits + i0;
        TRY(plan_group(h, ln, groups[gi], locals + at, anchors + at, momenta + at, ln.stream, gplans[k]));
      }
      for (int step = 0; step < kNumSteps; ++step)
        for (int k = 0; k < nh; ++k) {
          if (nh > 1) CUDA_TRY(hs[k], cudaSetDevice(hs[k]->cfg.device));
          const NvtxRange range(hs[k]->nvtx && step == kStepBegin, "edit_sync group of %d units", (int)groups[gi].size());
          TRY(enqueue_group_step(hs[k], gplans[k], step));
        }
      continue;
    }
    const int i = first[gi];
    const int32_t layer = layers[i];
    for (int k = 0; k < nh; ++k) {
      edit_sync_t h = hs[k];
      Lane& ln = use_lanes ? h->lanes[gi % h->lanes.size()] : h->lanes[0];
      Mode mode{};
      mode.peer_ctas = h->peer_ctas;
      const size_t at = (size_t)k * nunits + i;
      TRY(plan_unit(h, ln, layer, locals[at], anchors[at], momenta[at], use_lanes ? ln.stream : streams[k], mode,
                    plans[k]));
    }
    for (int step = 0; step < kNumSteps; ++step)
      for (int k = 0; k < nh; ++k) {
        if (nh > 1) CUDA_TRY(hs[k], cudaSetDevice(hs[k]->cfg.device));
        const NvtxRange range(hs[k]->nvtx && step == kStepBegin, "edit_sync unit %d", layer);
        TRY(enqueue_step(hs[k], plans[k], step));
      }
  }
  if (use_lanes)
    for (int k = 0; k < nh; ++k) {
      edit_sync_t h = hs[k];
      for (Lane& ln : h->lanes) {
        CUDA_TRY(h, cudaEventRecord(ln.tail, ln.stream));
        CUDA_TRY(h, cudaStreamWaitEvent(streams[k], ln.tail, 0));
      }
    }
  return EDIT_OK;
}

// Warm-up all-reduce (Alg. 1 l.422-424), peer variant, step-major over nh handles: stage the
// gradient where the row can read it; barrier; each member averages its 1/N slice from every
// member; barrier; every member pulls each averaged slice from its owner.
edit_status_t enqueue_warmup(edit_sync_t const* hs, int nh, int32_t layer, void* const* grads,
                             const cudaStream_t* streams, bool force_peer, bool on_lane) {
  const char* wa = getenv("EDIT_WARMUP_ALGO");
  // on_lane: unit `layer` runs on lane layer % lanes, on the lane's stream (the round API
  // forked the caller's stream to the lanes); else lane 0 on the caller's stream
  auto lane_of = [&](edit_sync_t h) -> Lane& { return on_lane ? h->lanes[layer % h->lanes.size()] : h->lanes[0]; };
  auto stream_of = [&](edit_sync_t h, int k) { return on_lane ? lane_of(h).stream : streams[k]; };
  for (int k = 0; k < nh; ++k) {
    edit_sync_t h = hs[k];
    TRY(check_unit_args(h, layer, grads[k], grads[k], grads[k]));
    if (h->N == 1) return EDIT_OK;
    const bool warm_peer = h->peer && (force_peer || (wa && !strcmp(wa, "peer")));
    if (!warm_peer) {
      if (nh > 1) return fail(EDIT_ERR_INVALID_ARG, "the simulated mesh runs the peer warm-up only");
      const int dt = h->cfg.param_dtype;
      CUDA_TRY(h, cudaSetDevice(h->cfg.device));
      Lane& ln = lane_of(h);
      cudaStream_t st = stream_of(h, 0);
      CUDA_TRY(h, cudaStreamWaitEvent(st, ln.last, 0));
      NCCL_TRY(h, ncclAllReduce(grads[0], grads[0], (size_t)h->numel[layer],
                                dt == EDIT_BF16 ? ncclBfloat16 : ncclFloat32, ncclAvg, ln.sync, st));
      CUDA_TRY(h, cudaEventRecord(ln.last, st));
      return EDIT_OK;
    }
  }
  auto barrier = [&](edit_sync_t h, Lane& ln, cudaStream_t st) -> edit_status_t {
    if (h->dev_xchg) {
      h->launches += launch_xchg(xchg_args(h, ln, 2), ln.bar, ln.bar + 1, nullptr, st);
      CUDA_TRY(h, cudaGetLastError());
    } else {
      NCCL_TRY(h, ncclAllGather(ln.bar, ln.bar + 1, 1, ncclFloat64, ln.sync, st));
    }
    return EDIT_OK;
  };
  for (int step = 0; step < 6; ++step)
    for (int k = 0; k < nh; ++k) {
      edit_sync_t h = hs[k];
      Lane& ln = lane_of(h);
      cudaStream_t st = stream_of(h, k);
      const int dt = h->cfg.param_dtype;
      const size_t esz = dt == EDIT_BF16 ? 2 : 4;
      const Slicing sl = slicing_of(h->numel[layer], h->N, h->sync_idx, h->peer_tile);
      if (nh > 1) CUDA_TRY(h, cudaSetDevice(h->cfg.device));
      switch (step) {
        case 0:
          CUDA_TRY(h, cudaStreamWaitEvent(st, ln.last, 0));
          CUDA_TRY(h, cudaMemcpyAsync(ln.Lown, grads[k], (size_t)h->numel[layer] * esz, cudaMemcpyDeviceToDevice, st));
          break;
        case 1:  // staging complete on every member before any RS reads it
        case 3:  // every averaged slice complete before any AG pulls it
          TRY(barrier(h, ln, st));
          break;
        case 2:
          h->launches += launch_warm_rs(dt, ln.pp, sl, ln.Down, h->err_dev, st);
          CUDA_TRY(h, cudaGetLastError());
          break;
        case 4:
          h->launches += launch_warm_ag(dt, ln.pp, sl, grads[k], h->err_dev, st);
          CUDA_TRY(h, cudaGetLastError());
          break;
        case 5:
          CUDA_TRY(h, cudaEventRecord(ln.last, st));
          break;
      }
    }
  return EDIT_OK;
}

edit_status_t enqueue_warmup_units(edit_sync_t const* hs, int nh, int nunits, void* const* grads,
                                   const cudaStream_t* streams, bool force_peer) {
  for (int k = 0; k < nh; ++k) {
    edit_sync_t h = hs[k];
    TRY(check_err(h));
    CUDA_TRY(h, cudaSetDevice(h->cfg.device));
    CUDA_TRY(h, cudaEventRecord(h->fork, streams[k]));
    for (Lane& ln : h->lanes) CUDA_TRY(h, cudaStreamWaitEvent(ln.stream, h->fork, 0));
  }
  std::vector<void*> g(nh);
  for (int u = 0; u < nunits; ++u) {
    if (hs[0]->numel[u] == 0) continue;
    for (int k = 0; k < nh; ++k) g[k] = grads[(size_t)k * nunits + u];
    TRY(enqueue_warmup(hs, nh, u, g.data(), streams, force_peer, true));
  }
  for (int k = 0; k < nh; ++k) {
    edit_sync_t h = hs[k];
    if (nh > 1) CUDA_TRY(h, cudaSetDevice(h->cfg.device));
    for (Lane& ln : h->lanes) {
      CUDA_TRY(h, cudaEventRecord(ln.tail, ln.stream));
      CUDA_TRY(h, cudaStreamWaitEvent(streams[k], ln.tail, 0));
    }
  }
  return EDIT_OK;
}

}  // namespace edit

extern "C" {
static edit_status_t exchange_ipc(edit_sync_t h, void* const* ptrs, const size_t* bytes, int L, ncclComm_t comm,
                                  int P, int me, cudaStream_t st, std::vector<std::vector<void*>>& out,
                                  std::vector<void*>& opened);

const char* edit_sync_last_error(void) { return g_last_error.c_str(); }

const char* edit_sync_version(void) { return "edit_sync 0.2 (sm_100a)"; }

edit_status_t edit_sync_get_unique_id(uint8_t id[EDIT_UNIQUE_ID_BYTES]) {
  static_assert(sizeof(ncclUniqueId) == EDIT_UNIQUE_ID_BYTES, "ncclUniqueId size");
  if (!id) return fail(EDIT_ERR_INVALID_ARG, "null id");
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) return fail(EDIT_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  memcpy(id, &u, sizeof u);
  return EDIT_OK;
}

edit_status_t edit_sync_workspace_bytes(const edit_sync_config_t* cfg, size_t* bytes) {
  TRY(validate(cfg));
  if (!bytes) return fail(EDIT_ERR_INVALID_ARG, "null bytes");
  *bytes = layout_of(*cfg).total;
  return EDIT_OK;
}

// Settings every rank must agree on (slice layout, lane mapping, exchange protocol, units):
// a digest of them is all-gathered at init and compared.
struct ConfigDigest {
  int32_t nlanes, peer_tile, dev_xchg, graph, algo, L, M, N, dtype, flags, peer_ldg, group_numel;
  uint64_t numel_hash;
};

edit_status_t edit_sync_init(const edit_sync_config_t* cfg, const uint8_t id[EDIT_UNIQUE_ID_BYTES],
                             void* workspace, size_t workspace_bytes, edit_sync_t* out) {
  TRY(validate(cfg));
  if (!out) return fail(EDIT_ERR_INVALID_ARG, "null out");
  *out = nullptr;
  const int K = cfg->shard_dim * cfg->sync_dim;
  if (K > 1 && !id) return fail(EDIT_ERR_INVALID_ARG, "null unique id for a multi-rank mesh");
  edit_sync_t h = nullptr;
  edit_status_t st = create_local(cfg, workspace, workspace_bytes, &h);
  auto bail = [&](edit_status_t s) {
    if (h) edit_sync_destroy(h);
    return s;
  };
  if (st != EDIT_OK) return bail(st);
#define INIT_CUDA(expr)                                                                     \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return bail(fail(EDIT_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)));   \
  } while (0)
#define INIT_NCCL(expr)                                                                     \
  do {                                                                                      \
    ncclResult_t r_ = (expr);                                                               \
    if (r_ != ncclSuccess)                                                                  \
      return bail(fail(EDIT_ERR_NCCL, std::string(#expr ": ") + ncclGetErrorString(r_)));   \
  } while (0)
  const int nlanes = (int)h->lanes.size();
  for (int li = 0; li < nlanes && K > 1; ++li) {
    Lane& ln = h->lanes[li];
    if (li == 0) {
      ncclUniqueId u;
      memcpy(&u, id, sizeof u);
      INIT_NCCL(ncclCommInitRank(&ln.global, K, u, cfg->rank));
      // every rank must agree on the settings that fix slice layout, lane mapping and the
      // exchange protocol (read per rank from the environment): compare digests
      ConfigDigest mine;
      memset(&mine, 0, sizeof mine);  // (padding too: the digests are compared bytewise)
      const int32_t vals[12] = {nlanes, h->peer_tile, h->dev_xchg ? 1 : 0, h->graph ? 1 : 0, cfg->algo,
                                cfg->num_layers, h->M, h->N, cfg->param_dtype, (int32_t)cfg->flags, h->peer_ldg,
                                (int32_t)h->group_numel};
      memcpy(&mine, vals, sizeof vals);
      mine.numel_hash = 1469598103934665603ull;
      for (int64_t x : h->numel) mine.numel_hash = (mine.numel_hash ^ (uint64_t)x) * 1099511628211ull;
      char* dev = nullptr;
      INIT_CUDA(cudaMalloc(&dev, sizeof(ConfigDigest) * (K + 1)));
      INIT_CUDA(cudaMemcpy(dev, &mine, sizeof mine, cudaMemcpyHostToDevice));
      INIT_NCCL(ncclAllGather(dev, dev + sizeof mine, sizeof mine, ncclChar, ln.global, ln.stream));
      INIT_CUDA(cudaStreamSynchronize(ln.stream));
      std::vector<ConfigDigest> all(K);
      INIT_CUDA(cudaMemcpy(all.data(), dev + sizeof mine, sizeof mine * K, cudaMemcpyDeviceToHost));
      INIT_CUDA(cudaFree(dev));
      for (int r = 0; r < K; ++r)
        if (memcmp(&all[r], &all[0], sizeof mine) != 0)
          return bail(fail(EDIT_ERR_INVALID_ARG,
                           "ranks disagree on EDIT_LANES / EDIT_PEER_TILE / EDIT_XCHG / EDIT_GRAPH / algo / "
                           "units / dtype / flags (rank " + std::to_string(r) + " differs from rank 0)"));
    } else {
      INIT_NCCL(ncclCommSplit(h->lanes[0].global, 0, cfg->rank, &ln.global, nullptr));  // a dup
    }
    // sync group (row): same shard index m, ordered by n; shard group (column): same n.
    INIT_NCCL(ncclCommSplit(ln.global, h->shard_idx, h->sync_idx, &ln.sync, nullptr));
    INIT_NCCL(ncclCommSplit(ln.global, h->sync_idx, h->shard_idx, &ln.shard, nullptr));
    if (ln.mailbox) {
      void* mine = ln.mailbox;
      size_t mb = mailbox_bytes(K);
      std::vector<std::vector<void*>> boxes;
      edit_status_t rc = exchange_ipc(h, &mine, &mb, 1, ln.global, K, cfg->rank, ln.stream, boxes, ln.opened);
      if (rc != EDIT_OK) return bail(rc);
      for (int r = 0; r < K; ++r) ln.mp.box[r] = static_cast<unsigned long long*>(boxes[0][r]);
    }
    if (h->peer) {
      // exchange the IPC handles over the lane's sync comm (row): [N][2] cudaIpcMemHandle_t
      cudaIpcMemHandle_t mine[2];
      INIT_CUDA(cudaIpcGetMemHandle(&mine[0], ln.Lown));
      INIT_CUDA(cudaIpcGetMemHandle(&mine[1], ln.Down));
      const size_t hb = sizeof(mine);
      char* dev = nullptr;
      INIT_CUDA(cudaMalloc(&dev, hb * (h->N + 1)));
      INIT_CUDA(cudaMemcpy(dev, mine, hb, cudaMemcpyHostToDevice));
      INIT_NCCL(ncclAllGather(dev, dev + hb, hb, ncclChar, ln.sync, ln.stream));
      INIT_CUDA(cudaStreamSynchronize(ln.stream));
      std::vector<cudaIpcMemHandle_t> all(2 * h->N);
      INIT_CUDA(cudaMemcpy(all.data(), dev + hb, hb * h->N, cudaMemcpyDeviceToHost));
      INIT_CUDA(cudaFree(dev));
      for (int j = 0; j < h->N; ++j) {
        if (j == h->sync_idx) continue;
        void *pl = nullptr, *pd = nullptr;
        INIT_CUDA(cudaIpcOpenMemHandle(&pl, all[2 * j], cudaIpcMemLazyEnablePeerAccess));
        ln.opened.push_back(pl);
        INIT_CUDA(cudaIpcOpenMemHandle(&pd, all[2 * j + 1], cudaIpcMemLazyEnablePeerAccess));
        ln.opened.push_back(pd);
        ln.pp.L[j] = pl;
        ln.pp.D[j] = static_cast<float*>(pd);
      }
    } else if (h->N > 1) {
      ln.ops.assign(cfg->num_layers, ncclRedOp_t{});
      for (int l = 0; l < cfg->num_layers; ++l)
        INIT_NCCL(ncclRedOpCreatePreMulSum(&ln.ops[l], &h->scratch[l].w, ncclFloat32, ncclScalarDevice, ln.sync));
    }
  }
  INIT_CUDA(cudaDeviceSynchronize());
#undef INIT_CUDA
#undef INIT_NCCL
  h->ready = true;
  *out = h;
  return EDIT_OK;
}

edit_status_t edit_layer_sync(edit_sync_t h, int32_t layer, void* local, float* anchor, float* momentum,
                              void* stream) {
  TRY(check_unit_args(h, layer, local, anchor, momentum));
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return enqueue_units(&h, 1, 1, &layer, &local, &anchor, &momentum, &st, false);
}

typedef CUresult_t (*AddrRangeFn)(unsigned long long*, size_t*, unsigned long long);

// Map `ptrs` (L device pointers of this rank, inside cudaMalloc allocations) on every member of
// `comm` (size P, this rank = `me`): out[u][j] = member j's pointer for unit u in this process.
static edit_status_t exchange_ipc(edit_sync_t h, void* const* ptrs, const size_t* bytes, int L, ncclComm_t comm,
                                  int P, int me, cudaStream_t st, std::vector<std::vector<void*>>& out,
                                  std::vector<void*>& opened) {
  const bool dbg = getenv("EDIT_DEBUG") != nullptr;
  // cuMemGetAddressRange_v2 from the driver itself (dlopen: the library must load on
  // machines without a driver, and the unversioned entry point may resolve to the 32-bit v1)
  static AddrRangeFn range = [] {
    void* lib = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
    if (!lib) lib = dlopen("libcuda.so.1", RTLD_NOW);
    return lib ? reinterpret_cast<AddrRangeFn>(dlsym(lib, "cuMemGetAddressRange_v2")) : nullptr;
  }();
  if (!range) return fail(EDIT_ERR_CUDA, "cuMemGetAddressRange_v2 unavailable");
  struct Rec {
    cudaIpcMemHandle_t handle;
    uint64_t offset;
    uint64_t valid;
  };
  std::vector<Rec> mine(L);
  for (int u = 0; u < L; ++u) {
    memset(&mine[u], 0, sizeof(Rec));
    if (!ptrs[u]) continue;
    unsigned long long base = 0;
    size_t size = 0;
    if (range(&base, &size, (unsigned long long)(uintptr_t)ptrs[u]) != 0)
      return fail(EDIT_ERR_CUDA, "cuMemGetAddressRange failed for a registered buffer");
    const uintptr_t p = (uintptr_t)ptrs[u];
    if (p < base || p + bytes[u] > base + size)
      return fail(EDIT_ERR_INVALID_ARG, "registered buffer does not lie inside one device allocation");
    CUDA_TRY(h, cudaIpcGetMemHandle(&mine[u].handle, ptrs[u]));
    mine[u].offset = (uint64_t)(p - (uintptr_t)base);
    if (dbg)
      fprintf(stderr, "[edit_sync] ipc export unit %d ptr %p base %#llx size %zu offset %llu\n", u, ptrs[u], base,
              size, (unsigned long long)mine[u].offset);
    mine[u].valid = 1;
  }
  const size_t rb = sizeof(Rec) * (size_t)L;
  char* dev = nullptr;
  CUDA_TRY(h, cudaMalloc(&dev, rb * (P + 1)));
  CUDA_TRY(h, cudaMemcpy(dev, mine.data(), rb, cudaMemcpyHostToDevice));
  NCCL_TRY(h, ncclAllGather(dev, dev + rb, rb, ncclChar, comm, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  std::vector<Rec> all((size_t)L * P);
  CUDA_TRY(h, cudaMemcpy(all.data(), dev + rb, rb * P, cudaMemcpyDeviceToHost));
  CUDA_TRY(h, cudaFree(dev));
  out.assign(L, std::vector<void*>(P, nullptr));
  std::vector<std::pair<std::string, void*>> mapped;  // one mapping per distinct handle
  for (int j = 0; j < P; ++j)
    for (int u = 0; u < L; ++u) {
      if (j == me) {
        out[u][j] = ptrs[u];
        continue;
      }
      const Rec& r = all[(size_t)j * L + u];
      if (!r.valid) continue;
      const std::string key(reinterpret_cast<const char*>(&r.handle), sizeof r.handle);
      void* basep = nullptr;
      for (auto& m : mapped)
        if (m.first == key) basep = m.second;
      if (!basep) {
        CUDA_TRY(h, cudaIpcOpenMemHandle(&basep, r.handle, cudaIpcMemLazyEnablePeerAccess));
        mapped.emplace_back(key, basep);
        opened.push_back(basep);
      }
      out[u][j] = static_cast<char*>(basep) + r.offset;
      if (dbg)
        fprintf(stderr, "[edit_sync] ipc import unit %d member %d base %p offset %llu -> %p\n", u, j, basep,
                (unsigned long long)r.offset, out[u][j]);
    }
  return EDIT_OK;
}

edit_status_t edit_sync_register_gather(edit_sync_t h, void* const* full_bufs) {
  if (!h) return fail(EDIT_ERR_INVALID_ARG, "null handle");
  TRY(check_err(h));
  if (!full_bufs) return fail(EDIT_ERR_INVALID_ARG, "null buffer array");
  if (h->M == 1) return EDIT_OK;
  if (!h->reg_gather.empty()) return fail(EDIT_ERR_INVALID_ARG, "gather buffers already registered");
  const int L = h->cfg.num_layers;
  for (int u = 0; u < L; ++u)
    if ((h->numel[u] > 0 && !full_bufs[u]) || ((uintptr_t)full_bufs[u] & 15u))
      return fail(EDIT_ERR_INVALID_ARG, "null or misaligned gather buffer");
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  std::vector<void*> ptrs(full_bufs, full_bufs + L);
  std::vector<size_t> bytes(L);
  const size_t esz = h->cfg.param_dtype == EDIT_BF16 ? 2 : 4;
  for (int u = 0; u < L; ++u) {
    if (h->numel[u] == 0) ptrs[u] = nullptr;
    bytes[u] = (size_t)h->M * h->numel[u] * esz;
  }
  Lane& ln = h->lanes[0];
  TRY(exchange_ipc(h, ptrs.data(), bytes.data(), L, ln.shard, h->M, h->shard_idx, ln.stream, h->reg_gather,
                   h->gather_opened));
  CUDA_TRY(h, cudaMalloc(reinterpret_cast<void**>(&h->gather_dev), sizeof(double) * (size_t)L * (h->M + 1)));
  clear_graphs(h);  // a captured round holds the non-gathering update kernels
  return EDIT_OK;
}

edit_status_t edit_sync_register_locals(edit_sync_t h, void* const* locals) {
  if (!h) return fail(EDIT_ERR_INVALID_ARG, "null handle");
  TRY(check_err(h));
  if (!locals) return fail(EDIT_ERR_INVALID_ARG, "null buffer array");
  if (!h->peer) return EDIT_OK;
  if (!h->reg_local.empty()) return fail(EDIT_ERR_INVALID_ARG, "locals already registered");
  const int L = h->cfg.num_layers;
  for (int u = 0; u < L; ++u)
    if ((h->numel[u] > 0 && !locals[u]) || ((uintptr_t)locals[u] & 15u))
      return fail(EDIT_ERR_INVALID_ARG, "null or misaligned local");
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  std::vector<void*> ptrs(locals, locals + L);
  std::vector<size_t> bytes(L);
  const size_t esz = h->cfg.param_dtype == EDIT_BF16 ? 2 : 4;
  for (int u = 0; u < L; ++u) {
    if (h->numel[u] == 0) ptrs[u] = nullptr;
    bytes[u] = (size_t)h->numel[u] * esz;
  }
  std::vector<std::vector<void*>> peers;
  Lane& ln = h->lanes[0];
  TRY(exchange_ipc(h, ptrs.data(), bytes.data(), L, ln.sync, h->N, h->sync_idx, ln.stream, peers, h->reg_opened));
  h->reg_peer.assign(L, std::vector<const void*>(h->N, nullptr));
  for (int u = 0; u < L; ++u)
    for (int j = 0; j < h->N; ++j) h->reg_peer[u][j] = peers[u][j];
  h->reg_local.assign(locals, locals + L);
  clear_graphs(h);  // a captured round reads the staging copies
  return EDIT_OK;
}

edit_status_t edit_sync_round(edit_sync_t h, void* const* locals, float* const* anchors, float* const* momenta,
                              void* stream) {
  if (!h) return fail(EDIT_ERR_INVALID_ARG, "null handle");
  TRY(check_err(h));
  if (!locals || !anchors || !momenta) return fail(EDIT_ERR_INVALID_ARG, "null buffer arrays");
  if (h->sched_active) return fail(EDIT_ERR_INVALID_ARG, "a scheduled round is active");
  const int L = h->cfg.num_layers;
  for (int u = 0; u < L; ++u) TRY(check_unit_args(h, u, locals[u], anchors[u], momenta[u]));
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  const NvtxRange range(h->nvtx, "edit_sync_round (%d units)", L);
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  std::vector<int32_t> layers(L);
  for (int u = 0; u < L; ++u) layers[u] = u;
  const bool use_graph = h->graph && (h->K == 1 || h->lanes[0].dseq != nullptr);
  if (!use_graph) return enqueue_units(&h, 1, L, layers.data(), locals, (float* const*)anchors, (float* const*)momenta,
                                       &cs, true);
  std::vector<uintptr_t> key;
  key.reserve(3 * (size_t)L + 1);
  for (int u = 0; u < L; ++u) {
    key.push_back(reinterpret_cast<uintptr_t>(locals[u]));
    key.push_back(reinterpret_cast<uintptr_t>(anchors[u]));
    key.push_back(reinterpret_cast<uintptr_t>(momenta[u]));
  }
  key.push_back(h->profiling ? 1u : 0u);  // a profiled capture holds the phase events
  // a replay (or the first launch) is ordered after every earlier use of the lanes' buffers
  // and of the units' scratch, on whatever stream it ran
  auto launch = [&](RoundGraph& g) -> edit_status_t {
    for (Lane& ln : h->lanes) CUDA_TRY(h, cudaStreamWaitEvent(cs, ln.last, 0));
    for (int u = 0; u < L; ++u) CUDA_TRY(h, cudaStreamWaitEvent(cs, h->done[u], 0));
    CUDA_TRY(h, cudaGraphLaunch(g.exec, cs));
    h->launches += g.launches;
    if (h->profiling)
      for (int u = 0; u < L; ++u) h->pending.push_back(u);
    return EDIT_OK;
  };
  for (RoundGraph& g : h->graphs)
    if (g.key == key) return launch(g);
  // capture on a library stream (the caller's may be the legacy default stream, which
  // cannot be captured); the graph is then launched on the caller's stream
  if (!h->cap_stream) CUDA_TRY(h, cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
  CUDA_TRY(h, cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeRelaxed));
  const int64_t launches0 = h->launches;
  const std::vector<int32_t> pending0 = h->pending;
  edit_status_t rc = enqueue_units(&h, 1, L, layers.data(), locals, (float* const*)anchors, (float* const*)momenta,
                                   &h->cap_stream, true);
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(h->cap_stream, &graph);
  if (rc != EDIT_OK) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  CUDA_TRY(h, ec);
  RoundGraph g;
  g.key = std::move(key);
  g.launches = h->launches - launches0;
  h->launches = launches0;  // capture launched nothing; the replay below does
  h->pending = pending0;
  const cudaError_t ei = cudaGraphInstantiate(&g.exec, graph, 0);
  cudaGraphDestroy(graph);
  CUDA_TRY(h, ei);
  if (h->graphs.size() >= 4) {
    cudaGraphExecDestroy(h->graphs.front().exec);
    h->graphs.erase(h->graphs.begin());
  }
  h->graphs.push_back(std::move(g));
  return launch(h->graphs.back());
}

edit_status_t edit_warmup_allreduce(edit_sync_t h, int32_t layer, void* grad, void* stream) {
  TRY(check_unit_args(h, layer, grad, grad, grad));
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return enqueue_warmup(&h, 1, layer, &grad, &st, false);
}

edit_status_t edit_warmup_allreduce_round(edit_sync_t h, void* const* grads, void* stream) {
  if (!h) return fail(EDIT_ERR_INVALID_ARG, "null handle");
  if (!grads) return fail(EDIT_ERR_INVALID_ARG, "null grads");
  TRY(check_err(h));
  if (h->N == 1) return EDIT_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return enqueue_warmup_units(&h, 1, h->cfg.num_layers, grads, &st, false);
}

edit_status_t edit_layer_sync_host(edit_sync_t h, int32_t layer, void* local_host, float* anchor_host,
                                   float* momentum_host, void* stream) {
  if (!h) return fail(EDIT_ERR_INVALID_ARG, "null handle");
  TRY(check_err(h));
  if (layer < 0 || layer >= h->cfg.num_layers) return fail(EDIT_ERR_INVALID_ARG, "layer out of range");
  const int64_t n = h->numel[layer];
  if (n > 0 && (!local_host || !anchor_host || !momentum_host)) return fail(EDIT_ERR_INVALID_ARG, "null buffer");
  const size_t esz = h->cfg.param_dtype == EDIT_BF16 ? 2 : 4;
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  if (!h->staging) {
    int64_t max_numel = 0;
    for (int64_t x : h->numel) max_numel = std::max(max_numel, x);
    // per slot: anchor | momentum | local, each 256-byte aligned
    h->slot_bytes = align_up((size_t)max_numel * 4, 256) * 2 + align_up((size_t)max_numel * esz, 256);
    CUDA_TRY(h, cudaMalloc(reinterpret_cast<void**>(&h->staging), edit_sync::kHostSlots * h->slot_bytes));
    CUDA_TRY(h, cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking));
    CUDA_TRY(h, cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking));
    for (int i = 0; i < edit_sync::kHostSlots; ++i) {
      CUDA_TRY(h, cudaEventCreateWithFlags(&h->slot_in[i], cudaEventDisableTiming));
      CUDA_TRY(h, cudaEventCreateWithFlags(&h->slot_done[i], cudaEventDisableTiming));
      CUDA_TRY(h, cudaEventCreateWithFlags(&h->slot_free[i], cudaEventDisableTiming));
      CUDA_TRY(h, cudaEventRecord(h->slot_free[i], h->d2h));
    }
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int slot = h->next_slot;
  h->next_slot = (h->next_slot + 1) % edit_sync::kHostSlots;
  char* base = h->staging + (size_t)slot * h->slot_bytes;
  const size_t fbytes = align_up((size_t)std::max<int64_t>(n, 1) * 4, 256);
  float* anc = reinterpret_cast<float*>(base);
  float* mom = reinterpret_cast<float*>(base + fbytes);
  void* loc = base + 2 * fbytes;
  // copy-in once the slot's previous copy-out has drained
  CUDA_TRY(h, cudaStreamWaitEvent(h->h2d, h->slot_free[slot], 0));
  CUDA_TRY(h, cudaMemcpyAsync(anc, anchor_host, (size_t)n * 4, cudaMemcpyHostToDevice, h->h2d));
  CUDA_TRY(h, cudaMemcpyAsync(mom, momentum_host, (size_t)n * 4, cudaMemcpyHostToDevice, h->h2d));
  CUDA_TRY(h, cudaMemcpyAsync(loc, local_host, (size_t)n * esz, cudaMemcpyHostToDevice, h->h2d));
  CUDA_TRY(h, cudaEventRecord(h->slot_in[slot], h->h2d));
  CUDA_TRY(h, cudaStreamWaitEvent(st, h->slot_in[slot], 0));
  TRY(edit_layer_sync(h, layer, loc, anc, mom, stream));
  CUDA_TRY(h, cudaEventRecord(h->slot_done[slot], st));
  CUDA_TRY(h, cudaStreamWaitEvent(h->d2h, h->slot_done[slot], 0));
  CUDA_TRY(h, cudaMemcpyAsync(anchor_host, anc, (size_t)n * 4, cudaMemcpyDeviceToHost, h->d2h));
  CUDA_TRY(h, cudaMemcpyAsync(momentum_host, mom, (size_t)n * 4, cudaMemcpyDeviceToHost, h->d2h));
  CUDA_TRY(h, cudaMemcpyAsync(local_host, loc, (size_t)n * esz, cudaMemcpyDeviceToHost, h->d2h));
  CUDA_TRY(h, cudaEventRecord(h->slot_free[slot], h->d2h));
  return EDIT_OK;
}

edit_status_t edit_sync_host_wait(edit_sync_t h, void* stream) {
  if (!h) return fail(EDIT_ERR_INVALID_ARG, "null handle");
  TRY(check_err(h));
  if (!h->staging) return EDIT_OK;
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int i = 0; i < edit_sync::kHostSlots; ++i) CUDA_TRY(h, cudaStreamWaitEvent(st, h->slot_free[i], 0));
  return EDIT_OK;
}

// HBM bytes per param one unit sync streams through the SMs (the dataflow's, not the
// algorithmic minimum): N == 1: K1 (b_l + 4) + K4 (16 + 2 b_l); peer path: K1 (+ staging copy
// unless registered) + RS (b_l + 8/N) + AG (20 + b_l).
static double unit_bytes_per_param(edit_sync_t h, int u) {
  const double bl = h->cfg.param_dtype == EDIT_BF16 ? 2.0 : 4.0;
  if (h->N == 1) return (bl + 4) + (16 + 2 * bl);
  const bool direct = h->peer && !h->reg_local.empty() && h->reg_local[u] == h->sched_local[u];
  return (bl + 4) + (direct ? 0 : bl) + (bl + 8.0 / h->N) + (20 + bl);
}

// ---------------------------------------------------------------- the scheduler's auto mode
// A self-tuning controller over a few candidate plans, chosen per round by the measured
// round time (compute stream, begin_round -> end_round; the caller's forward is the same work
// every round, so the round time IS the objective):
//   candidate 0 = serial: the whole round first, exactly as edit_sync_round runs it (every
//                 unit enqueued at begin_round, pipelined over the lanes on full grids), and
//                 the forward's first acquire waits for all of it -- no overlap, and the same
//                 cost as running the round and the forward back to back (a per-unit gate,
//                 the earlier form, exposed every small unit's whole latency chain: 350M 1x4
//                 3.28 ms against 3.08 for the pipelined round, profiles/r2_4gpu_350M_1x4.json);
//   candidate c > 0 = partition: unit u's sync (enqueued depth_c units ahead, depth_c =
//                 max(caller's depth, 2, 2, 1 for c = 1, 2, 3)) gets f_c = 1.0, 1.6, 1.0 x the
//                 fewest SMs that stream its bytes within the forward time it overlaps (units
//                 u-depth_c .. u-1, measured per unit between acquire calls) at EDIT_SM_GBPS
//                 per SM; units < full_units keep full grids.
// Each candidate is measured kTuneSamples times (serial first: it also measures the forward
// cleanly), then the one with the lowest median round time is kept; if its newest sample
// drifts > 15 % from its median (the workload changed) every candidate is re-measured.
static const double kTuneFactors[kTuneCands] = {0.0, 1.0, 1.6, 1.0};
static const int kTuneMinDepth[kTuneCands] = {1, 2, 2, 1};  // prefetch depth >= this (and >= the caller's)

static int partition_sms(edit_sync_t h, int u, double factor) {
  double budget_ms = 0.0;
  for (int k = std::max(0, u - h->sched_depth); k < u; ++k) budget_ms += h->fwd_ms[k];
  const double bytes = unit_bytes_per_param(h, u) * (double)h->numel[u];
  if (budget_ms <= 0.0) return h->num_sms;
  const double sms = factor * bytes / (h->sm_gbps * 1e9 * budget_ms * 1e-3);
  return std::max(4, std::min(h->num_sms, (int)std::ceil(sms)));
}

static double median_of(std::vector<float> v) {
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  const size_t n = v.size();
  return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

// begin_round: fold the previous round's measurements in (without blocking: only if its
// events have completed), then pick this round's candidate.
static void tune_begin(edit_sync_t h) {
  const int L = h->cfg.num_layers;
  if (h->rnd_pending && cudaEventQuery(h->rnd_ev1) == cudaSuccess) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, h->rnd_ev0, h->rnd_ev1) == cudaSuccess && h->round_cand >= 0)
      h->tune_ms[h->round_cand].push_back(ms);
    bool ok = true;
    for (int u = 0; u < L && ok; ++u) {
      float f = 0.f;
      ok = cudaEventElapsedTime(&f, h->post_ev[u], u + 1 < L ? h->pre_ev[u + 1] : h->end_ev) == cudaSuccess;
      h->fwd_ms[u] = f;
    }
    // the forward times of a serial round are clean (nothing else runs next to them)
    if (ok && (h->round_cand == 0 || !h->fwd_valid)) h->fwd_valid = true;
    cudaGetLastError();  // (clear a failed elapsed-time query)
    h->rnd_pending = false;
  }
  if (h->sched_part != kSchedAuto) {
    h->round_cand = -1;
    return;
  }
  // the partition plans only reshape single-unit items (unit groups run at full speed under
  // every plan); with none past full_units (every small unit grouped) they can only lose --
  // measured 1B 2x2: h = -0.34 / -0.58 -- so the plan is serial, identically on every rank
  bool partitionable = false;
  for (const auto& item : h->sched_items)
    if (item.size() == 1 && item[0] >= h->sched_full_units) partitionable = true;
  if (!partitionable) {
    h->round_cand = 0;
    return;
  }
  int cand = -1;
  if (!h->fwd_valid) {
    cand = 0;  // measure the forward first
  } else {
    for (int c = 0; c < kTuneCands && cand < 0; ++c)
      if ((int)h->tune_ms[c].size() < kTuneSamples) cand = c;
    if (cand < 0) {
      double best = 0.0;
      for (int c = 0; c < kTuneCands; ++c) {
        const double m = median_of(h->tune_ms[c]);
        if (cand < 0 || m < best) {
          cand = c;
          best = m;
        }
      }
      // the workload changed (3 rounds in a row > 15 % above the choice's median; one slow
      // round -- a straggling peer, a clock dip -- is noise): measure again
      h->tune_drift = h->tune_ms[cand].back() > 1.15 * best ? h->tune_drift + 1 : 0;
      if (h->tune_drift >= 3) {
        for (auto& v : h->tune_ms) v.clear();
        h->tune_drift = 0;
      }
      for (auto& v : h->tune_ms)  // keep a sliding window
        if (v.size() > 8) v.erase(v.begin(), v.begin() + (v.size() - 8));
    }
  }
  h->round_cand = cand;
}

static bool round_serial(edit_sync_t h) { return h->sched_part == kSchedAuto && h->round_cand == 0; }

// The scheduler's work items are the round API's: runs of small units form unit groups
// (form_groups, deterministic from the numel list), every other unit is its own item; item i
// runs on lane i % lanes.  So every plan -- whichever one a rank's tuner picked for this round
// -- enqueues the same exchanges in the same order on every rank: plans differ only in how
// many SMs a single-unit item's kernels get and in when items are enqueued.
static int item_first(edit_sync_t h, int i) { return h->sched_items[i][0]; }

static edit_status_t sched_enqueue_next(edit_sync_t h, cudaStream_t gate = nullptr) {
  const int i = h->sched_next_sync++;
  const std::vector<int32_t>& item = h->sched_items[i];
  Lane& ln = h->lanes[i % h->lanes.size()];
  const int u = item[0];
  if (gate && h->sched_gate && !round_serial(h)) {
    CUDA_TRY(h, cudaEventRecord(h->gate_ev[u], gate));
    CUDA_TRY(h, cudaStreamWaitEvent(ln.stream, h->gate_ev[u], 0));
  }
  if (item.size() > 1) {
    // a unit group: the group kernels at full speed under every plan (small units lose with
    // any overlapped plan, DESIGN 7)
    for (int32_t v : item) h->sched_sms[v] = round_serial(h) ? -1 : 0;
    GroupPlan gp;
    TRY(plan_group(h, ln, item, h->sched_local.data() + u, h->sched_anchor.data() + u, h->sched_mom.data() + u,
                   ln.stream, gp));
    const NvtxRange range(h->nvtx, "edit_sync group of %d units (scheduled)", (int)item.size());
    for (int step = 0; step < kNumSteps; ++step) TRY(enqueue_group_step(h, gp, step));
    return EDIT_OK;
  }
  Mode mode{h->sched_ctas, h->sched_ctas > 0 ? h->sched_ctas : h->peer_ctas, h->sched_ctas > 0 ? h->sched_smem_kb : 0,
            0};
  int per = 0;
  if (h->sched_part > 0 && u >= h->sched_full_units) {
    // partition mode: persistent TMA pipelines with full rings; the lanes run concurrently,
    // so each lane's kernels get an equal share of the sched_part SMs
    const int nl = (int)h->lanes.size();
    per = std::max(1, (h->sched_part + nl - 1) / nl);
  } else if (h->sched_part == kSchedAuto && h->round_cand > 0 && u >= h->sched_full_units) {
    per = partition_sms(h, u, kTuneFactors[h->round_cand]);
  }
  if (per > 0) {
    mode.cap = 0;
    mode.peer_ctas = per;
    mode.smem_kb = 0;
    mode.part = per;
  }
  h->sched_sms[u] = round_serial(h) ? -1 : per;
  UnitPlan p;
  TRY(plan_unit(h, ln, u, h->sched_local[u], h->sched_anchor[u], h->sched_mom[u], ln.stream, mode, p));
  const NvtxRange range(h->nvtx, "edit_sync unit %d (scheduled)", u);
  for (int step = 0; step < kNumSteps; ++step) TRY(enqueue_step(h, p, step));
  return EDIT_OK;
}

edit_status_t edit_sched_begin_round(edit_sync_t h, void* const* locals, float* const* anchors,
                                     float* const* momenta, int32_t depth, void* compute_stream) {
  if (!h) return fail(EDIT_ERR_INVALID_ARG, "null handle");
  TRY(check_err(h));
  if (!locals || !anchors || !momenta) return fail(EDIT_ERR_INVALID_ARG, "null buffer arrays");
  if (depth < 1) return fail(EDIT_ERR_INVALID_ARG, "depth must be >= 1");
  if (h->sched_active) return fail(EDIT_ERR_INVALID_ARG, "a round is already active");
  const int L = h->cfg.num_layers;
  for (int u = 0; u < L; ++u) TRY(check_unit_args(h, u, locals[u], anchors[u], momenta[u]));
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  h->sched_local.assign(locals, locals + L);
  h->sched_anchor.assign(anchors, anchors + L);
  h->sched_mom.assign(momenta, momenta + L);
  h->sched_next_sync = 0;
  h->sched_next_acquire = 0;
  {
    std::vector<int32_t> all(L);
    for (int u = 0; u < L; ++u) all[u] = u;
    h->sched_items = form_groups(h, all.data(), L);
  }
  h->sched_active = true;
  tune_begin(h);
  h->sched_depth = h->round_cand > 0 ? std::max(depth, kTuneMinDepth[h->round_cand]) : depth;
  cudaStream_t cs = static_cast<cudaStream_t>(compute_stream);
  CUDA_TRY(h, cudaEventRecord(h->rnd_ev0, cs));
  // the side streams (lanes) start after everything already on the compute stream (the
  // inner steps that produced the locals)
  CUDA_TRY(h, cudaEventRecord(h->fork, cs));
  for (Lane& ln : h->lanes) CUDA_TRY(h, cudaStreamWaitEvent(ln.stream, h->fork, 0));
  const int nitems = (int)h->sched_items.size();
  if (round_serial(h)) {
    // the whole round ahead of the forward, as edit_sync_round runs it (the same items and
    // lanes); the compute stream then waits for all of it
    while (h->sched_next_sync < nitems) TRY(sched_enqueue_next(h));
    for (Lane& ln : h->lanes) {
      CUDA_TRY(h, cudaEventRecord(ln.tail, ln.stream));
      CUDA_TRY(h, cudaStreamWaitEvent(cs, ln.tail, 0));
    }
  } else {
    while (h->sched_next_sync < nitems && item_first(h, h->sched_next_sync) < depth) TRY(sched_enqueue_next(h));
  }
  return EDIT_OK;
}

edit_status_t edit_sched_acquire(edit_sync_t h, int32_t layer, void* compute_stream) {
  if (!h) return fail(EDIT_ERR_INVALID_ARG, "null handle");
  TRY(check_err(h));
  if (!h->sched_active) return fail(EDIT_ERR_INVALID_ARG, "no active round");
  if (layer != h->sched_next_acquire) return fail(EDIT_ERR_INVALID_ARG, "acquire units in order 0..L-1");
  const int L = h->cfg.num_layers;
  cudaStream_t cs = static_cast<cudaStream_t>(compute_stream);
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  // the forward of unit layer-1 ends here on the compute stream (auto mode's measurement)
  CUDA_TRY(h, cudaEventRecord(h->pre_ev[layer], cs));
  // serial: the whole round was enqueued at begin_round, the forward starts after all of it;
  // otherwise unit `layer` was enqueued `depth` units ahead (depth can only lag if acquire
  // skipped ahead)
  const int nitems = (int)h->sched_items.size();
  while (h->sched_next_sync < nitems && item_first(h, h->sched_next_sync) <= layer) TRY(sched_enqueue_next(h));
  CUDA_TRY(h, cudaStreamWaitEvent(cs, h->done[layer], 0));
  CUDA_TRY(h, cudaEventRecord(h->post_ev[layer], cs));  // the forward of `layer` starts here
  h->sched_next_acquire = layer + 1;
  while (!round_serial(h) && h->sched_next_sync < nitems && item_first(h, h->sched_next_sync) <= layer + h->sched_depth)
    TRY(sched_enqueue_next(h, cs));
  return EDIT_OK;
}

edit_status_t edit_sched_end_round(edit_sync_t h, void* compute_stream) {
  if (!h) return fail(EDIT_ERR_INVALID_ARG, "null handle");
  TRY(check_err(h));
  if (!h->sched_active) return fail(EDIT_ERR_INVALID_ARG, "no active round");
  const int L = h->cfg.num_layers;
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  cudaStream_t cs = static_cast<cudaStream_t>(compute_stream);
  const bool complete = h->sched_next_acquire == L;  // every unit acquired: the round is measurable
  if (complete) CUDA_TRY(h, cudaEventRecord(h->end_ev, cs));
  while (h->sched_next_sync < (int)h->sched_items.size()) TRY(sched_enqueue_next(h));
  for (Lane& ln : h->lanes) {
    CUDA_TRY(h, cudaEventRecord(ln.tail, ln.stream));
    CUDA_TRY(h, cudaStreamWaitEvent(cs, ln.tail, 0));
  }
  if (complete) {
    CUDA_TRY(h, cudaEventRecord(h->rnd_ev1, cs));
    h->rnd_pending = true;
  }
  h->sched_active = false;
  return EDIT_OK;
}

edit_status_t edit_sched_get_plan(edit_sync_t h, int32_t* candidate, int32_t* sms, double* median_ms) {
  if (!h) return fail(EDIT_ERR_INVALID_ARG, "null handle");
  if (candidate) *candidate = h->round_cand;
  if (sms)
    for (int u = 0; u < h->cfg.num_layers; ++u) sms[u] = h->sched_sms[u];
  if (median_ms)
    for (int c = 0; c < kTuneCands; ++c) median_ms[c] = median_of(h->tune_ms[c]);
  return EDIT_OK;
}

edit_status_t edit_sched_set_partition(edit_sync_t h, int32_t sms, int32_t full_units) {
  if (!h) return fail(EDIT_ERR_INVALID_ARG, "null handle");
  TRY(check_err(h));
  if (h->sched_active) return fail(EDIT_ERR_INVALID_ARG, "a scheduled round is active");
  if (sms < kSchedAuto || sms > h->num_sms || full_units < 0)
    return fail(EDIT_ERR_INVALID_ARG, "sms must be -1 (auto) or in [0, #SMs], full_units >= 0");
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  int prio_lo = 0, prio_hi = 0;
  CUDA_TRY(h, cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  // partition mode: the lanes' persistent CTAs should take each SM a forward CTA releases,
  // so the lanes run at the highest priority; otherwise back to the priority of init
  const int prio = sms != 0 ? h->lane_prio : prio_lo;
  for (Lane& ln : h->lanes) {
    int cur = 0;
    CUDA_TRY(h, cudaStreamGetPriority(ln.stream, &cur));
    if (cur == prio) continue;
    // a lane's stream orders its buffers and communicators: drain it, then replace it
    CUDA_TRY(h, cudaStreamSynchronize(ln.stream));
    CUDA_TRY(h, cudaStreamDestroy(ln.stream));
    ln.stream = nullptr;
    CUDA_TRY(h, cudaStreamCreateWithPriority(&ln.stream, cudaStreamNonBlocking, prio));
  }
  clear_graphs(h);  // captured rounds reference the old lane streams' work order
  if (sms == kSchedAuto && h->sched_part != kSchedAuto)
    for (auto& v : h->tune_ms) v.clear();  // re-tune from scratch
  h->sched_part = sms;
  h->sched_full_units = full_units;
  return EDIT_OK;
}

edit_status_t edit_sync_stats(edit_sync_t h, int32_t layer, edit_layer_stats_t* out) {
  if (!h || !out) return fail(EDIT_ERR_INVALID_ARG, "null argument");
  TRY(check_err(h));
  if (layer < 0 || layer >= h->cfg.num_layers) return fail(EDIT_ERR_INVALID_ARG, "layer out of range");
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  CUDA_TRY(h, cudaEventSynchronize(h->done[layer]));
  TRY(check_err(h));  // an exchange of this (or an earlier) unit timed out
  for (Lane& ln : h->lanes) {
    if (!ln.global) continue;
    ncclResult_t async_err = ncclSuccess;
    NCCL_TRY(h, ncclCommGetAsyncError(ln.global, &async_err));
    if (async_err != ncclSuccess) {
      h->poisoned = true;
      return fail(EDIT_ERR_NCCL, std::string("async NCCL error: ") + ncclGetErrorString(async_err));
    }
  }
  CUDA_TRY(h, cudaMemcpy(out, h->rec + layer, sizeof *out, cudaMemcpyDeviceToHost));
  return EDIT_OK;
}

edit_status_t edit_sync_get_state(edit_sync_t h, void* host_buf, size_t* bytes) {
  if (!h || !bytes) return fail(EDIT_ERR_INVALID_ARG, "null argument");
  TRY(check_err(h));
  const size_t need = sizeof(edit_ema_t) * (size_t)h->cfg.num_layers * h->N;
  if (!host_buf || *bytes < need) {
    *bytes = need;
    return host_buf ? fail(EDIT_ERR_NO_MEMORY, "state buffer too small") : EDIT_OK;
  }
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  CUDA_TRY(h, cudaDeviceSynchronize());
  CUDA_TRY(h, cudaMemcpy(host_buf, h->ema, need, cudaMemcpyDeviceToHost));
  *bytes = need;
  return EDIT_OK;
}

edit_status_t edit_sync_set_state(edit_sync_t h, const void* host_buf, size_t bytes) {
  if (!h || !host_buf) return fail(EDIT_ERR_INVALID_ARG, "null argument");
  TRY(check_err(h));
  const size_t need = sizeof(edit_ema_t) * (size_t)h->cfg.num_layers * h->N;
  if (bytes != need) return fail(EDIT_ERR_INVALID_ARG, "state size must be L*N*sizeof(edit_ema_t)");
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  CUDA_TRY(h, cudaDeviceSynchronize());
  CUDA_TRY(h, cudaMemcpy(h->ema, host_buf, need, cudaMemcpyHostToDevice));
  return EDIT_OK;
}

edit_status_t edit_sync_set_profiling(edit_sync_t h, int32_t enable) {
  if (!h) return fail(EDIT_ERR_INVALID_ARG, "null handle");
  TRY(check_err(h));
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  if (enable && h->prof.empty()) {
    h->prof.assign((size_t)h->cfg.num_layers * (EDIT_NUM_PHASES + 1), nullptr);
    for (auto& e : h->prof) CUDA_TRY(h, cudaEventCreate(&e));
  }
  h->profiling = enable != 0;
  h->pending.clear();
  return EDIT_OK;
}

edit_status_t edit_sync_profile_collect(edit_sync_t h, double phase_ms[EDIT_NUM_PHASES], double busy_ms[EDIT_NUM_PHASES],
                                        int64_t* syncs, int64_t* elements) {
  if (!h || !phase_ms) return fail(EDIT_ERR_INVALID_ARG, "null argument");
  TRY(check_err(h));
  for (int p = 0; p < EDIT_NUM_PHASES; ++p) phase_ms[p] = 0.0;
  int64_t elems = 0;
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  // per phase: the [start, end) interval of every unit, in ms from the first unit's start
  std::vector<std::vector<std::pair<double, double>>> iv(EDIT_NUM_PHASES);
  cudaEvent_t ref = nullptr;
  for (int32_t layer : h->pending) {
    cudaEvent_t* ev = &h->prof[(size_t)layer * (EDIT_NUM_PHASES + 1)];
    CUDA_TRY(h, cudaEventSynchronize(ev[EDIT_NUM_PHASES]));
    if (!ref) ref = ev[0];
    // N == 1 records no events for the empty phases 2 and 3 (no all-reduce, no K3)
    const int seq[6] = {0, 1, 2, 3, 4, 5}, seq1[4] = {0, 1, 2, 5};
    const int* q = h->N > 1 ? seq : seq1;
    const int nq = h->N > 1 ? 6 : 4;
    for (int k = 0; k + 1 < nq; ++k) {
      float ms = 0.f, t0 = 0.f, t1 = 0.f;
      CUDA_TRY(h, cudaEventElapsedTime(&ms, ev[q[k]], ev[q[k + 1]]));
      const int ph = q[k + 1] == 5 ? 4 : q[k];
      phase_ms[ph] += ms;
      if (busy_ms) {
        CUDA_TRY(h, cudaEventElapsedTime(&t0, ref, ev[q[k]]));
        CUDA_TRY(h, cudaEventElapsedTime(&t1, ref, ev[q[k + 1]]));
        iv[ph].emplace_back(t0, t1);
      }
    }
    elems += h->numel[layer];
  }
  // busy time of a phase = the union of its units' intervals (units on different lanes
  // overlap, so the plain sum over-counts the time the phase's kernels occupied the GPU)
  if (busy_ms)
    for (int p = 0; p < EDIT_NUM_PHASES; ++p) {
      auto& v = iv[p];
      std::sort(v.begin(), v.end());
      double total = 0.0, lo = 0.0, hi = 0.0;
      bool open = false;
      for (const auto& x : v) {
        if (!open || x.first > hi) {
          if (open) total += hi - lo;
          lo = x.first;
          hi = x.second;
          open = true;
        } else if (x.second > hi) {
          hi = x.second;
        }
      }
      if (open) total += hi - lo;
      busy_ms[p] = total;
    }
  if (syncs) *syncs = (int64_t)h->pending.size();
  if (elements) *elements = elems;
  h->pending.clear();
  return EDIT_OK;
}

edit_status_t edit_sync_nvlink_probe(edit_sync_t h, int64_t bytes_per_peer, int32_t reps, double* gbps) {
  if (!h || !gbps) return fail(EDIT_ERR_INVALID_ARG, "null argument");
  TRY(check_err(h));
  if (!h->peer || !h->dev_xchg || h->N < 2 || h->simulated)
    return fail(EDIT_ERR_INVALID_ARG, "the NVLink probe needs the peer path with N > 1 (mailbox exchange)");
  if (bytes_per_peer < 16 || reps < 1) return fail(EDIT_ERR_INVALID_ARG, "bytes_per_peer >= 16, reps >= 1");
  CUDA_TRY(h, cudaSetDevice(h->cfg.device));
  Lane& ln = h->lanes[0];
  int64_t max_numel = 0;
  for (int64_t x : h->numel) max_numel = std::max(max_numel, x);
  const int64_t esz = h->cfg.param_dtype == EDIT_BF16 ? 2 : 4;
  const int64_t cap = std::max<int64_t>(max_numel, 8) * esz / 16 * 16;
  bytes_per_peer = std::min(bytes_per_peer, cap) / 16 * 16;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  struct EventGuard {  // destroyed on every return path
    cudaEvent_t* a;
    cudaEvent_t* b;
    ~EventGuard() {
      if (*a) cudaEventDestroy(*a);
      if (*b) cudaEventDestroy(*b);
    }
  } guard{&e0, &e1};
  CUDA_TRY(h, cudaEventCreate(&e0));
  CUDA_TRY(h, cudaEventCreate(&e1));
  cudaStream_t st = ln.stream;
  CUDA_TRY(h, cudaStreamWaitEvent(st, ln.last, 0));
  // barriers: every member starts (and is known to have finished) pulling together
  h->launches += launch_xchg(xchg_args(h, ln, 2), ln.bar, ln.bar + 1, nullptr, st);
  CUDA_TRY(h, cudaEventRecord(e0, st));
  for (int r = 0; r < reps; ++r)
    h->launches += launch_nvlink_probe(ln.pp, h->N, h->sync_idx, bytes_per_peer,
                                       reinterpret_cast<unsigned*>(ln.Down), st);
  CUDA_TRY(h, cudaEventRecord(e1, st));
  h->launches += launch_xchg(xchg_args(h, ln, 2), ln.bar, ln.bar + 1, nullptr, st);
  CUDA_TRY(h, cudaEventRecord(ln.last, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  TRY(check_err(h));
  float ms = 0.f;
  CUDA_TRY(h, cudaEventElapsedTime(&ms, e0, e1));
  *gbps = ms > 0 ? (double)reps * (h->N - 1) * (double)bytes_per_peer / (ms * 1e-3) / 1e9 : 0.0;
  return EDIT_OK;
}

int64_t edit_sync_kernel_launches(edit_sync_t h) { return h ? h->launches : -1; }

edit_status_t edit_sync_destroy(edit_sync_t h) {
  if (!h) return EDIT_OK;
  edit_status_t st = EDIT_OK;
  cudaSetDevice(h->cfg.device);
  if (h->err_host && *reinterpret_cast<volatile int*>(h->err_host)) h->poisoned = true;
  // (a poisoned handle may have exchange kernels spinning until their timeout: do not block)
  if (!h->poisoned) cudaDeviceSynchronize();
  // captured rounds first: a graph holding NCCL collectives references the communicators,
  // which must outlive it (the NCCL-exchange graph case once stalled in teardown with the
  // graphs destroyed after the comms)
  clear_graphs(h);
  // (the simulated mesh's members are destroyed together after a device synchronize)
  bool ipc_safe = true;
  const bool exported = h->peer || !h->reg_gather.empty() || h->dev_xchg;
  if (exported && h->K > 1 && !h->simulated) {
    ipc_safe = false;
    if (h->ready && !h->poisoned && !h->lanes.empty() && h->lanes[0].global) {
      // barrier: no member may free its IPC-exported buffers while a peer still reads them.
      // Device mailbox exchange, bounded (30 s or the exchange timeout if shorter): a rank
      // unwinding after a peer died must not hang here
      Lane& ln = h->lanes[0];
      if (h->dev_xchg && ln.mailbox) {
        XchgArgs x = xchg_args(h, ln, 2);
        const unsigned long long cap = 30ull * 1000000000ull;
        x.timeout_ns = (h->timeout_ns && h->timeout_ns < cap) ? h->timeout_ns : cap;
        launch_xchg(x, ln.bar, ln.bar + 1, nullptr, ln.stream);
        cudaStreamSynchronize(ln.stream);
        int e = 0;
        cudaMemcpy(&e, h->err_dev, sizeof e, cudaMemcpyDeviceToHost);
        ipc_safe = e == 0;
      } else {
        double* tmpd = nullptr;
        if (cudaMalloc(&tmpd, sizeof(double) * (h->K + 1)) == cudaSuccess) {
          if (ncclAllGather(tmpd, tmpd + 1, 1, ncclFloat64, ln.global, ln.stream) != ncclSuccess) st = EDIT_ERR_NCCL;
          ipc_safe = cudaStreamSynchronize(ln.stream) == cudaSuccess && st == EDIT_OK;
          cudaFree(tmpd);
        }
      }
    }
  }
  for (void* p : h->reg_opened) cudaIpcCloseMemHandle(p);
  for (void* p : h->gather_opened) cudaIpcCloseMemHandle(p);
  if (h->gather_dev) cudaFree(h->gather_dev);
  for (Lane& ln : h->lanes) {
    for (size_t l = 0; l < ln.ops.size(); ++l)
      if (ln.sync) ncclRedOpDestroy(ln.ops[l], ln.sync);
    for (void* p : ln.opened) cudaIpcCloseMemHandle(p);
    // IPC-exported buffers a peer may still be reading (no completed barrier): leaked, not
    // freed -- freeing them could fault the peers' GPUs
    if (ipc_safe) {
      if (ln.Lown) cudaFree(ln.Lown);
      if (ln.Down) cudaFree(ln.Down);
      if (ln.mailbox) cudaFree(ln.mailbox);
    }
    if (ln.S) cudaFree(ln.S);
    if (ln.dseq) cudaFree(ln.dseq);
    if (ln.bar) cudaFree(ln.bar);
    // a poisoned handle's communicators may have collectives that never complete: abort them
    auto drop = [&](ncclComm_t c) {
      if (!c) return;
      if (h->poisoned) ncclCommAbort(c);
      else ncclCommDestroy(c);
    };
    drop(ln.shard);
    drop(ln.sync);
    drop(ln.global);
    if (ln.tail) cudaEventDestroy(ln.tail);
    if (ln.last) cudaEventDestroy(ln.last);
    if (ln.stream && !h->poisoned) cudaStreamDestroy(ln.stream);
  }
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  if (h->fork) cudaEventDestroy(h->fork);
  if (h->warm_dev) cudaFree(h->warm_dev);
  for (auto e : h->done)
    if (e) cudaEventDestroy(e);
  for (auto e : h->gate_ev)
    if (e) cudaEventDestroy(e);
  for (auto e : h->pre_ev)
    if (e) cudaEventDestroy(e);
  for (auto e : h->post_ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : {h->end_ev, h->rnd_ev0, h->rnd_ev1})
    if (e) cudaEventDestroy(e);
  for (auto e : h->prof)
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < edit_sync::kHostSlots; ++i) {
    if (h->slot_in[i]) cudaEventDestroy(h->slot_in[i]);
    if (h->slot_done[i]) cudaEventDestroy(h->slot_done[i]);
    if (h->slot_free[i]) cudaEventDestroy(h->slot_free[i]);
  }
  if (h->h2d) cudaStreamDestroy(h->h2d);
  if (h->d2h) cudaStreamDestroy(h->d2h);
  if (h->staging) cudaFree(h->staging);
  if (!h->poisoned) {
    if (h->err_dev) cudaFree(h->err_dev);
    if (h->err_host) cudaFreeHost(h->err_host);
  }
  delete h;
  return st;
}

}  // extern "C"
