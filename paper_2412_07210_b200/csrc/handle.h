// handle.h -- the library's handle and its per-unit enqueue steps (not part of the C ABI).
//
// Shared by api.cpp (the C ABI of include/edit_sync.h) and the single-GPU simulated mesh of
// tests/sim/edit_sim.cpp, which builds K member handles in one process on one device and
// drives them through the SAME plan/step functions, step-major across the members (so no
// member's exchange kernel waits behind another member's dependent work).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <string>
#include <vector>

#include "internal.h"

namespace edit {

// A lane = one in-order pipeline of unit syncs: its stream (internal; the caller's stream for
// edit_layer_sync), its own NCCL communicators (so two lanes' collectives never interleave on
// one comm) and its own exchange buffers.  edit_sync_round / the prefetch scheduler deal
// units round-robin over the lanes, so unit u+1's norm pass and scalar gathers run while unit
// u's exchange and update run.  Every rank maps unit u to lane u % nlanes: the collective
// order per communicator (and per mailbox phase) is identical on all ranks.
struct Lane {
  cudaStream_t stream = nullptr;
  cudaEvent_t tail = nullptr;  // join event
  // recorded after every unit sync that used this lane's buffers, on whatever stream it ran;
  // every later use waits on it first (edit_layer_sync may be called on any caller stream)
  cudaEvent_t last = nullptr;
  ncclComm_t global = nullptr, sync = nullptr, shard = nullptr;
  std::vector<ncclRedOp_t> ops;  // NCCL algo: per unit PreMulSum with that unit's device weight
  float* S = nullptr;            // NCCL algo: fp32 Delta exchange buffer
  // peer algo: own staging copy of the local (L) and own Dbar slice (D), cudaMalloc'd and
  // exported by CUDA IPC to the sync row; pp holds every member's mapped pointers
  void* Lown = nullptr;
  float* Down = nullptr;
  PeerPtrs pp{};
  std::vector<void*> opened;  // IPC mappings to close
  // device-side scalar exchange (EDIT_XCHG=nccl disables): own mailbox, all ranks' mapped
  unsigned long long* mailbox = nullptr;
  MailPtrs mp{};
  unsigned long long seq[kXchgPhases] = {0, 0, 0};
  unsigned long long* dseq = nullptr;  // graph mode: device-side sequence counters [kXchgPhases]
  double* bar = nullptr;               // barrier exchanges: [1 + kMaxRanks] fp64 (send, recv)
};

// EDIT_GRAPH=1: edit_sync_round captures the round once per set of buffer pointers into a
// CUDA graph and replays it.  Requires the mailbox sequence numbers on the device
// (Lane::dseq); must be equal on every rank.
struct RoundGraph {
  std::vector<uintptr_t> key;  // the 3L buffer pointers + the profiling flag
  cudaGraphExec_t exec = nullptr;
  int64_t launches = 0;        // kernels per replay
};

// How a unit's kernels are shaped (default full grids; the scheduler's modes).
constexpr int kSchedAuto = -1;  // edit_sched_set_partition(sms = -1): the self-tuning default
constexpr int kTuneCands = 4;   // serial + 3 partition plans
constexpr int kTuneSamples = 3; // rounds measured per candidate before choosing

struct Mode {
  int cap = 0;        // max CTAs of the LDG streaming kernels (0 = full grid)
  int peer_ctas = 0;  // persistent grid of the TMA peer kernels
  int smem_kb = 0;    // shared-memory ring of the TMA peer kernels (0 = default)
  int part = 0;       // > 0: partition mode, K1 / K4 / peer kernels on <= part persistent CTAs
};

// EDIT_PEER_KERNELS=ldg|ldg2|ldgall|tma (default ldg): the kernels of full-speed rounds.
// ldg: AG + update as a non-persistent LDG full grid (measured on 2 B200s, 7B unit, N = 2:
// 0.70 ms vs 0.77 ms for the TMA pipeline; equal at N = 4 where both pull at the NVLink
// ceiling, profiles/r2_peer_kbench_ag.txt), RS as the persistent TMA pipeline; ldg2: 2 vectors
// per thread in AG; ldgall: RS as an LDG full grid too (slower in full rounds); tma: both as
// the persistent warp-specialised TMA pipelines, which the scheduler's partition and
// co-resident modes always use (capped grids).  Bits: 1 = AG LDG, 2 = 2 vectors, 4 = RS LDG.

}  // namespace edit

struct edit_sync {
  edit_sync_config_t cfg{};
  std::vector<int64_t> numel;
  int M = 1, N = 1, K = 1, sync_idx = 0, shard_idx = 0;
  int num_sms = 0;
  std::vector<double*> part1, part2;  // per-unit per-CTA partial slots (workspace)
  std::vector<edit::Lane> lanes;
  bool peer = false;                  // N > 1 and algo == EDIT_ALGO_PEER
  bool simulated = false;             // a member of the single-GPU simulated mesh (tests/sim)
  int peer_ctas = 148;                // persistent grid of the peer kernels (EDIT_PEER_CTAS env overrides)
  int peer_tile = edit::kPeerTileVec; // vectors per TMA tile (EDIT_PEER_TILE env; must match on all ranks)
  bool dev_xchg = true;               // scalar chain over NVLink mailboxes (EDIT_XCHG=nccl: NCCL gathers)
  int peer_ldg = 1;                   // EDIT_PEER_KERNELS bits (full-speed rounds): 1 AG LDG, 2 x2, 4 RS LDG
  // unit groups (internal.h GroupArgs): edit_sync_round syncs runs of consecutive units up to
  // this many elements in total as one group (EDIT_GROUP_NUMEL; 0 = off; must match on all
  // ranks).  Measured 350M 1x2 (2 B200s): 2.60 ms per round without groups, 2.44 / 2.34 / 2.24
  // with 16 / 32 / 64 Mi (profiles/r2_groups_sweep_2gpu.txt)
  int64_t group_numel = 64ll << 20;
  unsigned long long timeout_ns = 0;  // mailbox wait bound (EDIT_XCHG_TIMEOUT_S; 0 = forever)
  // sticky exchange error: device flag read by every exchange, and its mapped-host mirror the
  // library polls at every call (no device sync needed to notice a dead peer)
  int* err_dev = nullptr;
  int* err_host = nullptr;      // host pointer of the mapped page
  int* err_host_dev = nullptr;  // its device alias
  // scheduler (co-resident) mode: at most sched_ctas CTAs per streaming kernel (EDIT_SCHED_CTAS)
  // (default 0 = full grids: measured, capping does not buy overlap on B200 -- DESIGN.md 7)
  int sched_ctas = 0;
  int sched_smem_kb = 18;
  // partition mode (edit_sched_set_partition): scheduled units u >= sched_full_units run
  // as persistent TMA pipelines on sched_part CTAs (one per SM), lanes at high priority.
  // sched_part == kSchedAuto (the default): per unit, the fewest SMs that finish the unit's
  // sync within the forward time it overlaps (measured in the previous round from events at
  // acquire), at sm_gbps per SM (EDIT_SM_GBPS, measured ~100 GB/s per SM, DESIGN 6)
  int sched_part = -1;
  int sched_full_units = 2;
  double sm_gbps = 100.0;
  // auto mode = a self-tuning choice among kTuneCands plans per round (api.cpp): timing events
  // on the compute stream at each acquire (before / after its wait), at end_round, and around
  // the whole round
  std::vector<cudaEvent_t> pre_ev, post_ev;  // [L]
  cudaEvent_t end_ev = nullptr, rnd_ev0 = nullptr, rnd_ev1 = nullptr;
  bool rnd_pending = false;                  // a measurable round is in flight
  std::vector<double> fwd_ms;                // [L] forward time of each unit (last measurement)
  bool fwd_valid = false;
  int round_cand = -1;                       // candidate of the current round (-1: fixed setting)
  int tune_drift = 0;                        // consecutive rounds far above the choice's median
  std::vector<std::vector<float>> tune_ms;   // [kTuneCands] measured round times
  std::vector<int> sched_sms;                // [L] SMs given to each unit's sync (0 full grid, -1 serial)
  int lane_prio = 0;             // priority the lanes were created with (env default)
  // gate (EDIT_SCHED_GATE=1): the sync of unit u+depth starts only when the forward of unit
  // u may start (an event on the compute stream at acquire(u)), not as soon as its lane frees
  bool sched_gate = false;
  std::vector<cudaEvent_t> gate_ev;
  bool ready = false;            // init completed (destroy may then barrier with the peers)
  char* ws = nullptr;
  edit::LayerScratch* scratch = nullptr;
  edit_ema_t* ema = nullptr;
  edit_layer_stats_t* rec = nullptr;
  std::vector<cudaEvent_t> done;  // per unit: recorded after its last kernel
  cudaEvent_t fork = nullptr;     // round API / scheduler: "the caller's inputs are ready"
  // profiling: EDIT_NUM_PHASES + 1 timing events per unit, and the units pending collection
  bool profiling = false;
  bool graph = false;               // EDIT_GRAPH=1 (round replay from CUDA graphs)
  bool nvtx = false;                // EDIT_NVTX=1 (NVTX ranges per unit / round)
  cudaStream_t cap_stream = nullptr;  // the capture origin (the caller's may be the legacy one)
  std::vector<edit::RoundGraph> graphs;  // small cache, most recent last
  std::vector<cudaEvent_t> prof;
  std::vector<int32_t> pending;
  // host-buffer variant: staging slots + copy-in / copy-out streams
  char* staging = nullptr;
  size_t slot_bytes = 0;
  int next_slot = 0;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  // kHostSlots staging slots: copy-in of unit u+2 need not wait for copy-out of unit u
  static constexpr int kHostSlots = 3;
  cudaEvent_t slot_in[kHostSlots] = {}, slot_done[kHostSlots] = {}, slot_free[kHostSlots] = {};
  double* warm_dev = nullptr;  // warm-up all-reduce (NCCL-exchange mode): barrier scalars (N + 1)
  // NEXT-2 registered gather buffers: [L][M] (member q's full-module buffer, mapped)
  std::vector<std::vector<void*>> reg_gather;
  std::vector<void*> gather_opened;
  double* gather_dev = nullptr;  // gather barrier scalars per unit [L][M + 1] (NCCL-exchange mode)
  // registered caller locals (peer path): my pointers and every member's mapped pointer
  std::vector<void*> reg_local;                     // [L]
  std::vector<std::vector<const void*>> reg_peer;   // [L][N]
  std::vector<void*> reg_opened;                    // distinct IPC mappings to close
  // prefetch scheduler state
  std::vector<void*> sched_local;
  std::vector<float*> sched_anchor, sched_mom;
  std::vector<std::vector<int32_t>> sched_items;  // the round's work items (form_groups)
  int sched_depth = 0, sched_next_sync = 0, sched_next_acquire = 0;  // next_sync: item index
  bool sched_active = false;
  bool poisoned = false;
  int64_t launches = 0;
};

namespace edit {

// Everything one unit sync needs, fixed before its first kernel is enqueued.
struct UnitPlan {
  Lane* ln = nullptr;
  int32_t layer = 0;
  void* local = nullptr;
  float* anchor = nullptr;
  float* momentum = nullptr;
  cudaStream_t st = nullptr;
  Mode mode{};
  bool direct = false;    // peer path reads the members' registered locals
  bool gathered = false;  // NEXT-2 fused shard all-gather
  PeerPtrs pp{};
  float* S = nullptr;     // NCCL path's fp32 exchange buffer
  DecideArgs d{};
  UpdateArgs u{};
  Slicing sl{};
  cudaEvent_t* ev = nullptr;  // profiling events [EDIT_NUM_PHASES + 1] or null
};

// The steps of one unit sync (Alg. 2), in enqueue order.  Each may enqueue nothing on a path
// where it has no work.  Across ranks, step s of a unit only waits for steps <= s of the same
// unit on the other ranks, so enqueueing step-major over several handles on one device
// (the simulated mesh) can never block a member behind another member's later step.
enum Step {
  kStepBegin,     // wait for the previous use of the lane and of the unit; profiling event
  kStepNorm,      // K1: Delta + shard norm (+ folded norm exchange and K2)
  kStepDecide,    // NCCL scalar gather + K2 (when not folded)
  kStepExchange,  // Eq. 3: peer RS (+ folded Dbar-norm exchange) / NCCL PreMulSum all-reduce + K3
  kStepDbarNorm,  // NCCL gathers of the Dbar-norm partials (when not folded)
  kStepUpdate,    // K4 / AG + update (+ NEXT-2 gather stores)
  kStepGather,    // NEXT-2: barrier after which every member's gathered module is complete
  kStepEnd,       // done / lane events
  kNumSteps
};

edit_status_t plan_unit(edit_sync_t h, Lane& ln, int32_t layer, void* local, float* anchor, float* momentum,
                        cudaStream_t st, const Mode& mode, UnitPlan& p);
edit_status_t enqueue_step(edit_sync_t h, UnitPlan& p, int step);

// A group of small units synced by the three group kernels (peer path, full-speed rounds):
// the units' plans (for their events), the kernel arguments and the lane.
struct GroupPlan {
  Lane* ln = nullptr;
  cudaStream_t st = nullptr;
  std::vector<UnitPlan> units;
  GroupArgs g{};
};
// Partition of a round's unit list into groups (deterministic from the numel list and the
// settings, so identical on every rank); a group of one unit takes the single-unit path.
std::vector<std::vector<int32_t>> form_groups(edit_sync_t h, const int32_t* layers, int nunits);
edit_status_t plan_group(edit_sync_t h, Lane& ln, const std::vector<int32_t>& layers, void* const* locals,
                         float* const* anchors, float* const* momenta, cudaStream_t st, GroupPlan& gp);
edit_status_t enqueue_group_step(edit_sync_t h, GroupPlan& gp, int step);

// Enqueue syncs of `nunits` units on each of nh handles (production: nh == 1; the simulated
// mesh: nh == K members), unit by unit and, inside a unit, step-major across the handles.
//   use_lanes == false: every unit on lane 0, on streams[k] (edit_layer_sync).
//   use_lanes == true: unit u on lane u % nlanes, on the lane's stream, after a fork from
//     streams[k]; streams[k] then waits for all lanes (edit_sync_round).
// locals/anchors/momenta: [nh][nunits] (row k = handle k).
edit_status_t enqueue_units(edit_sync_t const* hs, int nh, int nunits, const int32_t* layers,
                            void* const* locals, float* const* anchors, float* const* momenta,
                            const cudaStream_t* streams, bool use_lanes);
// Warm-up all-reduce of one unit on nh handles (same step-major rule); force_peer selects the
// peer-memory variant regardless of EDIT_WARMUP_ALGO.
edit_status_t enqueue_warmup(edit_sync_t const* hs, int nh, int32_t layer, void* const* grads,
                             const cudaStream_t* streams, bool force_peer, bool on_lane = false);
// Warm-up all-reduce of every unit (grads [nh][nunits]), unit u on lane u % lanes after a
// fork from streams[k]; streams[k] then joins every lane (edit_warmup_allreduce_round).
edit_status_t enqueue_warmup_units(edit_sync_t const* hs, int nh, int nunits, void* const* grads,
                                   const cudaStream_t* streams, bool force_peer);

// Init split: everything that needs no other rank (validation, workspace carving, streams,
// events, exchange buffers, the mapped error flag); then, for a real mesh, the NCCL
// communicators and CUDA IPC wiring (api.cpp).  The simulated mesh wires its members with
// plain device pointers instead.
edit_status_t create_local(const edit_sync_config_t* cfg, void* workspace, size_t workspace_bytes, edit_sync_t* out);
edit_status_t fail(edit_status_t st, const std::string& msg);
edit_status_t check_err(edit_sync_t h);  // EDIT_ERR_STATE if the handle is (or just got) poisoned

}  // namespace edit
