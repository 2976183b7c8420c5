/*
 * edit_sync.h -- C ABI of the B200-native EDiT layer-wise sync library
 * (libedit_sync.so, built from paper_2412_07210_b200/csrc).
 *
 * What it computes: Sync() of PAPER.md Algorithm 2, the model
 * synchronisation of EDiT with the pseudo-gradient penalty (Section 3.2,
 * P:84-123), for ONE rank of an M x N device mesh (Section 3.1, P:61:
 * M model sync groups of N workers = rows; N model shard groups of M workers =
 * columns; K = M*N ranks, rank = sync_idx*M + shard_idx, reading R20 of
 * DESIGN.md).  Per sync unit ("module") and call:
 *
 *   Delta   = anchor - local                             (Alg.2 l.442; sign R1)
 *   G_n     = ||Delta_n||_2 over the whole module         (l.443, R5)
 *   z-test against EMA (mu, sigma), G_n := inf if z > delta (l.444-446)
 *   EMA update of every finite G_n (Eq. 1)
 *   rollback iff no G_n finite (l.447-449, R11)
 *   w_n     = exp(-G_n) / sum_j exp(-G_j)                 (Eq. 2, l.451)
 *   Dbar    = sum_n w_n Delta_n over the sync group       (Eq. 3, l.452)
 *   beta    = min(phi / (||Dbar|| + eps), 1)              (Eq. 4, l.453)
 *   m       = mu m + beta Dbar ; anchor = anchor - nu (beta Dbar + mu m)
 *                                                         (Eq. 5 + OuterOpt, l.454, R2)
 *   local   = round_to_local_dtype(anchor)                (l.455)
 *
 * All device work is enqueued on the caller's stream; nothing here blocks the
 * host except edit_sync_stats / get_state / set_state / destroy and init.
 * There is no CPU fallback: without a CUDA device every call that needs one
 * returns EDIT_ERR_CUDA.
 *
 * Cross-rank exchange (N > 1 or M > 1, default): the K-scalar gathers of the module norms and
 * of the ||Dbar|| partials run over NVLink mailboxes inside the LAST CTA of the producing
 * kernel (K1, the reduce-scatter), so a unit is 3 dependent kernels on the peer path and 2 at
 * N == 1.  A rank that waits longer than EDIT_XCHG_TIMEOUT_S seconds (default 600; 0 = wait
 * forever, as NCCL does) for a peer marks its handle failed: from then on every exchange of
 * the handle returns at once without publishing, no kernel of an affected unit writes any
 * buffer (no update from stale peer data), the peers in turn time out the same way, and
 * every later call on the handle returns EDIT_ERR_STATE (polled from mapped host memory, no
 * device sync).  The state is then that of the last unit that completed everywhere: restore
 * from a checkpoint.
 */
#ifndef EDIT_SYNC_H_
#define EDIT_SYNC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EDIT_MAX_SYNC 8          /* N <= 8: one NVSwitch node                      */
#define EDIT_MAX_SHARD 8         /* M <= 8                                         */
#define EDIT_UNIQUE_ID_BYTES 128 /* == sizeof(ncclUniqueId)                        */

typedef struct edit_sync* edit_sync_t;

typedef enum {
  EDIT_OK = 0,
  EDIT_ERR_INVALID_ARG = 1, /* bad config / pointer / layer index / alignment    */
  EDIT_ERR_CUDA = 2,        /* CUDA runtime error (text: edit_sync_last_error)   */
  EDIT_ERR_NCCL = 3,        /* NCCL error                                        */
  EDIT_ERR_STATE = 4,       /* handle poisoned by an earlier CUDA/NCCL error     */
  EDIT_ERR_NO_MEMORY = 5    /* workspace too small / host allocation failed      */
} edit_status_t;

typedef enum { EDIT_BF16 = 0, EDIT_F32 = 1 } edit_dtype_t;

/* Ablations of Section 4.5. */
#define EDIT_NO_AE 1u /* w/o anomaly elimination: no z-test (non-finite G still excluded, R9) */
#define EDIT_NO_WA 2u /* w/o weighted averaging: uniform 1/#finite                              */
#define EDIT_NO_GC 4u /* w/o gradient clip: beta = 1                                            */

typedef struct {
  int32_t shard_dim;             /* M                                              */
  int32_t sync_dim;              /* N; M*N = world size                             */
  int32_t rank;                  /* 0 <= rank < M*N; sync_idx = rank / M, shard_idx = rank % M */
  int32_t device;                /* CUDA ordinal this rank runs on                         */
  int32_t num_layers;            /* L sync units                                           */
  int32_t param_dtype;           /* edit_dtype_t of `local`; anchor/momentum are fp32      */
  const int64_t* layer_numel;    /* [L] per-rank padded shard length (host memory, copied) */
  float outer_lr;                /* nu    (0.8 / 1.0)                               */
  float outer_momentum;          /* mu    (0.85 / 0.8)                              */
  float clip_threshold;          /* phi   (10)                                      */
  float clip_eps;                /* eps   (value unstated -> 1e-6, R12)             */
  float anomaly_threshold;       /* delta (3)                                        */
  float ema_alpha;               /* alpha (0.02)                                     */
  int32_t ema_warmup_rounds;     /* EMA warm-up length (unstated -> 10, R8)          */
  uint32_t flags;                /* EDIT_NO_AE | EDIT_NO_WA | EDIT_NO_GC                   */
  int32_t algo;                  /* N > 1 exchange (Eq. 3): EDIT_ALGO_PEER (default) or EDIT_ALGO_NCCL */
} edit_sync_config_t;

/* How Eq. 3's weighted sum crosses the sync group when N > 1:
 *  EDIT_ALGO_PEER: fused peer-memory kernels over NVLink (CUDA IPC within one node): each
 *    member reduces one 1/N slice straight from the peers' bf16/fp32 params
 *    (Dbar = sum_j w_j (anchor - local_j)) and every member then pulls the reduced slices
 *    while applying the update -- (b_l + 4)(N-1)/N bytes per param per direction.
 *  EDIT_ALGO_NCCL: Delta in an fp32 buffer, ncclAllReduce with PreMulSum(w on device),
 *    then the update -- 8(N-1)/N bytes per param per direction plus NCCL's HBM traffic. */
#define EDIT_ALGO_PEER 0
#define EDIT_ALGO_NCCL 1

/* Outcome of the last completed sync of one unit (device-written, D5). */
typedef struct {
  int64_t round;                     /* number of syncs of this unit so far            */
  double G[EDIT_MAX_SYNC];           /* module-level ||Delta_n||, +inf if flagged       */
  double z[EDIT_MAX_SYNC];           /* EMA z-score, NaN when the test was not applied */
  double w[EDIT_MAX_SYNC];           /* Eq. 2 weights                                   */
  int32_t anomalous[EDIT_MAX_SYNC];  /* 1 if G_n was set to infinity                    */
  double G_bar;                      /* ||Dbar|| (module level), 0 on rollback          */
  double beta;                       /* Eq. 4, 1 on rollback                            */
  int32_t rollback;                  /* Alg. 2 l.448-449 taken                          */
  int32_t num_sync;                  /* N                                               */
  double ema_mu[EDIT_MAX_SYNC];      /* EMA after this sync, per replica n              */
  double ema_sigma[EDIT_MAX_SYNC];
  int64_t ema_count[EDIT_MAX_SYNC];
} edit_layer_stats_t;

/* EMA record of one (unit, replica): used by get_state / set_state. */
typedef struct {
  double mu;
  double sigma;
  int64_t count;
  int64_t reserved;
} edit_ema_t;

/* Rank 0 creates the NCCL unique id; the caller broadcasts it to every rank
 * (e.g. over a torch.distributed process group).  Not needed when M*N == 1. */
edit_status_t edit_sync_get_unique_id(uint8_t id[EDIT_UNIQUE_ID_BYTES]);

/* Device workspace the caller must provide to edit_sync_init (256-byte aligned, on
 * cfg->device): per-unit scratch and per-CTA partial slots, the EMA state [L][N] and the
 * outcome records [L].  The exchange buffers of the N > 1 paths (peer: a staging copy of
 * the local + a 1/N Dbar slice, exported by CUDA IPC; NCCL: an fp32 Delta buffer) are
 * library-owned, one set per lane (see edit_sync_round), cudaMalloc'd by init. */
edit_status_t edit_sync_workspace_bytes(const edit_sync_config_t* cfg, size_t* bytes);

/* Collective over all M*N ranks (blocks until every rank has joined).
 * Validates cfg (EDIT_ERR_INVALID_ARG for: null pointers; M, N < 1; M > 8;
 * N > 8; rank outside [0, M*N); L < 1; negative numel; nu <= 0; mu outside
 * [0, 1); phi <= 0; eps <= 0; alpha outside (0, 1]; delta <= 0; W < 0),
 * creates the NCCL comms (global, sync = row, shard = column) and zeroes the
 * EMA state (mu = sigma = 0, count = 0; R8).  The workspace stays owned by the
 * caller and must outlive the handle.
 * Every rank must agree on the settings that fix slice layout, lane mapping and the exchange
 * protocol (EDIT_LANES, EDIT_PEER_TILE, EDIT_XCHG, EDIT_GRAPH, algo, the units, dtype,
 * flags): init all-gathers a digest of them and fails with EDIT_ERR_INVALID_ARG on a mismatch.
 * EMA warm-up (R8, PAPER P:98 gives no initialisation): with mu = sigma = 0 and the paper's
 * alpha = 0.02, mu reaches only ~18 % of a constant G after W = 10 rounds, so z stays near 2
 * at the end of the warm-up and a ~1.35x rise of G then flags every replica (a rollback
 * whose skipped Eq. 1 update freezes the EMA).  Callers should either seed the EMA with
 * edit_sync_set_state (e.g. mu = G of the first sync, sigma = 0.1 mu, count = W) or use a
 * warm-up of about 3 / alpha rounds. */
edit_status_t edit_sync_init(const edit_sync_config_t* cfg, const uint8_t id[EDIT_UNIQUE_ID_BYTES],
                             void* workspace, size_t workspace_bytes, edit_sync_t* out);

/* Sync one unit (Alg. 2) in place:
 *   local    [layer_numel[layer]] param_dtype, device  theta_{t,tau} in, theta_{t+1,0} out
 *   anchor   [layer_numel[layer]] fp32, device         theta_t in, theta_{t+1} out
 *   momentum [layer_numel[layer]] fp32, device         outer momentum, in/out
 *   stream   cudaStream_t (NULL = legacy default stream)
 * Buffers must be 16-byte aligned, must not alias each other or the workspace,
 * and the zero-padded shard tail must be zero.  Every rank must call this for
 * every unit in the same order (collective).  Enqueues only: no host sync, no
 * data-dependent host branch (the rollback branch is taken on the device).
 * Stream order: any stream may be passed, a different one per call.  The call runs on
 * `stream` after (i) the work already enqueued there, (ii) the previous sync of the same unit
 * and (iii) the previous user of the exchange buffers of lane 0 (which every per-unit call
 * shares), whatever streams those ran on (internal events) -- so calls on different streams
 * or host threads cannot race on the library's buffers.  The ORDER of the calls (the host
 * order in which they were made) must still be the same on every rank: it fixes the pairing
 * of the exchanges across ranks; calls from several host threads must be serialised.
 * EDIT_ERR_INVALID_ARG: null handle/pointer, layer outside [0, L), misalignment.
 * EDIT_ERR_STATE: the handle is poisoned (CUDA/NCCL error, or an exchange timed out). */
edit_status_t edit_layer_sync(edit_sync_t h, int32_t layer, void* local, float* anchor, float* momentum,
                              void* stream);

/* Peer path only (N > 1, EDIT_ALGO_PEER), optional: register the caller's L local buffers
 * (device pointers, the same ones later passed to edit_layer_sync / edit_sync_round /
 * the scheduler) so the members of a sync row read each other's params straight from
 * those buffers (CUDA IPC of their allocations) instead of from a staging copy the norm
 * pass writes -- saves b_l bytes per param of HBM writes.  Collective over all ranks.
 * The buffers must stay allocated (not moved or freed) until edit_sync_destroy; a sync
 * called with a different pointer for a unit falls back to the staging copy.
 * No-op returning EDIT_OK when N == 1 or algo == EDIT_ALGO_NCCL. */
edit_status_t edit_sync_register_locals(edit_sync_t h, void* const* locals);

/* NEXT-2, fused write-back -> shard-group all-gather (Alg. 1 l.411: after the sync, "gather
 * module parameters in G^s_n" for the forward).  Register, per unit, a device buffer of
 * M * layer_numel[u] elements (param_dtype) that receives the whole module: shard m at
 * [m * layer_numel[u], (m+1) * layer_numel[u]).  From then on every sync of a unit stores
 * its updated local ALSO into that slot of every shard-group member's buffer (NVLink stores
 * through CUDA IPC mappings, fused into the update kernel), followed by one scalar gather on
 * the shard comm, so when the unit's sync has completed on a rank its gathered module is
 * complete there -- no separate all-gather pass.  Collective over all ranks; buffers must
 * stay allocated until edit_sync_destroy.  M == 1: nothing to gather, returns EDIT_OK. */
edit_status_t edit_sync_register_gather(edit_sync_t h, void* const* full_bufs);

/* One full sync round: every unit 0..L-1 (arrays of L device pointers), equivalent to
 * calling edit_layer_sync for u = 0..L-1 in order but pipelined: work items (units, or the
 * unit groups below) are dealt round-robin over the library's lanes (EDIT_LANES; default 4 for N > 1, 2 for N == 1;
 * each lane = an internal stream + its own NCCL communicators + exchange buffers), so unit u+1's norm pass and
 * scalar gathers overlap unit u's exchange and update.  Starts after the work already on
 * `stream`; `stream` waits for the whole round.
 * Unit groups (peer path, N > 1, mailbox exchange, no registered gather buffers): runs of
 * consecutive units up to EDIT_GROUP_NUMEL elements in total (default 67,108,864; 0 = off;
 * equal on every rank) are synced as one work item -- one norm, one reduce-scatter and one
 * update launch for the group, and one exchange message per phase carrying every unit's
 * scalars; per-unit semantics (norms, z-tests, EMA, weights, rollback, clip) unchanged.
 * Results: N == 1 (no groups) bit for bit those of the sequential calls; within a group the
 * reduce-scatter's per-CTA partition of ||Dbar||^2 differs from the single-unit kernel's, so
 * beta (hence anchor/momentum/local) can differ from the sequential calls in the last bits
 * (within the R17 tolerance; decisions identical), and is identical on every rank.
 * EDIT_GRAPH=1 in the environment at init (equal on every rank; opt-in): the round is
 * captured into a CUDA graph on the first call with a given set of 3L pointers and replayed
 * on later calls with the same set (up to 4 sets cached); same results. */
edit_status_t edit_sync_round(edit_sync_t h, void* const* locals, float* const* anchors, float* const* momenta,
                              void* stream);

/* Host-buffer variant (the paper's CPU offload of the extra parameters and outer
 * momentum): local/anchor/momentum live in host memory (page-locked for the
 * copies to be asynchronous).  Per call: H2D of the three shards into one of three
 * library-owned device staging slots (on an internal copy stream), the same device
 * sync as edit_layer_sync on `stream`, then D2H of the three results back into the
 * host buffers (on a second copy stream), so consecutive units overlap copy-in,
 * compute and copy-out.  Staging is allocated on the first call (3 x max numel x
 * (elem + 8) bytes).  The host buffers must stay valid and untouched until
 * edit_sync_host_wait() on a stream has been reached. */
edit_status_t edit_layer_sync_host(edit_sync_t h, int32_t layer, void* local_host, float* anchor_host,
                                   float* momentum_host, void* stream);
/* Makes `stream` wait until every outstanding host-variant copy-out has landed. */
edit_status_t edit_sync_host_wait(edit_sync_t h, void* stream);

/* Layer-wise prefetch scheduler (Alg. 1 l.408-412): "sync parameters for the
 * upcoming module concurrently with ongoing computations".  The syncs run in unit order on
 * a library-owned side stream; the caller's forward (on `compute_stream`) acquires each unit
 * before using its params.
 *   begin_round: registers the round's L buffers (arrays of L device pointers, copied),
 *     makes the side stream wait for everything already enqueued on compute_stream (the
 *     inner steps that produced the locals), and enqueues the syncs of units 0..depth-1.
 *   acquire(layer): makes compute_stream wait until unit `layer` is synced and enqueues the
 *     sync of unit layer+depth.  Call for layer = 0, 1, ..., L-1 in order.
 *   end_round: enqueues any unit not yet synced and makes compute_stream wait for all.
 * depth >= 1 (the paper prefetches "the upcoming module": depth 1).
 * EDIT_ERR_INVALID_ARG: null arrays, depth < 1, acquire out of order / outside a round. */
edit_status_t edit_sched_begin_round(edit_sync_t h, void* const* locals, float* const* anchors,
                                     float* const* momenta, int32_t depth, void* compute_stream);
edit_status_t edit_sched_acquire(edit_sync_t h, int32_t layer, void* compute_stream);
edit_status_t edit_sched_end_round(edit_sync_t h, void* compute_stream);
/* Partition mode of the scheduler (how the overlap of P:70 is obtained on one GPU whose
 * forward is tensor-bound on every SM).  The syncs of units u >= full_units run as persistent
 * TMA pipelines on a few SMs, each CTA holding a ~200 KB shared-memory ring so that it owns
 * its SM; the concurrent forward keeps the other SMs.  Units u < full_units (the ones a
 * forward reaches before its first GEMM, e.g. the embedding: 2) keep full grids.
 *   sms == -1 (the DEFAULT, "auto"): self-tuning.  Each round runs one of four plans and
 *     is timed on the compute stream (begin_round -> end_round): SERIAL (the whole round
 *     first, pipelined over the lanes on full grids exactly as edit_sync_round runs it, and
 *     acquire(0) waits for all of it: no overlap, the cost of the two back to back) or PARTITION with (f, depth) = (1.0, >= 2), (1.6, >= 2),
 *     (1.0, the caller's depth): f x the fewest SMs that stream unit u's bytes within the
 *     forward time its sync overlaps (units u-depth .. u-1, measured per unit between acquire
 *     calls; EDIT_SM_GBPS, default 100 GB/s per SM, the measured per-SM streaming rate), in
 *     [4, #SMs].  Every plan is measured 3 times (serial first), then the fastest median is
 *     kept; a > 15 % drift of its newest round time re-measures all.  So after 12 rounds the
 *     default is the best of serial and the partitions for this forward (edit_sched_get_plan
 *     reports the choice).  The depth passed to begin_round is a minimum in this mode.
 *   sms > 0: fixed, ceil(sms / lanes) CTAs per lane's kernels (the lanes run concurrently).
 *   sms == 0: full grids at the lowest stream priority (the sync fills what the forward
 *     leaves free; measured worse than serial on a tensor-bound forward, DESIGN 7).
 * The side streams run at the highest priority for sms != 0 (a freed SM goes to a sync CTA
 * first).  Covers K1 and the N == 1 update (peer path: also RS and AG); the NCCL path's
 * K1/K3/K4 and the NEXT-2 gathering update keep their full-grid kernels.  Results are those
 * of the default mode within R17 (only the reduction grouping of K1 differs).  Not during a
 * round.  EDIT_ERR_INVALID_ARG: sms < -1 or > #SMs, full_units < 0, a round is active. */
edit_status_t edit_sched_set_partition(edit_sync_t h, int32_t sms, int32_t full_units);
/* The scheduler's plan of its last round (host values, no device sync): *candidate = -1 for a
 * fixed setting (sms >= 0), else the auto mode's choice: 0 = serial, 1..3 = partition with
 * (1.0, depth >= 2) / (1.6, depth >= 2) / (1.0, caller's depth) x the minimum SMs; sms[u] (nullable, [L]) = SMs given to unit u's sync
 * (0 = full grid, -1 = serial); median_ms (nullable, [4]) = the measured median round time of
 * each candidate so far (0 = not measured). */
edit_status_t edit_sched_get_plan(edit_sync_t h, int32_t* candidate, int32_t* sms, double* median_ms);

/* Warm-up phase (Alg. 1 l.422-424): while (t*tau + p) <= t_warm the gradients
 * of the synchronous mini-batch phase are all-reduced within the model sync group, after the
 * shard group's reduce-scatter.  grad [layer_numel[layer]] param_dtype, device: this rank's
 * gradient shard of the unit, replaced in place by the MEAN over the N members of its sync
 * row, bit-identical on every member.  Collective over the sync row
 * (every rank calls it for the same units in the same order).  Default: ncclAllReduce
 * (ncclAvg) on the library's sync comm -- a pure mean with nothing to fuse, where NCCL
 * measured faster.  EDIT_WARMUP_ALGO=peer (with EDIT_ALGO_PEER): the gradient is staged into
 * the IPC-exported buffer, each member averages its 1/N slice straight from the others over
 * NVLink and rounds it once, then pulls every averaged slice from its owner.  N == 1: no-op. */
edit_status_t edit_warmup_allreduce(edit_sync_t h, int32_t layer, void* grad, void* stream);

/* The warm-up all-reduce of EVERY unit in one call: grads [num_layers] (the same layout and
 * meaning as above, one per unit; units with layer_numel == 0 are skipped), unit u on the
 * library's lane u % lanes after a fork from `stream`, which then waits for all lanes -- so
 * unit u+1's staging and barriers overlap unit u's NVLink pulls (a per-unit call on one stream
 * serialises them).  Same algorithm choice as edit_warmup_allreduce (EDIT_WARMUP_ALGO).
 * Collective over the sync row.  N == 1: no-op. */
edit_status_t edit_warmup_allreduce_round(edit_sync_t h, void* const* grads, void* stream);

/* Blocks until this unit's last enqueued sync has completed, then copies its
 * outcome record to *out. */
edit_status_t edit_sync_stats(edit_sync_t h, int32_t layer, edit_layer_stats_t* out);

/* EMA state of every (unit, replica), row-major [L][N] edit_ema_t (host memory).
 * get: *bytes in = capacity, out = size needed; set: bytes must equal L*N*sizeof(edit_ema_t).
 * Both synchronise the device.  Used for checkpoint/resume and to seed tests. */
edit_status_t edit_sync_get_state(edit_sync_t h, void* host_buf, size_t* bytes);
edit_status_t edit_sync_set_state(edit_sync_t h, const void* host_buf, size_t bytes);

/* Phase timing with CUDA events on the stream each unit runs on (bench evidence, off by
 * default).  Phases: 0 = K1 pg_norm, 1 = norm gather + K2 decide, 2 = weighted all-reduce /
 * peer RS (N > 1), 3 = K3 / Dbar-norm gather (N > 1), 4 = K4 outer_update / peer AG+update.
 * collect() blocks until every unit synced since the last collect has completed and returns
 * the per-phase sums (ms) over those syncs; busy_ms (nullable) = per phase, the union of the
 * units' intervals (units on different lanes overlap: the time the phase's kernels were
 * running at all); plus the number of syncs and of elements the K4 launches processed. */
#define EDIT_NUM_PHASES 5
edit_status_t edit_sync_set_profiling(edit_sync_t h, int32_t enable);
edit_status_t edit_sync_profile_collect(edit_sync_t h, double phase_ms[EDIT_NUM_PHASES],
                                        double busy_ms[EDIT_NUM_PHASES], int64_t* syncs, int64_t* elements);

/* NVLink calibration (the roofline denominator of the peer kernels, measured
 * in the run instead of quoted).  Collective over the sync row: every member pulls
 * bytes_per_peer from each of the other N - 1 members' staging buffers at the same time (the
 * AG kernel's access pattern), `reps` times between two mailbox barriers, on lane 0's stream.
 * *gbps = per-direction ingress GB/s of this rank = reps (N - 1) bytes_per_peer / elapsed.
 * Peer path with N > 1 only (EDIT_ERR_INVALID_ARG otherwise); bytes_per_peer is clamped to
 * the staging buffer (the largest unit); blocks until done (call outside timed regions). */
edit_status_t edit_sync_nvlink_probe(edit_sync_t h, int64_t bytes_per_peer, int32_t reps, double* gbps);

/* Number of kernels the library launched so far on this handle (bench evidence). */
int64_t edit_sync_kernel_launches(edit_sync_t h);

/* Frees library-owned resources (NCCL comms, ops, events); never the workspace.  With N > 1
 * it first waits (device mailbox barrier, at most 30 s) until every rank has stopped reading
 * this rank's exported buffers; if that barrier fails or the handle is poisoned, the
 * IPC-exported buffers are leaked rather than freed (a peer may still be reading them) and
 * the communicators are aborted.  Call it explicitly (close()) rather than from a finaliser. */
edit_status_t edit_sync_destroy(edit_sync_t h);

/* ---------------------------------------------------------------------------------------
 * When to sync (host logic only; no device work).
 *   EDIT_TRIGGER_STEPS: EDiT, Alg. 1 l.408 -- the forward of global inner step s = t*tau + p
 *     syncs iff s > t_warm and p == 0 (s % tau == 0).
 *   EDIT_TRIGGER_TIME:  A-EDiT, §3.3 -- after the warm-up, each rank runs whole inner
 *     steps until its own time since its last sync reaches tau_time, then syncs; ranks may
 *     complete different numbers of inner steps; no extra communication (the sync's first
 *     collective is where early ranks wait, at most one step of the slowest rank).
 * sync_now(step, now) is asked at the start of every inner step `step` (a running step count)
 * with the caller's clock in seconds; mark_synced(now) restarts the A-EDiT time base after
 * the sync completed.  in_warmup(step): Alg. 1 l.422 "(t*tau + p) <= t_warm" -- the
 * synchronous mini-batch phase whose gradients are all-reduced over the sync group. */
typedef struct edit_trigger* edit_trigger_t;
#define EDIT_TRIGGER_STEPS 0
#define EDIT_TRIGGER_TIME 1
edit_status_t edit_trigger_create(int32_t kind, int64_t tau_steps, double tau_time_s, int64_t t_warm,
                                  double start_time_s, edit_trigger_t* out);
int32_t edit_trigger_sync_now(edit_trigger_t t, int64_t step, double now_s);
int32_t edit_trigger_in_warmup(edit_trigger_t t, int64_t step);
edit_status_t edit_trigger_mark_synced(edit_trigger_t t, double now_s);
int64_t edit_trigger_syncs(edit_trigger_t t);
edit_status_t edit_trigger_destroy(edit_trigger_t t);

/* Text of the last error on the calling thread ("" if none). */
const char* edit_sync_last_error(void);

/* Library version string. */
const char* edit_sync_version(void);

#ifdef __cplusplus
}
#endif
#endif /* EDIT_SYNC_H_ */
