// Internal declarations shared by api.cpp and kernels.cu (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "edit_sync.h"

namespace edit {

constexpr int kThreads = 256;   // threads per CTA of the streaming kernels
// 8-element vectors per thread.  Grids are NOT persistent: one CTA per kThreads*U vectors
// (measured on B200: a full grid streams at 6.9-7.4 TB/s where a grid-stride persistent
// grid of occupancy x 148 CTAs stalls at 5.3-5.5 TB/s; profiles/r1_k4_variants_microbench.txt).
// {U, I}: a thread handles I steps of U vectors (loads of the U vectors issued together).
constexpr int kReduceShape[2] = {2, 4};  // K1, K3 (read-only streams): 6.8 TB/s incl. the fp64 combine
constexpr int kUpdateShape[2] = {1, 1};  // K4 (3 read + 3 write streams)
constexpr int kVecReduce = kReduceShape[0] * kReduceShape[1];
constexpr int kVecUpdate = kUpdateShape[0] * kUpdateShape[1];
constexpr int kMaxRanks = EDIT_MAX_SYNC * EDIT_MAX_SHARD;

inline int64_t grid_of(int64_t n, int vec_per_thread) {
  const int64_t per_cta = (int64_t)kThreads * vec_per_thread * 8;
  const int64_t g = (n + per_cta - 1) / per_cta;
  return g < 1 ? 1 : g;
}

// Per-unit device scratch: partial sums, gathered scalars, the PreMulSum weight and
// the rollback decision of the unit's last sync.  One per unit so that the scalar
// chains of different units never share a slot.
struct alignas(256) LayerScratch {
  double send1;               // this rank's ||Delta_shard||^2            (K1 output)
  double gsq;                 // N == 1: G^2 of the module (= G_bar^2)    (K2 output)
  double send2;               // this rank's ||Dbar_shard||^2             (K3 output)
  double pad0;
  double recv1[kMaxRanks];    // gathered send1 of all K ranks, index n*M + m
  double recv2[kMaxRanks];    // gathered send2 (M shard ranks; all K ranks on the peer path)
  float w;                    // own Eq. 2 weight: the PreMulSum scalar
  int32_t rollback;           // Alg. 2 l.448
  float w_all[EDIT_MAX_SYNC]; // every replica's Eq. 2 weight (peer-memory reduce-scatter)
  uint32_t counter1;          // last-CTA tickets
  uint32_t counter2;
};

struct DecideArgs {
  const double* parts;        // [M*N] gathered per-rank partial sums of squares
  int32_t M, N, my_n;
  edit_ema_t* ema;            // [N] EMA of this unit
  edit_layer_stats_t* rec;    // outcome record of this unit
  float* w_out;
  float* w_all_out;
  int32_t* rollback_out;
  double* gsq_out;
  double alpha, delta;
  int64_t warmup;
  uint32_t flags;
};

struct UpdateArgs {
  void* local;                // T*
  float* anchor;
  float* momentum;
  const float* dbar;          // N > 1: the all-reduced Dbar shard (nullptr for N == 1)
  int64_t n;
  const double* gparts;       // partial sums of ||Dbar||^2 to combine in order
  int32_t n_gparts;
  const int32_t* rollback;
  float nu, mu;
  double phi, eps;
  uint32_t flags;
  edit_layer_stats_t* rec;
  // NEXT-2 fused write-back -> shard-group all-gather: the updated local is also stored at
  // element offset gather_off of every shard-group member's full-module buffer (gather[q],
  // q < gather_M; peers' buffers are NVLink/IPC mappings).  gather_M == 0: no gather.
  void* gather[EDIT_MAX_SHARD];
  int32_t gather_M;
  int64_t gather_off;
};

// Peer-memory view of a sync row (the N members sharing shard index m): every member's
// staging copy of its local (L) and its slice of Dbar (D), mapped through CUDA IPC.
struct PeerPtrs {
  const void* L[EDIT_MAX_SYNC];
  const float* D[EDIT_MAX_SYNC];
};

// Slicing of a unit's shard for the peer-memory reduce-scatter: nv = ceil(n/8) vectors,
// owner j of vectors [j*slice, min((j+1)*slice, nv)); the last vector may be partial.
struct Slicing {
  int64_t n, nv, slice;
  int32_t N, me;
  int32_t tile;  // vectors per TMA tile (slices are whole tiles)
};
constexpr int kPeerTileVec = 512;  // default vectors (of 8 elements) per TMA tile of the peer kernels
constexpr int kMaxStages = 8;      // shared-memory ring depth cap
constexpr int kMaxPeerCtas = 1024; // persistent grid cap of the peer kernels (per-CTA partial slots)
// slices are whole tiles, so every AG tile has exactly one owner
inline Slicing slicing_of(int64_t n, int N, int me, int tile = kPeerTileVec) {
  Slicing s;
  s.n = n;
  s.nv = (n + 7) / 8;
  const int64_t per = (s.nv + N - 1) / N;
  s.slice = (per + tile - 1) / tile * tile;
  if (s.slice < tile) s.slice = tile;
  s.N = N;
  s.me = me;
  s.tile = tile;
  return s;
}

// Device-side scalar exchange over NVLink (replaces the tiny NCCL all-gathers of the scalar
// chain): every rank's mailbox, mapped in every rank through CUDA IPC (or, in the single-GPU
// simulated mesh of tests/sim, plain device pointers of the other members' mailboxes).
// A message carries up to kMaxGroup fp64 values (one per unit of a group, below).
// Slot layout: box[((phase * 2 + (seq & 1)) * K + src) * kSlotWords + {0: seq, 1 + s: value s}].
// Phases: 0 = module norms (fused into K1), 1 = ||Dbar|| partials (fused into RS),
// 2 = barriers (fused shard all-gather, warm-up all-reduce).
constexpr int kXchgPhases = 3;
constexpr int kMaxGroup = 16;
constexpr int kSlotWords = 1 + kMaxGroup;
struct MailPtrs {
  unsigned long long* box[kMaxRanks];
};
inline size_t mailbox_bytes(int K) { return sizeof(unsigned long long) * kSlotWords * 2 * kXchgPhases * (size_t)K; }

// One exchange of one fp64 per rank: publish to every rank's mailbox, wait for all K.
//  seq:  host-passed sequence number (dseq == nullptr), else the lane's device counter
//        dseq[phase] is advanced by the exchanging CTA (graph-replayable).
//  err:  the handle's sticky device error flag.  A wait longer than timeout_ns (0 = forever)
//        sets it (and *err_host, mapped host memory the library polls at every call); once
//        set, every later exchange of the handle returns at once without publishing, and the
//        unit's data kernels skip all writes (LayerScratch::rollback = kAbort).  So a peer that
//        stops syncing poisons every rank instead of letting them apply stale data.
struct XchgArgs {
  MailPtrs mp;
  int32_t K, me, phase;
  unsigned long long seq;
  unsigned long long* dseq;
  int* err;
  int* err_host;
  unsigned long long timeout_ns;
};
constexpr int32_t kAbort = 2;  // LayerScratch::rollback value: skip the unit entirely

// K1 / RS fold: the kernel's last CTA (the one adding the per-CTA partials) runs the exchange
// of its result (and, for K1, K2 right after) -- one dependent launch fewer per exchange.
//  K1: K == 1 -> K2 on the own partial; K > 1 -> exchange phase 0 into recv1, then K2.
//  RS: exchange phase 1 of send2 into recv2.
struct FoldArgs {
  XchgArgs x;
  DecideArgs dec;
  int32_t on;       // 0: no fold (NCCL scalar gathers), 1: fold
};

int launch_xchg(const XchgArgs& x, const double* src, double* out, int32_t* rollback, cudaStream_t st,
                const DecideArgs* dec = nullptr);

// ---------------------------------------------------------------- unit groups
// Small units (350M / 1B shards: 7-28 M params per rank) are latency-bound when each runs its
// own chain K1 -> RS -> AG with two scalar exchanges.  edit_sync_round therefore syncs runs
// of consecutive small units as a GROUP: one K1, one RS and one AG launch for the whole
// group (each CTA finds its unit in the segment table), and ONE exchange message per phase
// carrying the group's values.  Per-unit semantics are unchanged (module norms, z-tests,
// weights, beta are per unit, from each unit's own scratch; R4).  Peer path only.
struct GroupSeg {
  const void* L[EDIT_MAX_SYNC];   // every member's local of this unit (registered) or staging copy
  const float* D[EDIT_MAX_SYNC];  // every member's D buffer at this unit's offset
  void* local;
  float* anchor;
  float* momentum;
  void* Lcopy;                    // non-registered local: my staging copy at this unit's offset
  float* Dmine;                   // my D buffer at this unit's offset
  int64_t n, slice;               // elements; vectors per owner slice (slicing_of)
  LayerScratch* scr;
  double* parts1;                 // per-CTA partials of K1 / RS
  double* parts2;
  edit_ema_t* ema;                // [N] of this unit
  edit_layer_stats_t* rec;
  int32_t c1, c2, c3;             // first CTA of this unit in the K1 / RS / AG grids
};
struct GroupArgs {
  GroupSeg seg[kMaxGroup];
  int32_t B, M, N, my_n, K;
  int32_t c1_end, c2_end, c3_end;
  XchgArgs x;                     // the exchange of the launching kernel (phase 0: K1, 1: RS)
  double alpha, delta;            // K2
  int64_t warmup;
  float nu, mu;                   // K4
  double phi, eps;
  uint32_t flags;
};
// passed by value as __grid_constant__ kernel parameters (4,496 B; CUDA 12.1+ on sm_70+ allows
// 32,764 B of kernel parameters)
static_assert(sizeof(GroupArgs) <= 32764, "GroupArgs exceeds the kernel parameter limit");
int launch_group_norm(int dtype, const GroupArgs& g, cudaStream_t st);
int launch_group_rs(int dtype, const GroupArgs& g, cudaStream_t st);
int launch_group_ag(int dtype, const GroupArgs& g, cudaStream_t st);
// CTA counts of a unit of n elements in the three group kernels (c1/c2/c3 strides)
inline int64_t group_k1_ctas(int64_t n) { return grid_of(n, kVecReduce); }
constexpr int kGroupAgVec = 1;  // vectors per thread of the group AG
inline int64_t group_ag_ctas(int64_t slice, int N) {
  const int64_t cv = (int64_t)kThreads * kGroupAgVec;
  return (int64_t)N * ((slice + cv - 1) / cv);
}

// Launchers (kernels.cu).  Each returns the number of kernels launched.
// cta_parts: grid_of(n, kVecReduce) fp64 slots for the per-CTA partials.
// cap > 0: at most `cap` CTAs (grid-stride over chunks) -- the co-resident mode next to a
// forward's GEMMs.
int launch_pg_norm(int dtype, const void* local, const float* anchor, float* S, int64_t n,
                   LayerScratch* scr, double* cta_parts, int cap, const FoldArgs& f, cudaStream_t st);
int launch_sumsq(const float* x, int64_t n, LayerScratch* scr, double* cta_parts, int cap, cudaStream_t st);
int launch_decide(const DecideArgs& a, cudaStream_t st);
// K1 variant for the peer-memory path: also copies the local into this rank's staging L.
int launch_pg_norm_copy(int dtype, const void* local, const float* anchor, void* Lcopy, int64_t n,
                        LayerScratch* scr, double* cta_parts, int cap, const FoldArgs& f, cudaStream_t st);
// RS (peer_kernels.cu): Dbar = sum_j w_j (anchor - L_j) over this rank's slice, written to its D;
// ||Dbar_slice||^2 -> scr->send2 (persistent grid <= max_ctas; cta_parts needs that many slots).
// smem_kb > 0: shared-memory ring budget per CTA (tiles shrink to fit; co-resident mode).
// ldg: 0 = the persistent TMA pipeline on <= max_ctas CTAs (smem_kb ring budget); 1 = the
// non-persistent LDG full grid (2: two vectors per thread in AG) -- EDIT_PEER_KERNELS.
int launch_rs(int dtype, const PeerPtrs& pp, const Slicing& sl, const float* anchor, float* Dmine,
              LayerScratch* scr, double* cta_parts, int max_ctas, int smem_kb, int ldg, const FoldArgs& f,
              cudaStream_t st);
// AG + update: Dbar pulled from each slice's owner, then the K4 math on the whole shard.
int launch_ag_update(int dtype, const UpdateArgs& a, const PeerPtrs& pp, const Slicing& sl, int max_ctas,
                     int smem_kb, int ldg, cudaStream_t st);
// Partition mode of the prefetch scheduler (peer_kernels.cu): K1 (no S, no copy) and the
// N == 1 K4 as persistent TMA pipelines on <= max_ctas CTAs, each with the full ~200 KB
// ring (one CTA per SM, no GEMM CTA beside it).
int launch_pg_norm_tma(int dtype, const void* local, const float* anchor, int64_t n, LayerScratch* scr,
                       double* cta_parts, int max_ctas, const FoldArgs& f, cudaStream_t st);
int launch_update_tma(int dtype, const UpdateArgs& a, int max_ctas, cudaStream_t st);
// The LDG reduce-scatter's grid over a slice of `cnt` vectors: one CTA per kThreads x
// kRsLdgIters vectors; its per-CTA partial slots are sized by rs_partial_slots.
constexpr int kRsLdgIters = 4;
inline int64_t rs_ldg_grid(int64_t cnt) {
  const int64_t per = (int64_t)kThreads * kRsLdgIters;
  const int64_t g = (cnt + per - 1) / per;
  return g < 1 ? 1 : g;
}
inline int64_t rs_partial_slots(int64_t n, int N) {
  const int64_t nv = (n + 7) / 8, slice = (nv + N - 1) / N + 4096;  // >= any tile-rounded slice
  const int64_t g = rs_ldg_grid(slice);
  return g > kMaxPeerCtas ? g : kMaxPeerCtas;
}

// Warm-up gradient all-reduce (mean) over the sync row, peer path (peer_kernels.cu).
int launch_warm_rs(int dtype, const PeerPtrs& pp, const Slicing& sl, void* Dmine, const int* err, cudaStream_t st);
int launch_warm_ag(int dtype, const PeerPtrs& pp, const Slicing& sl, void* out, const int* err, cudaStream_t st);
int launch_update(int dtype, const UpdateArgs& a, int cap, cudaStream_t st);
// NVLink calibration: pull bytes_per_peer from every other member's staging buffer (pp.L).
int launch_nvlink_probe(const PeerPtrs& pp, int N, int me, int64_t bytes_per_peer, unsigned* sink, cudaStream_t st);

}  // namespace edit
