// peer_kernels.cu -- the N > 1 exchange of Eq. 3 (Alg. 2 l.452) as two
// fused compute+communication kernels over NVLink peer memory (CUDA IPC within a node),
// instead of an all-reduce of an fp32 pseudo-gradient buffer:
//
//   RS  (reduce-scatter): member n owns a 1/N slice of the shard; it pulls that slice of
//       every member's staged local (bf16: 2 B/param) and computes
//           Dbar = sum_j w_j (anchor - L_j)             (fixed j order; w_j == 0 skipped, R9)
//       into its D buffer, plus ||Dbar_slice||^2 for the clip (Eq. 4).
//   AG  (all-gather + update): every member pulls each slice of Dbar from its owner (fp32)
//       and applies beta, the Nesterov step and the write-back (Eq. 5, l.454-455) -- the K4
//       math -- on its whole shard.  All members read the same Dbar bits: bitwise-identical
//       anchors along the sync row.
//
// Both are persistent, warp-specialised TMA pipelines: one producer thread streams tiles
// (local HBM and peers alike) with 1-D bulk copies (cp.async.bulk ... complete_tx) into a
// ring of shared-memory stages; 8 consumer warps compute from shared memory (4-element units:
// conflict-free LDS) and store with coalesced STG.  Measured on B200 (profiles/r1_peer_bench_2gpu.txt): 16-32 CTAs of bulk
// copies already pull ~780 GB/s from a peer, where plain LDG needs the whole GPU.
#include <cuda_bf16.h>
#include <math.h>

#include <stdlib.h>

#include <algorithm>

#include "device_common.cuh"
#include "internal.h"

namespace edit {
namespace {
using namespace dev;

#ifndef EDIT_CONSUMER_WARPS
#define EDIT_CONSUMER_WARPS 8
#endif
constexpr int kConsumerWarps = EDIT_CONSUMER_WARPS;
constexpr int kPeerThreads = 32 * (1 + kConsumerWarps);  // warp 0 = producer
constexpr int kSmemBudget = 200 * 1024;

struct RingBars {
  uint64_t full[kMaxStages];
  uint64_t empty[kMaxStages];
};

__device__ __forceinline__ void ring_init(RingBars* b, int K) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < K; ++s) {
      mbar_init(&b->full[s], 1);
      mbar_init(&b->empty[s], kConsumerWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
}

// ------------------------------------------------------------------------------ RS
template <typename T, bool kEF>
__global__ void __launch_bounds__(kPeerThreads) rs_tma_kernel(const __grid_constant__ PeerPtrs pp, Slicing sl,
                                                              const float* __restrict__ anchor,
                                                              float* __restrict__ Dmine,
                                                              LayerScratch* __restrict__ scr,
                                                              double* __restrict__ cta_parts, int K, int V) {
  extern __shared__ __align__(128) char smem[];
  __shared__ RingBars bars;
  const int N = sl.N;
  float w[EDIT_MAX_SYNC];
  int nact = 0;
#pragma unroll
  for (int j = 0; j < EDIT_MAX_SYNC; ++j) {
    w[j] = scr->w_all[j];
    nact += (j < N && w[j] != 0.f) ? 1 : 0;
  }
  const int lbytes = (int)sizeof(T);
  const bool skip = scr->rollback != 0;
  const uint64_t pol = kEF ? l2_evict_first_policy() : 0;
  const int64_t n8 = sl.n >> 3;
  const int64_t s0 = (int64_t)sl.me * sl.slice;                       // first vector of my slice
  const int64_t s1 = min(s0 + sl.slice, n8);                           // end (full vectors only)
  const int64_t ntiles = s1 > s0 ? (s1 - s0 + V - 1) / V : 0;
  // stage layout: [anchor V*8 f32][L_0 V*8 T]...[L_{N-1}]; slots of w_j == 0 stay unused
  const int stage_bytes = V * 8 * (4 + N * lbytes);
  ring_init(&bars, K);
  float acc = 0.f;
  if (!skip) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
      if (lane == 0) {  // producer
        int it = 0;
        for (int64_t q = blockIdx.x; q < ntiles; q += gridDim.x, ++it) {
          const int s = it % K, use = it / K;
          if (use > 0) mbar_wait(&bars.empty[s], (use - 1) & 1);
          const int64_t v0 = s0 + q * V;
          const int nv = (int)min((int64_t)V, s1 - v0);
          char* st = smem + (size_t)s * stage_bytes;
          mbar_arrive_expect_tx(&bars.full[s], (uint32_t)(nv * 8 * (4 + nact * lbytes)));
          tma_load_1d<kEF>(st, anchor + 8 * v0, nv * 32, &bars.full[s], pol);
          for (int j = 0; j < N; ++j) {
            if (w[j] == 0.f) continue;
            tma_load_1d<kEF>(st + V * 32 + j * V * 8 * lbytes, static_cast<const T*>(pp.L[j]) + 8 * v0,
                             (uint32_t)(nv * 8 * lbytes), &bars.full[s], pol);
          }
        }
      }
    } else {  // consumers
      const int t = threadIdx.x - 32;
      int it = 0;
      for (int64_t q = blockIdx.x; q < ntiles; q += gridDim.x, ++it) {
        const int s = it % K, use = it / K;
        mbar_wait(&bars.full[s], use & 1);
        const int64_t v0 = s0 + q * V;
        const int nv = (int)min((int64_t)V, s1 - v0);
        const char* st = smem + (size_t)s * stage_bytes;
        for (int v = t; v < 2 * nv; v += 32 * kConsumerWarps) {  // 4-element units
          float a[4], d[4];
          load4(reinterpret_cast<const float*>(st) + 4 * v, a);
#pragma unroll
          for (int k = 0; k < 4; ++k) d[k] = 0.f;
#pragma unroll
          for (int j = 0; j < EDIT_MAX_SYNC; ++j) {
            if (j >= N || w[j] == 0.f) continue;
            float l[4];
            load4(reinterpret_cast<const T*>(st + V * 32 + j * V * 8 * lbytes) + 4 * v, l);
#pragma unroll
            for (int k = 0; k < 4; ++k) d[k] = fmaf(w[j], a[k] - l[k], d[k]);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) acc = fmaf(d[k], d[k], acc);
          store4<kEF>(Dmine + 8 * (v0 - s0) + 4 * v, d, pol);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.empty[s]);
      }
    }
  }
  double accd = (double)acc;
  // the partial last vector (n % 8 elements) belongs to the owner of vector n8
  const int64_t tail = sl.n & 7;
  if (!skip && tail && n8 >= s0 && n8 < s0 + sl.slice && blockIdx.x == 0 && threadIdx.x >= 32 &&
      threadIdx.x < 32 + tail) {
    const int64_t k = 8 * n8 + (threadIdx.x - 32);
    const float a = anchor[k];
    float d = 0.f;
    for (int j = 0; j < N; ++j)
      if (w[j] != 0.f) d = fmaf(w[j], a - load1(static_cast<const T*>(pp.L[j]) + k), d);
    accd += (double)(d * d);
    Dmine[k - 8 * s0] = d;
  }
  accd = block_sum_n<kPeerThreads>(accd);
  finish_partials_n<kPeerThreads>(accd, cta_parts, &scr->counter2, &scr->send2);
}

// ------------------------------------------------------------------------------ AG + update
template <typename T, bool kEF, bool kG>
__global__ void __launch_bounds__(kPeerThreads) ag_update_tma_kernel(UpdateArgs p,
                                                                     const __grid_constant__ PeerPtrs pp,
                                                                     Slicing sl, int K, int V) {
  extern __shared__ __align__(128) char smem[];
  __shared__ RingBars bars;
  __shared__ float s_beta;
  __shared__ int s_rollback;
  T* __restrict__ local = static_cast<T*>(p.local);
  float* __restrict__ anchor = p.anchor;
  float* __restrict__ mom = p.momentum;
  if (threadIdx.x == 0) {  // Eq. 4 once per CTA (fp64)
    double gsq = 0.0;
    for (int i = 0; i < p.n_gparts; ++i) gsq += p.gparts[i];  // every slice of every shard, rank order
    const double gbar = sqrt(gsq);
    double beta_d = p.phi / (gbar + p.eps);
    beta_d = beta_d < 1.0 ? beta_d : 1.0;
    if (p.flags & EDIT_NO_GC) beta_d = 1.0;
    const int rb = *p.rollback;
    if (blockIdx.x == 0) {
      p.rec->G_bar = rb ? 0.0 : gbar;
      p.rec->beta = rb ? 1.0 : beta_d;
      p.rec->rollback = rb;
      p.rec->round += 1;
    }
    s_beta = (float)beta_d;
    s_rollback = rb;
  }
  ring_init(&bars, K);  // (contains __syncthreads)
  const float beta = s_beta, mu = p.mu, nu = p.nu;
  const uint64_t pol = kEF ? l2_evict_first_policy() : 0;
  const int64_t n8 = p.n >> 3;
  const int N = sl.N;
  const int64_t tps = sl.slice / V;                      // tiles per slice (slices are tile-aligned)
  const int64_t nq = (int64_t)N * tps;                   // owner-interleaved tile sequence
  const int stage_bytes = V * 8 * 12;                    // Dbar | anchor | momentum, fp32
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // q -> (owner o = (q + me) mod N, k = q / N): at any moment a member's CTAs read from all
  // N owners at once, and each owner serves all readers evenly.
  auto tile_of = [&](int64_t q, int64_t& v0, int& nv, int& owner) {
    owner = (int)((q + sl.me) % N);
    v0 = owner * sl.slice + (q / N) * V;
    nv = (int)max((int64_t)0, min((int64_t)V, n8 - v0));
  };
  if (s_rollback) {  // Alg. 2 l.449: local = rne(anchor), plain LDG/STG
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride) {
      float a[8];
      load8<kEF>(anchor + 8 * i, a, pol);
      store8<kEF>(local + 8 * i, a, pol);
      if (kG) gather_store8_t<kEF, T>(p, 8 * i, a, pol);
    }
    if (blockIdx.x == 0 && threadIdx.x < (p.n & 7)) {
      const int64_t k = 8 * n8 + threadIdx.x;
      store1(local + k, anchor[k]);
      if (kG) gather_store1_t<T>(p, k, anchor[k]);
    }
    return;
  }
  if (warp == 0) {
    if (lane == 0) {  // producer
      int it = 0;
      for (int64_t q = blockIdx.x; q < nq; q += gridDim.x) {
        int64_t v0;
        int nv, owner;
        tile_of(q, v0, nv, owner);
        if (nv <= 0) continue;
        const int s = it % K, use = it / K;
        if (use > 0) mbar_wait(&bars.empty[s], (use - 1) & 1);
        char* st = smem + (size_t)s * stage_bytes;
        mbar_arrive_expect_tx(&bars.full[s], (uint32_t)(nv * 96));
        tma_load_1d<kEF>(st, pp.D[owner] + 8 * (v0 - owner * sl.slice), nv * 32, &bars.full[s], pol);
        tma_load_1d<kEF>(st + V * 32, anchor + 8 * v0, nv * 32, &bars.full[s], pol);
        tma_load_1d<kEF>(st + V * 64, mom + 8 * v0, nv * 32, &bars.full[s], pol);
        ++it;
      }
    }
  } else {  // consumers
    const int t = threadIdx.x - 32;
    int it = 0;
    for (int64_t q = blockIdx.x; q < nq; q += gridDim.x) {
      int64_t v0;
      int nv, owner;
      tile_of(q, v0, nv, owner);
      if (nv <= 0) continue;
      const int s = it % K, use = it / K;
      mbar_wait(&bars.full[s], use & 1);
      const float* st = reinterpret_cast<const float*>(smem + (size_t)s * stage_bytes);
      // 4-element units, consecutive threads on consecutive 16 B: conflict-free shared-memory
      // reads, fully coalesced stores (tools/sm_stream_bench.cu)
      const int n4 = 2 * nv;
      for (int v = t; v < n4; v += 32 * kConsumerWarps) {
        float d[4], a[4], m[4];
        load4(st + 4 * v, d);
        load4(st + V * 8 + 4 * v, a);
        load4(st + V * 16 + 4 * v, m);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float g = beta * d[k];                // Eq. 5
          m[k] = fmaf(mu, m[k], g);                   // m' = mu m + g
          a[k] = a[k] - nu * fmaf(mu, m[k], g);       // a' = a - nu (g + mu m')
        }
        const int64_t i = 8 * v0 + 4 * v;             // first element of the unit
        store4<kEF>(mom + i, m, pol);
        store4<kEF>(anchor + i, a, pol);
        store4<kEF>(local + i, a, pol);
        if (kG) gather_store4_t<kEF, T>(p, i, a, pol);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.empty[s]);
      ++it;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x >= 32 && threadIdx.x < 32 + (p.n & 7)) {  // partial last vector
    const int64_t k = 8 * n8 + (threadIdx.x - 32);
    const int64_t j = n8 / sl.slice;
    const float dk = pp.D[j][k - 8 * j * sl.slice];
    const float g = beta * dk;
    const float m1 = fmaf(mu, mom[k], g);
    const float a1 = anchor[k] - nu * fmaf(mu, m1, g);
    mom[k] = m1;
    anchor[k] = a1;
    store1(local + k, a1);
    if (kG) gather_store1_t<T>(p, k, a1);
  }
}

// ------------------------------------------------------------------------------ partition mode
// The prefetch scheduler's partition mode (a8): while a forward runs on the compute
// stream, a unit's K1 and (N == 1) K4 run as persistent TMA pipelines on a FEW CTAs, each
// holding the whole ~200 KB ring -- so no GEMM CTA (213 KB) can share its SM and the forward
// keeps the other SMs undisturbed.  Per-SM bandwidth comes from the bulk-copy ring depth
// rather than from thread count.  Same math and reduction structure as kernels.cu's K1/K4
// (fixed tile -> CTA map for a given grid, fp32 per-thread sums, fp64 CTA tree, partials
// added in CTA order by the last CTA): deterministic for a given grid.

// K1 (Alg. 2 l.442-443): partial ||anchor - local||^2 of the shard -> scr->send1.
template <typename T>
__global__ void __launch_bounds__(kPeerThreads) pg_norm_tma_kernel(const T* __restrict__ local,
                                                                   const float* __restrict__ anchor, int64_t n,
                                                                   LayerScratch* __restrict__ scr,
                                                                   double* __restrict__ cta_parts, int K, int V) {
  extern __shared__ __align__(128) char smem[];
  __shared__ RingBars bars;
  const int lbytes = (int)sizeof(T);
  const int64_t n8 = n >> 3;
  const int64_t ntiles = (n8 + V - 1) / V;
  const int stage_bytes = V * 8 * (4 + lbytes);  // [anchor V*8 f32][local V*8 T]
  ring_init(&bars, K);
  float acc = 0.f;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {  // producer
      int it = 0;
      for (int64_t q = blockIdx.x; q < ntiles; q += gridDim.x, ++it) {
        const int s = it % K, use = it / K;
        if (use > 0) mbar_wait(&bars.empty[s], (use - 1) & 1);
        const int64_t v0 = q * V;
        const int nv = (int)min((int64_t)V, n8 - v0);
        char* st = smem + (size_t)s * stage_bytes;
        mbar_arrive_expect_tx(&bars.full[s], (uint32_t)(nv * 8 * (4 + lbytes)));
        tma_load_1d(st, anchor + 8 * v0, nv * 32, &bars.full[s]);
        tma_load_1d(st + V * 32, local + 8 * v0, (uint32_t)(nv * 8 * lbytes), &bars.full[s]);
      }
    }
  } else {  // consumers
    const int t = threadIdx.x - 32;
    int it = 0;
    for (int64_t q = blockIdx.x; q < ntiles; q += gridDim.x, ++it) {
      const int s = it % K, use = it / K;
      mbar_wait(&bars.full[s], use & 1);
      const int n4 = 2 * (int)min((int64_t)V, n8 - q * V);  // 4-element units of the tile
      const char* st = smem + (size_t)s * stage_bytes;
      for (int v = t; v < n4; v += 32 * kConsumerWarps) {
        float a[4], l[4];
        load4(reinterpret_cast<const float*>(st) + 4 * v, a);
        load4(reinterpret_cast<const T*>(st + V * 32) + 4 * v, l);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float d = a[k] - l[k];
          acc = fmaf(d, d, acc);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.empty[s]);
    }
  }
  double accd = (double)acc;
  if (blockIdx.x == 0 && threadIdx.x >= 32 && threadIdx.x < 32 + (n & 7)) {  // ragged tail
    const int64_t k = 8 * n8 + (threadIdx.x - 32);
    const float d = anchor[k] - load1(local + k);
    accd += (double)(d * d);
  }
  accd = block_sum_n<kPeerThreads>(accd);
  finish_partials_n<kPeerThreads>(accd, cta_parts, &scr->counter1, &scr->send1);
}

// K4 at N == 1 (Eq. 4-5, Alg. 2 l.449, l.454-455): Dbar = Delta = anchor - local, beta from
// the module norm; m = mu m + beta Dbar; a = a - nu (beta Dbar + mu m); local = rne(a).
// Tiles are walked from the unit's end (K1 streamed it forward: its tail is still in L2).
template <typename T>
__global__ void __launch_bounds__(kPeerThreads) update_tma_kernel(UpdateArgs p, int K, int V) {
  extern __shared__ __align__(128) char smem[];
  __shared__ RingBars bars;
  __shared__ float s_beta;
  __shared__ int s_rollback;
  T* __restrict__ local = static_cast<T*>(p.local);
  float* __restrict__ anchor = p.anchor;
  float* __restrict__ mom = p.momentum;
  if (threadIdx.x == 0) {  // Eq. 4 once per CTA (fp64)
    double gsq = 0.0;
    for (int i = 0; i < p.n_gparts; ++i) gsq += p.gparts[i];
    const double gbar = sqrt(gsq);
    double beta_d = p.phi / (gbar + p.eps);
    beta_d = beta_d < 1.0 ? beta_d : 1.0;
    if (p.flags & EDIT_NO_GC) beta_d = 1.0;
    const int rb = *p.rollback;
    if (blockIdx.x == 0) {
      p.rec->G_bar = rb ? 0.0 : gbar;
      p.rec->beta = rb ? 1.0 : beta_d;
      p.rec->rollback = rb;
      p.rec->round += 1;
    }
    s_beta = (float)beta_d;
    s_rollback = rb;
  }
  ring_init(&bars, K);  // (contains __syncthreads)
  const float beta = s_beta, mu = p.mu, nu = p.nu;
  const int lbytes = (int)sizeof(T);
  const int64_t n8 = p.n >> 3;
  const int64_t ntiles = (n8 + V - 1) / V;
  const int stage_bytes = V * 8 * (8 + lbytes);  // [anchor V*8 f32][mom V*8 f32][local V*8 T]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (s_rollback) {  // Alg. 2 l.449: local = rne(anchor) (R14)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride) {
      float a[8];
      load8(anchor + 8 * i, a);
      store8(local + 8 * i, a);
    }
    if (blockIdx.x == 0 && threadIdx.x < (p.n & 7)) store1(local + 8 * n8 + threadIdx.x, anchor[8 * n8 + threadIdx.x]);
    return;
  }
  if (warp == 0) {
    if (lane == 0) {  // producer
      int it = 0;
      for (int64_t q = blockIdx.x; q < ntiles; q += gridDim.x, ++it) {
        const int s = it % K, use = it / K;
        if (use > 0) mbar_wait(&bars.empty[s], (use - 1) & 1);
        const int64_t v0 = (ntiles - 1 - q) * V;
        const int nv = (int)min((int64_t)V, n8 - v0);
        char* st = smem + (size_t)s * stage_bytes;
        mbar_arrive_expect_tx(&bars.full[s], (uint32_t)(nv * 8 * (8 + lbytes)));
        tma_load_1d(st, anchor + 8 * v0, nv * 32, &bars.full[s]);
        tma_load_1d(st + V * 32, mom + 8 * v0, nv * 32, &bars.full[s]);
        tma_load_1d(st + V * 64, local + 8 * v0, (uint32_t)(nv * 8 * lbytes), &bars.full[s]);
      }
    }
  } else {  // consumers
    const int t = threadIdx.x - 32;
    int it = 0;
    for (int64_t q = blockIdx.x; q < ntiles; q += gridDim.x, ++it) {
      const int s = it % K, use = it / K;
      mbar_wait(&bars.full[s], use & 1);
      const int64_t v0 = (ntiles - 1 - q) * V;
      const int n4 = 2 * (int)min((int64_t)V, n8 - v0);  // 4-element units of the tile
      const char* st = smem + (size_t)s * stage_bytes;
      for (int v = t; v < n4; v += 32 * kConsumerWarps) {
        float a[4], m[4], l[4];
        load4(reinterpret_cast<const float*>(st) + 4 * v, a);
        load4(reinterpret_cast<const float*>(st + V * 32) + 4 * v, m);
        load4(reinterpret_cast<const T*>(st + V * 64) + 4 * v, l);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float g = beta * (a[k] - l[k]);     // Eq. 5, Dbar = Delta at N == 1
          m[k] = fmaf(mu, m[k], g);                 // m' = mu m + g
          a[k] = a[k] - nu * fmaf(mu, m[k], g);     // a' = a - nu (g + mu m')
        }
        const int64_t i = 8 * v0 + 4 * v;           // first element of the unit
        store4(mom + i, m);
        store4(anchor + i, a);
        store4(local + i, a);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.empty[s]);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x >= 32 && threadIdx.x < 32 + (p.n & 7)) {  // ragged tail
    const int64_t k = 8 * n8 + (threadIdx.x - 32);
    const float g = beta * (anchor[k] - load1(local + k));
    const float m1 = fmaf(mu, mom[k], g);
    const float a1 = anchor[k] - nu * fmaf(mu, m1, g);
    mom[k] = m1;
    anchor[k] = a1;
    store1(local + k, a1);
  }
}

// ------------------------------------------------------------------------------ warm-up
// Alg. 1 l.422-424: during the warm-up the sync group all-reduces the gradients
// (mean, R-warm).  Same two-kernel shape as the sync's exchange, with uniform weights and no
// anchor: member n averages its 1/N slice straight from every member's staged gradient
// (fixed member order), then every member pulls each averaged slice from its owner.
// Full-grid LDG (the gradient is consumed right after; plain loads reach ~780 GB/s from a
// peer with the whole GPU, profiles/r1_peer_bench_2gpu.txt).
template <typename T>
__global__ void __launch_bounds__(kThreads) warm_rs_kernel(const __grid_constant__ PeerPtrs pp, Slicing sl,
                                                           T* __restrict__ Dmine) {
  // the owner averages its slice in fp32 (fixed member order) and rounds ONCE to the
  // gradient type, so the pull below moves b_l bytes per element and every member ends
  // with the owner's bits
  const int64_t s0 = (int64_t)sl.me * sl.slice;
  const int64_t n8 = sl.n >> 3;
  const int64_t s1 = min(s0 + sl.slice, n8);
  const int64_t i = s0 + (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const float inv = 1.f / (float)sl.N;
  if (i < s1) {
    float g[EDIT_MAX_SYNC][8];
#pragma unroll
    for (int j = 0; j < EDIT_MAX_SYNC; ++j)  // all members' loads in flight together
      if (j < sl.N) load8(static_cast<const T*>(pp.L[j]) + 8 * i, g[j]);
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < EDIT_MAX_SYNC; ++j)
      if (j < sl.N) {
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] += g[j][k];
      }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] *= inv;
    store8(Dmine + 8 * (i - s0), acc);
  }
  // the partial last vector (n % 8 elements) belongs to the owner of vector n8
  if ((sl.n & 7) && n8 >= s0 && n8 < s0 + sl.slice && blockIdx.x == 0 && threadIdx.x < (sl.n & 7)) {
    const int64_t k = 8 * n8 + threadIdx.x;
    float acc = 0.f;
    for (int j = 0; j < sl.N; ++j) acc += load1(static_cast<const T*>(pp.L[j]) + k);
    store1(Dmine + (k - 8 * s0), acc * inv);
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) warm_ag_kernel(const __grid_constant__ PeerPtrs pp, Slicing sl,
                                                           T* __restrict__ out) {
  const int64_t n8 = sl.n >> 3;
  const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (i < n8) {  // a pure copy of the owner's rounded mean (16 B per bf16 vector)
    const int64_t j = i / sl.slice;
    const T* src = reinterpret_cast<const T*>(pp.D[j]) + 8 * (i - j * sl.slice);
    if (sizeof(T) == 2) {
      *reinterpret_cast<uint4*>(out + 8 * i) = *reinterpret_cast<const uint4*>(src);
    } else {
      *reinterpret_cast<uint4*>(out + 8 * i) = *reinterpret_cast<const uint4*>(src);
      *reinterpret_cast<uint4*>(out + 8 * i + 4) = *reinterpret_cast<const uint4*>(src + 4);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < (sl.n & 7)) {
    const int64_t k = 8 * n8 + threadIdx.x;
    const int64_t j = n8 / sl.slice;
    out[k] = reinterpret_cast<const T*>(pp.D[j])[k - 8 * j * sl.slice];
  }
}

// ------------------------------------------------------------------------------ scalar exchange
// Publish this rank's scalar into every rank's mailbox (value, then seq with release
// semantics at system scope), then wait for all K senders in its own mailbox (acquire).
// Slots alternate by seq parity: a rank can only write seq+2 into a slot after the reader
// published seq+1, i.e. after it finished reading seq -- no slot is overwritten early.
// with_decide: K2 (decide_body) runs right after the gather in the same 1-CTA kernel (the
// phase-0 exchange feeds it), saving one dependent launch per unit.
// dseq != nullptr: the sequence number is this lane's device counter for the phase, incremented
// here (so a captured CUDA graph can be replayed: every replay takes the next number; only this
// 1-CTA kernel on the lane's stream touches the counter); else the host-passed seq.
__global__ void xchg_kernel(const __grid_constant__ MailPtrs mp, int K, int me, int phase,
                            unsigned long long seq_arg, unsigned long long* dseq, const double* src, double* out,
                            int* err, const __grid_constant__ DecideArgs dec, int with_decide) {
  const int t = threadIdx.x;
  __shared__ unsigned long long s_seq;
  if (dseq) {
    if (t == 0) {
      s_seq = dseq[phase] + 1;
      dseq[phase] = s_seq;
    }
    __syncthreads();
  }
  const unsigned long long seq = dseq ? s_seq : seq_arg;
  const int base = (phase * 2 + (int)(seq & 1)) * K;
  if (t < K) {
    const double v = *src;
    unsigned long long* slot = mp.box[t] + 2 * (base + me);
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(slot), "l"((unsigned long long)__double_as_longlong(v))
                 : "memory");
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(slot + 1), "l"(seq) : "memory");
  }
  if (t < K) {
    unsigned long long* slot = mp.box[me] + 2 * (base + t);
    unsigned long long s = 0, t0, now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(s) : "l"(slot + 1) : "memory");
      if (s == seq) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > 10000000000ull) {  // 10 s: a peer is gone; fail loudly instead of hanging
        atomicExch(err, 1);
        break;
      }
    }
    unsigned long long vb;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(vb) : "l"(slot) : "memory");
    out[t] = __longlong_as_double((long long)vb);
  }
  if (with_decide) {
    __syncthreads();  // out[0..K) written by threads 0..K-1 of this CTA
    if (t == 0) decide_body(dec);
  }
}

int default_smem_budget() {
  static int b = [] {
    const char* e = getenv("EDIT_PEER_SMEM_KB");  // shared-memory ring per CTA (default 200 KB)
    const int v = e ? atoi(e) : 0;
    return v > 0 ? v * 1024 : kSmemBudget;
  }();
  return b;
}

// Kernel tile V (vectors) and ring depth K for a shared-memory budget: the largest V that
// divides the slicing tile and leaves >= 3 stages (V >= 32), K = as many stages as fit (<= 8).
struct Ring {
  int V, K, stage_bytes;
};
Ring ring_for(int tile, int bytes_per_vec, int smem_kb) {
  const int budget = smem_kb > 0 ? smem_kb * 1024 : default_smem_budget();
  int V = tile;
  while (V > 32 && 3 * V * bytes_per_vec > budget) V /= 2;
  Ring r;
  r.V = V;
  r.stage_bytes = V * bytes_per_vec;
  r.K = std::max(2, std::min(kMaxStages, budget / r.stage_bytes));
  return r;
}

template <typename KernelT>
void set_smem(KernelT kernel, int bytes) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

}  // namespace

template <typename T, bool kEF>
void rs_go(unsigned grid, const Ring& r, cudaStream_t st, const PeerPtrs& pp, const Slicing& sl, const float* anchor,
           float* Dmine, LayerScratch* scr, double* cta_parts) {
  set_smem(rs_tma_kernel<T, kEF>, r.K * r.stage_bytes);
  rs_tma_kernel<T, kEF><<<grid, kPeerThreads, r.K * r.stage_bytes, st>>>(pp, sl, anchor, Dmine, scr, cta_parts,
                                                                          r.K, r.V);
}

int launch_rs(int dtype, const PeerPtrs& pp, const Slicing& sl, const float* anchor, float* Dmine,
              LayerScratch* scr, double* cta_parts, int max_ctas, bool ef, int smem_kb, cudaStream_t st) {
  const int esz = dtype == EDIT_BF16 ? 2 : 4;
  const Ring r = ring_for(sl.tile, 8 * (4 + sl.N * esz), smem_kb);
  const int64_t n8 = sl.n >> 3;
  const int64_t s0 = (int64_t)sl.me * sl.slice;
  const int64_t s1 = n8 < s0 + sl.slice ? n8 : s0 + sl.slice;
  const int64_t ntiles = s1 > s0 ? (s1 - s0 + r.V - 1) / r.V : 0;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ntiles, max_ctas));
  if (dtype == EDIT_BF16) {
    if (ef) rs_go<__nv_bfloat16, true>(grid, r, st, pp, sl, anchor, Dmine, scr, cta_parts);
    else rs_go<__nv_bfloat16, false>(grid, r, st, pp, sl, anchor, Dmine, scr, cta_parts);
  } else {
    if (ef) rs_go<float, true>(grid, r, st, pp, sl, anchor, Dmine, scr, cta_parts);
    else rs_go<float, false>(grid, r, st, pp, sl, anchor, Dmine, scr, cta_parts);
  }
  return 1;
}

template <typename T, bool kEF>
void ag_go(unsigned grid, const Ring& r, cudaStream_t st, const UpdateArgs& a, const PeerPtrs& pp, const Slicing& sl) {
  if (a.gather_M > 0) {
    set_smem(ag_update_tma_kernel<T, kEF, true>, r.K * r.stage_bytes);
    ag_update_tma_kernel<T, kEF, true><<<grid, kPeerThreads, r.K * r.stage_bytes, st>>>(a, pp, sl, r.K, r.V);
  } else {
    set_smem(ag_update_tma_kernel<T, kEF, false>, r.K * r.stage_bytes);
    ag_update_tma_kernel<T, kEF, false><<<grid, kPeerThreads, r.K * r.stage_bytes, st>>>(a, pp, sl, r.K, r.V);
  }
}

int launch_ag_update(int dtype, const UpdateArgs& a, const PeerPtrs& pp, const Slicing& sl, int max_ctas,
                     bool ef, int smem_kb, cudaStream_t st) {
  const Ring r = ring_for(sl.tile, 8 * 12, smem_kb);
  const int64_t nq = (int64_t)sl.N * (sl.slice / r.V);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nq, max_ctas));
  if (dtype == EDIT_BF16) {
    if (ef) ag_go<__nv_bfloat16, true>(grid, r, st, a, pp, sl);
    else ag_go<__nv_bfloat16, false>(grid, r, st, a, pp, sl);
  } else {
    if (ef) ag_go<float, true>(grid, r, st, a, pp, sl);
    else ag_go<float, false>(grid, r, st, a, pp, sl);
  }
  return 1;
}

template <typename T>
void pg_norm_tma_go(unsigned grid, const Ring& r, cudaStream_t st, const void* local, const float* anchor, int64_t n,
                    LayerScratch* scr, double* cta_parts) {
  set_smem(pg_norm_tma_kernel<T>, r.K * r.stage_bytes);
  pg_norm_tma_kernel<T><<<grid, kPeerThreads, r.K * r.stage_bytes, st>>>(static_cast<const T*>(local), anchor, n,
                                                                         scr, cta_parts, r.K, r.V);
}

int launch_pg_norm_tma(int dtype, const void* local, const float* anchor, int64_t n, LayerScratch* scr,
                       double* cta_parts, int max_ctas, cudaStream_t st) {
  const int esz = dtype == EDIT_BF16 ? 2 : 4;
  const Ring r = ring_for(2 * kPeerTileVec, 8 * (4 + esz), 0);  // bf16: 1024-vector tiles x 4 stages
  const int64_t ntiles = ((n >> 3) + r.V - 1) / r.V;
  // never more CTAs than the unit's partial slots (grid_of(n, kVecReduce), the full-grid K1's)
  const int64_t g = std::min<int64_t>({ntiles, (int64_t)max_ctas, grid_of(n, kVecReduce)});
  const unsigned grid = (unsigned)std::max<int64_t>(1, g);
  if (dtype == EDIT_BF16) pg_norm_tma_go<__nv_bfloat16>(grid, r, st, local, anchor, n, scr, cta_parts);
  else pg_norm_tma_go<float>(grid, r, st, local, anchor, n, scr, cta_parts);
  return 1;
}

int launch_update_tma(int dtype, const UpdateArgs& a, int max_ctas, cudaStream_t st) {
  const int esz = dtype == EDIT_BF16 ? 2 : 4;
  const Ring r = ring_for(kPeerTileVec, 8 * (8 + esz), 0);
  const int64_t ntiles = ((a.n >> 3) + r.V - 1) / r.V;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ntiles, max_ctas));
  if (dtype == EDIT_BF16) {
    set_smem(update_tma_kernel<__nv_bfloat16>, r.K * r.stage_bytes);
    update_tma_kernel<__nv_bfloat16><<<grid, kPeerThreads, r.K * r.stage_bytes, st>>>(a, r.K, r.V);
  } else {
    set_smem(update_tma_kernel<float>, r.K * r.stage_bytes);
    update_tma_kernel<float><<<grid, kPeerThreads, r.K * r.stage_bytes, st>>>(a, r.K, r.V);
  }
  return 1;
}

int launch_xchg(const MailPtrs& mp, int K, int me, int phase, unsigned long long seq, const double* src,
                double* out, int* err, cudaStream_t st, const DecideArgs* dec, unsigned long long* dseq) {
  DecideArgs d{};
  if (dec) d = *dec;
  xchg_kernel<<<1, 64, 0, st>>>(mp, K, me, phase, seq, dseq, src, out, err, d, dec ? 1 : 0);
  return 1;
}

int launch_warm_rs(int dtype, const PeerPtrs& pp, const Slicing& sl, void* Dmine, cudaStream_t st) {
  const int64_t n8 = sl.n >> 3;
  const int64_t s0 = (int64_t)sl.me * sl.slice;
  const int64_t cnt = std::max<int64_t>(0, std::min(s0 + sl.slice, n8) - s0);
  const unsigned grid = (unsigned)std::max<int64_t>(1, (cnt + kThreads - 1) / kThreads);
  if (dtype == EDIT_BF16)
    warm_rs_kernel<__nv_bfloat16><<<grid, kThreads, 0, st>>>(pp, sl, static_cast<__nv_bfloat16*>(Dmine));
  else
    warm_rs_kernel<float><<<grid, kThreads, 0, st>>>(pp, sl, static_cast<float*>(Dmine));
  return 1;
}

int launch_warm_ag(int dtype, const PeerPtrs& pp, const Slicing& sl, void* out, cudaStream_t st) {
  const unsigned grid = (unsigned)std::max<int64_t>(1, ((sl.n >> 3) + kThreads - 1) / kThreads);
  if (dtype == EDIT_BF16) warm_ag_kernel<__nv_bfloat16><<<grid, kThreads, 0, st>>>(pp, sl, static_cast<__nv_bfloat16*>(out));
  else warm_ag_kernel<float><<<grid, kThreads, 0, st>>>(pp, sl, static_cast<float*>(out));
  return 1;
}

}  // namespace edit
