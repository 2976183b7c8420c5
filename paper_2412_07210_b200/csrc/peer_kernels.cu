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
#include <string.h>

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
template <typename T>
__global__ void __launch_bounds__(kPeerThreads) rs_tma_kernel(const __grid_constant__ PeerPtrs pp, Slicing sl,
                                                              const float* __restrict__ anchor,
                                                              float* __restrict__ Dmine,
                                                              LayerScratch* __restrict__ scr,
                                                              double* __restrict__ cta_parts, int K, int V,
                                                              const __grid_constant__ FoldArgs f) {
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
  const bool skip = scr->rollback != 0;  // rollback (l.449) or an aborted unit
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
          tma_load_1d(st, anchor + 8 * v0, nv * 32, &bars.full[s]);
          for (int j = 0; j < N; ++j) {
            if (w[j] == 0.f) continue;
            tma_load_1d(st + V * 32 + j * V * 8 * lbytes, static_cast<const T*>(pp.L[j]) + 8 * v0,
                        (uint32_t)(nv * 8 * lbytes), &bars.full[s]);
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
          store4(Dmine + 8 * (v0 - s0) + 4 * v, d);
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
  // the last CTA: ||Dbar||^2 partials of every rank (module level, Eq. 4), also the barrier
  // after which every member's D slice is complete
  if (finish_partials_n<kPeerThreads>(accd, cta_parts, &scr->counter2, &scr->send2) && f.on) fold_dbar_norm(f, scr);
}

// RS, LDG variant (EDIT_PEER_KERNELS=ldgall, experimental): a non-persistent full grid over this
// rank's slice, CTA b owning vectors [b T I, (b+1) T I) of it; each thread loads its vector of
// the anchor and of every member's local (16-B LDG, the peers' over NVLink; members with
// w_j == 0 are not read, R9) before any arithmetic.  Same math and fixed member order as the
// TMA kernel; per-CTA partials of ||Dbar||^2 added in CTA order by the last CTA.
// NM = the row size rounded up to 2 / 4 / 8 (register arrays sized at compile time: with the
// EDIT_MAX_SYNC-sized arrays the kernel needed 128 registers, 2 CTAs per SM); P = vectors per
// thread whose loads are issued together.
template <typename T, int I, int NM, int P>
__global__ void __launch_bounds__(kThreads) rs_ldg_kernel(const __grid_constant__ PeerPtrs pp, Slicing sl,
                                                          const float* __restrict__ anchor, float* __restrict__ Dmine,
                                                          LayerScratch* __restrict__ scr,
                                                          double* __restrict__ cta_parts,
                                                          const __grid_constant__ FoldArgs f) {
  const int N = sl.N;
  float w[NM];
#pragma unroll
  for (int j = 0; j < NM; ++j) w[j] = j < N ? scr->w_all[j] : 0.f;
  const bool skip = scr->rollback != 0;  // rollback (l.449) or an aborted unit
  const int64_t n8 = sl.n >> 3;
  const int64_t s0 = (int64_t)sl.me * sl.slice;
  const int64_t s1 = min(s0 + sl.slice, n8);
  float acc = 0.f;
  if (!skip) {
#pragma unroll 1
    for (int it = 0; it < I; it += P) {
      float a[P][8], l[P][NM][8];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int64_t v = s0 + ((int64_t)blockIdx.x * I + it + p) * kThreads + threadIdx.x;
        if (v < s1) {
          load8(anchor + 8 * v, a[p]);
#pragma unroll
          for (int j = 0; j < NM; ++j)
            if (w[j] != 0.f) load8(static_cast<const T*>(pp.L[j]) + 8 * v, l[p][j]);
        }
      }
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int64_t v = s0 + ((int64_t)blockIdx.x * I + it + p) * kThreads + threadIdx.x;
        if (v < s1) {
          float d[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int j = 0; j < NM; ++j)
            if (w[j] != 0.f) {
#pragma unroll
              for (int k = 0; k < 8; ++k) d[k] = fmaf(w[j], a[p][k] - l[p][j][k], d[k]);
            }
#pragma unroll
          for (int k = 0; k < 8; ++k) acc = fmaf(d[k], d[k], acc);
          store8(Dmine + 8 * (v - s0), d);
        }
      }
    }
  }
  double accd = (double)acc;
  // the partial last vector (n % 8 elements) belongs to the owner of vector n8
  const int64_t tail = sl.n & 7;
  if (!skip && tail && n8 >= s0 && n8 < s0 + sl.slice && blockIdx.x == 0 && threadIdx.x < tail) {
    const int64_t k = 8 * n8 + threadIdx.x;
    const float a = anchor[k];
    float d = 0.f;
    for (int j = 0; j < N; ++j)
      if (w[j] != 0.f) d = fmaf(w[j], a - load1(static_cast<const T*>(pp.L[j]) + k), d);
    accd += (double)(d * d);
    Dmine[k - 8 * s0] = d;
  }
  accd = block_sum(accd);
  if (finish_partials(accd, cta_parts, &scr->counter2, &scr->send2) && f.on) fold_dbar_norm(f, scr);
}

// ------------------------------------------------------------------------------ AG + update
template <typename T, bool kG>
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
    if (blockIdx.x == 0 && rb != kAbort) {
      p.rec->G_bar = rb ? 0.0 : gbar;
      p.rec->beta = rb ? 1.0 : beta_d;
      p.rec->rollback = rb;
      p.rec->round += 1;
    }
    s_beta = (float)beta_d;
    s_rollback = rb;
  }
  ring_init(&bars, K);  // (contains __syncthreads)
  if (s_rollback == kAbort) return;  // the unit's exchange failed: no write at all
  const float beta = s_beta, mu = p.mu, nu = p.nu;
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
      load8(anchor + 8 * i, a);
      store8(local + 8 * i, a);
      if (kG) gather_store8_t<false, T>(p, 8 * i, a, 0);
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
        tma_load_1d(st, pp.D[owner] + 8 * (v0 - owner * sl.slice), nv * 32, &bars.full[s]);
        tma_load_1d(st + V * 32, anchor + 8 * v0, nv * 32, &bars.full[s]);
        tma_load_1d(st + V * 64, mom + 8 * v0, nv * 32, &bars.full[s]);
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
        store4(mom + i, m);
        store4(anchor + i, a);
        store4(local + i, a);
        if (kG) gather_store4_t<false, T>(p, i, a, 0);
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

// AG + update, LDG variant (EDIT_AG=ldg): a non-persistent full grid like K4 -- each CTA
// one chunk of kThreads x U vectors inside one owner's slice, Dbar loaded straight from the
// owner (16-B LDG over NVLink, no shared-memory staging), anchor / momentum from local HBM.
// Chunks are dealt owner-interleaved (block b -> owner (b + me) mod N), so the CTAs resident
// at any moment pull from every owner at once.
template <typename T, bool kG, int U>
__global__ void __launch_bounds__(kThreads) ag_update_ldg_kernel(UpdateArgs p, const __grid_constant__ PeerPtrs pp,
                                                                 Slicing sl) {
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
    if (blockIdx.x == 0 && rb != kAbort) {
      p.rec->G_bar = rb ? 0.0 : gbar;
      p.rec->beta = rb ? 1.0 : beta_d;
      p.rec->rollback = rb;
      p.rec->round += 1;
    }
    s_beta = (float)beta_d;
    s_rollback = rb;
  }
  __syncthreads();
  if (s_rollback == kAbort) return;
  const float beta = s_beta, mu = p.mu, nu = p.nu;
  const int64_t n8 = p.n >> 3;
  const int N = sl.N;
  if (s_rollback) {  // Alg. 2 l.449: local = rne(anchor)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride) {
      float a[8];
      load8(anchor + 8 * i, a);
      store8(local + 8 * i, a);
      if (kG) gather_store8_t<false, T>(p, 8 * i, a, 0);
    }
    if (blockIdx.x == 0 && threadIdx.x < (p.n & 7)) {
      const int64_t k = 8 * n8 + threadIdx.x;
      store1(local + k, anchor[k]);
      if (kG) gather_store1_t<T>(p, k, anchor[k]);
    }
    return;
  }
  const int64_t cv = (int64_t)kThreads * U;
  const int64_t cps = (sl.slice + cv - 1) / cv;  // chunks per slice
  const int owner = (int)((blockIdx.x % N + sl.me) % N);
  const int64_t k = blockIdx.x / N;
  const int64_t s_lo = (int64_t)owner * sl.slice;
  const int64_t v_lo = s_lo + k * cv;
  const int64_t v_hi = min(min(v_lo + cv, s_lo + sl.slice), n8);
  const float* __restrict__ D = pp.D[owner] - 8 * s_lo;  // indexed by the global vector
  (void)cps;
  float d[U][8], a[U][8], m[U][8];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t v = v_lo + threadIdx.x + (int64_t)u * kThreads;
    if (v < v_hi) {
      load8(D + 8 * v, d[u]);
      load8(anchor + 8 * v, a[u]);
      load8(mom + 8 * v, m[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t v = v_lo + threadIdx.x + (int64_t)u * kThreads;
    if (v < v_hi) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float g = beta * d[u][j];               // Eq. 5
        m[u][j] = fmaf(mu, m[u][j], g);               // m' = mu m + g
        a[u][j] = a[u][j] - nu * fmaf(mu, m[u][j], g);  // a' = a - nu (g + mu m')
      }
      store8(mom + 8 * v, m[u]);
      store8(anchor + 8 * v, a[u]);
      store8(local + 8 * v, a[u]);
      if (kG) gather_store8_t<false, T>(p, 8 * v, a[u], 0);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < (p.n & 7)) {  // partial last vector
    const int64_t kk = 8 * n8 + threadIdx.x;
    const int64_t j = n8 / sl.slice;
    const float dk = pp.D[j][kk - 8 * j * sl.slice];
    const float g = beta * dk;
    const float m1 = fmaf(mu, mom[kk], g);
    const float a1 = anchor[kk] - nu * fmaf(mu, m1, g);
    mom[kk] = m1;
    anchor[kk] = a1;
    store1(local + kk, a1);
    if (kG) gather_store1_t<T>(p, kk, a1);
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
                                                                   double* __restrict__ cta_parts, int K, int V,
                                                                   const __grid_constant__ FoldArgs f) {
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
  if (finish_partials_n<kPeerThreads>(accd, cta_parts, &scr->counter1, &scr->send1) && f.on) fold_norm_decide(f, scr);
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
    if (blockIdx.x == 0 && rb != kAbort) {
      p.rec->G_bar = rb ? 0.0 : gbar;
      p.rec->beta = rb ? 1.0 : beta_d;
      p.rec->rollback = rb;
      p.rec->round += 1;
    }
    s_beta = (float)beta_d;
    s_rollback = rb;
  }
  ring_init(&bars, K);  // (contains __syncthreads)
  if (s_rollback == kAbort) return;
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
// NM = the row size rounded up to 2 / 4 / 8 (register arrays sized at compile time)
template <typename T, int NM>
__global__ void __launch_bounds__(kThreads) warm_rs_kernel(const __grid_constant__ PeerPtrs pp, Slicing sl,
                                                           T* __restrict__ Dmine, const int* __restrict__ err) {
  if (*err) return;  // the barrier before this kernel failed: peers' staging may be stale
  // the owner averages its slice in fp32 (fixed member order) and rounds ONCE to the
  // gradient type, so the pull below moves b_l bytes per element and every member ends
  // with the owner's bits
  const int64_t s0 = (int64_t)sl.me * sl.slice;
  const int64_t n8 = sl.n >> 3;
  const int64_t s1 = min(s0 + sl.slice, n8);
  const int64_t i = s0 + (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const float inv = 1.f / (float)sl.N;
  if (i < s1) {
    float g[NM][8];
#pragma unroll
    for (int j = 0; j < NM; ++j)  // all members' loads in flight together
      if (j < sl.N) load8(static_cast<const T*>(pp.L[j]) + 8 * i, g[j]);
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < NM; ++j)
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

// A pure copy of each owner's rounded mean.  CTAs interleave the owners (CTA b pulls chunk
// b / N of owner (b % N + me) % N), so every member reads from all N owners at once -- the AG
// kernel's pattern; consecutive CTAs pulling from one owner leave the other links idle.
template <typename T>
__global__ void __launch_bounds__(kThreads) warm_ag_kernel(const __grid_constant__ PeerPtrs pp, Slicing sl,
                                                           T* __restrict__ out, const int* __restrict__ err) {
  if (*err) return;
  const int64_t n8 = sl.n >> 3;
  const int N = sl.N;
  const int owner = (int)((blockIdx.x % N + sl.me) % N);
  const int64_t s_lo = (int64_t)owner * sl.slice;
  const int64_t i = s_lo + (int64_t)(blockIdx.x / N) * kThreads + threadIdx.x;
  if (i < min(s_lo + sl.slice, n8)) {
    const T* src = reinterpret_cast<const T*>(pp.D[owner]) + 8 * (i - s_lo);
    if (sizeof(T) == 2) {
      *reinterpret_cast<uint4*>(out + 8 * i) = *reinterpret_cast<const uint4*>(src);
    } else {
      const uint4 a = *reinterpret_cast<const uint4*>(src), b = *reinterpret_cast<const uint4*>(src + 4);
      *reinterpret_cast<uint4*>(out + 8 * i) = a;
      *reinterpret_cast<uint4*>(out + 8 * i + 4) = b;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < (sl.n & 7)) {
    const int64_t k = 8 * n8 + threadIdx.x;
    const int64_t j = n8 / sl.slice;
    out[k] = reinterpret_cast<const T*>(pp.D[j])[k - 8 * j * sl.slice];
  }
}

// NVLink calibration (edit_sync_nvlink_probe): every member of the sync row pulls `nv`
// 16-B vectors from each other member's staging buffer at once (owner-interleaved CTAs, the
// AG kernel's pattern) -- the per-direction ingress ceiling the peer kernels work against.
// The loaded words are folded into one store per CTA so no load is dead.
__global__ void __launch_bounds__(kThreads) nvlink_probe_kernel(const __grid_constant__ PeerPtrs pp, int N, int me,
                                                                int64_t nv, unsigned* sink) {
  constexpr int U = 4;
  const int peers = N - 1;
  const int owner = (me + 1 + (int)(blockIdx.x % peers)) % N;
  const int64_t v0 = (int64_t)(blockIdx.x / peers) * kThreads * U + threadIdx.x;
  const uint4* src = static_cast<const uint4*>(pp.L[owner]);
  uint4 r[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t v = v0 + (int64_t)u * kThreads;
    r[u] = v < nv ? __ldcg(src + v) : make_uint4(0, 0, 0, 0);
  }
  unsigned x = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) x ^= r[u].x ^ r[u].y ^ r[u].z ^ r[u].w;
  if (x == 0x9e3779b9u) sink[blockIdx.x & 1023] = x;  // practically never taken; keeps the loads
}

// ------------------------------------------------------------------------------ scalar exchange
// One CTA: the mailbox exchange (xchg_body, device_common.cuh) as its own launch -- used for
// the barrier phase (fused shard all-gather, warm-up) and by the NCCL-exchange-free paths that
// have no producing kernel to fold it into.  dec_on: K2 right after the gather.  On failure
// *rollback (if given) := kAbort so the unit's data kernels write nothing.
__global__ void xchg_kernel(const __grid_constant__ XchgArgs x, const double* src, double* out,
                            int32_t* rollback, const __grid_constant__ DecideArgs dec, int dec_on) {
  const bool ok = xchg_body(x, src, out);
  if (threadIdx.x == 0) {
    if (!ok && rollback) *rollback = kAbort;
    if (ok && dec_on) decide_body(dec);
  }
}

}  // namespace

namespace {

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

template <typename T>
void rs_go(unsigned grid, const Ring& r, cudaStream_t st, const PeerPtrs& pp, const Slicing& sl, const float* anchor,
           float* Dmine, LayerScratch* scr, double* cta_parts, const FoldArgs& f) {
  set_smem(rs_tma_kernel<T>, r.K * r.stage_bytes);
  rs_tma_kernel<T><<<grid, kPeerThreads, r.K * r.stage_bytes, st>>>(pp, sl, anchor, Dmine, scr, cta_parts, r.K, r.V, f);
}

template <typename T>
void rs_ldg_go(unsigned grid, cudaStream_t st, const PeerPtrs& pp, const Slicing& sl, const float* anchor,
               float* Dmine, LayerScratch* scr, double* cta_parts, const FoldArgs& f) {
  constexpr int I = kRsLdgIters;
  // EDIT_RS_LDG_P=2: two vectors per thread in flight (experiment knob; measured slower: 7B unit
  // at N = 2 541 vs 600 GB/s NVLink in, profiles/r2_rs_variants_4gpu.txt)
  static const int two = [] {
    const char* e = getenv("EDIT_RS_LDG_P");
    return e && atoi(e) == 2 ? 1 : 0;
  }();
  if (sl.N <= 2) {
    if (two) rs_ldg_kernel<T, I, 2, 2><<<grid, kThreads, 0, st>>>(pp, sl, anchor, Dmine, scr, cta_parts, f);
    else rs_ldg_kernel<T, I, 2, 1><<<grid, kThreads, 0, st>>>(pp, sl, anchor, Dmine, scr, cta_parts, f);
  } else if (sl.N <= 4) {
    if (two) rs_ldg_kernel<T, I, 4, 2><<<grid, kThreads, 0, st>>>(pp, sl, anchor, Dmine, scr, cta_parts, f);
    else rs_ldg_kernel<T, I, 4, 1><<<grid, kThreads, 0, st>>>(pp, sl, anchor, Dmine, scr, cta_parts, f);
  } else {
    rs_ldg_kernel<T, I, 8, 1><<<grid, kThreads, 0, st>>>(pp, sl, anchor, Dmine, scr, cta_parts, f);
  }
}

int launch_rs(int dtype, const PeerPtrs& pp, const Slicing& sl, const float* anchor, float* Dmine,
              LayerScratch* scr, double* cta_parts, int max_ctas, int smem_kb, int ldg, const FoldArgs& f,
              cudaStream_t st) {
  if (ldg & 4) {  // EDIT_PEER_KERNELS=ldgall: the LDG reduce-scatter (measured slower than the
                  // TMA pipeline in full rounds: one vector's loads in flight per thread)
    const int64_t n8 = sl.n >> 3;
    const int64_t s0 = (int64_t)sl.me * sl.slice;
    const int64_t cnt = std::max<int64_t>(0, std::min(s0 + sl.slice, n8) - s0);
    const unsigned grid = (unsigned)rs_ldg_grid(cnt);
    if (dtype == EDIT_BF16) rs_ldg_go<__nv_bfloat16>(grid, st, pp, sl, anchor, Dmine, scr, cta_parts, f);
    else rs_ldg_go<float>(grid, st, pp, sl, anchor, Dmine, scr, cta_parts, f);
    return 1;
  }
  const int esz = dtype == EDIT_BF16 ? 2 : 4;
  const Ring r = ring_for(sl.tile, 8 * (4 + sl.N * esz), smem_kb);
  const int64_t n8 = sl.n >> 3;
  const int64_t s0 = (int64_t)sl.me * sl.slice;
  const int64_t s1 = n8 < s0 + sl.slice ? n8 : s0 + sl.slice;
  const int64_t ntiles = s1 > s0 ? (s1 - s0 + r.V - 1) / r.V : 0;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ntiles, max_ctas));
  if (dtype == EDIT_BF16) rs_go<__nv_bfloat16>(grid, r, st, pp, sl, anchor, Dmine, scr, cta_parts, f);
  else rs_go<float>(grid, r, st, pp, sl, anchor, Dmine, scr, cta_parts, f);
  return 1;
}

template <typename T>
void ag_go(unsigned grid, const Ring& r, cudaStream_t st, const UpdateArgs& a, const PeerPtrs& pp, const Slicing& sl) {
  if (a.gather_M > 0) {
    set_smem(ag_update_tma_kernel<T, true>, r.K * r.stage_bytes);
    ag_update_tma_kernel<T, true><<<grid, kPeerThreads, r.K * r.stage_bytes, st>>>(a, pp, sl, r.K, r.V);
  } else {
    set_smem(ag_update_tma_kernel<T, false>, r.K * r.stage_bytes);
    ag_update_tma_kernel<T, false><<<grid, kPeerThreads, r.K * r.stage_bytes, st>>>(a, pp, sl, r.K, r.V);
  }
}

template <typename T, int U>
void ag_ldg_go(cudaStream_t st, const UpdateArgs& a, const PeerPtrs& pp, const Slicing& sl) {
  const int64_t cv = (int64_t)kThreads * U;
  const int64_t cps = (sl.slice + cv - 1) / cv;
  const unsigned grid = (unsigned)std::max<int64_t>(1, (int64_t)sl.N * cps);
  if (a.gather_M > 0) ag_update_ldg_kernel<T, true, U><<<grid, kThreads, 0, st>>>(a, pp, sl);
  else ag_update_ldg_kernel<T, false, U><<<grid, kThreads, 0, st>>>(a, pp, sl);
}


int launch_ag_update(int dtype, const UpdateArgs& a, const PeerPtrs& pp, const Slicing& sl, int max_ctas,
                     int smem_kb, int ldg, cudaStream_t st) {
  if (ldg) {
    if (dtype == EDIT_BF16) {
      if (ldg & 2) ag_ldg_go<__nv_bfloat16, 2>(st, a, pp, sl);
      else ag_ldg_go<__nv_bfloat16, 1>(st, a, pp, sl);
    } else {
      if (ldg & 2) ag_ldg_go<float, 2>(st, a, pp, sl);
      else ag_ldg_go<float, 1>(st, a, pp, sl);
    }
    return 1;
  }
  const Ring r = ring_for(sl.tile, 8 * 12, smem_kb);
  const int64_t nq = (int64_t)sl.N * (sl.slice / r.V);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nq, max_ctas));
  if (dtype == EDIT_BF16) ag_go<__nv_bfloat16>(grid, r, st, a, pp, sl);
  else ag_go<float>(grid, r, st, a, pp, sl);
  return 1;
}

template <typename T>
void pg_norm_tma_go(unsigned grid, const Ring& r, cudaStream_t st, const void* local, const float* anchor, int64_t n,
                    LayerScratch* scr, double* cta_parts, const FoldArgs& f) {
  set_smem(pg_norm_tma_kernel<T>, r.K * r.stage_bytes);
  pg_norm_tma_kernel<T><<<grid, kPeerThreads, r.K * r.stage_bytes, st>>>(static_cast<const T*>(local), anchor, n,
                                                                         scr, cta_parts, r.K, r.V, f);
}

int launch_pg_norm_tma(int dtype, const void* local, const float* anchor, int64_t n, LayerScratch* scr,
                       double* cta_parts, int max_ctas, const FoldArgs& f, cudaStream_t st) {
  const int esz = dtype == EDIT_BF16 ? 2 : 4;
  const Ring r = ring_for(2 * kPeerTileVec, 8 * (4 + esz), 0);  // bf16: 1024-vector tiles x 4 stages
  const int64_t ntiles = ((n >> 3) + r.V - 1) / r.V;
  // never more CTAs than the unit's partial slots (grid_of(n, kVecReduce), the full-grid K1's)
  const int64_t g = std::min<int64_t>({ntiles, (int64_t)max_ctas, grid_of(n, kVecReduce)});
  const unsigned grid = (unsigned)std::max<int64_t>(1, g);
  if (dtype == EDIT_BF16) pg_norm_tma_go<__nv_bfloat16>(grid, r, st, local, anchor, n, scr, cta_parts, f);
  else pg_norm_tma_go<float>(grid, r, st, local, anchor, n, scr, cta_parts, f);
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

int launch_xchg(const XchgArgs& x, const double* src, double* out, int32_t* rollback, cudaStream_t st,
                const DecideArgs* dec) {
  DecideArgs d{};
  if (dec) d = *dec;
  xchg_kernel<<<1, 64, 0, st>>>(x, src, out, rollback, d, dec ? 1 : 0);
  return 1;
}

int launch_nvlink_probe(const PeerPtrs& pp, int N, int me, int64_t bytes_per_peer, unsigned* sink, cudaStream_t st) {
  const int64_t nv = bytes_per_peer / 16;
  const int64_t per = (int64_t)kThreads * 4;
  const unsigned grid = (unsigned)std::max<int64_t>(1, (N - 1) * ((nv + per - 1) / per));
  nvlink_probe_kernel<<<grid, kThreads, 0, st>>>(pp, N, me, nv, sink);
  return 1;
}

template <typename T>
void warm_rs_go(unsigned grid, cudaStream_t st, const PeerPtrs& pp, const Slicing& sl, T* Dmine, const int* err) {
  if (sl.N <= 2) warm_rs_kernel<T, 2><<<grid, kThreads, 0, st>>>(pp, sl, Dmine, err);
  else if (sl.N <= 4) warm_rs_kernel<T, 4><<<grid, kThreads, 0, st>>>(pp, sl, Dmine, err);
  else warm_rs_kernel<T, 8><<<grid, kThreads, 0, st>>>(pp, sl, Dmine, err);
}

int launch_warm_rs(int dtype, const PeerPtrs& pp, const Slicing& sl, void* Dmine, const int* err, cudaStream_t st) {
  const int64_t n8 = sl.n >> 3;
  const int64_t s0 = (int64_t)sl.me * sl.slice;
  const int64_t cnt = std::max<int64_t>(0, std::min(s0 + sl.slice, n8) - s0);
  const unsigned grid = (unsigned)std::max<int64_t>(1, (cnt + kThreads - 1) / kThreads);
  if (dtype == EDIT_BF16) warm_rs_go<__nv_bfloat16>(grid, st, pp, sl, static_cast<__nv_bfloat16*>(Dmine), err);
  else warm_rs_go<float>(grid, st, pp, sl, static_cast<float*>(Dmine), err);
  return 1;
}

int launch_warm_ag(int dtype, const PeerPtrs& pp, const Slicing& sl, void* out, const int* err, cudaStream_t st) {
  // N owners x ceil(slice / kThreads) chunks (owner-interleaved, see warm_ag_kernel)
  const unsigned grid = (unsigned)std::max<int64_t>(1, (int64_t)sl.N * ((sl.slice + kThreads - 1) / kThreads));
  if (dtype == EDIT_BF16)
    warm_ag_kernel<__nv_bfloat16><<<grid, kThreads, 0, st>>>(pp, sl, static_cast<__nv_bfloat16*>(out), err);
  else warm_ag_kernel<float><<<grid, kThreads, 0, st>>>(pp, sl, static_cast<float*>(out), err);
  return 1;
}

}  // namespace edit
