// group_kernels.cu -- the peer path's three data kernels for a GROUP of small units
// (internal.h: GroupArgs): one launch per step for the whole group instead of one per unit.
//
//   K1  group_norm_kernel  Delta and ||Delta_shard||^2 of every unit (Alg. 2 l.442-443); the
//                          last CTA of the launch adds each unit's per-CTA partials in CTA
//                          order, exchanges ALL the group's partials in one mailbox message
//                          ("one scalar communication") and runs K2 (l.443-451) for
//                          every unit -- one thread per unit.
//   RS  group_rs_kernel    Dbar = sum_j w_j (anchor - L_j) on this rank's slice of every unit
//                          (Eq. 3, l.452), ||Dbar_slice||^2 per unit, one exchange message.
//   AG  group_ag_kernel    beta (Eq. 4) per unit, then pulls each slice of Dbar from its owner
//                          and applies the Nesterov step + write-back (Eq. 5, l.454-455).
//
// Each CTA finds its unit in the segment table (<= kMaxGroup entries, kernel parameters) and
// runs the same per-element math as the single-unit kernels (kernels.cu K1, peer_kernels.cu
// rs_ldg / ag_update_ldg): full non-persistent grids of 16-B LDG/STG, fp32 per-thread sums,
// fp64 CTA trees, the last CTA adding partials in CTA order -- deterministic for a given
// group.  A unit's slices and its D buffer region are laid out identically on every member
// (offsets from the numel list only), so peers read each other's regions directly.
#include <cuda_bf16.h>
#include <math.h>

#include "device_common.cuh"
#include "internal.h"

namespace edit {
namespace {
using namespace dev;

constexpr int kRedU = kReduceShape[0], kRedI = kReduceShape[1];

// the unit of CTA b: the last segment whose first CTA is <= b (c = c1 / c2 / c3)
template <int C>
__device__ __forceinline__ int seg_of(const GroupArgs& g, int b) {
  int s = 0;
  for (int k = 1; k < g.B; ++k) {
    const int c = C == 1 ? g.seg[k].c1 : (C == 2 ? g.seg[k].c2 : g.seg[k].c3);
    if (c <= b) s = k;
  }
  return s;
}
template <int C>
__device__ __forceinline__ int seg_end(const GroupArgs& g, int s) {
  if (s + 1 < g.B) return C == 1 ? g.seg[s + 1].c1 : (C == 2 ? g.seg[s + 1].c2 : g.seg[s + 1].c3);
  return C == 1 ? g.c1_end : (C == 2 ? g.c2_end : g.c3_end);
}

// The launch's last CTA: unit s's partials [0, cnt_s) added in CTA order (fp64) -> *out_s.
// Returns true in every thread of the last CTA.  The ticket is the first unit's counter.
template <int C>
__device__ bool group_finish(const GroupArgs& g, double cta_total, int s, int bid, bool second) {
  __shared__ bool is_last;
  const GroupSeg& q = g.seg[s];
  uint32_t* ticket = second ? &g.seg[0].scr->counter2 : &g.seg[0].scr->counter1;
  const int total = C == 1 ? g.c1_end : g.c2_end;
  if (threadIdx.x == 0) {
    (second ? q.parts2 : q.parts1)[bid] = cta_total;
    __threadfence();
    is_last = atomicAdd(ticket, 1u) == (uint32_t)total - 1;
  }
  __syncthreads();
  if (!is_last) return false;
  __threadfence();
  for (int k = 0; k < g.B; ++k) {
    const GroupSeg& r = g.seg[k];
    const double* parts = second ? r.parts2 : r.parts1;
    const int cnt = seg_end<C>(g, k) - (C == 1 ? r.c1 : r.c2);
    double v = 0.0;
    for (int i = threadIdx.x; i < cnt; i += kThreads) v += __ldcg(parts + i);
    v = block_sum(v);
    if (threadIdx.x == 0) *(second ? &r.scr->send2 : &r.scr->send1) = v;
  }
  if (threadIdx.x == 0) *ticket = 0u;
  __syncthreads();
  return true;
}

// ---------------------------------------------------------------- K1
template <typename T>
__global__ void __launch_bounds__(kThreads) group_norm_kernel(const __grid_constant__ GroupArgs g) {
  const int s = seg_of<1>(g, blockIdx.x);
  const GroupSeg& q = g.seg[s];
  const int bid = blockIdx.x - q.c1;
  const T* __restrict__ local = static_cast<const T*>(q.local);
  const float* __restrict__ anchor = q.anchor;
  T* __restrict__ Lcopy = static_cast<T*>(q.Lcopy);
  const int64_t n = q.n, n8 = n >> 3;
  float acc = 0.f;
  const int64_t cta0 = (int64_t)bid * kThreads * kRedU * kRedI + threadIdx.x;
#pragma unroll 1
  for (int it = 0; it < kRedI; ++it) {
    const int64_t base = cta0 + (int64_t)it * kThreads * kRedU;
    float l[kRedU][8], a[kRedU][8];
#pragma unroll
    for (int u = 0; u < kRedU; ++u) {
      const int64_t i = base + (int64_t)u * kThreads;
      if (i < n8) {
        load8(local + 8 * i, l[u]);
        load8(anchor + 8 * i, a[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < kRedU; ++u) {
      const int64_t i = base + (int64_t)u * kThreads;
      if (i < n8) {
        if (Lcopy) store8(Lcopy + 8 * i, l[u]);  // exact round trip
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float d = a[u][j] - l[u][j];
          acc = fmaf(d, d, acc);
        }
      }
    }
  }
  double accd = (double)acc;
  if (bid == 0 && threadIdx.x < (n & 7)) {  // ragged tail (< 8 elements)
    const int64_t k = 8 * n8 + threadIdx.x;
    const float lk = load1(local + k);
    const float d = anchor[k] - lk;
    accd += (double)(d * d);
    if (Lcopy) store1(Lcopy + k, lk);
  }
  accd = block_sum(accd);
  if (!group_finish<1>(g, accd, s, bid, false)) return;
  // one message with every unit's module-norm partial, then K2 per unit (R6)
  XchgIO io;
  io.B = g.B;
  for (int k = 0; k < g.B; ++k) {
    io.src[k] = &g.seg[k].scr->send1;
    io.out[k] = g.seg[k].scr->recv1;
  }
  const bool ok = xchg_body_n(g.x, io);
  if (threadIdx.x < g.B) {
    const GroupSeg& r = g.seg[threadIdx.x];
    LayerScratch* scr = r.scr;
    if (!ok) {
      scr->rollback = kAbort;
    } else {
      DecideArgs d;
      d.parts = scr->recv1;
      d.M = g.M;
      d.N = g.N;
      d.my_n = g.my_n;
      d.ema = r.ema;
      d.rec = r.rec;
      d.w_out = &scr->w;
      d.w_all_out = scr->w_all;
      d.rollback_out = &scr->rollback;
      d.gsq_out = &scr->gsq;
      d.alpha = g.alpha;
      d.delta = g.delta;
      d.warmup = g.warmup;
      d.flags = g.flags;
      decide_body(d);
    }
  }
}

// ---------------------------------------------------------------- RS
// NM = the sync-row size rounded up to 2 / 4 / 8 (register arrays sized at compile time)
template <typename T, int NM>
__global__ void __launch_bounds__(kThreads) group_rs_kernel(const __grid_constant__ GroupArgs g) {
  const int s = seg_of<2>(g, blockIdx.x);
  const GroupSeg& q = g.seg[s];
  const int bid = blockIdx.x - q.c2;
  const int N = g.N;
  const LayerScratch* scr = q.scr;
  float w[NM];
#pragma unroll
  for (int j = 0; j < NM; ++j) w[j] = j < N ? scr->w_all[j] : 0.f;
  const bool skip = scr->rollback != 0;  // rollback (l.449) or an aborted unit
  const int64_t n8 = q.n >> 3;
  const int64_t s0 = (int64_t)g.my_n * q.slice;
  const int64_t s1 = min(s0 + q.slice, n8);
  const float* __restrict__ anchor = q.anchor;
  float* __restrict__ Dmine = q.Dmine;
  float acc = 0.f;
  if (!skip) {
#pragma unroll 1
    for (int it = 0; it < kRsLdgIters; ++it) {
      const int64_t v = s0 + ((int64_t)bid * kRsLdgIters + it) * kThreads + threadIdx.x;
      if (v < s1) {
        float a[8], d[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        float l[NM][8];
        load8(anchor + 8 * v, a);
#pragma unroll
        for (int j = 0; j < NM; ++j)
          if (w[j] != 0.f) load8(static_cast<const T*>(q.L[j]) + 8 * v, l[j]);
#pragma unroll
        for (int j = 0; j < NM; ++j)
          if (w[j] != 0.f) {
#pragma unroll
            for (int k = 0; k < 8; ++k) d[k] = fmaf(w[j], a[k] - l[j][k], d[k]);
          }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc = fmaf(d[k], d[k], acc);
        store8(Dmine + 8 * (v - s0), d);
      }
    }
  }
  double accd = (double)acc;
  // the partial last vector (n % 8 elements) belongs to the owner of vector n8
  const int64_t tail = q.n & 7;
  if (!skip && tail && n8 >= s0 && n8 < s0 + q.slice && bid == 0 && threadIdx.x < tail) {
    const int64_t k = 8 * n8 + threadIdx.x;
    const float a = anchor[k];
    float d = 0.f;
    for (int j = 0; j < N; ++j)
      if (w[j] != 0.f) d = fmaf(w[j], a - load1(static_cast<const T*>(q.L[j]) + k), d);
    accd += (double)(d * d);
    Dmine[k - 8 * s0] = d;
  }
  accd = block_sum(accd);
  if (!group_finish<2>(g, accd, s, bid, true)) return;
  // ||Dbar slice||^2 of every unit of the group, one message (also the barrier after which
  // every member's D regions are complete)
  XchgIO io;
  io.B = g.B;
  for (int k = 0; k < g.B; ++k) {
    io.src[k] = &g.seg[k].scr->send2;
    io.out[k] = g.seg[k].scr->recv2;
  }
  const bool ok = xchg_body_n(g.x, io);
  if (!ok && threadIdx.x < g.B) g.seg[threadIdx.x].scr->rollback = kAbort;
}

// ---------------------------------------------------------------- AG + update
template <typename T>
__global__ void __launch_bounds__(kThreads) group_ag_kernel(const __grid_constant__ GroupArgs g) {
  const int s = seg_of<3>(g, blockIdx.x);
  const GroupSeg& q = g.seg[s];
  const int bid = blockIdx.x - q.c3;
  __shared__ float s_beta;
  __shared__ int s_rollback;
  T* __restrict__ local = static_cast<T*>(q.local);
  float* __restrict__ anchor = q.anchor;
  float* __restrict__ mom = q.momentum;
  if (threadIdx.x == 0) {  // Eq. 4 once per CTA (fp64), module level over every rank's slice
    double gsq = 0.0;
    for (int i = 0; i < g.K; ++i) gsq += q.scr->recv2[i];
    const double gbar = sqrt(gsq);
    double beta_d = g.phi / (gbar + g.eps);
    beta_d = beta_d < 1.0 ? beta_d : 1.0;
    if (g.flags & EDIT_NO_GC) beta_d = 1.0;
    const int rb = q.scr->rollback;
    if (bid == 0 && rb != kAbort) {
      q.rec->G_bar = rb ? 0.0 : gbar;
      q.rec->beta = rb ? 1.0 : beta_d;
      q.rec->rollback = rb;
      q.rec->round += 1;
    }
    s_beta = (float)beta_d;
    s_rollback = rb;
  }
  __syncthreads();
  if (s_rollback == kAbort) return;
  const float beta = s_beta, mu = g.mu, nu = g.nu;
  const int64_t n8 = q.n >> 3;
  const int N = g.N;
  const int nb = seg_end<3>(g, s) - q.c3;
  if (s_rollback) {  // Alg. 2 l.449: local = rne(anchor)
    const int64_t stride = (int64_t)nb * kThreads;
    for (int64_t i = (int64_t)bid * kThreads + threadIdx.x; i < n8; i += stride) {
      float a[8];
      load8(anchor + 8 * i, a);
      store8(local + 8 * i, a);
    }
    if (bid == 0 && threadIdx.x < (q.n & 7)) {
      const int64_t k = 8 * n8 + threadIdx.x;
      store1(local + k, anchor[k]);
    }
    return;
  }
  constexpr int U = kGroupAgVec;
  const int64_t cv = (int64_t)kThreads * U;
  // CTAs interleave the owners (consecutive CTAs read different members)
  const int owner = (int)((bid % N + g.my_n) % N);
  const int64_t k = bid / N;
  const int64_t s_lo = (int64_t)owner * q.slice;
  const int64_t v_lo = s_lo + k * cv;
  const int64_t v_hi = min(min(v_lo + cv, s_lo + q.slice), n8);
  const float* __restrict__ D = q.D[owner] - 8 * s_lo;  // indexed by the unit's vector
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
        const float gj = beta * d[u][j];                // Eq. 5
        m[u][j] = fmaf(mu, m[u][j], gj);                // m' = mu m + g
        a[u][j] = a[u][j] - nu * fmaf(mu, m[u][j], gj);  // a' = a - nu (g + mu m')
      }
      store8(mom + 8 * v, m[u]);
      store8(anchor + 8 * v, a[u]);
      store8(local + 8 * v, a[u]);
    }
  }
  if (bid == 0 && threadIdx.x < (q.n & 7)) {  // partial last vector
    const int64_t kk = 8 * n8 + threadIdx.x;
    const int64_t j = n8 / q.slice;
    const float dk = q.D[j][kk - 8 * j * q.slice];
    const float gk = beta * dk;
    const float m1 = fmaf(mu, mom[kk], gk);
    const float a1 = anchor[kk] - nu * fmaf(mu, m1, gk);
    mom[kk] = m1;
    anchor[kk] = a1;
    store1(local + kk, a1);
  }
}

}  // namespace

int launch_group_norm(int dtype, const GroupArgs& g, cudaStream_t st) {
  const unsigned grid = (unsigned)g.c1_end;
  if (dtype == EDIT_BF16) group_norm_kernel<__nv_bfloat16><<<grid, kThreads, 0, st>>>(g);
  else group_norm_kernel<float><<<grid, kThreads, 0, st>>>(g);
  return 1;
}

template <typename T>
void group_rs_go(const GroupArgs& g, cudaStream_t st) {
  const unsigned grid = (unsigned)g.c2_end;
  if (g.N <= 2) group_rs_kernel<T, 2><<<grid, kThreads, 0, st>>>(g);
  else if (g.N <= 4) group_rs_kernel<T, 4><<<grid, kThreads, 0, st>>>(g);
  else group_rs_kernel<T, 8><<<grid, kThreads, 0, st>>>(g);
}

int launch_group_rs(int dtype, const GroupArgs& g, cudaStream_t st) {
  if (dtype == EDIT_BF16) group_rs_go<__nv_bfloat16>(g, st);
  else group_rs_go<float>(g, st);
  return 1;
}

int launch_group_ag(int dtype, const GroupArgs& g, cudaStream_t st) {
  const unsigned grid = (unsigned)g.c3_end;
  if (dtype == EDIT_BF16) group_ag_kernel<__nv_bfloat16><<<grid, kThreads, 0, st>>>(g);
  else group_ag_kernel<float><<<grid, kThreads, 0, st>>>(g);
  return 1;
}

}  // namespace edit
