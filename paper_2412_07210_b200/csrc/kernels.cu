// kernels.cu -- sm_100a kernels of the EDiT layer-wise sync (Alg. 2).
//
// The path is HBM-bound streaming plus reductions (no tensor cores):
//   K1 pg_norm       Delta = anchor - local, sum Delta^2 (Alg.2 l.442-443); N > 1 also
//                    writes Delta (non-finite -> 0, R9) into the fp32 exchange buffer S.
//   K2 decide        one thread: module norms G_n, EMA z-test, Eq. 1, Eq. 2 weights,
//                    rollback test (l.447-451).
//   K3 sumsq         sum Dbar^2 of the all-reduced S (Eq. 4 numerator input).
//   K4 outer_update  beta (Eq. 4) in the prologue; m = mu m + beta Dbar;
//                    a = a - nu (beta Dbar + mu m); local = rne(a) (Eq. 5, l.454-455);
//                    rollback branch local = rne(a) (l.449).  N == 1 recomputes
//                    Dbar = Delta = a - local from the inputs (2-pass sync).
// Every reduction is deterministic: a fixed grid for a given length, fixed per-thread
// element sets (fp32 sum of a thread's 8*U squares), warp-shuffle/CTA trees in fp64, and
// the last CTA adding the per-CTA partials in index order in fp64.
#include <cuda_bf16.h>
#include <math.h>

#include "device_common.cuh"
#include "internal.h"

namespace edit {
namespace {
using namespace dev;

// ---------------------------------------------------------------- K1
// Alg. 2 l.442-443: Delta = anchor - local; partial ||Delta||^2 of this shard.
// Shape: CTA b owns vectors [b*T*U*I, (b+1)*T*U*I); a thread walks I steps of U vectors
// (stride T), issuing the U vectors' loads before any arithmetic.
// kCopy: also store the local unchanged into Lcopy (the peer-memory path's staging buffer).
// f.on: the last CTA also runs the norm exchange (K > 1) and K2 (fold_norm_decide).
template <typename T, bool kWriteS, int U, int I, bool kCopy = false>
__global__ void __launch_bounds__(kThreads) pg_norm_kernel(const T* __restrict__ local,
                                                           const float* __restrict__ anchor,
                                                           float* __restrict__ S, int64_t n,
                                                           LayerScratch* __restrict__ scr,
                                                           double* __restrict__ cta_parts,
                                                           T* __restrict__ Lcopy,
                                                           const __grid_constant__ FoldArgs f) {
  const int64_t n8 = n >> 3;
  const int64_t nchunks = (n8 + kThreads * U * I - 1) / (kThreads * U * I);
  float acc = 0.f;
  // one chunk per CTA with the full grid; grid-stride over chunks when the grid is capped
  // (the scheduler's co-resident mode, 1 CTA per SM)
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
  const int64_t cta0 = c * kThreads * U * I + threadIdx.x;
#pragma unroll 1
  for (int it = 0; it < I; ++it) {
    const int64_t base = cta0 + (int64_t)it * kThreads * U;
    float l[U][8], a[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * kThreads;
      if (i < n8) {
        load8(local + 8 * i, l[u]);
        load8(anchor + 8 * i, a[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * kThreads;
      if (i < n8) {
        if (kCopy) store8(Lcopy + 8 * i, l[u]);  // exact: bf16 -> f32 -> bf16 round-trips
        float d[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          d[j] = a[u][j] - l[u][j];
          acc = fmaf(d[j], d[j], acc);
        }
        if (kWriteS) {
#pragma unroll
          for (int j = 0; j < 8; ++j) d[j] = isfinite(d[j]) ? d[j] : 0.f;  // R9: w = 0 must give 0
          store8(S + 8 * i, d);
        }
      }
    }
  }
  }
  double accd = (double)acc;
  if (blockIdx.x == 0 && threadIdx.x < (n & 7)) {  // ragged tail (< 8 elements)
    const int64_t k = 8 * n8 + threadIdx.x;
    const float lk = load1(local + k);
    const float d = anchor[k] - lk;
    accd += (double)(d * d);
    if (kWriteS) S[k] = isfinite(d) ? d : 0.f;
    if (kCopy) store1(Lcopy + k, lk);
  }
  accd = block_sum(accd);
  if (finish_partials(accd, cta_parts, &scr->counter1, &scr->send1) && f.on) fold_norm_decide(f, scr);
}

// ---------------------------------------------------------------- K3
// Eq. 4: partial ||Dbar||^2 of this shard of the all-reduced pseudo-gradient.
template <int U, int I>
__global__ void __launch_bounds__(kThreads) sumsq_kernel(const float* __restrict__ x, int64_t n,
                                                         LayerScratch* __restrict__ scr,
                                                         double* __restrict__ cta_parts) {
  const int64_t n8 = n >> 3;
  const int64_t nchunks = (n8 + kThreads * U * I - 1) / (kThreads * U * I);
  float acc = 0.f;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
  const int64_t cta0 = c * kThreads * U * I + threadIdx.x;
#pragma unroll 1
  for (int it = 0; it < I; ++it) {
    const int64_t base = cta0 + (int64_t)it * kThreads * U;
    float v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * kThreads;
      if (i < n8) load8(x + 8 * i, v[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * kThreads;
      if (i < n8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) acc = fmaf(v[u][j], v[u][j], acc);
      }
    }
  }
  }
  double accd = (double)acc;
  if (blockIdx.x == 0 && threadIdx.x < (n & 7)) {
    const float t = x[8 * n8 + threadIdx.x];
    accd += (double)(t * t);
  }
  accd = block_sum(accd);
  finish_partials(accd, cta_parts, &scr->counter2, &scr->send2);
}

// ---------------------------------------------------------------- K2
// Alg. 2 l.443-451 on the gathered scalars, identically on every rank (R6): all N
// replicas' norms, z-tests, EMA updates (Eq. 1) and weights (Eq. 2).  One thread:
// N <= 8 scalars, fp64, fixed order.
__global__ void decide_kernel(DecideArgs p) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  decide_body(p);
}

// ---------------------------------------------------------------- K4
// beta (Eq. 4), then OuterOpt = Nesterov (R2) on (anchor, momentum) and the
// write-back local = rne(anchor) (Alg. 2 l.454-455).  Rollback: local = rne(anchor).
template <typename T, bool kFromS, int U, int I, bool kG = false>
__global__ void __launch_bounds__(kThreads) outer_update_kernel(UpdateArgs p) {
  T* __restrict__ local = static_cast<T*>(p.local);
  float* __restrict__ anchor = p.anchor;
  float* __restrict__ mom = p.momentum;
  const float* __restrict__ dbar = p.dbar;
  __shared__ float s_beta;
  __shared__ int s_rollback;
  if (threadIdx.x == 0) {  // Eq. 4 once per CTA (fp64), broadcast through shared memory
    double gsq = 0.0;
    for (int i = 0; i < p.n_gparts; ++i) gsq += p.gparts[i];  // module level, m order
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
  if (s_rollback == kAbort) return;  // the unit's exchange failed: no write at all
  const float beta = s_beta, mu = p.mu, nu = p.nu;
  const int64_t n8 = p.n >> 3;
  const int64_t nchunks = (n8 + kThreads * U * I - 1) / (kThreads * U * I);
  const bool tail = blockIdx.x == 0 && threadIdx.x < (p.n & 7);
  if (s_rollback) {  // Alg. 2 l.449: theta_{t+1,0} = theta_t (R14)
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int64_t cta0 = c * kThreads * U * I + threadIdx.x;
#pragma unroll 1
    for (int it = 0; it < I; ++it)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = cta0 + (int64_t)(it * U + u) * kThreads;
        if (i < n8) {
          float a[8];
          load8(anchor + 8 * i, a);
          store8(local + 8 * i, a);
          if (kG) gather_store8_t<false, T>(p, 8 * i, a, 0);
        }
      }
    }
    if (tail) {
      const int64_t k = 8 * n8 + threadIdx.x;
      store1(local + k, anchor[k]);
      if (kG) gather_store1_t<T>(p, k, anchor[k]);
    }
    return;
  }
  // chunks are walked from the unit's END: the producer pass right before (K1 at N == 1,
  // K3 at N > 1) streamed it forward, so its last ~100 MB are still in the 126 MB L2
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
  const int64_t cta0 = (nchunks - 1 - c) * kThreads * U * I + threadIdx.x;
#pragma unroll 1
  for (int it = 0; it < I; ++it) {
    const int64_t base = cta0 + (int64_t)it * kThreads * U;
    float a[U][8], m[U][8], d[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * kThreads;
      if (i < n8) {
        if (kFromS) {
          load8(dbar + 8 * i, d[u]);
        } else {
          load8(local + 8 * i, d[u]);  // the local; Delta formed below
        }
        load8(anchor + 8 * i, a[u]);
        load8(mom + 8 * i, m[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * kThreads;
      if (i < n8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float dj = kFromS ? d[u][j] : a[u][j] - d[u][j];  // N == 1: Dbar = Delta
          const float g = beta * dj;                    // Eq. 5
          m[u][j] = fmaf(mu, m[u][j], g);               // m' = mu m + g
          a[u][j] = a[u][j] - nu * fmaf(mu, m[u][j], g);  // a' = a - nu (g + mu m')
        }
        store8(mom + 8 * i, m[u]);
        store8(anchor + 8 * i, a[u]);
        store8(local + 8 * i, a[u]);
        if (kG) gather_store8_t<false, T>(p, 8 * i, a[u], 0);
      }
    }
  }
  }
  if (tail) {
    const int64_t k = 8 * n8 + threadIdx.x;
    const float d = kFromS ? dbar[k] : anchor[k] - load1(local + k);
    const float g = beta * d;
    const float m1 = fmaf(mu, mom[k], g);
    const float a1 = anchor[k] - nu * fmaf(mu, m1, g);
    mom[k] = m1;
    anchor[k] = a1;
    store1(local + k, a1);
    if (kG) gather_store1_t<T>(p, k, a1);
  }
}

}  // namespace

// ---------------------------------------------------------------- launchers
// Production shapes (profiles/r1_kbench_shapes.txt, tools/kbench.cu).
constexpr int kRedU = kReduceShape[0], kRedI = kReduceShape[1];
constexpr int kUpdU = kUpdateShape[0], kUpdI = kUpdateShape[1];

template <typename T, bool kWriteS, bool kCopy>
void pg_norm_go(unsigned grid, cudaStream_t st, const void* local, const float* anchor, float* S, int64_t n,
                LayerScratch* scr, double* cta_parts, void* Lcopy, const FoldArgs& f) {
  pg_norm_kernel<T, kWriteS, kRedU, kRedI, kCopy><<<grid, kThreads, 0, st>>>(
      static_cast<const T*>(local), anchor, S, n, scr, cta_parts, static_cast<T*>(Lcopy), f);
}

static unsigned capped(int64_t g, int cap) { return (unsigned)(cap > 0 && g > cap ? cap : g); }

int launch_pg_norm(int dtype, const void* local, const float* anchor, float* S, int64_t n,
                   LayerScratch* scr, double* cta_parts, int cap, const FoldArgs& f, cudaStream_t st) {
  const unsigned grid = capped(grid_of(n, kRedU * kRedI), cap);
  if (dtype == EDIT_BF16) {
    if (S) pg_norm_go<__nv_bfloat16, true, false>(grid, st, local, anchor, S, n, scr, cta_parts, nullptr, f);
    else pg_norm_go<__nv_bfloat16, false, false>(grid, st, local, anchor, S, n, scr, cta_parts, nullptr, f);
  } else {
    if (S) pg_norm_go<float, true, false>(grid, st, local, anchor, S, n, scr, cta_parts, nullptr, f);
    else pg_norm_go<float, false, false>(grid, st, local, anchor, S, n, scr, cta_parts, nullptr, f);
  }
  return 1;
}

int launch_pg_norm_copy(int dtype, const void* local, const float* anchor, void* Lcopy, int64_t n,
                        LayerScratch* scr, double* cta_parts, int cap, const FoldArgs& f, cudaStream_t st) {
  const unsigned grid = capped(grid_of(n, kRedU * kRedI), cap);
  if (dtype == EDIT_BF16) pg_norm_go<__nv_bfloat16, false, true>(grid, st, local, anchor, nullptr, n, scr, cta_parts, Lcopy, f);
  else pg_norm_go<float, false, true>(grid, st, local, anchor, nullptr, n, scr, cta_parts, Lcopy, f);
  return 1;
}

int launch_sumsq(const float* x, int64_t n, LayerScratch* scr, double* cta_parts, int cap, cudaStream_t st) {
  const unsigned grid = capped(grid_of(n, kRedU * kRedI), cap);
  sumsq_kernel<kRedU, kRedI><<<grid, kThreads, 0, st>>>(x, n, scr, cta_parts);
  return 1;
}

int launch_decide(const DecideArgs& a, cudaStream_t st) {
  decide_kernel<<<1, 32, 0, st>>>(a);
  return 1;
}

template <typename T, bool kFromS>
void update_go(unsigned grid, cudaStream_t st, const UpdateArgs& a) {
  if (a.gather_M > 0)  // NEXT-2 stores compiled only into the gathering variant
    outer_update_kernel<T, kFromS, kUpdU, kUpdI, true><<<grid, kThreads, 0, st>>>(a);
  else
    outer_update_kernel<T, kFromS, kUpdU, kUpdI, false><<<grid, kThreads, 0, st>>>(a);
}

int launch_update(int dtype, const UpdateArgs& a, int cap, cudaStream_t st) {
  const unsigned grid = capped(grid_of(a.n, kUpdU * kUpdI), cap);
  if (dtype == EDIT_BF16) {
    if (a.dbar) update_go<__nv_bfloat16, true>(grid, st, a);
    else update_go<__nv_bfloat16, false>(grid, st, a);
  } else {
    if (a.dbar) update_go<float, true>(grid, st, a);
    else update_go<float, false>(grid, st, a);
  }
  return 1;
}

}  // namespace edit
