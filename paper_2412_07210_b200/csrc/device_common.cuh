// device_common.cuh -- device helpers shared by kernels.cu and peer_kernels.cu:
// 8-element vector IO, deterministic CTA reductions, mbarrier / TMA (cp.async.bulk) wrappers.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "internal.h"

namespace edit {
namespace dev {

// ---------------------------------------------------------------- vector IO
// 8 elements per vector: one 16-byte access of bf16 or two of fp32.
// kEF = stream with an L2 evict_first policy (createpolicy ... L2::evict_first +
// ld/st .L2::cache_hint): the sync's bytes are then the first to leave the 126 MB L2, so a
// concurrent forward keeps its GEMM operand tiles resident (profiles/r1_coresidency_*).
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
template <bool kEF>
__device__ __forceinline__ uint4 ldg16(const void* p, uint64_t pol) {
  uint4 r;
  if (kEF)
    asm volatile("ld.global.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  else
    r = *reinterpret_cast<const uint4*>(p);
  return r;
}
template <bool kEF>
__device__ __forceinline__ void stg16(void* p, uint4 v, uint64_t pol) {
  if (kEF)
    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w), "l"(pol)
                 : "memory");
  else
    *reinterpret_cast<uint4*>(p) = v;
}
template <bool kEF = false>
__device__ __forceinline__ void load8(const float* __restrict__ p, float (&v)[8], uint64_t pol = 0) {
  const uint4 a = ldg16<kEF>(p, pol), b = ldg16<kEF>(p + 4, pol);
  v[0] = __uint_as_float(a.x); v[1] = __uint_as_float(a.y); v[2] = __uint_as_float(a.z); v[3] = __uint_as_float(a.w);
  v[4] = __uint_as_float(b.x); v[5] = __uint_as_float(b.y); v[6] = __uint_as_float(b.z); v[7] = __uint_as_float(b.w);
}
template <bool kEF = false>
__device__ __forceinline__ void load8(const __nv_bfloat16* __restrict__ p, float (&v)[8], uint64_t pol = 0) {
  const uint4 r = ldg16<kEF>(p, pol);
  const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __uint_as_float(w[i] << 16);
    v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
template <bool kEF = false>
__device__ __forceinline__ void store8(float* __restrict__ p, const float (&v)[8], uint64_t pol = 0) {
  stg16<kEF>(p, make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]), __float_as_uint(v[3])),
             pol);
  stg16<kEF>(p + 4,
             make_uint4(__float_as_uint(v[4]), __float_as_uint(v[5]), __float_as_uint(v[6]), __float_as_uint(v[7])),
             pol);
}
template <bool kEF = false>
__device__ __forceinline__ void store8(__nv_bfloat16* __restrict__ p, const float (&v)[8], uint64_t pol = 0) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);  // RNE (R16)
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  stg16<kEF>(p, make_uint4(w[0], w[1], w[2], w[3]), pol);
}
// 4 elements: 16 B (fp32) / 8 B (bf16) per thread, consecutive threads at consecutive
// addresses -- conflict-free shared-memory reads and fully coalesced global stores (the
// partition-mode kernels, where per-SM datapath bandwidth is the limit: tools/sm_stream_bench.cu)
__device__ __forceinline__ void load4(const float* __restrict__ p, float (&v)[4]) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
}
__device__ __forceinline__ void load4(const __nv_bfloat16* __restrict__ p, float (&v)[4]) {
  const uint2 r = *reinterpret_cast<const uint2*>(p);
  v[0] = __uint_as_float(r.x << 16); v[1] = __uint_as_float(r.x & 0xffff0000u);
  v[2] = __uint_as_float(r.y << 16); v[3] = __uint_as_float(r.y & 0xffff0000u);
}
template <bool kEF = false>
__device__ __forceinline__ void store4(float* __restrict__ p, const float (&v)[4], uint64_t pol = 0) {
  stg16<kEF>(p, make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]), __float_as_uint(v[3])),
             pol);
}
template <bool kEF = false>
__device__ __forceinline__ void store4(__nv_bfloat16* __restrict__ p, const float (&v)[4], uint64_t pol = 0) {
  __nv_bfloat162 h0 = __floats2bfloat162_rn(v[0], v[1]), h1 = __floats2bfloat162_rn(v[2], v[3]);  // RNE (R16)
  const uint32_t x = *reinterpret_cast<uint32_t*>(&h0), y = *reinterpret_cast<uint32_t*>(&h1);
  if (kEF)
    asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1,%2}, %3;" ::"l"(p), "r"(x), "r"(y), "l"(pol) : "memory");
  else
    *reinterpret_cast<uint2*>(p) = make_uint2(x, y);
}
__device__ __forceinline__ float load1(const float* p) { return *p; }
__device__ __forceinline__ float load1(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ void store1(float* p, float v) { *p = v; }
__device__ __forceinline__ void store1(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

// NEXT-2: the updated local, also stored into every shard-group member's full-module buffer
// (UpdateArgs::gather; no-op when gather_M == 0).  The element type follows the local's.
// A shard's slot in the full module starts at element m * numel, which is 16-byte aligned
// only when numel is a multiple of 8: otherwise the 8 elements are stored one by one.
template <bool kEF, typename T>
__device__ __forceinline__ void gather_store8_t(const UpdateArgs& p, int64_t k, const float (&v)[8], uint64_t pol) {
  if ((p.gather_off & 7) == 0) {
#pragma unroll
    for (int q = 0; q < EDIT_MAX_SHARD; ++q)
      if (q < p.gather_M) store8<kEF>(static_cast<T*>(p.gather[q]) + p.gather_off + k, v, pol);
  } else {
    for (int q = 0; q < p.gather_M; ++q)
#pragma unroll
      for (int j = 0; j < 8; ++j) store1(static_cast<T*>(p.gather[q]) + p.gather_off + k + j, v[j]);
  }
}
// 4-element variant (slot aligned for a 4-element store iff gather_off % 4 == 0)
template <bool kEF, typename T>
__device__ __forceinline__ void gather_store4_t(const UpdateArgs& p, int64_t k, const float (&v)[4], uint64_t pol) {
  if ((p.gather_off & 3) == 0) {
#pragma unroll
    for (int q = 0; q < EDIT_MAX_SHARD; ++q)
      if (q < p.gather_M) store4<kEF>(static_cast<T*>(p.gather[q]) + p.gather_off + k, v, pol);
  } else {
    for (int q = 0; q < p.gather_M; ++q)
#pragma unroll
      for (int j = 0; j < 4; ++j) store1(static_cast<T*>(p.gather[q]) + p.gather_off + k + j, v[j]);
  }
}
template <typename T>
__device__ __forceinline__ void gather_store1_t(const UpdateArgs& p, int64_t k, float v) {
  for (int q = 0; q < p.gather_M; ++q) store1(static_cast<T*>(p.gather[q]) + p.gather_off + k, v);
}

// ---------------------------------------------------------------- K2 (scalar chain)
// K2 body (one thread): Alg. 2 l.443-451 on the gathered scalars, identically on every rank
// (R6).  Used by decide_kernel and, fused after the exchange, by xchg_kernel (phase 0).
static __device__ __noinline__ void decide_body(const DecideArgs& p) {
  double G[EDIT_MAX_SYNC];
  const int M = p.M, N = p.N;
  edit_layer_stats_t* rec = p.rec;
  for (int n = 0; n < N; ++n) {
    double s = 0.0;
    for (int m = 0; m < M; ++m) s += p.parts[n * M + m];  // module-level norm (R5)
    G[n] = sqrt(s);
  }
  // IsAnomaly (R7-R10) with the pre-update EMA, then Eq. 1 for finite G.
  for (int n = 0; n < N; ++n) {
    edit_ema_t e = p.ema[n];
    double z = nan("");
    bool flagged = !isfinite(G[n]);  // R9: always excluded
    if (!flagged && !(p.flags & EDIT_NO_AE) && e.count >= p.warmup && e.sigma > 0.0) {
      z = (G[n] - e.mu) / e.sigma;
      flagged = z > p.delta;
    }
    rec->z[n] = z;
    rec->anomalous[n] = flagged ? 1 : 0;
    if (flagged) {
      G[n] = INFINITY;  // Alg. 2 l.445; Eq. 1 skipped
    } else {
      const double mu_new = p.alpha * G[n] + (1.0 - p.alpha) * e.mu;
      const double dev = G[n] - mu_new;
      e.sigma = sqrt((1.0 - p.alpha) * e.sigma * e.sigma + p.alpha * dev * dev);
      e.mu = mu_new;
      e.count += 1;
      p.ema[n] = e;
    }
    rec->G[n] = G[n];
    rec->ema_mu[n] = e.mu;
    rec->ema_sigma[n] = e.sigma;
    rec->ema_count[n] = e.count;
  }
  // gamma == 0 <=> no finite G (R11); Eq. 2 with exp(G_min) cancelled.
  int nfinite = 0;
  double gmin = INFINITY;
  for (int n = 0; n < N; ++n)
    if (isfinite(G[n])) {
      ++nfinite;
      gmin = fmin(gmin, G[n]);
    }
  double w[EDIT_MAX_SYNC];
  double gamma = 0.0;
  for (int n = 0; n < N; ++n) {
    if (!isfinite(G[n])) w[n] = 0.0;
    else w[n] = (p.flags & EDIT_NO_WA) ? 1.0 : exp(-(G[n] - gmin));
    gamma += w[n];
  }
  const int rollback = nfinite == 0;
  for (int n = 0; n < N; ++n) {
    w[n] = rollback ? 0.0 : w[n] / gamma;
    rec->w[n] = w[n];
  }
  for (int n = N; n < EDIT_MAX_SYNC; ++n) {
    rec->G[n] = 0.0; rec->z[n] = 0.0; rec->w[n] = 0.0; rec->anomalous[n] = 0;
  }
  rec->num_sync = N;
  *p.w_out = (float)w[p.my_n];
  if (p.w_all_out)
    for (int n = 0; n < EDIT_MAX_SYNC; ++n) p.w_all_out[n] = n < N ? (float)w[n] : 0.f;
  *p.rollback_out = rollback;
  *p.gsq_out = rollback ? 0.0 : G[p.my_n] * G[p.my_n];  // N == 1: G_bar = G
}

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Sum over a CTA of NT threads (result valid in thread 0).  Fixed tree: deterministic.
template <int NT>
__device__ double block_sum_n(double v) {
  __shared__ double ws[NT / 32];
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) ws[warp] = v;
  __syncthreads();
  v = 0.0;
  if (warp == 0) {
    v = lane < (NT / 32) ? ws[lane] : 0.0;
    v = warp_sum(v);
  }
  __syncthreads();
  return v;
}
__device__ __forceinline__ double block_sum(double v) { return block_sum_n<kThreads>(v); }

// Writes this CTA's partial; the last CTA to finish adds all partials in index order
// (fp64) and stores the total in *out, then re-arms the ticket counter.  Returns (in every
// thread of the CTA) whether this CTA was the last one; *out is then visible to the whole CTA.
template <int NT>
__device__ bool finish_partials_n(double cta_total, double* cta_parts, uint32_t* counter, double* out) {
  __shared__ bool is_last;
  if (threadIdx.x == 0) {
    cta_parts[blockIdx.x] = cta_total;
    __threadfence();
    is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!is_last) return false;
  __threadfence();
  // thread t adds partials t, t+NT, t+2NT, ... in that order; 8 loads in flight per step
  const int G = (int)gridDim.x;
  double v = 0.0;
  int i = threadIdx.x;
  for (; i + 7 * NT < G; i += 8 * NT) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __ldcg(cta_parts + i + k * NT);
#pragma unroll
    for (int k = 0; k < 8; ++k) v += x[k];
  }
  for (; i < G; i += NT) v += __ldcg(cta_parts + i);
  v = block_sum_n<NT>(v);
  if (threadIdx.x == 0) {
    *out = v;
    *counter = 0u;
  }
  __syncthreads();
  return true;
}
__device__ __forceinline__ bool finish_partials(double cta_total, double* cta_parts, uint32_t* counter,
                                                double* out) {
  return finish_partials_n<kThreads>(cta_total, cta_parts, counter, out);
}

// ---------------------------------------------------------------- scalar exchange (mailboxes)
// Called by every thread of ONE CTA (>= K threads): threads t < K store the B values
// (*src[0..B-1]) into rank t's mailbox (the values, then the sequence number with
// st.release.sys), then wait for sender t in this rank's own mailbox (ld.acquire.sys) and
// write out[s][t].  Slots alternate by sequence parity: a rank can only write seq+2 into a
// slot after the reader published seq+1, i.e. after it finished reading seq -- no slot is
// overwritten early.  Returns false (in every thread) if the handle already had an error or
// this wait timed out (the error is then set).
struct XchgIO {
  int B;                          // values per message (1, or a group's units)
  const double* src[kMaxGroup];
  double* out[kMaxGroup];         // out[s][t] = sender t's value s
};
static __device__ __noinline__ bool xchg_body_n(const XchgArgs& x, const XchgIO& io) {
  __shared__ unsigned long long s_seq;
  __shared__ int s_ok;
  const int t = threadIdx.x;
  if (t == 0) {
    s_ok = *reinterpret_cast<volatile int*>(x.err) == 0;
    unsigned long long seq = x.seq;
    if (x.dseq) {
      seq = x.dseq[x.phase] + 1;
      x.dseq[x.phase] = seq;
    }
    s_seq = seq;
  }
  __syncthreads();
  if (!s_ok) return false;  // silent after an earlier error of this handle
  const unsigned long long seq = s_seq;
  const int K = x.K, me = x.me, B = io.B;
  const int base = (x.phase * 2 + (int)(seq & 1)) * K;
  if (t < K) {
    unsigned long long* slot = x.mp.box[t] + (size_t)kSlotWords * (base + me);
    for (int s = 0; s < B; ++s) {
      const double v = *io.src[s];
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(slot + 1 + s),
                   "l"((unsigned long long)__double_as_longlong(v))
                   : "memory");
    }
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(slot), "l"(seq) : "memory");
  }
  __syncthreads();  // (all publishes issued before anyone may leave on a timeout)
  if (t < K) {
    unsigned long long* slot = x.mp.box[me] + (size_t)kSlotWords * (base + t);
    unsigned long long s = 0, t0, now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    bool ok = true;
    while (true) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(s) : "l"(slot) : "memory");
      if (s == seq) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (x.timeout_ns && now - t0 > x.timeout_ns) {  // a peer stopped syncing: fatal
        ok = false;
        break;
      }
    }
    if (ok) {
      for (int v = 0; v < B; ++v) {
        unsigned long long vb;
        asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(vb) : "l"(slot + 1 + v) : "memory");
        io.out[v][t] = __longlong_as_double((long long)vb);
      }
    } else {
      atomicExch(x.err, 1);
      if (x.err_host) {
        *reinterpret_cast<volatile int*>(x.err_host) = 1;
        __threadfence_system();
      }
      s_ok = 0;
    }
  }
  __syncthreads();
  return s_ok != 0;
}
// One value per rank.
static __device__ __forceinline__ bool xchg_body(const XchgArgs& x, const double* src, double* out) {
  XchgIO io;
  io.B = 1;
  io.src[0] = src;
  io.out[0] = out;
  return xchg_body_n(x, io);
}

// K1's last CTA (after finish_partials): the phase-0 exchange of the module-norm partials
// (K > 1), then K2 on the gathered values -- what xchg_kernel + decide_kernel do as two
// launches.  An exchange failure leaves the EMA untouched and aborts the unit (kAbort).
static __device__ __forceinline__ void fold_norm_decide(const FoldArgs& f, LayerScratch* scr) {
  bool ok = true;
  if (f.x.K > 1) ok = xchg_body(f.x, &scr->send1, scr->recv1);
  if (threadIdx.x == 0) {
    if (ok) decide_body(f.dec);
    else scr->rollback = kAbort;
  }
}
// RS's last CTA: the phase-1 exchange of the ||Dbar slice||^2 partials (every rank's).
static __device__ __forceinline__ void fold_dbar_norm(const FoldArgs& f, LayerScratch* scr) {
  const bool ok = xchg_body(f.x, &scr->send2, scr->recv2);
  if (!ok && threadIdx.x == 0) scr->rollback = kAbort;
}

// ---------------------------------------------------------------- mbarrier + TMA (sm_90+/sm_100a)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// arrive (count 1) and add `bytes` to the expected transaction count of the current phase
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global (local HBM or an NVLink peer's memory) -> shared, completing on `bar`
template <bool kEF = false>
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar,
                                            uint64_t pol = 0) {
  if (kEF)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(dst_smem)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
  else
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst_smem)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

}  // namespace dev
}  // namespace edit
