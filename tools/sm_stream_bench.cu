// tools/sm_stream_bench.cu -- dev microbenchmark (1 GPU): per-SM streaming bandwidth of the
// N == 1 sync passes on a FEW persistent CTAs (the scheduler's partition mode, a8).  How
// many bytes/s can one SM move when the rest of the GPU is left to a forward?
//   K1-like: read local (bf16) + anchor (f32), sum of squares        (6 B/param)
//   K4-like: read local, anchor, mom; write mom, anchor, local        (20 B/param)
// Variants: TMA bulk loads + STG stores (the library's update_tma_kernel), TMA loads + TMA
// bulk STORES from shared memory (cp.async.bulk.global.shared::cta), and plain LDG/STG with
// 1024 threads per CTA.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/sm_stream_bench tools/sm_stream_bench.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

constexpr int CW = 8;                  // consumer warps
constexpr int NT = 32 * (1 + CW);
constexpr int MAXK = 8;

__device__ __forceinline__ void ld8f(const float* p, float (&v)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void st8f(float* p, const float (&v)[8]) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void ld8h(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 r = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __uint_as_float(w[i] << 16);
    v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
__device__ __forceinline__ void st8h(__nv_bfloat16* p, const float (&v)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
}

// K1-like: TMA ring, consumers reduce
__global__ void __launch_bounds__(NT) k1_tma(const __nv_bfloat16* local, const float* anchor, int64_t n8, float* out,
                                             int K, int V) {
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t full[MAXK], empty[MAXK];
  if (threadIdx.x == 0) {
    for (int s = 0; s < K; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], CW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nt = (n8 + V - 1) / V;
  const int sb = V * 48;
  float acc = 0.f;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int64_t q = blockIdx.x; q < nt; q += gridDim.x, ++it) {
        const int s = it % K, use = it / K;
        if (use) mbar_wait(&empty[s], (use - 1) & 1);
        const int64_t v0 = q * V;
        const int nv = (int)min((int64_t)V, n8 - v0);
        char* st = smem + (size_t)s * sb;
        mbar_expect_tx(&full[s], nv * 48);
        tma_load(st, anchor + 8 * v0, nv * 32, &full[s]);
        tma_load(st + V * 32, local + 8 * v0, nv * 16, &full[s]);
      }
    }
  } else {
    const int t = threadIdx.x - 32;
    int it = 0;
    for (int64_t q = blockIdx.x; q < nt; q += gridDim.x, ++it) {
      const int s = it % K, use = it / K;
      mbar_wait(&full[s], use & 1);
      const int nv = (int)min((int64_t)V, n8 - q * V);
      const char* st = smem + (size_t)s * sb;
      for (int v = t; v < nv; v += 32 * CW) {
        float a[8], l[8];
        ld8f(reinterpret_cast<const float*>(st) + 8 * v, a);
        ld8h(reinterpret_cast<const __nv_bfloat16*>(st + V * 32) + 8 * v, l);
#pragma unroll
        for (int k = 0; k < 8; ++k) { const float d = a[k] - l[k]; acc = fmaf(d, d, acc); }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}

// K4-like: TMA loads; kBulkStore: results written in place into the stage, then stored with
// cp.async.bulk (one thread), stage released after the store has READ shared memory
template <bool kBulkStore>
__global__ void __launch_bounds__(NT) k4_tma(__nv_bfloat16* local, float* anchor, float* mom, int64_t n8, int K,
                                             int V) {
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t full[MAXK], empty[MAXK];
  if (threadIdx.x == 0) {
    for (int s = 0; s < K; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kBulkStore ? 1 : CW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const float beta = 0.5f, mu = 0.85f, nu = 0.8f;
  const int64_t nt = (n8 + V - 1) / V;
  const int sb = V * 80;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int64_t q = blockIdx.x; q < nt; q += gridDim.x, ++it) {
        const int s = it % K, use = it / K;
        if (use) mbar_wait(&empty[s], (use - 1) & 1);
        const int64_t v0 = q * V;
        const int nv = (int)min((int64_t)V, n8 - v0);
        char* st = smem + (size_t)s * sb;
        mbar_expect_tx(&full[s], nv * 80);
        tma_load(st, anchor + 8 * v0, nv * 32, &full[s]);
        tma_load(st + V * 32, mom + 8 * v0, nv * 32, &full[s]);
        tma_load(st + V * 64, local + 8 * v0, nv * 16, &full[s]);
      }
    }
  } else {
    const int t = threadIdx.x - 32;
    int it = 0, prev = -1;
    for (int64_t q = blockIdx.x; q < nt; q += gridDim.x, ++it) {
      const int s = it % K, use = it / K;
      mbar_wait(&full[s], use & 1);
      const int64_t v0 = q * V;
      const int nv = (int)min((int64_t)V, n8 - v0);
      char* st = smem + (size_t)s * sb;
      for (int v = t; v < nv; v += 32 * CW) {
        float a[8], m[8], l[8];
        ld8f(reinterpret_cast<const float*>(st) + 8 * v, a);
        ld8f(reinterpret_cast<const float*>(st + V * 32) + 8 * v, m);
        ld8h(reinterpret_cast<const __nv_bfloat16*>(st + V * 64) + 8 * v, l);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float g = beta * (a[k] - l[k]);
          m[k] = fmaf(mu, m[k], g);
          a[k] = a[k] - nu * fmaf(mu, m[k], g);
        }
        if (kBulkStore) {
          st8f(reinterpret_cast<float*>(st) + 8 * v, a);
          st8f(reinterpret_cast<float*>(st + V * 32) + 8 * v, m);
          st8h(reinterpret_cast<__nv_bfloat16*>(st + V * 64) + 8 * v, a);
        } else {
          const int64_t i = v0 + v;
          st8f(mom + 8 * i, m);
          st8f(anchor + 8 * i, a);
          st8h(local + 8 * i, a);
        }
      }
      if (kBulkStore) {
        fence_async_smem();
        named_bar(1, 32 * CW);
        if (t == 0) {
          tma_store(anchor + 8 * v0, st, nv * 32);
          tma_store(mom + 8 * v0, st + V * 32, nv * 32);
          tma_store(local + 8 * v0, st + V * 64, nv * 16);
          bulk_commit();
          bulk_wait_read<1>();  // the previous stage's stores have read their smem
          if (prev >= 0) mbar_arrive(&empty[prev]);
        }
        prev = s;
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    }
    if (kBulkStore && t == 0) bulk_wait_all();
  }
}

// LDG/STG K4 with 1024 threads, U vectors per thread in flight, grid-stride
template <int U>
__global__ void __launch_bounds__(1024) k4_ldg(__nv_bfloat16* local, float* anchor, float* mom, int64_t n8) {
  const float beta = 0.5f, mu = 0.85f, nu = 0.8f;
  const int64_t stride = (int64_t)gridDim.x * 1024 * U;
  for (int64_t base = (int64_t)blockIdx.x * 1024 * U + threadIdx.x; base < n8; base += stride) {
    float a[U][8], m[U][8], l[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * 1024;
      if (i < n8) { ld8f(anchor + 8 * i, a[u]); ld8f(mom + 8 * i, m[u]); ld8h(local + 8 * i, l[u]); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * 1024;
      if (i < n8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float g = beta * (a[u][k] - l[u][k]);
          m[u][k] = fmaf(mu, m[u][k], g);
          a[u][k] = a[u][k] - nu * fmaf(mu, m[u][k], g);
        }
        st8f(mom + 8 * i, m[u]); st8f(anchor + 8 * i, a[u]); st8h(local + 8 * i, a[u]);
      }
    }
  }
}

// ---- 4-element units: thread t of a warp touches 16 B (f32) / 8 B (bf16) at consecutive
// addresses -> conflict-free LDS and fully coalesced LDG/STG
__device__ __forceinline__ void ld4h(const __nv_bfloat16* p, float (&v)[4]) {
  const uint2 r = *reinterpret_cast<const uint2*>(p);
  v[0] = __uint_as_float(r.x << 16); v[1] = __uint_as_float(r.x & 0xffff0000u);
  v[2] = __uint_as_float(r.y << 16); v[3] = __uint_as_float(r.y & 0xffff0000u);
}
__device__ __forceinline__ void st4h(__nv_bfloat16* p, const float (&v)[4]) {
  __nv_bfloat162 h0 = __floats2bfloat162_rn(v[0], v[1]), h1 = __floats2bfloat162_rn(v[2], v[3]);
  *reinterpret_cast<uint2*>(p) = make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
}

template <int CWn>
__global__ void __launch_bounds__(32 * (1 + CWn)) k1_tma4(const __nv_bfloat16* local, const float* anchor, int64_t n8,
                                                         float* out, int K, int V) {
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t full[MAXK], empty[MAXK];
  if (threadIdx.x == 0) {
    for (int s = 0; s < K; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], CWn); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nt = (n8 + V - 1) / V;
  const int sb = V * 48;
  float acc = 0.f;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int64_t q = blockIdx.x; q < nt; q += gridDim.x, ++it) {
        const int s = it % K, use = it / K;
        if (use) mbar_wait(&empty[s], (use - 1) & 1);
        const int64_t v0 = q * V;
        const int nv = (int)min((int64_t)V, n8 - v0);
        char* st = smem + (size_t)s * sb;
        mbar_expect_tx(&full[s], nv * 48);
        tma_load(st, anchor + 8 * v0, nv * 32, &full[s]);
        tma_load(st + V * 32, local + 8 * v0, nv * 16, &full[s]);
      }
    }
  } else {
    const int t = threadIdx.x - 32;
    int it = 0;
    for (int64_t q = blockIdx.x; q < nt; q += gridDim.x, ++it) {
      const int s = it % K, use = it / K;
      mbar_wait(&full[s], use & 1);
      const int n4 = 2 * (int)min((int64_t)V, n8 - q * V);
      const char* st = smem + (size_t)s * sb;
      for (int v = t; v < n4; v += 32 * CWn) {
        const float4 a = reinterpret_cast<const float4*>(st)[v];
        float l[4];
        ld4h(reinterpret_cast<const __nv_bfloat16*>(st + V * 32) + 4 * v, l);
        float d = a.x - l[0]; acc = fmaf(d, d, acc);
        d = a.y - l[1]; acc = fmaf(d, d, acc);
        d = a.z - l[2]; acc = fmaf(d, d, acc);
        d = a.w - l[3]; acc = fmaf(d, d, acc);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}

template <int CWn>
__global__ void __launch_bounds__(32 * (1 + CWn)) k4_tma4(__nv_bfloat16* local, float* anchor, float* mom, int64_t n8,
                                                         int K, int V) {
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t full[MAXK], empty[MAXK];
  if (threadIdx.x == 0) {
    for (int s = 0; s < K; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], CWn); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const float beta = 0.5f, mu = 0.85f, nu = 0.8f;
  const int64_t nt = (n8 + V - 1) / V;
  const int sb = V * 80;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int64_t q = blockIdx.x; q < nt; q += gridDim.x, ++it) {
        const int s = it % K, use = it / K;
        if (use) mbar_wait(&empty[s], (use - 1) & 1);
        const int64_t v0 = q * V;
        const int nv = (int)min((int64_t)V, n8 - v0);
        char* st = smem + (size_t)s * sb;
        mbar_expect_tx(&full[s], nv * 80);
        tma_load(st, anchor + 8 * v0, nv * 32, &full[s]);
        tma_load(st + V * 32, mom + 8 * v0, nv * 32, &full[s]);
        tma_load(st + V * 64, local + 8 * v0, nv * 16, &full[s]);
      }
    }
  } else {
    const int t = threadIdx.x - 32;
    int it = 0;
    for (int64_t q = blockIdx.x; q < nt; q += gridDim.x, ++it) {
      const int s = it % K, use = it / K;
      mbar_wait(&full[s], use & 1);
      const int64_t v0 = q * V;
      const int n4 = 2 * (int)min((int64_t)V, n8 - v0);
      const char* st = smem + (size_t)s * sb;
      for (int v = t; v < n4; v += 32 * CWn) {
        float4 a = reinterpret_cast<const float4*>(st)[v];
        float4 m = reinterpret_cast<const float4*>(st + V * 32)[v];
        float l[4];
        ld4h(reinterpret_cast<const __nv_bfloat16*>(st + V * 64) + 4 * v, l);
        float g;
        g = beta * (a.x - l[0]); m.x = fmaf(mu, m.x, g); a.x = a.x - nu * fmaf(mu, m.x, g);
        g = beta * (a.y - l[1]); m.y = fmaf(mu, m.y, g); a.y = a.y - nu * fmaf(mu, m.y, g);
        g = beta * (a.z - l[2]); m.z = fmaf(mu, m.z, g); a.z = a.z - nu * fmaf(mu, m.z, g);
        g = beta * (a.w - l[3]); m.w = fmaf(mu, m.w, g); a.w = a.w - nu * fmaf(mu, m.w, g);
        const int64_t i = 2 * v0 + v;  // 4-element unit index
        reinterpret_cast<float4*>(mom)[i] = m;
        reinterpret_cast<float4*>(anchor)[i] = a;
        const float o[4] = {a.x, a.y, a.z, a.w};
        st4h(local + 4 * i, o);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
}

template <int U>
__global__ void __launch_bounds__(1024) k4_ldg4(__nv_bfloat16* local, float* anchor, float* mom, int64_t n4) {
  const float beta = 0.5f, mu = 0.85f, nu = 0.8f;
  const int64_t stride = (int64_t)gridDim.x * 1024 * U;
  for (int64_t base = (int64_t)blockIdx.x * 1024 * U + threadIdx.x; base < n4; base += stride) {
    float4 a[U], m[U];
    float l[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * 1024;
      if (i < n4) {
        a[u] = reinterpret_cast<const float4*>(anchor)[i];
        m[u] = reinterpret_cast<const float4*>(mom)[i];
        ld4h(local + 4 * i, l[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * 1024;
      if (i < n4) {
        float g;
        g = beta * (a[u].x - l[u][0]); m[u].x = fmaf(mu, m[u].x, g); a[u].x = a[u].x - nu * fmaf(mu, m[u].x, g);
        g = beta * (a[u].y - l[u][1]); m[u].y = fmaf(mu, m[u].y, g); a[u].y = a[u].y - nu * fmaf(mu, m[u].y, g);
        g = beta * (a[u].z - l[u][2]); m[u].z = fmaf(mu, m[u].z, g); a[u].z = a[u].z - nu * fmaf(mu, m[u].z, g);
        g = beta * (a[u].w - l[u][3]); m[u].w = fmaf(mu, m[u].w, g); a[u].w = a[u].w - nu * fmaf(mu, m[u].w, g);
        reinterpret_cast<float4*>(mom)[i] = m[u];
        reinterpret_cast<float4*>(anchor)[i] = a[u];
        const float o[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
        st4h(local + 4 * i, o);
      }
    }
  }
}

template <int U>
__global__ void __launch_bounds__(1024) k1_ldg4(const __nv_bfloat16* local, const float* anchor, int64_t n4, float* out) {
  const int64_t stride = (int64_t)gridDim.x * 1024 * U;
  float acc = 0.f;
  for (int64_t base = (int64_t)blockIdx.x * 1024 * U + threadIdx.x; base < n4; base += stride) {
    float4 a[U];
    float l[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * 1024;
      if (i < n4) { a[u] = reinterpret_cast<const float4*>(anchor)[i]; ld4h(local + 4 * i, l[u]); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * 1024;
      if (i < n4) {
        float d = a[u].x - l[u][0]; acc = fmaf(d, d, acc);
        d = a[u].y - l[u][1]; acc = fmaf(d, d, acc);
        d = a[u].z - l[u][2]; acc = fmaf(d, d, acc);
        d = a[u].w - l[u][3]; acc = fmaf(d, d, acc);
      }
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}

// 4-element layout + TMA bulk STORES: results written in place into the stage (conflict-free
// 16-B / 8-B shared stores), one elected consumer thread stores the tile with cp.async.bulk
// (fewer, wider write requests than 16-B STG), the stage is released once the stores READ it.
template <int CWn>
__global__ void __launch_bounds__(32 * (1 + CWn)) k4_tma4_bulk(__nv_bfloat16* local, float* anchor, float* mom,
                                                              int64_t n8, int K, int V) {
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t full[MAXK], empty[MAXK];
  if (threadIdx.x == 0) {
    for (int s = 0; s < K; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const float beta = 0.5f, mu = 0.85f, nu = 0.8f;
  const int64_t nt = (n8 + V - 1) / V;
  const int sb = V * 80;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int64_t q = blockIdx.x; q < nt; q += gridDim.x, ++it) {
        const int s = it % K, use = it / K;
        if (use) mbar_wait(&empty[s], (use - 1) & 1);
        const int64_t v0 = q * V;
        const int nv = (int)min((int64_t)V, n8 - v0);
        char* st = smem + (size_t)s * sb;
        mbar_expect_tx(&full[s], nv * 80);
        tma_load(st, anchor + 8 * v0, nv * 32, &full[s]);
        tma_load(st + V * 32, mom + 8 * v0, nv * 32, &full[s]);
        tma_load(st + V * 64, local + 8 * v0, nv * 16, &full[s]);
      }
    }
  } else {
    const int t = threadIdx.x - 32;
    int it = 0, prev = -1;
    for (int64_t q = blockIdx.x; q < nt; q += gridDim.x, ++it) {
      const int s = it % K, use = it / K;
      mbar_wait(&full[s], use & 1);
      const int64_t v0 = q * V;
      const int nv = (int)min((int64_t)V, n8 - v0);
      char* st = smem + (size_t)s * sb;
      for (int v = t; v < 2 * nv; v += 32 * CWn) {
        float4* ap = reinterpret_cast<float4*>(st) + v;
        float4* mp = reinterpret_cast<float4*>(st + V * 32) + v;
        __nv_bfloat16* lp = reinterpret_cast<__nv_bfloat16*>(st + V * 64) + 4 * v;
        float4 a = *ap, m = *mp;
        float l[4];
        ld4h(lp, l);
        float g;
        g = beta * (a.x - l[0]); m.x = fmaf(mu, m.x, g); a.x = a.x - nu * fmaf(mu, m.x, g);
        g = beta * (a.y - l[1]); m.y = fmaf(mu, m.y, g); a.y = a.y - nu * fmaf(mu, m.y, g);
        g = beta * (a.z - l[2]); m.z = fmaf(mu, m.z, g); a.z = a.z - nu * fmaf(mu, m.z, g);
        g = beta * (a.w - l[3]); m.w = fmaf(mu, m.w, g); a.w = a.w - nu * fmaf(mu, m.w, g);
        *ap = a;
        *mp = m;
        const float o[4] = {a.x, a.y, a.z, a.w};
        st4h(lp, o);
      }
      fence_async_smem();
      named_bar(1, 32 * CWn);
      if (t == 0) {
        tma_store(anchor + 8 * v0, st, nv * 32);
        tma_store(mom + 8 * v0, st + V * 32, nv * 32);
        tma_store(local + 8 * v0, st + V * 64, nv * 16);
        bulk_commit();
        bulk_wait_read<1>();
        if (prev >= 0) mbar_arrive(&empty[prev]);
      }
      prev = s;
    }
    if (t == 0) bulk_wait_all();
  }
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 202383360;  // a 7B decoder unit
  const int64_t n8 = n / 8;
  __nv_bfloat16* local;
  float *anchor, *mom, *out;
  CK(cudaMalloc(&local, n * 2));
  CK(cudaMalloc(&anchor, n * 4));
  CK(cudaMalloc(&mom, n * 4));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(local, 0, n * 2));
  CK(cudaMemset(anchor, 0, n * 4));
  CK(cudaMemset(mom, 0, n * 4));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](auto fn) {
    fn();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    const int R = 3;
    for (int r = 0; r < R; ++r) fn();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    CK(cudaGetLastError());
    return ms / R;
  };
  const int grids[] = {8, 16, 32, 148};
  printf("n=%lld params\n", (long long)n);
  for (int V : {512, 1024, 2048}) {
    const int bk = 200;
    const int K1 = std::min(MAXK, bk * 1024 / (V * 48));
    const int K4 = std::min(MAXK, bk * 1024 / (V * 80));
    if (K4 < 2) continue;
    CK(cudaFuncSetAttribute(k1_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, K1 * V * 48));
    CK(cudaFuncSetAttribute(k4_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, K4 * V * 80));
    CK(cudaFuncSetAttribute(k1_tma4<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, K1 * V * 48));
    CK(cudaFuncSetAttribute(k4_tma4<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, K4 * V * 80));
    CK(cudaFuncSetAttribute(k1_tma4<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, K1 * V * 48));
    CK(cudaFuncSetAttribute(k4_tma4<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, K4 * V * 80));
    CK(cudaFuncSetAttribute(k4_tma4_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, K4 * V * 80));
    for (int g : grids) {
      const float a1 = timeit([&] { k1_tma<<<g, NT, K1 * V * 48>>>(local, anchor, n8, out, K1, V); });
      const float b1 = timeit([&] { k1_tma4<8><<<g, 288, K1 * V * 48>>>(local, anchor, n8, out, K1, V); });
      const float c1 = timeit([&] { k1_tma4<16><<<g, 544, K1 * V * 48>>>(local, anchor, n8, out, K1, V); });
      const float a4 = timeit([&] { k4_tma<false><<<g, NT, K4 * V * 80>>>(local, anchor, mom, n8, K4, V); });
      const float b4 = timeit([&] { k4_tma4<8><<<g, 288, K4 * V * 80>>>(local, anchor, mom, n8, K4, V); });
      const float c4 = timeit([&] { k4_tma4<16><<<g, 544, K4 * V * 80>>>(local, anchor, mom, n8, K4, V); });
      auto ps = [&](double bpp, float ms) { return bpp * n / ms / 1e6 / g; };
      const float d4 = timeit([&] { k4_tma4_bulk<8><<<g, 288, K4 * V * 80>>>(local, anchor, mom, n8, K4, V); });
      printf("V %4d grid %3d | K4 v4 + TMA bulk store %5.1f GB/s/SM\n", V, g, ps(20, d4));
      printf("V %4d K1st %d K4st %d grid %3d | GB/s/SM  K1: v8 %5.1f  v4w8 %5.1f  v4w16 %5.1f | K4: v8 %5.1f  v4w8 %5.1f  "
             "v4w16 %5.1f | total@grid K1 %6.0f K4 %6.0f\n",
             V, K1, K4, g, ps(6, a1), ps(6, b1), ps(6, c1), ps(20, a4), ps(20, b4), ps(20, c4),
             6.0 * n / std::min({a1, b1, c1}) / 1e6, 20.0 * n / std::min({a4, b4, c4}) / 1e6);
    }
  }
  const int64_t n4 = n / 4;
  for (int g : grids) {
    const float u1 = timeit([&] { k4_ldg4<1><<<g, 1024>>>(local, anchor, mom, n4); });
    const float u2 = timeit([&] { k4_ldg4<2><<<g, 1024>>>(local, anchor, mom, n4); });
    const float u4 = timeit([&] { k4_ldg4<4><<<g, 1024>>>(local, anchor, mom, n4); });
    const float r2 = timeit([&] { k1_ldg4<2><<<g, 1024>>>(local, anchor, n4, out); });
    const float r4 = timeit([&] { k1_ldg4<4><<<g, 1024>>>(local, anchor, n4, out); });
    const float r8 = timeit([&] { k1_ldg4<8><<<g, 1024>>>(local, anchor, n4, out); });
    auto ps = [&](double bpp, float ms) { return bpp * n / ms / 1e6 / g; };
    printf("LDG4 1024thr grid %3d | GB/s/SM K4: U1 %5.1f U2 %5.1f U4 %5.1f | K1: U2 %5.1f U4 %5.1f U8 %5.1f\n", g,
           ps(20, u1), ps(20, u2), ps(20, u4), ps(6, r2), ps(6, r4), ps(6, r8));
  }
  return 0;
}
