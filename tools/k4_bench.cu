// tools/k4_bench.cu -- dev microbenchmark of streaming-kernel variants for K4 (outer_update,
// N == 1 form: read bf16 local + fp32 anchor + fp32 momentum, write all three) and K1.
// Not part of the product; used to pick the load/store scheme on sm_100a.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o k4_bench tools/k4_bench.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));      \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

enum { LD_PLAIN = 0, LD_CS = 1, LD_NA = 2, LD_LU = 3 };

template <int LD>
__device__ __forceinline__ float4 ldf4(const float4* p) {
  if (LD == LD_CS) return __ldcs(p);
  if (LD == LD_LU) return __ldlu(p);
  if (LD == LD_NA) {
    float4 r;
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
  }
  return *p;
}
template <int LD>
__device__ __forceinline__ uint4 ldu4(const uint4* p) {
  if (LD == LD_CS) return __ldcs(p);
  if (LD == LD_LU) return __ldlu(p);
  if (LD == LD_NA) {
    uint4 r;
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
  }
  return *p;
}
template <int ST>
__device__ __forceinline__ void stf4(float4* p, float4 v) {
  if (ST == 1) __stcs(p, v);
  else if (ST == 2) asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
  else *p = v;
}
template <int ST>
__device__ __forceinline__ void stu4(uint4* p, uint4 v) {
  if (ST == 1) __stcs(p, v);
  else if (ST == 2) asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
  else *p = v;
}

__device__ __forceinline__ void unpack(uint4 r, float (&v)[8]) {
  const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __uint_as_float(w[i] << 16);
    v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
__device__ __forceinline__ uint4 pack(const float (&v)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// K4 N==1 body with U vectors (of 8 elements) per thread-iteration, loads issued first.
template <int U, int LD, int ST, int T>
__global__ void __launch_bounds__(T) k4(uint4* __restrict__ local, float4* __restrict__ anchor,
                                        float4* __restrict__ mom, int64_t n8, float beta, float mu, float nu) {
  const int64_t stride = (int64_t)gridDim.x * T * U;
  for (int64_t base = (int64_t)blockIdx.x * T * U + threadIdx.x; base < n8; base += stride) {
    uint4 l[U];
    float4 a0[U], a1[U], m0[U], m1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * T;
      if (i < n8) {
        l[u] = ldu4<LD>(local + i);
        a0[u] = ldf4<LD>(anchor + 2 * i);
        a1[u] = ldf4<LD>(anchor + 2 * i + 1);
        m0[u] = ldf4<LD>(mom + 2 * i);
        m1[u] = ldf4<LD>(mom + 2 * i + 1);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * T;
      if (i < n8) {
        float lv[8], a[8] = {a0[u].x, a0[u].y, a0[u].z, a0[u].w, a1[u].x, a1[u].y, a1[u].z, a1[u].w};
        float m[8] = {m0[u].x, m0[u].y, m0[u].z, m0[u].w, m1[u].x, m1[u].y, m1[u].z, m1[u].w};
        unpack(l[u], lv);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float g = beta * (a[j] - lv[j]);
          m[j] = fmaf(mu, m[j], g);
          a[j] = a[j] - nu * fmaf(mu, m[j], g);
        }
        stf4<ST>(mom + 2 * i, make_float4(m[0], m[1], m[2], m[3]));
        stf4<ST>(mom + 2 * i + 1, make_float4(m[4], m[5], m[6], m[7]));
        stf4<ST>(anchor + 2 * i, make_float4(a[0], a[1], a[2], a[3]));
        stf4<ST>(anchor + 2 * i + 1, make_float4(a[4], a[5], a[6], a[7]));
        stu4<ST>(local + i, pack(a));
      }
    }
  }
}

// reference copy: fp32 read + write
template <int U, int T>
__global__ void __launch_bounds__(T) copyk(const float4* __restrict__ x, float4* __restrict__ y, int64_t n4) {
  const int64_t stride = (int64_t)gridDim.x * T * U;
  for (int64_t base = (int64_t)blockIdx.x * T * U + threadIdx.x; base < n4; base += stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * T < n4) v[u] = x[base + u * T];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * T < n4) y[base + u * T] = v[u];
  }
}

// K1 N==1: read local + anchor, sum of squares (simplified: per-thread fp32 -> atomic per CTA not needed for timing)
template <int U, int LD, int T>
__global__ void __launch_bounds__(T) k1(const uint4* __restrict__ local, const float4* __restrict__ anchor,
                                        int64_t n8, double* out) {
  const int64_t stride = (int64_t)gridDim.x * T * U;
  double acc = 0.0;
  for (int64_t base = (int64_t)blockIdx.x * T * U + threadIdx.x; base < n8; base += stride) {
    uint4 l[U];
    float4 a0[U], a1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * T;
      if (i < n8) {
        l[u] = ldu4<LD>(local + i);
        a0[u] = ldf4<LD>(anchor + 2 * i);
        a1[u] = ldf4<LD>(anchor + 2 * i + 1);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * T;
      if (i < n8) {
        float lv[8], a[8] = {a0[u].x, a0[u].y, a0[u].z, a0[u].w, a1[u].x, a1[u].y, a1[u].z, a1[u].w};
        unpack(l[u], lv);
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float d = a[j] - lv[j];
          s = fmaf(d, d, s);
        }
        acc += s;
      }
    }
  }
  if (acc == 12345.0) *out = acc;  // keep the loads alive
}

template <typename F>
float time_it(F f, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int r = 0; r < reps; ++r) f();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 202383360;  // one 7B decoder unit
  const int64_t n8 = n / 8;
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint4* local;
  float4 *anchor, *mom, *x, *y;
  double* out;
  CK(cudaMalloc(&local, n * 2));
  CK(cudaMalloc(&anchor, n * 4));
  CK(cudaMalloc(&mom, n * 4));
  CK(cudaMalloc(&x, n * 4));
  CK(cudaMalloc(&y, n * 4));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(local, 0, n * 2));
  CK(cudaMemset(anchor, 0, n * 4));
  CK(cudaMemset(mom, 0, n * 4));
  CK(cudaMemset(x, 0, n * 4));
  const int reps = 10;
  const double k4_bytes = 20.0 * n, k1_bytes = 6.0 * n, cp_bytes = 8.0 * n;
  printf("n=%lld sms=%d\n", (long long)n, sms);
#define RUNCOPY(U, T, G)                                                                              \
  {                                                                                                   \
    int grid = (G) > 0 ? (G) * sms : (int)((n / 4 + (int64_t)T * U - 1) / ((int64_t)T * U));         \
    float ms = time_it([&] { copyk<U, T><<<grid, T>>>(x, y, n / 4); }, reps);                         \
    printf("copy   U=%d T=%d grid=%d: %.3f ms %.1f GB/s\n", U, T, grid, ms, cp_bytes / ms / 1e6);    \
  }
#define RUNK4(U, LD, ST, T, G)                                                                        \
  {                                                                                                   \
    int grid = (G) > 0 ? (G) * sms : (int)((n8 + (int64_t)T * U - 1) / ((int64_t)T * U));            \
    float ms = time_it([&] { k4<U, LD, ST, T><<<grid, T>>>(local, anchor, mom, n8, 0.3f, 0.85f, 0.8f); }, reps); \
    printf("k4 U=%d LD=%d ST=%d T=%d grid=%d: %.3f ms %.1f GB/s\n", U, LD, ST, T, grid, ms, k4_bytes / ms / 1e6); \
  }
#define RUNK1(U, LD, T, G)                                                                            \
  {                                                                                                   \
    int grid = (G) > 0 ? (G) * sms : (int)((n8 + (int64_t)T * U - 1) / ((int64_t)T * U));            \
    float ms = time_it([&] { k1<U, LD, T><<<grid, T>>>(local, anchor, n8, out); }, reps);             \
    printf("k1 U=%d LD=%d T=%d grid=%d: %.3f ms %.1f GB/s\n", U, LD, T, grid, ms, k1_bytes / ms / 1e6); \
  }
  RUNCOPY(1, 256, 0);
  RUNCOPY(4, 256, 0);
  RUNCOPY(4, 256, 8);
  RUNK4(1, LD_CS, 1, 256, 6);
  RUNK4(1, LD_PLAIN, 0, 256, 6);
  RUNK4(1, LD_PLAIN, 0, 256, 0);
  RUNK4(2, LD_PLAIN, 0, 256, 0);
  RUNK4(2, LD_PLAIN, 0, 256, 4);
  RUNK4(2, LD_NA, 2, 256, 4);
  RUNK4(2, LD_CS, 1, 256, 4);
  RUNK4(2, LD_LU, 0, 256, 4);
  RUNK4(4, LD_PLAIN, 0, 256, 2);
  RUNK4(4, LD_PLAIN, 0, 256, 0);
  RUNK4(2, LD_PLAIN, 0, 512, 2);
  RUNK4(2, LD_PLAIN, 0, 128, 8);
  RUNK4(1, LD_PLAIN, 0, 1024, 2);
  RUNK1(1, LD_CS, 256, 6);
  RUNK1(2, LD_PLAIN, 256, 4);
  RUNK1(4, LD_PLAIN, 256, 4);
  RUNK1(4, LD_NA, 256, 4);
  RUNK1(2, LD_PLAIN, 256, 0);
  RUNK1(4, LD_PLAIN, 256, 0);
  return 0;
}
