// tools/kbench.cu -- dev microbenchmark of the PRODUCTION kernels (kernels.cu included
// verbatim) at other {U, I} thread shapes, on one 7B decoder unit (202,383,360 params).
// Picks kReduceShape / kUpdateShape in internal.h.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -I paper_2412_07210_b200/csrc -o tools/kbench tools/kbench.cu
#include "../paper_2412_07210_b200/csrc/kernels.cu"

#include <stdio.h>
#include <stdlib.h>

using namespace edit;

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

template <typename F>
float time_it(F f, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  float total = 0.f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    total += ms;
  }
  return total / reps;
}

__global__ void fill(float* x, int64_t n, float scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = scale * (float)((i * 2654435761ull) % 1000003) / 1000003.f;
}
__global__ void fillb(__nv_bfloat16* x, const float* a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = __float2bfloat16_rn(a[i] * 0.999f);
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 202383360;
  const int reps = 10;
  __nv_bfloat16* local;
  float *anchor, *mom, *S;
  LayerScratch* scr;
  double *parts, *gparts;
  int32_t* rb;
  edit_layer_stats_t* rec;
  CK(cudaMalloc(&local, n * 2));
  CK(cudaMalloc(&anchor, n * 4));
  CK(cudaMalloc(&mom, n * 4));
  CK(cudaMalloc(&S, n * 4));
  CK(cudaMalloc(&scr, sizeof(LayerScratch)));
  CK(cudaMalloc(&parts, (n / 8 + 1) * sizeof(double)));
  CK(cudaMalloc(&gparts, 8 * sizeof(double)));
  CK(cudaMalloc(&rb, 4));
  CK(cudaMalloc(&rec, sizeof(edit_layer_stats_t)));
  CK(cudaMemset(scr, 0, sizeof(LayerScratch)));
  CK(cudaMemset(rb, 0, 4));
  CK(cudaMemset(gparts, 0, 8 * sizeof(double)));
  fill<<<4096, 256>>>(anchor, n, 0.02f);
  fill<<<4096, 256>>>(mom, n, 5e-4f);
  fill<<<4096, 256>>>(S, n, 2e-3f);
  fillb<<<4096, 256>>>(local, anchor, n);
  CK(cudaDeviceSynchronize());
  printf("n=%lld\n", (long long)n);
#define K1(U, I, WS)                                                                                   \
  {                                                                                                    \
    unsigned g = (unsigned)grid_of(n, U * I);                                                          \
    float ms = time_it([&] { pg_norm_kernel<__nv_bfloat16, WS, U, I><<<g, kThreads>>>(local, anchor,   \
                                                                       WS ? S : nullptr, n, scr, parts); }, reps); \
    double bytes = (6.0 + (WS ? 4.0 : 0.0)) * n;                                                       \
    printf("K1 pg_norm bf16 S=%d U=%d I=%d grid=%u: %.1f us %.0f GB/s\n", WS, U, I, g, ms * 1e3, bytes / ms / 1e6); \
  }
#define K3(U, I)                                                                                       \
  {                                                                                                    \
    unsigned g = (unsigned)grid_of(n, U * I);                                                          \
    float ms = time_it([&] { sumsq_kernel<U, I><<<g, kThreads>>>(S, n, scr, parts); }, reps);          \
    printf("K3 sumsq U=%d I=%d grid=%u: %.1f us %.0f GB/s\n", U, I, g, ms * 1e3, 4.0 * n / ms / 1e6);  \
  }
#define K4(U, I, FS)                                                                                   \
  {                                                                                                    \
    UpdateArgs a{};                                                                                    \
    a.local = local; a.anchor = anchor; a.momentum = mom; a.dbar = FS ? S : nullptr; a.n = n;         \
    a.gparts = gparts; a.n_gparts = 1; a.rollback = rb; a.nu = 0.8f; a.mu = 0.85f; a.phi = 10.0;       \
    a.eps = 1e-6; a.flags = 0; a.rec = rec;                                                            \
    unsigned g = (unsigned)grid_of(n, U * I);                                                          \
    float ms = time_it([&] { outer_update_kernel<__nv_bfloat16, FS, U, I><<<g, kThreads>>>(a); }, reps); \
    double bytes = (FS ? 22.0 : 20.0) * n;                                                             \
    printf("K4 update bf16 fromS=%d U=%d I=%d grid=%u: %.1f us %.0f GB/s\n", FS, U, I, g, ms * 1e3, bytes / ms / 1e6); \
  }
  K1(1, 1, false) K1(2, 1, false) K1(2, 2, false) K1(4, 1, false) K1(2, 4, false) K1(4, 2, false) K1(1, 4, false)
  K1(4, 4, false) K1(2, 8, false)
  K1(1, 1, true) K1(2, 1, true) K1(2, 2, true) K1(4, 1, true) K1(2, 4, true)
  K3(2, 1) K3(2, 2) K3(4, 1) K3(4, 2) K3(2, 4)
  K4(1, 1, false) K4(2, 1, false) K4(1, 2, false) K4(2, 2, false) K4(1, 4, false) K4(4, 1, false)
  K4(1, 1, true) K4(2, 1, true) K4(1, 2, true)
  {  // L2 evict_first streaming variants of the production shapes
    UpdateArgs a{};
    a.local = local; a.anchor = anchor; a.momentum = mom; a.dbar = nullptr; a.n = n;
    a.gparts = gparts; a.n_gparts = 1; a.rollback = rb; a.nu = 0.8f; a.mu = 0.85f; a.phi = 10.0;
    a.eps = 1e-6; a.flags = 0; a.rec = rec;
    unsigned g = (unsigned)grid_of(n, 1);
    float ms = time_it([&] { outer_update_kernel<__nv_bfloat16, false, 1, 1, true><<<g, kThreads>>>(a); }, reps);
    printf("K4 update bf16 EF U=1 I=1: %.1f us %.0f GB/s\n", ms * 1e3, 20.0 * n / ms / 1e6);
    unsigned g1 = (unsigned)grid_of(n, 8);
    float ms1 = time_it([&] { pg_norm_kernel<__nv_bfloat16, false, 2, 4, false, true><<<g1, kThreads>>>(local, anchor, nullptr, n, scr, parts); }, reps);
    printf("K1 pg_norm bf16 EF U=2 I=4: %.1f us %.0f GB/s\n", ms1 * 1e3, 6.0 * n / ms1 / 1e6);
  }
  return 0;
}
