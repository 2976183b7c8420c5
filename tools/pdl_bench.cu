// tools/pdl_bench.cu -- dev microbenchmark (1 GPU): the cost of a dependent kernel boundary on
// B200, for the sync's per-unit chain (K1 -> exchange+K2 -> RS -> exchange -> AG) on small units.
// A chain of C dependent kernels (each: 148 CTAs streaming `bytes_per_kernel`) launched
//   (a) plainly on one stream,
//   (b) with programmatic dependent launch (PDL: cudaLaunchAttributeProgrammaticStreamSerialization,
//       the kernel waits with griddepcontrol.wait before touching its input and lets the next one
//       launch early with griddepcontrol.launch_dependents),
//   (c) as a CUDA graph of the plain launches.
// Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/pdl_bench tools/pdl_bench.cu
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

template <bool kPDL>
__global__ void __launch_bounds__(256) step(const float4* __restrict__ in, float4* __restrict__ out, int64_t n4) {
  if (kPDL) asm volatile("griddepcontrol.wait;" ::: "memory");  // predecessor's writes visible
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 v = in[i];
    v.x += 1.f;
    out[i] = v;
  }
  if (kPDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

int main(int argc, char** argv) {
  const int C = 170;  // 5 dependent kernels x 34 units
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int64_t bytes : {(int64_t)0, (int64_t)1 << 20, (int64_t)8 << 20, (int64_t)64 << 20}) {
    const int64_t n4 = bytes / 16 > 0 ? bytes / 16 : 1;
    float4 *a, *b;
    CK(cudaMalloc(&a, n4 * 16));
    CK(cudaMalloc(&b, n4 * 16));
    CK(cudaMemset(a, 0, n4 * 16));
    const unsigned grid = bytes == 0 ? 148 : (unsigned)std::min<int64_t>(148 * 8, (n4 + 255) / 256);
    auto plain = [&] {
      for (int c = 0; c < C; ++c) step<false><<<grid, 256, 0, st>>>(c & 1 ? b : a, c & 1 ? a : b, bytes ? n4 : 0);
    };
    auto pdl = [&] {
      for (int c = 0; c < C; ++c) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const float4* in = c & 1 ? b : a;
        float4* out = c & 1 ? a : b;
        const int64_t nn = bytes ? n4 : 0;
        CK(cudaLaunchKernelEx(&cfg, step<true>, in, out, nn));
      }
    };
    auto timeit = [&](auto fn) {
      fn();
      CK(cudaStreamSynchronize(st));
      CK(cudaEventRecord(e0, st));
      for (int r = 0; r < 5; ++r) fn();
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      return ms / 5 * 1000.f / C;  // us per kernel
    };
    const float tp = timeit(plain), tq = timeit(pdl);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
    plain();
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    const float tg = timeit([&] { CK(cudaGraphLaunch(ge, st)); });
    printf("bytes/kernel %9lld: plain %6.2f us/kernel  PDL %6.2f  graph %6.2f  (stream of %d dependent kernels, grid %u)\n",
           (long long)bytes, tp, tq, tg, C, grid);
    CK(cudaGraphExecDestroy(ge));
    CK(cudaGraphDestroy(g));
    CK(cudaFree(a));
    CK(cudaFree(b));
  }
  return 0;
}
