// tools/a2a_bench.cu -- dev microbenchmark: all GPUs of the box pull from every peer at once
// (the traffic pattern of the peer path's RS / AG), LDG full grid; per-GPU inbound GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/a2a_bench tools/a2a_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

struct Srcs { const uint4* p[8]; int n; };

// vector i is read from source (i % n): a member's kernel reads every peer (and itself) evenly
__global__ void pull(Srcs s, int64_t n16, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = s.p[i % s.n][i];
    acc.x ^= v.x;
  }
  if (acc.x == 0x1234567u) sink[0] = acc;
}

int main() {
  int ng;
  CK(cudaGetDeviceCount(&ng));
  const int64_t bytes = 1LL << 30, n16 = bytes / 16;
  char* buf[8];
  uint4* sink[8];
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < ng; ++h)
      if (h != g) CK(cudaDeviceEnablePeerAccess(h, 0));
    CK(cudaMalloc(&buf[g], bytes));
    CK(cudaMemset(buf[g], 1, bytes));
    CK(cudaMalloc(&sink[g], 64));
  }
  for (int mode = 0; mode < 2; ++mode) {  // 0: peers only, 1: peers + self (like the RS/AG mix)
    cudaEvent_t a[8], b[8];
    for (int rep = 0; rep < 3; ++rep) {
      for (int g = 0; g < ng; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaDeviceSynchronize());
      }
      for (int g = 0; g < ng; ++g) {
        CK(cudaSetDevice(g));
        Srcs s{};
        for (int h = 0; h < ng; ++h)
          if (mode == 1 || h != g) s.p[s.n++] = reinterpret_cast<const uint4*>(buf[h]);
        if (rep == 2) {
          CK(cudaEventCreate(&a[g]));
          CK(cudaEventCreate(&b[g]));
          CK(cudaEventRecord(a[g]));
        }
        pull<<<(unsigned)(n16 / 256), 256>>>(s, n16, sink[g]);
        if (rep == 2) CK(cudaEventRecord(b[g]));
      }
    }
    for (int g = 0; g < ng; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaEventSynchronize(b[g]));
      float ms;
      CK(cudaEventElapsedTime(&ms, a[g], b[g]));
      const double remote = mode == 1 ? bytes * (double)(ng - 1) / ng : (double)bytes;
      printf("mode %s gpu %d: %.2f ms, inbound NVLink %.0f GB/s\n", mode ? "peers+self" : "peers", g, ms,
             remote / ms / 1e6);
    }
  }
  return 0;
}
