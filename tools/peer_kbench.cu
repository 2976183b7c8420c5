// tools/peer_kbench.cu -- the PRODUCTION peer-path kernels (peer_kernels.cu included verbatim),
// driven in ONE process over 2 GPUs with peer access (instead of two ranks + CUDA IPC), so they
// can be timed and profiled with ncu (which must not wrap a multi-rank command).  One 7B
// decoder unit (202,383,360 params per rank), N = 2 sync row, bf16 locals.  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include \
//        -I paper_2412_07210_b200/csrc -o tools/peer_kbench tools/peer_kbench.cu
#include "../paper_2412_07210_b200/csrc/peer_kernels.cu"

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

__global__ void fill(float* x, int64_t n, float scale, float off) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = off + scale * (float)((i * 2654435761ull) % 1000003) / 1000003.f;
}
__global__ void fillb(__nv_bfloat16* x, const float* a, int64_t n, float d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = __float2bfloat16_rn(a[i] - d * (float)((i * 40503ull) % 997) / 997.f);
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 202383360;
  const int N = 2, reps = argc > 2 ? atoi(argv[2]) : 5;
  int ng = 0;
  CK(cudaGetDeviceCount(&ng));
  if (ng < 2) {
    printf("needs 2 GPUs\n");
    return 0;
  }
  const Slicing sl0 = slicing_of(n, N, 0);
  __nv_bfloat16* local[2];
  float *anchor[2], *mom[2], *D[2];
  LayerScratch* scr[2];
  double* parts[2];
  double* gparts[2];
  edit_layer_stats_t* rec[2];
  cudaStream_t st[2];
  for (int g = 0; g < N; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&local[g], n * 2));
    CK(cudaMalloc(&anchor[g], n * 4));
    CK(cudaMalloc(&mom[g], n * 4));
    CK(cudaMalloc(&D[g], sl0.slice * 8 * 4));
    CK(cudaMalloc(&scr[g], sizeof(LayerScratch)));
    CK(cudaMalloc(&parts[g], kMaxPeerCtas * sizeof(double)));
    CK(cudaMalloc(&gparts[g], 2 * sizeof(double)));
    CK(cudaMalloc(&rec[g], sizeof(edit_layer_stats_t)));
    CK(cudaMemset(scr[g], 0, sizeof(LayerScratch)));
    CK(cudaMemset(gparts[g], 0, 2 * sizeof(double)));
    LayerScratch h{};
    h.w_all[0] = 0.6f;
    h.w_all[1] = 0.4f;
    CK(cudaMemcpy(scr[g], &h, sizeof h, cudaMemcpyHostToDevice));
    fill<<<4096, 256>>>(anchor[g], n, 0.02f, 0.f);
    fill<<<4096, 256>>>(mom[g], n, 5e-4f, 0.f);
    fillb<<<4096, 256>>>(local[g], anchor[g], n, 2e-3f * (1 + g));
    CK(cudaStreamCreate(&st[g]));
    CK(cudaDeviceSynchronize());
  }
  PeerPtrs pp{};
  for (int g = 0; g < N; ++g) {
    pp.L[g] = local[g];
    pp.D[g] = D[g];
  }
  float rs_ms[2] = {0, 0}, ag_ms[2] = {0, 0};
  for (int r = 0; r < reps + 1; ++r) {
    cudaEvent_t evs[2][3];
    for (int g = 0; g < N; ++g) {
      CK(cudaSetDevice(g));
      for (int k = 0; k < 3; ++k) CK(cudaEventCreate(&evs[g][k]));
      CK(cudaEventRecord(evs[g][0], st[g]));
      launch_rs(EDIT_BF16, pp, slicing_of(n, N, g), anchor[g], D[g], scr[g], parts[g], 148, false, 0, st[g]);
      CK(cudaEventRecord(evs[g][1], st[g]));
    }
    for (int g = 0; g < N; ++g) {  // the barrier the scalar exchange provides in the library
      CK(cudaSetDevice(g));
      CK(cudaStreamSynchronize(st[g]));
    }
    for (int g = 0; g < N; ++g) {
      CK(cudaSetDevice(g));
      UpdateArgs a{};
      a.local = local[g];
      a.anchor = anchor[g];
      a.momentum = mom[g];
      a.n = n;
      a.gparts = gparts[g];
      a.n_gparts = 2;
      a.rollback = &scr[g]->rollback;
      a.nu = 0.8f;
      a.mu = 0.85f;
      a.phi = 10.0;
      a.eps = 1e-6;
      a.rec = rec[g];
      launch_ag_update(EDIT_BF16, a, pp, slicing_of(n, N, g), 148, false, 0, st[g]);
      CK(cudaEventRecord(evs[g][2], st[g]));
    }
    for (int g = 0; g < N; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaStreamSynchronize(st[g]));
      float a, b;
      CK(cudaEventElapsedTime(&a, evs[g][0], evs[g][1]));
      CK(cudaEventElapsedTime(&b, evs[g][1], evs[g][2]));
      if (r > 0) {
        rs_ms[g] += a / reps;
        ag_ms[g] += b / reps;
      }
    }
  }
  for (int g = 0; g < N; ++g) {
    const double nvl_rs = 2.0 * n * (N - 1) / N, nvl_ag = 4.0 * n * (N - 1) / N;
    printf("gpu %d: RS %.3f ms (NVLink in %.0f GB/s, HBM %.0f GB/s)  AG %.3f ms (NVLink in %.0f GB/s, HBM %.0f GB/s)\n",
           g, rs_ms[g], nvl_rs / rs_ms[g] / 1e6, (2.0 + 8.0 / N) * n / rs_ms[g] / 1e6, ag_ms[g],
           nvl_ag / ag_ms[g] / 1e6, 22.0 * n / ag_ms[g] / 1e6);
  }
  return 0;
}
