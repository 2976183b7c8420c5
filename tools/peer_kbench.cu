// tools/peer_kbench.cu -- the PRODUCTION peer-path kernels (peer_kernels.cu included verbatim),
// driven in ONE process over G GPUs with peer access (instead of G ranks + CUDA IPC), so they
// can be timed in isolation and profiled with ncu (which must not wrap a multi-rank command).
// One 7B decoder unit (202,383,360 params per rank) by default, sync row of N = G members,
// bf16 locals.  RS on every GPU, a host barrier (the scalar exchange's role), then AG + update.
// Environment knobs of the library apply (EDIT_PEER_TILE via argv[3], EDIT_PEER_SMEM_KB,
// EDIT_PEER_CTAS via argv[4]).  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include \
//        -I paper_2412_07210_b200/csrc -o tools/peer_kbench tools/peer_kbench.cu
//   tools/peer_kbench [numel] [reps] [tile] [ctas] [gpus] [local_only]
// local_only = 1: every member's AG reads ITS OWN D buffer for every slice (no NVLink: the
// kernel's HBM-side ceiling; results meaningless)
#include "../paper_2412_07210_b200/csrc/peer_kernels.cu"

#include <stdio.h>
#include <stdlib.h>

#include <vector>

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
  const int reps = argc > 2 ? atoi(argv[2]) : 5;
  const int tile = argc > 3 ? atoi(argv[3]) : kPeerTileVec;
  const int ctas = argc > 4 ? atoi(argv[4]) : 148;
  int ng = 0;
  CK(cudaGetDeviceCount(&ng));
  const int N = argc > 5 ? atoi(argv[5]) : (ng >= 4 ? 4 : 2);
  if (ng < N || N < 2 || N > EDIT_MAX_SYNC) {
    printf("needs %d GPUs, have %d\n", N, ng);
    return 0;
  }
  const Slicing sl0 = slicing_of(n, N, 0, tile);
  std::vector<__nv_bfloat16*> local(N);
  std::vector<float*> anchor(N), mom(N), D(N);
  std::vector<LayerScratch*> scr(N);
  std::vector<double*> parts(N), gparts(N);
  std::vector<edit_layer_stats_t*> rec(N);
  std::vector<cudaStream_t> st(N);
  for (int g = 0; g < N; ++g) {
    CK(cudaSetDevice(g));
    for (int o = 0; o < N; ++o)
      if (o != g) CK(cudaDeviceEnablePeerAccess(o, 0));
    CK(cudaMalloc(&local[g], n * 2));
    CK(cudaMalloc(&anchor[g], n * 4));
    CK(cudaMalloc(&mom[g], n * 4));
    CK(cudaMalloc(&D[g], sl0.slice * 8 * 4));
    CK(cudaMalloc(&scr[g], sizeof(LayerScratch)));
    CK(cudaMalloc(&parts[g], rs_partial_slots(n, N) * sizeof(double)));
    CK(cudaMalloc(&gparts[g], 8 * sizeof(double)));
    CK(cudaMalloc(&rec[g], sizeof(edit_layer_stats_t)));
    CK(cudaMemset(gparts[g], 0, 8 * sizeof(double)));
    LayerScratch h{};
    for (int j = 0; j < N; ++j) h.w_all[j] = 1.0f / N;
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
  const bool local_only = argc > 6 && atoi(argv[6]) != 0;
  const char* ke = getenv("EDIT_PEER_KERNELS");  // as the library: ldg (default) | ldg2 | ldgall | tma
  const int kern = ke && !strcmp(ke, "tma") ? 0 : ke && !strcmp(ke, "ldg2") ? 3 : ke && !strcmp(ke, "ldgall") ? 5 : 1;
  std::vector<float> rs_ms(N, 0.f), ag_ms(N, 0.f);
  FoldArgs nofold{};
  for (int r = 0; r < reps + 1; ++r) {
    std::vector<cudaEvent_t> e0(N), e1(N), e2(N);
    for (int g = 0; g < N; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaEventCreate(&e0[g]));
      CK(cudaEventCreate(&e1[g]));
      CK(cudaEventCreate(&e2[g]));
      CK(cudaEventRecord(e0[g], st[g]));
      launch_rs(EDIT_BF16, pp, slicing_of(n, N, g, tile), anchor[g], D[g], scr[g], parts[g], ctas, 0, kern, nofold, st[g]);
      CK(cudaEventRecord(e1[g], st[g]));
    }
    for (int g = 0; g < N; ++g) {  // the barrier the scalar exchange provides in the library
      CK(cudaSetDevice(g));
      CK(cudaStreamSynchronize(st[g]));
    }
    for (int g = 0; g < N; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaEventRecord(e1[g], st[g]));
      UpdateArgs a{};
      a.local = local[g];
      a.anchor = anchor[g];
      a.momentum = mom[g];
      a.n = n;
      a.gparts = gparts[g];
      a.n_gparts = N;
      a.rollback = &scr[g]->rollback;
      a.nu = 0.8f;
      a.mu = 0.85f;
      a.phi = 10.0;
      a.eps = 1e-6;
      a.rec = rec[g];
      PeerPtrs pa = pp;
      if (local_only)
        for (int j = 0; j < N; ++j) pa.D[j] = D[g];
      launch_ag_update(EDIT_BF16, a, pa, slicing_of(n, N, g, tile), ctas, 0, kern, st[g]);
      CK(cudaEventRecord(e2[g], st[g]));
    }
    for (int g = 0; g < N; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaStreamSynchronize(st[g]));
      CK(cudaGetLastError());
      float a, b;
      CK(cudaEventElapsedTime(&a, e0[g], e1[g]));
      CK(cudaEventElapsedTime(&b, e1[g], e2[g]));
      if (r > 0) {
        rs_ms[g] += a / reps;
        ag_ms[g] += b / reps;
      }
    }
  }
  for (int g = 0; g < N; ++g) {
    const double nvl_rs = 2.0 * n * (N - 1) / N, nvl_ag = 4.0 * n * (N - 1) / N;
    printf("%s N=%d tile=%d ctas=%d gpu %d: RS %.3f ms (NVLink in %.0f GB/s, HBM %.0f GB/s)  AG %.3f ms (NVLink in %.0f "
           "GB/s, HBM %.0f GB/s incl. served D, %.0f GB/s algorithmic 20 B)\n",
           kern == 0 ? "tma" : kern == 3 ? "ldg2" : kern == 5 ? "ldgall" : "ldg", N, tile, ctas, g, rs_ms[g], nvl_rs / rs_ms[g] / 1e6, (2.0 + 8.0 / N) * n / rs_ms[g] / 1e6, ag_ms[g],
           nvl_ag / ag_ms[g] / 1e6, 22.0 * n / ag_ms[g] / 1e6, 20.0 * n / ag_ms[g] / 1e6);
  }
  return 0;
}
