// tools/peer_bench.cu -- dev microbenchmark (2 GPUs, one process, peer access): how fast
// can a kernel pull a peer's memory over NVLink 5, and with how many SMs?  LDG.128 at
// various grids vs TMA 1-D bulk copies (cp.async.bulk, mbarrier complete_tx) with few
// persistent CTAs; also TMA on local HBM and cudaMemcpyPeerAsync.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/peer_bench tools/peer_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__global__ void ldg_read(const uint4* __restrict__ src, int64_t n16, uint4* sink, int per_thread) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x * per_thread + threadIdx.x; base < n16;
       base += stride * per_thread) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (u < per_thread && base + (int64_t)u * blockDim.x < n16) v[u] = src[base + (int64_t)u * blockDim.x];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (u < per_thread && base + (int64_t)u * blockDim.x < n16) acc.x ^= v[u].x ^ v[u].w;
  }
  if (acc.x == 0x12345678u) sink[0] = acc;
}

// LDG copy peer -> local
__global__ void ldg_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t n16) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) dst[i] = src[i];
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}\n" ::"r"(smem_u32(bar)), "r"(parity));
}
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst_smem)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// persistent TMA reader: each CTA walks chunks blockIdx.x, +grid, ... with K stages of CH bytes
template <int K>
__global__ void tma_read(const char* __restrict__ src, int64_t bytes, int chunk, uint4* sink) {
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t bars[K];
  const int64_t nchunks = bytes / chunk;
  if (threadIdx.x == 0) {
    for (int s = 0; s < K; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int64_t c = blockIdx.x;
  int issued = 0;
  for (int s = 0; s < K && c + (int64_t)s * gridDim.x < nchunks; ++s) {
    mbar_expect_tx(&bars[s], chunk);
    tma_load_1d(smem + s * chunk, src + (c + (int64_t)s * gridDim.x) * chunk, chunk, &bars[s]);
    ++issued;
  }
  uint32_t acc = 0;
  int64_t next = c + (int64_t)issued * gridDim.x;
  for (int64_t k = 0; c + k * gridDim.x < nchunks; ++k) {
    const int s = k % K;
    mbar_wait(&bars[s], (k / K) & 1);
    acc ^= *reinterpret_cast<volatile uint32_t*>(smem + s * chunk);
    if (next < nchunks) {
      mbar_expect_tx(&bars[s], chunk);
      tma_load_1d(smem + s * chunk, src + next * chunk, chunk, &bars[s]);
      next += gridDim.x;
    }
  }
  if (acc == 0x12345678u) sink[0] = make_uint4(acc, 0, 0, 0);
}

template <typename F>
float time_it(F f, int reps = 5) {
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

int main() {
  int ndev;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("need 2 GPUs\n");
    return 0;
  }
  const int64_t bytes = 2LL << 30;  // 2 GiB
  char *buf0, *buf1, *dst0;
  uint4* sink;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&buf1, bytes));
  CK(cudaMemset(buf1, 1, bytes));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&buf0, bytes));
  CK(cudaMalloc(&dst0, bytes));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMemset(buf0, 1, bytes));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t n16 = bytes / 16;
  printf("bytes=%lld sms=%d\n", (long long)bytes, sms);
  for (int grid : {16, 32, 64, 148, 296, 592, 0}) {
    for (int pt : {1, 4, 8}) {
      int g = grid ? grid : (int)((n16 + 256 * pt - 1) / (256 * pt));
      const char* src = buf1;
      float ms = time_it([&] { ldg_read<<<g, 256>>>((const uint4*)src, n16, sink, pt); });
      float msl = time_it([&] { ldg_read<<<g, 256>>>((const uint4*)buf0, n16, sink, pt); });
      printf("LDG read  grid=%6d per_thread=%d: peer %7.1f GB/s   local %7.1f GB/s\n", g, pt, bytes / ms / 1e6,
             bytes / msl / 1e6);
    }
  }
  {
    int g = (int)(n16 / 256);
    float ms = time_it([&] { ldg_copy<<<g, 256>>>((const uint4*)buf1, (uint4*)dst0, n16); });
    printf("LDG copy peer->local full grid: %.1f GB/s\n", bytes / ms / 1e6);
  }
  for (int chunk : {8192, 16384, 32768}) {
    for (int grid : {8, 16, 32, 64, 148}) {
      const int K = 4;
      const int sm = K * chunk;
      CK(cudaFuncSetAttribute(tma_read<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      float ms = time_it([&] { tma_read<4><<<grid, 32, sm>>>(buf1, bytes, chunk, sink); });
      float msl = time_it([&] { tma_read<4><<<grid, 32, sm>>>(buf0, bytes, chunk, sink); });
      printf("TMA read K=4 chunk=%6d grid=%4d: peer %7.1f GB/s   local %7.1f GB/s\n", chunk, grid,
             bytes / ms / 1e6, bytes / msl / 1e6);
    }
  }
  for (int grid : {8, 16, 32, 64, 148}) {
    const int K = 8, chunk = 16384, sm = K * chunk;
    CK(cudaFuncSetAttribute(tma_read<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    float ms = time_it([&] { tma_read<8><<<grid, 32, sm>>>(buf1, bytes, chunk, sink); });
    float msl = time_it([&] { tma_read<8><<<grid, 32, sm>>>(buf0, bytes, chunk, sink); });
    printf("TMA read K=8 chunk=%6d grid=%4d: peer %7.1f GB/s   local %7.1f GB/s\n", chunk, grid, bytes / ms / 1e6,
           bytes / msl / 1e6);
  }
  {
    float ms = time_it([&] { CK(cudaMemcpyPeerAsync(dst0, 0, buf1, 1, bytes, 0)); });
    printf("cudaMemcpyPeerAsync 1->0: %.1f GB/s\n", bytes / ms / 1e6);
  }
  return 0;
}
