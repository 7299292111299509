// Micro: does a 16-byte (not 128-byte) aligned start address of a no-swizzle
// K-major A operand (the shifted-view conv's per-tap offset) slow
// tcgen05.mma.kind::tf32 M=128 K=8?  One thread issues `iters` MMAs whose A
// start advances by `unit` 16-byte units per MMA (1: misaligned shifts, 8:
// 128-byte aligned).  Diagnostic only.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_align.cu -o mma_align
#include <cstdint>
#include <cstdio>

#include "../../paper_1501_07338_b200/csrc/tc_ptx.cuh"
using namespace vcnn_b200;

template <int N, int M = 128>
__global__ void bench(int unit, int iters, unsigned long long* out, int nacc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 100 * 1024 / 4; i += blockDim.x) ((float*)s)[i] = 0.f;
  if (threadIdx.x < 32) {
    ptx::tmem_alloc(&tbase, 512);
    ptx::tmem_relinquish();
  }
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t a = ptx::smem_u32(s), b = a + 64 * 1024;
    const uint32_t id = ptx::idesc_tf32(M, N);
    const uint64_t ad0 = ptx::interleave_desc(a, 2048u * 16u, 128u);
    const uint64_t bd = ptx::interleave_desc(b, 128u, 256u);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
      ptx::mma_tf32(tbase + (uint32_t)((i % nacc) * N), ad0 + (uint64_t)(unit * (i % 64)), bd, id, i >= nacc);
    unsigned long long t1 = clock64();
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    unsigned long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc(tbase, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  unsigned long long h[2];
  const int smem = 104 * 1024;
  int grid = 1, nacc = 1;
  auto run = [&](auto kern, const char* name, int unit, int iters) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int r = 0; r < 3; ++r) kern<<<grid, 128, smem>>>(unit, iters, d, nacc);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("nacc %d grid %3d %-6s unit %d iters %4d: issue %6llu cyc, done %6llu cyc -> %.1f cyc/mma %s\n", nacc, grid, name,
           unit, iters, h[0], h[1], (double)h[1] / iters, cudaGetErrorString(e));
  };
  for (int g : {1, 296})
    for (int na : {1, 2, 4}) {
      grid = g;
      nacc = na;
      run(bench<32>, "N=32", 1, 400);
      run(bench<64>, "N=64", 1, 400);
      run(bench<128>, "N=128", 1, 400);
    }
  return 0;
}
