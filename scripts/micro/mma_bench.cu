// Microbenchmark: cycles per tcgen05.mma.kind::tf32 (M=128, K=8) issued
// back to back by one thread from shared memory, for no-swizzle K-major and
// SW128 K-major operands and several N.  Diagnostic only.
#include <cstdio>
#include <cstdint>
#include "../../paper_1501_07338_b200/csrc/tc_ptx.cuh"
using namespace vcnn_b200;

template <int N>
__global__ void bench(int mode, int iters, unsigned long long* out, uint32_t lbo_a) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) ((float*)s)[i] = 0.f;
  if (threadIdx.x < 32) { ptx::tmem_alloc(&tbase, 256); ptx::tmem_relinquish(); }
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const bool issuer = mode >= 2 ? (threadIdx.x < 32 && ptx::elect_one()) : threadIdx.x == 0;
  if (mode >= 2 && threadIdx.x < 32) {
    const uint32_t a = ptx::smem_u32(s), b = a + 96 * 1024;
    const uint32_t id = ptx::idesc_tf32(128, N);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      uint64_t ad = ptx::interleave_desc(a + (i % 64) * 16, lbo_a, 128);
      uint64_t bd = ptx::interleave_desc(b, 128, 256);
      if (mode == 2) {
        if (ptx::elect_one()) ptx::mma_tf32(tbase, ad, bd, id, i > 0);
        __syncwarp();
      } else {
        if (issuer) ptx::mma_tf32(tbase, ad, bd, id, i > 0);
      }
    }
    unsigned long long t1 = clock64();
    if (ptx::elect_one()) ptx::mma_commit(&bar);
    __syncwarp();
    ptx::mbar_wait(&bar, 0);
    unsigned long long t2 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  const uint32_t tmem_l = tbase;
  if (mode == 4 && threadIdx.x == 0) {
    const uint32_t a = ptx::smem_u32(s), b = a + 96 * 1024;
    const uint32_t id = ptx::idesc_tf32(128, N);
    const uint64_t ad0 = ptx::interleave_desc(a, lbo_a, 128);
    const uint64_t bd = ptx::interleave_desc(b, 128, 256);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
      ptx::mma_tf32(tmem_l, ad0 + (uint64_t)(i % 64), bd, id, i > 0);
    unsigned long long t1 = clock64();
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    unsigned long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  if (mode < 2 && threadIdx.x == 0) {
    const uint32_t a = ptx::smem_u32(s), b = a + 96 * 1024;
    const uint32_t id = ptx::idesc_tf32(128, N);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      uint64_t ad, bd;
      if (mode == 0) {  // no-swizzle K-major, shifted start (direct conv style)
        ad = ptx::interleave_desc(a + (i % 64) * 16, lbo_a, 128);
        bd = ptx::interleave_desc(b, 128, 256);
      } else {          // SW128 K-major
        ad = ptx::sw128_kmajor_desc(a + (i % 4) * 32);
        bd = ptx::sw128_kmajor_desc(b + (i % 4) * 32);
      }
      ptx::mma_tf32(tbase, ad, bd, id, i > 0);
    }
    unsigned long long t1 = clock64();
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    unsigned long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc(tbase, 256);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  unsigned long long h[2];
  const int smem = 170 * 1024;
  auto run = [&](auto kern, const char* name, int mode, int iters, uint32_t lbo) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int r = 0; r < 3; ++r) kern<<<1, 128, smem>>>(mode, iters, d, lbo);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-6s mode %d iters %4d lbo %5u: issue %6llu cyc, done %6llu cyc -> %.1f cyc/mma %s\n",
           name, mode, iters, lbo, h[0], h[1], (double)h[1] / iters, cudaGetErrorString(e));
  };
  for (int mode = 0; mode < 2; ++mode)
    for (int iters : {25, 100, 400}) {
      run(bench<32>, "N=32", mode, iters, 3072);
      run(bench<64>, "N=64", mode, iters, 3072);
      run(bench<128>, "N=128", mode, iters, 3072);
    }
  for (int mode = 4; mode < 5; ++mode)
    for (int iters : {25, 100, 400}) {
      run(bench<32>, "N=32", mode, iters, 3072);
      run(bench<64>, "N=64", mode, iters, 3072);
      run(bench<128>, "N=128", mode, iters, 3072);
    }
  for (int mode = 0; mode < 1; ++mode)
    for (int iters : {25, 100, 400}) {
      run(bench<32>, "N=32", mode, iters, 3072);
      run(bench<128>, "N=128", mode, iters, 3072);
    }
  return 0;
}
