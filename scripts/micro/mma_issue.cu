// Micro: single-CTA issue rate of tcgen05.mma.kind::tf32 (M=128, K=8) for
// three issue styles x accumulator rotation.  V0: one thread (divergent
// branch) issues; V1: warp 0 loops converged, elect_one() per MMA; V2: warp 0
// loops converged, elect.sync + predicated tcgen05.mma in ONE asm block.
// NACC: consecutive MMAs rotate over NACC TMEM accumulators (no RAW chain on
// one accumulator).  Diagnostic only.
#include <cstdint>
#include <cstdio>

#include "../../paper_1501_07338_b200/csrc/tc_ptx.cuh"
using namespace vcnn_b200;

__device__ __forceinline__ void mma_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t id,
                                          uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}

template <int N, int V, int NACC>
__global__ void bench(int iters, unsigned long long* out) {
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
  const uint32_t a = ptx::smem_u32(s), b = a + 64 * 1024;
  const uint32_t id = ptx::idesc_tf32(128, N);
  const uint64_t ad0 = ptx::interleave_desc(a, 2048u * 16u, 128u);
  const uint64_t bd = ptx::interleave_desc(b, 128u, 256u);
  const uint32_t tm = tbase;
  unsigned long long t0 = 0, t1 = 0;
  if (V == 0) {
    if (threadIdx.x == 0) {
      t0 = clock64();
      for (int i = 0; i < iters; i += NACC)
#pragma unroll
        for (int r = 0; r < NACC; ++r)
          ptx::mma_tf32(tm + r * N, ad0 + (uint64_t)((i + r) & 63), bd, id, i > 0);
      t1 = clock64();
      ptx::mma_commit(&bar);
    }
  } else if (threadIdx.x < 32) {
    t0 = clock64();
    for (int i = 0; i < iters; i += NACC)
#pragma unroll
      for (int r = 0; r < NACC; ++r) {
        if (V == 1) {
          if (ptx::elect_one()) ptx::mma_tf32(tm + r * N, ad0 + (uint64_t)((i + r) & 63), bd, id, i > 0);
          __syncwarp();
        } else {
          mma_elect(tm + r * N, ad0 + (uint64_t)((i + r) & 63), bd, id, i > 0);
        }
      }
    t1 = clock64();
    if (ptx::elect_one()) ptx::mma_commit(&bar);
    __syncwarp();
  }
  if (threadIdx.x == 0) {
    ptx::mbar_wait(&bar, 0);
    unsigned long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
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
  auto run = [&](auto kern, const char* name) {
    const int iters = 400;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int r = 0; r < 3; ++r) kern<<<1, 128, smem>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-16s issue %6llu cyc, done %6llu cyc -> %.1f cyc/mma %s\n", name, h[0], h[1],
           (double)h[1] / iters, cudaGetErrorString(e));
  };
  run(bench<32, 0, 1>, "N32 V0 acc1");
  run(bench<32, 0, 4>, "N32 V0 acc4");
  run(bench<32, 1, 1>, "N32 V1 acc1");
  run(bench<32, 1, 4>, "N32 V1 acc4");
  run(bench<32, 2, 1>, "N32 V2 acc1");
  run(bench<32, 2, 2>, "N32 V2 acc2");
  run(bench<32, 2, 4>, "N32 V2 acc4");
  run(bench<64, 2, 1>, "N64 V2 acc1");
  run(bench<64, 2, 4>, "N64 V2 acc4");
  run(bench<128, 0, 1>, "N128 V0 acc1");
  run(bench<128, 2, 1>, "N128 V2 acc1");
  run(bench<128, 2, 2>, "N128 V2 acc2");
  return 0;
}
