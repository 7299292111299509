// Micro: cost of one tcgen05.mma.kind::tf32 (M=128 or 64, K=8) by N, by the
// A start alignment (16-byte shifted views, as the direct conv's per-tap
// offsets, vs 128-byte aligned) and with 1 or 2 CTAs per SM.  One thread per
// CTA issues `iters` MMAs back to back (the direct kernels' issue style).
// Diagnostic only.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_align.cu -o mma_align
#include <cstdint>
#include <cstdio>

#include "../../paper_1501_07338_b200/csrc/tc_ptx.cuh"
using namespace vcnn_b200;

template <int N, int M, int UNIT>
__global__ void bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 100 * 1024 / 4; i += blockDim.x) ((float*)s)[i] = 0.f;
  if (threadIdx.x < 32) {
    ptx::tmem_alloc(&tbase, 256);
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
    const uint32_t tm = tbase;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
      ptx::mma_tf32(tm, ad0 + (uint64_t)(UNIT * (i & 63)), bd, id, i > 0);
    unsigned long long t1 = clock64();
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    unsigned long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc(tbase, 256);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  unsigned long long h[2];
  const int smem = 104 * 1024;  // two CTAs fit one SM
  int grid = 1;
  auto run = [&](auto kern, const char* name) {
    const int iters = 400;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int r = 0; r < 3; ++r) kern<<<grid, 128, smem>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("grid %3d %-22s issue %6llu cyc, done %6llu cyc -> %.1f cyc/mma per CTA %s\n", grid,
           name, h[0], h[1], (double)h[1] / iters, cudaGetErrorString(e));
  };
  for (int gsz : {1, 296}) {  // 296 = two CTAs on every SM
    grid = gsz;
    run(bench<32, 128, 1>, "M128 N32 16B-shift");
    run(bench<32, 128, 8>, "M128 N32 128B-shift");
    run(bench<64, 128, 1>, "M128 N64");
    run(bench<128, 128, 1>, "M128 N128");
    run(bench<144, 128, 1>, "M128 N144");
    run(bench<192, 128, 1>, "M128 N192");
    run(bench<256, 128, 1>, "M128 N256");
    run(bench<32, 64, 1>, "M64 N32");
    run(bench<128, 64, 1>, "M64 N128");
  }
  return 0;
}
