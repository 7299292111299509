// tcgen05.mma.kind::tf32 issue rate: 64 MMAs (M=128, K=8) per batch from one
// elected lane, descriptors advanced by additions (diagnostic only).
#include <cstdio>
#include <cstdint>
#include "../../paper_1501_07338_b200/csrc/tc_ptx.cuh"
using namespace vcnn_b200;

template <int N, int UNROLL, int STEP, int BSTEP = 0, int TC = 256, int LBOA = 4096,
          int LBOB = 128, int SBOB = 256, int NACC = 1>
__global__ void rate(unsigned long long* out, int batches) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((float*)s)[i] = 0.f;
  if (threadIdx.x < 32) { ptx::tmem_alloc(&tbase, TC); ptx::tmem_relinquish(); }
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = tbase;
  if (threadIdx.x < 32) {
    const uint32_t a = ptx::smem_u32(s);
    const uint64_t ad0 = ptx::interleave_desc(a, LBOA, 128);
    const uint64_t bd0 = ptx::interleave_desc(a + 32768, LBOB, SBOB);
    const uint32_t id = ptx::idesc_tf32(128, N);
    unsigned long long t0 = clock64();
    if (ptx::elect_one()) {
      for (int bt = 0; bt < batches; ++bt) {
#pragma unroll
        for (int i = 0; i < UNROLL; ++i)
          ptx::mma_tf32(tm + (uint32_t)((i % NACC) * N), ad0 + (uint64_t)((i * STEP) & 63), bd0 + (uint64_t)(BSTEP ? (i * BSTEP) & 1023 : (i >> 3) * 2), id, (bt | i) != 0);
      }
      ptx::mma_commit(&bar);
    }
    __syncwarp();
    unsigned long long t1 = clock64();
    ptx::mbar_wait(&bar, 0);
    unsigned long long t2 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc(tm, TC);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  unsigned long long h[2];
  auto run = [&](auto kern, const char* name, int batches, int per, int grid = 1) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
    for (int r = 0; r < 3; ++r) kern<<<grid, 128, 150 * 1024>>>(d, batches);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-10s %5d mmas: issue %7llu cyc, done %7llu cyc -> %.1f cyc/mma (%s)\n", name,
           batches * per, h[0], h[1], (double)h[1] / (batches * per), cudaGetErrorString(e));
    fflush(stdout);
  };
  // the wgrad kernel's operands: A lbo 2048 / sbo 128, B lbo 512 / sbo 128,
  // 10 accumulators, A advancing by granules
  run(rate<32, 16, 1, 64, 512, 2048, 512, 128, 10>, "wgrad-like g1", 32, 16, 1);
  run(rate<32, 16, 1, 64, 512, 2048, 512, 128, 10>, "wgrad-like g128", 32, 16, 128);
  run(rate<32, 16, 1, 64, 512, 2048, 512, 128, 1>, "wgrad-like 1acc", 32, 16, 1);
  run(rate<32, 16, 1, 64, 32, 3072>, "N=32 tc32 l3072 g148", 32, 16, 148);
  run(rate<32, 16, 1, 64, 32, 3072>, "N=32 tc32 l3072 g1", 32, 16, 1);
  run(rate<32, 16, 1, 64, 256, 3072>, "N=32 tc256 l3072", 32, 16, 1);
  run(rate<32, 16, 1, 64>, "N=32 s1 b1K", 32, 16);
  run(rate<32, 16, 0, 64>, "N=32 s0 b1K", 32, 16);
  run(rate<32, 16, 0>, "N=32 s0", 32, 16);
  run(rate<32, 16, 1>, "N=32 s1", 32, 16);
  run(rate<32, 16, 8>, "N=32 s8", 32, 16);
  run(rate<64, 16, 0>, "N=64 s0", 32, 16);
  run(rate<64, 16, 1>, "N=64 s1", 32, 16);
  run(rate<128, 16, 1>, "N=128 s1", 32, 16);
  return 0;
}
