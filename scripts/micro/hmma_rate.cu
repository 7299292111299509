// Micro: legacy mma.sync m16n8k8 TF32 issue rate and LDS latency on one SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 hmma_rate.cu -o hmma_rate
#include <cstdio>
#include <cstdint>

__global__ void hmma(int iters, float* out, long long* cyc) {
  float c[4][4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, "
          "{%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void lds_chain(int iters, float* out, long long* cyc) {
  __shared__ int buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x & 1023;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = buf[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void ffma(int iters, float* out, long long* cyc) {
  float c[16];
  for (int j = 0; j < 16; ++j) c[j] = threadIdx.x + j;
  const float x = threadIdx.x * 0.5f, y = 1.0001f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j] = fmaf(c[j], y, x);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 16; ++j) s += c[j];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 1024);
  const int iters = 1000;
  for (int threads : {32, 128, 256, 512}) {
    hmma<<<1, threads>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    hmma<<<1, threads>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    const double n = (double)iters * 4 * (threads / 32);
    printf("hmma tf32 m16n8k8: %4d threads  %.1f cycles per warp-mma per SM  (%.0f FMA/clk/SM)\n",
           threads, (double)cyc[0] / n * (threads / 32) / (threads / 32), n * 1024 / cyc[0]);
  }
  for (int threads : {32, 512}) {
    ffma<<<1, threads>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    ffma<<<1, threads>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    printf("ffma: %d threads  %.0f FMA/clk/SM\n", threads, (double)iters * 16 * threads / cyc[0]);
  }
  lds_chain<<<1, 32>>>(iters, out, cyc);
  cudaDeviceSynchronize();
  lds_chain<<<1, 32>>>(iters, out, cyc);
  cudaDeviceSynchronize();
  printf("lds dependent-chain latency: %.1f cycles\n", (double)cyc[0] / iters);
  return 0;
}
