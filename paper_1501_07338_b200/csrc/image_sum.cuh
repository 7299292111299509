// image_sum.cuh -- the fixed-order sum over per-image partials shared by the
// weight-gradient reduce kernel (wgrad.cu) and the SGD update that folds the
// last layer's reduce into itself (direct.cu): a block of 32 x kRedSlices
// threads owns 32 consecutive outputs; slice s sums images
// [s*per_s, (s+1)*per_s) (8 loads in flight), then lane-wise over the slices
// in order.  Deterministic; the same bits wherever it runs.
#pragma once

#include "common.cuh"

namespace vcnn_b200 {

constexpr int kRedSlices = 16;

// block-wide; returns the sum for output `i` (valid in slice 0, i < per)
__device__ __forceinline__ float image_sum(int nimg, int64_t per, int64_t stride, int64_t i,
                                           const float* __restrict__ part,
                                           float (&red)[kRedSlices][33]) {
  const int lane = threadIdx.x & 31, sl = threadIdx.x >> 5;
  const int per_s = (nimg + kRedSlices - 1) / kRedSlices;
  const int b0 = sl * per_s, b1 = b0 + per_s < nimg ? b0 + per_s : nimg;
  float acc = 0.f;
  if (i < per) {
    const float* p = part + i;
    int bb = b0;
    for (; bb + 8 <= b1; bb += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(p + (int64_t)(bb + u) * stride);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
    for (; bb < b1; ++bb) acc += __ldg(p + (int64_t)bb * stride);
  }
  red[sl][lane] = acc;
  __syncthreads();
  float t = 0.f;
  if (sl == 0) {
#pragma unroll
    for (int s2 = 0; s2 < kRedSlices; ++s2) t += red[s2][lane];
  }
  return t;
}

namespace direct {
// out[i] = image_sum over nimg partials (dW then db), wgrad.cu
__global__ void wgrad_reduce_kernel(int nimg, int64_t per, int64_t stride, int64_t nw,
                                    const float* __restrict__ part, float* __restrict__ dw,
                                    float* __restrict__ db);
}  // namespace direct

}  // namespace vcnn_b200
