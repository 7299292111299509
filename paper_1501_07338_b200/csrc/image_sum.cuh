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

// the same sum for 4 consecutive outputs at once (i4 = output / 4; per and
// stride multiples of 4, part 16-byte aligned): identical per-output order
// and bits, 4x fewer blocks and 16-byte loads
__device__ __forceinline__ float4 image_sum4(int nimg, int64_t per4, int64_t stride4, int64_t i4,
                                             const float4* __restrict__ part,
                                             float4 (&red)[kRedSlices][33]) {
  const int lane = threadIdx.x & 31, sl = threadIdx.x >> 5;
  const int per_s = (nimg + kRedSlices - 1) / kRedSlices;
  const int b0 = sl * per_s, b1 = b0 + per_s < nimg ? b0 + per_s : nimg;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (i4 < per4) {
    const float4* p = part + i4;
    int bb = b0;
    for (; bb + 8 <= b1; bb += 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(p + (int64_t)(bb + u) * stride4);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc.x += v[u].x;
        acc.y += v[u].y;
        acc.z += v[u].z;
        acc.w += v[u].w;
      }
    }
    for (; bb < b1; ++bb) {
      const float4 v = __ldg(p + (int64_t)bb * stride4);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
  }
  red[sl][lane] = acc;
  __syncthreads();
  float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
  if (sl == 0) {
#pragma unroll
    for (int s2 = 0; s2 < kRedSlices; ++s2) {
      t.x += red[s2][lane].x;
      t.y += red[s2][lane].y;
      t.z += red[s2][lane].z;
      t.w += red[s2][lane].w;
    }
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
