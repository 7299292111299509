// simt.cu -- memory-bound kernels (index maps, pooling, activations, losses,
// SGD) and the SIMT fp32 reference GEMM/conv path (VCNN_PREC_FP32).
//
// Every kernel is deterministic: reductions run in a fixed order (strided
// per-thread partials + a fixed shared-memory tree), scatters of the
// reference (col2im, pool_backward) are rewritten as gathers so no float
// atomics are needed.  Reference paths: /root/reference/proj/include/vcnn.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "kernels.cuh"

namespace vcnn_b200 {

namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(int64_t n, int threads = kThreads) {
  int64_t g = cdiv(n, threads);
  if (g > (1LL << 30)) g = 1LL << 30;
  return (unsigned)(g < 1 ? 1 : g);
}

inline bool fits32(int64_t v) { return v < (int64_t(1) << 31) - 1; }

// fixed-order block tree reduction (deterministic for a fixed blockDim)
template <int NT>
__device__ __forceinline__ float block_sum(float v, float* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
#pragma unroll
  for (int s = NT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  float r = sh[0];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------
// im2col (vectorize.hpp:54-79): one thread per patch cell, column fastest so
// the patch-matrix writes are coalesced.
__global__ void im2col_kernel(ConvDesc d, const float* __restrict__ x, float* __restrict__ P) {
  PDL_ENTRY();
  const int64_t cols = d.pixels();
  const int64_t total = d.kd() * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / cols, col = i - row * cols;
    const int kx = (int)(row % d.kw);
    const int ky = (int)((row / d.kw) % d.kh);
    const int c = (int)(row / ((int64_t)d.kw * d.kh));
    const int64_t b = col / d.ohw();
    const int64_t r = col - b * d.ohw();
    const int oy = (int)(r / d.OW), ox = (int)(r - (int64_t)oy * d.OW);
    P[i] = x[((b * d.C + c) * d.H + (int64_t)oy * d.s + ky) * d.W + (int64_t)ox * d.s + kx];
  }
}

// col2im (vectorize.hpp:111-120) in gather form: each input cell sums the
// patch cells it fed in (ky,kx) ascending order -- the same per-cell order
// as the reference's pair-ordered scatter (build_col2im_map enumerates
// c,ky,kx,b,oy,ox), so results are bit-identical to a sequential scatter.
template <class I>
__global__ void col2im_kernel(ConvDesc d, const float* __restrict__ dP, float* __restrict__ dX,
                              const float* __restrict__ yprev, int act_prev) {
  PDL_ENTRY();
  const I cols = (I)d.pixels();
  const I total = (I)d.in_size();
  const I ohw = (I)d.ohw();
  for (I i = blockIdx.x * (I)blockDim.x + threadIdx.x; i < total; i += (I)gridDim.x * blockDim.x) {
    const int x = (int)(i % d.W);
    const I t1 = i / d.W;
    const int y = (int)(t1 % d.H);
    const I t2 = t1 / d.H;
    const int c = (int)(t2 % d.C);
    const I b = t2 / d.C;
    float acc = 0.f;
    for (int ky = 0; ky < d.kh; ++ky) {
      const int ty = y - ky;
      if (ty < 0) break;
      if (ty % d.s) continue;
      const int oy = ty / d.s;
      if (oy >= d.OH) continue;
      for (int kx = 0; kx < d.kw; ++kx) {
        const int tx = x - kx;
        if (tx < 0) break;
        if (tx % d.s) continue;
        const int ox = tx / d.s;
        if (ox >= d.OW) continue;
        const I row = ((I)c * d.kh + ky) * d.kw + kx;
        acc += dP[row * cols + b * ohw + (I)oy * d.OW + ox];
      }
    }
    if (yprev) acc *= act_grad_from_out(act_prev, yprev[i]);
    dX[i] = acc;
  }
}

// build_col2im_map (vectorize.hpp:84-106): pair k enumerates
// (row=(c,ky,kx), b, oy, ox); its source is k itself.
__global__ void col2im_map_kernel(ConvDesc d, int64_t* __restrict__ src,
                                  int64_t* __restrict__ tgt) {
  PDL_ENTRY();
  const int64_t cols = d.pixels();
  const int64_t total = d.kd() * cols;
  const int64_t plane = (int64_t)d.H * d.W;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = k / cols, col = k - row * cols;
    const int kx = (int)(row % d.kw);
    const int ky = (int)((row / d.kw) % d.kh);
    const int64_t c = row / ((int64_t)d.kw * d.kh);
    const int64_t b = col / d.ohw();
    const int64_t r = col - b * d.ohw();
    const int64_t oy = r / d.OW, ox = r - oy * d.OW;
    src[k] = k;
    tgt[k] = (b * d.C + c) * plane + (oy * d.s + ky) * d.W + (ox * d.s + kx);
  }
}

// build_pool_map (vectorize.hpp:167-191): pairs (b,c,oy,ox,py,px)
__global__ void pool_map_kernel(PoolDesc d, int64_t* __restrict__ src,
                                int64_t* __restrict__ tgt) {
  PDL_ENTRY();
  const int64_t ws = (int64_t)d.ph * d.pw;
  const int64_t total = d.out_size() * ws;
  const int64_t plane = (int64_t)d.H * d.W;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = k / ws, w = k - t * ws;
    const int py = (int)(w / d.pw), px = (int)(w - (int64_t)py * d.pw);
    const int64_t ox = t % d.OW, oy = (t / d.OW) % d.OH, bc = t / ((int64_t)d.OW * d.OH);
    src[k] = bc * plane + (oy * d.s + py) * d.W + (ox * d.s + px);
    tgt[k] = t;
  }
}

// pool_forward (vectorize.hpp:197-210 -> tensor.hpp:240-289) + pool layer
// bias and activation (layers.hpp:305-321).  Max: the first window element
// seeds, then strict '>' in (py,px) order == ties to the lowest input index,
// and a NaN survives only if it is first (no fmaxf).
template <class IdxT, class I>
__global__ void pool_fwd_kernel(PoolDesc d, const float* __restrict__ x,
                                const float* __restrict__ bias, int act, float* __restrict__ y,
                                IdxT* __restrict__ arg) {
  PDL_ENTRY();
  const I total = (I)d.out_size();
  const I plane = (I)d.H * d.W;
  for (I t = blockIdx.x * (I)blockDim.x + threadIdx.x; t < total; t += (I)gridDim.x * blockDim.x) {
    const int ox = (int)(t % d.OW);
    const I t1 = t / d.OW;
    const int oy = (int)(t1 % d.OH);
    const I bc = t1 / d.OH;
    const I base = bc * plane + (I)oy * d.s * d.W + (I)ox * d.s;
    float v;
    if (d.mode == VCNN_POOL_MAX) {
      float best = x[base];
      I a = base;
      for (int py = 0; py < d.ph; ++py)
        for (int px = 0; px < d.pw; ++px) {
          const I s = base + (I)py * d.W + px;
          const float xv = x[s];
          if (xv > best) {
            best = xv;
            a = s;
          }
        }
      v = best;
      if (arg) arg[t] = (IdxT)a;
    } else {
      float acc = 0.f;
      for (int py = 0; py < d.ph; ++py)
        for (int px = 0; px < d.pw; ++px) acc += x[base + (I)py * d.W + px];
      v = acc / (float)(d.ph * d.pw);
      if (arg) arg[t] = (IdxT)-1;
    }
    if (bias) v += bias[(int)(bc % d.C)];
    y[t] = act_fwd(act, v);
  }
}

// pool_backward (vectorize.hpp:224-249) in gather form: each input cell
// visits its covering windows in window order (the reference's scatter
// order), then the upstream activation derivative is applied.
template <class IdxT, class I>
__global__ void pool_bwd_kernel(PoolDesc d, int bwd_mode, const float* __restrict__ g,
                                const IdxT* __restrict__ arg, float* __restrict__ dx,
                                const float* __restrict__ yprev, int act_prev) {
  PDL_ENTRY();
  const I total = (I)d.in_size();
  const float scale = 1.0f / (float)(d.ph * d.pw);
  for (I i = blockIdx.x * (I)blockDim.x + threadIdx.x; i < total; i += (I)gridDim.x * blockDim.x) {
    const int x = (int)(i % d.W);
    const I t1 = i / d.W;
    const int y = (int)(t1 % d.H);
    const I bc = t1 / d.H;
    int oy0 = y - d.ph + 1;
    oy0 = oy0 <= 0 ? 0 : (oy0 + d.s - 1) / d.s;
    int oy1 = y / d.s;
    if (oy1 > d.OH - 1) oy1 = d.OH - 1;
    int ox0 = x - d.pw + 1;
    ox0 = ox0 <= 0 ? 0 : (ox0 + d.s - 1) / d.s;
    int ox1 = x / d.s;
    if (ox1 > d.OW - 1) ox1 = d.OW - 1;
    float acc = 0.f;
    for (int oy = oy0; oy <= oy1; ++oy)
      for (int ox = ox0; ox <= ox1; ++ox) {
        const I t = (bc * d.OH + oy) * d.OW + ox;
        if (bwd_mode == VCNN_POOLBWD_PAPER_NN) {
          acc += g[t];
        } else if (d.mode == VCNN_POOL_MAX) {
          if ((I)arg[t] == i) acc += g[t];
        } else {
          acc += g[t] * scale;
        }
      }
    if (yprev) acc *= act_grad_from_out(act_prev, yprev[i]);
    dx[i] = acc;
  }
}

// pool bias gradient (layers.hpp:341-351): per-channel sum over batch and
// plane; one block per channel.
__global__ void pool_bias_grad_kernel(PoolDesc d, const float* __restrict__ g,
                                      float* __restrict__ db) {
  PDL_ENTRY();
  __shared__ float sh[kThreads];
  const int c = blockIdx.x;
  const int64_t plane = (int64_t)d.OH * d.OW;
  const int64_t n = plane * d.B;
  float acc = 0.f;
  for (int64_t i = threadIdx.x; i < n; i += kThreads) {
    const int64_t b = i / plane, p = i - b * plane;
    acc += g[(b * d.C + c) * plane + p];
  }
  acc = block_sum<kThreads>(acc, sh);
  if (threadIdx.x == 0) db[c] = acc;
}

__global__ void act_fwd_kernel(int64_t n, int act, const float* __restrict__ x,
                               float* __restrict__ y) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = act_fwd(act, x[i]);
}

__global__ void act_bwd_kernel(int64_t n, int act, const float* __restrict__ y, const float* dy,
                               float* g) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    g[i] = dy[i] * act_grad_from_out(act, y[i]);
}

// loss_forward + loss_backward, softmax-CE (layers.hpp:402-459): one warp
// per sample with shuffle max/sum; per-sample losses summed by thread 0 in
// sample order (the reference's order), then / B.
constexpr int kLossThreads = 1024;
__global__ void __launch_bounds__(kLossThreads) softmax_ce_kernel(
    int B, int units, const float* __restrict__ pred, const int* __restrict__ cls,
    float* __restrict__ loss, float* __restrict__ grad, int act_last, int* err) {
  PDL_ENTRY();
  __shared__ float red[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const float inv_b = 1.0f / (float)B;
  float mine = 0.f;  // lane 0: this warp's per-sample losses, in sample order
  for (int b = warp; b < B; b += nwarps) {
    const float* l = pred + (int64_t)b * units;
    const int c = cls[b];
    const bool bad = c < 0 || c >= units;
    if (bad && lane == 0 && err) atomicExch(err, 1);
    float m = -INFINITY;
    for (int u = lane; u < units; u += 32) m = fmaxf(m, l[u]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float s = 0.f;
    for (int u = lane; u < units; u += 32) s += expf(l[u] - m);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (grad) {
      const float inv = inv_b / s;
      for (int u = lane; u < units; u += 32) {
        float gv = expf(l[u] - m) * inv;
        if (u == c) gv -= inv_b;
        if (act_last != VCNN_ACT_IDENTITY) gv *= act_grad_from_out(act_last, l[u]);
        grad[(int64_t)b * units + u] = gv;
      }
    }
    if (!bad) mine += m + logf(s) - l[c];
  }
  // fixed-order reduction of the warps' partial sums -> deterministic
  if (lane == 0) red[warp] = mine;
  __syncthreads();
  if (warp == 0) {
    float v = lane < nwarps ? red[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0 && loss) *loss = v / (float)B;
  }
}

// MSE (layers.hpp:425-433, :461-467): loss = mean (p-t)^2, grad 2(p-t)/n
__global__ void __launch_bounds__(kLossThreads) mse_kernel(int64_t n, const float* __restrict__ p, const float* __restrict__ t,
                           float* __restrict__ loss, float* __restrict__ grad, int act_last) {
  PDL_ENTRY();
  __shared__ float sh[kLossThreads];
  const float scale = 2.0f / (float)n;
  float acc = 0.f;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const float dd = p[i] - t[i];
    acc += dd * dd;
    if (grad) {
      float gv = scale * dd;
      if (act_last != VCNN_ACT_IDENTITY) gv *= act_grad_from_out(act_last, p[i]);
      grad[i] = gv;
    }
  }
  acc = block_sum<kLossThreads>(acc, sh);
  if (threadIdx.x == 0 && loss) *loss = acc / (float)n;
}

// MSE over many CTAs: CTA i owns the contiguous chunk [i*chunk, (i+1)*chunk)
// (float4 when the pointers allow), writes its fixed-order partial, and the
// last CTA to finish sums the partials in CTA order and re-arms the counter.
// The chunking depends only on n, so the loss is deterministic.
constexpr int kMseThreads = 512;
__global__ void __launch_bounds__(kMseThreads) mse_multi_kernel(
    int64_t n, int64_t chunk, const float* __restrict__ p, const float* __restrict__ t,
    float* __restrict__ loss, float* __restrict__ grad, int act_last, float* ws, int vec) {
  PDL_ENTRY();
  __shared__ float sh[kMseThreads];
  __shared__ bool last;
  const float scale = 2.0f / (float)n;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = lo + chunk < n ? lo + chunk : n;
  float acc = 0.f;
  auto one = [&](float pv, float tv, float& gv) {
    const float dd = pv - tv;
    acc += dd * dd;
    gv = scale * dd;
    if (act_last != VCNN_ACT_IDENTITY) gv *= act_grad_from_out(act_last, pv);
  };
  if (vec) {  // lo, hi multiples of 4 except possibly hi == n
    const int64_t h4 = lo + ((hi - lo) & ~int64_t(3));
    for (int64_t i = lo + 4 * (int64_t)threadIdx.x; i < h4; i += 4 * kMseThreads) {
      const float4 pv = *reinterpret_cast<const float4*>(p + i);
      const float4 tv = *reinterpret_cast<const float4*>(t + i);
      float4 g;
      one(pv.x, tv.x, g.x);
      one(pv.y, tv.y, g.y);
      one(pv.z, tv.z, g.z);
      one(pv.w, tv.w, g.w);
      if (grad) *reinterpret_cast<float4*>(grad + i) = g;
    }
    for (int64_t i = h4 + threadIdx.x; i < hi; i += kMseThreads) {
      float g;
      one(p[i], t[i], g);
      if (grad) grad[i] = g;
    }
  } else {
    for (int64_t i = lo + threadIdx.x; i < hi; i += kMseThreads) {
      float g;
      one(p[i], t[i], g);
      if (grad) grad[i] = g;
    }
  }
  acc = block_sum<kMseThreads>(acc, sh);
  unsigned* counter = reinterpret_cast<unsigned*>(ws + kMseMaxCtas);
  if (threadIdx.x == 0) {
    ws[blockIdx.x] = acc;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  float v = 0.f;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += kMseThreads) v += ((volatile float*)ws)[i];
  v = block_sum<kMseThreads>(v, sh);
  if (threadIdx.x == 0) {
    if (loss) *loss = v / (float)n;
    *counter = 0u;
  }
}

// sgd_step (network.hpp:242-273): v = mom*v + g; w -= lr*v
__global__ void sgd_kernel(int64_t n, float* __restrict__ w, float* __restrict__ v,
                           const float* __restrict__ g, float lr, float mom, float scale,
                           int vec) {
  PDL_ENTRY();
  const int64_t n4 = vec ? (n >> 2) : 0;
  float4* w4 = reinterpret_cast<float4*>(w);
  float4* v4 = reinterpret_cast<float4*>(v);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 wv = w4[i], vv = v4[i], gv = g4[i];
    vv.x = mom * vv.x + scale * gv.x;
    vv.y = mom * vv.y + scale * gv.y;
    vv.z = mom * vv.z + scale * gv.z;
    vv.w = mom * vv.w + scale * gv.w;
    wv.x -= lr * vv.x;
    wv.y -= lr * vv.y;
    wv.z -= lr * vv.z;
    wv.w -= lr * vv.w;
    w4[i] = wv;
    v4[i] = vv;
  }
  for (int64_t i = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const float vv = mom * v[i] + scale * g[i];
    v[i] = vv;
    w[i] -= lr * vv;
  }
}

// generic accumulate_by_index / accumulate_max_arg (tensor.hpp:228-289):
// pairs stably sorted by target, so each bucket is reduced in map order.
__global__ void accumulate_kernel(const float* __restrict__ values,
                                  const int64_t* __restrict__ skeys,
                                  const int64_t* __restrict__ sidx,
                                  const int64_t* __restrict__ source, int64_t pairs,
                                  int64_t target_len, int reducer, float* __restrict__ out,
                                  int64_t* __restrict__ arg) {
  PDL_ENTRY();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < target_len;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = pairs;  // lower_bound(t)
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (skeys[mid] < t) lo = mid + 1; else hi = mid;
    }
    float acc = 0.f;
    int64_t a = -1, cnt = 0;
    for (int64_t p = lo; p < pairs && skeys[p] == t; ++p) {
      const int64_t s = source[sidx[p]];
      const float v = values[s];
      if (reducer == VCNN_REDUCE_MAX) {
        if (arg) {
          if (a < 0 || v > acc || (v == acc && s < a)) {
            acc = v;
            a = s;
          }
        } else if (cnt == 0 || v > acc) {
          acc = v;
        }
      } else {
        acc += v;
      }
      ++cnt;
    }
    if (reducer == VCNN_REDUCE_MEAN && cnt > 0) acc /= (float)cnt;
    if (cnt == 0) acc = 0.f;
    out[t] = acc;
    if (arg) arg[t] = a;
  }
}

__global__ void iota_kernel(int64_t n, int64_t* __restrict__ v) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = i;
}

// ---------------------------------------------------------------------------
// SIMT fp32 GEMM-shaped kernels (VCNN_PREC_FP32).  Straight restatements
// with ascending-k accumulation; block-tree reductions where the reduction
// dimension is the batch.
__global__ void conv_fwd_simt(ConvDesc d, const float* __restrict__ x,
                              const float* __restrict__ w, const float* __restrict__ b, int act,
                              float* __restrict__ y) {
  PDL_ENTRY();
  const int64_t total = d.out_size();
  const int64_t kd = d.kd();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int ox = (int)(i % d.OW), oy = (int)((i / d.OW) % d.OH);
    const int n = (int)((i / d.ohw()) % d.K);
    const int64_t bb = i / (d.ohw() * d.K);
    const float* wr = w + n * kd;
    const float* xb = x + bb * d.C * d.H * d.W + (int64_t)oy * d.s * d.W + (int64_t)ox * d.s;
    float acc = 0.f;
    for (int c = 0; c < d.C; ++c)
      for (int ky = 0; ky < d.kh; ++ky)
        for (int kx = 0; kx < d.kw; ++kx)
          acc += wr[((int64_t)c * d.kh + ky) * d.kw + kx] *
                 xb[((int64_t)c * d.H + ky) * d.W + kx];
    y[i] = act_fwd(act, acc + b[n]);
  }
}

// one block per (n, k) of dW, plus blocks k == kd computing db[n]
__global__ void conv_wgrad_simt(ConvDesc d, const float* __restrict__ x,
                                const float* __restrict__ g, float* __restrict__ dw,
                                float* __restrict__ db) {
  PDL_ENTRY();
  __shared__ float sh[kThreads];
  const int64_t kd = d.kd();
  const int64_t k = blockIdx.x;  // 0..kd (kd = bias)
  const int n = blockIdx.y;
  const int64_t pix = d.pixels();
  int c = 0, ky = 0, kx = 0;
  if (k < kd) {
    kx = (int)(k % d.kw);
    ky = (int)((k / d.kw) % d.kh);
    c = (int)(k / ((int64_t)d.kw * d.kh));
  }
  float acc = 0.f;
  for (int64_t p = threadIdx.x; p < pix; p += kThreads) {
    const int64_t bb = p / d.ohw(), r = p - bb * d.ohw();
    const int oy = (int)(r / d.OW), ox = (int)(r - (int64_t)oy * d.OW);
    const float gv = g[(bb * d.K + n) * d.ohw() + r];
    if (k < kd)
      acc += gv * x[((bb * d.C + c) * d.H + (int64_t)oy * d.s + ky) * d.W + (int64_t)ox * d.s + kx];
    else
      acc += gv;
  }
  acc = block_sum<kThreads>(acc, sh);
  if (threadIdx.x == 0) {
    if (k < kd) dw[(int64_t)n * kd + k] = acc;
    else db[n] = acc;
  }
}

__global__ void conv_dgrad_simt(ConvDesc d, const float* __restrict__ g,
                                const float* __restrict__ w, float* __restrict__ dx,
                                const float* __restrict__ yprev, int act_prev) {
  PDL_ENTRY();
  const int64_t total = d.in_size();
  const int64_t kd = d.kd();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % d.W), y = (int)((i / d.W) % d.H);
    const int c = (int)((i / ((int64_t)d.W * d.H)) % d.C);
    const int64_t bb = i / ((int64_t)d.W * d.H * d.C);
    float acc = 0.f;
    for (int n = 0; n < d.K; ++n) {
      const float* gb = g + (bb * d.K + n) * d.ohw();
      const float* wr = w + n * kd + (int64_t)c * d.kh * d.kw;
      for (int ky = 0; ky < d.kh; ++ky) {
        const int ty = y - ky;
        if (ty < 0 || ty % d.s) continue;
        const int oy = ty / d.s;
        if (oy >= d.OH) continue;
        for (int kx = 0; kx < d.kw; ++kx) {
          const int tx = x - kx;
          if (tx < 0 || tx % d.s) continue;
          const int ox = tx / d.s;
          if (ox >= d.OW) continue;
          acc += wr[ky * d.kw + kx] * gb[(int64_t)oy * d.OW + ox];
        }
      }
    }
    if (yprev) acc *= act_grad_from_out(act_prev, yprev[i]);
    dx[i] = acc;
  }
}

__global__ void full_fwd_simt(int B, int in, int out, const float* __restrict__ x,
                              const float* __restrict__ w, const float* __restrict__ b, int act,
                              float* __restrict__ y) {
  PDL_ENTRY();
  const int64_t total = (int64_t)B * out;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int o = (int)(i % out);
    const int64_t bb = i / out;
    const float* xr = x + bb * in;
    const float* wr = w + (int64_t)o * in;
    // 4 independent partial sums (loads of 4 iterations in flight), fixed
    // combination order -> deterministic
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int k = 0;
#pragma unroll 2
    for (; k + 3 < in; k += 4) {
      a0 += xr[k] * wr[k];
      a1 += xr[k + 1] * wr[k + 1];
      a2 += xr[k + 2] * wr[k + 2];
      a3 += xr[k + 3] * wr[k + 3];
    }
    for (; k < in; ++k) a0 += xr[k] * wr[k];
    y[i] = act_fwd(act, ((a0 + a1) + (a2 + a3)) + b[o]);
  }
}

// dW[o][i] = sum_b g[b][o] x[b][i]; column i == in gives db[o]
__global__ void full_wgrad_simt(int B, int in, int out, const float* __restrict__ x,
                                const float* __restrict__ g, float* __restrict__ dw,
                                float* __restrict__ db) {
  PDL_ENTRY();
  const int64_t total = (int64_t)out * (in + 1);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t % (in + 1));
    const int o = (int)(t / (in + 1));
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int bb = 0;
    if (i < in) {
#pragma unroll 2
      for (; bb + 3 < B; bb += 4) {
        a0 += g[(int64_t)bb * out + o] * x[(int64_t)bb * in + i];
        a1 += g[(int64_t)(bb + 1) * out + o] * x[(int64_t)(bb + 1) * in + i];
        a2 += g[(int64_t)(bb + 2) * out + o] * x[(int64_t)(bb + 2) * in + i];
        a3 += g[(int64_t)(bb + 3) * out + o] * x[(int64_t)(bb + 3) * in + i];
      }
      for (; bb < B; ++bb) a0 += g[(int64_t)bb * out + o] * x[(int64_t)bb * in + i];
      dw[(int64_t)o * in + i] = (a0 + a1) + (a2 + a3);
    } else {
#pragma unroll 2
      for (; bb + 3 < B; bb += 4) {
        a0 += g[(int64_t)bb * out + o];
        a1 += g[(int64_t)(bb + 1) * out + o];
        a2 += g[(int64_t)(bb + 2) * out + o];
        a3 += g[(int64_t)(bb + 3) * out + o];
      }
      for (; bb < B; ++bb) a0 += g[(int64_t)bb * out + o];
      db[o] = (a0 + a1) + (a2 + a3);
    }
  }
}

__global__ void full_dgrad_simt(int B, int in, int out, const float* __restrict__ g,
                                const float* __restrict__ w, float* __restrict__ dx,
                                const float* __restrict__ yprev, int act_prev) {
  PDL_ENTRY();
  const int64_t total = (int64_t)B * in;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t % in);
    const int64_t bb = t / in;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int o = 0;
#pragma unroll 2
    for (; o + 3 < out; o += 4) {
      a0 += g[bb * out + o] * w[(int64_t)o * in + i];
      a1 += g[bb * out + o + 1] * w[(int64_t)(o + 1) * in + i];
      a2 += g[bb * out + o + 2] * w[(int64_t)(o + 2) * in + i];
      a3 += g[bb * out + o + 3] * w[(int64_t)(o + 3) * in + i];
    }
    for (; o < out; ++o) a0 += g[bb * out + o] * w[(int64_t)o * in + i];
    float acc = (a0 + a1) + (a2 + a3);
    if (yprev) acc *= act_grad_from_out(act_prev, yprev[t]);
    dx[t] = acc;
  }
}

__global__ void matmul_simt(int64_t m, int64_t k, int64_t n, const float* __restrict__ a,
                            const float* __restrict__ b, float* __restrict__ c, bool transB) {
  PDL_ENTRY();
  const int64_t total = m * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t % n, i = t / n;
    float acc = 0.f;
    if (transB)
      for (int64_t q = 0; q < k; ++q) acc += a[i * k + q] * b[j * k + q];
    else
      for (int64_t q = 0; q < k; ++q) acc += a[i * k + q] * b[q * n + j];
    c[t] = acc;
  }
}

// general strided GEMM, fp32 FMA in ascending k (the reference matmul's
// order, tensor.hpp:131-174) + bias[n] + activation
__global__ void gemm_simt(int64_t m, int64_t n, int64_t k, const float* __restrict__ a,
                          int64_t as_m, int64_t as_k, const float* __restrict__ b, int64_t bs_k,
                          int64_t bs_n, float* __restrict__ c, int64_t ldc,
                          const float* __restrict__ bias, int act) {
  PDL_ENTRY();
  const int64_t total = m * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t % n, i = t / n;
    float acc = 0.f;
    for (int64_t q = 0; q < k; ++q) acc += a[i * as_m + q * as_k] * b[q * bs_k + j * bs_n];
    if (bias) acc += bias[j];
    c[i * ldc + j] = act_fwd(act, acc);
  }
}

}  // namespace

// ===========================================================================
// launchers
// ===========================================================================
int launch_im2col(const ConvDesc& d, const float* x, float* P, cudaStream_t st) {
  VCNN_CUDA_TRY(launch_pdl(im2col_kernel, dim3(grid_for(d.kd() * d.pixels())), dim3(kThreads), 0, st, d, x, P));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int launch_col2im(const ConvDesc& d, const float* dP, float* dX, cudaStream_t st,
                  const float* yprev, int act_prev) {
  if (fits32(d.in_size()) && fits32(d.kd() * d.pixels()))
    VCNN_CUDA_TRY(launch_pdl(col2im_kernel<int>, dim3(grid_for(d.in_size())), dim3(kThreads), 0, st, d, dP, dX, yprev, act_prev));
  else
    VCNN_CUDA_TRY(launch_pdl(col2im_kernel<int64_t>, dim3(grid_for(d.in_size())), dim3(kThreads), 0, st, d, dP, dX, yprev, act_prev));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int launch_col2im_map(const ConvDesc& d, int64_t* src, int64_t* tgt, cudaStream_t st) {
  VCNN_CUDA_TRY(launch_pdl(col2im_map_kernel, dim3(grid_for(d.kd() * d.pixels())), dim3(kThreads), 0, st, d, src, tgt));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int launch_pool_map(const PoolDesc& d, int64_t* src, int64_t* tgt, cudaStream_t st) {
  VCNN_CUDA_TRY(launch_pdl(pool_map_kernel, dim3(grid_for(d.out_size() * d.ph * d.pw)), dim3(kThreads), 0, st, d, src, tgt));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

template <class IdxT>
int launch_pool_fwd(const PoolDesc& d, const float* x, const float* bias, int act, float* y,
                    IdxT* arg, cudaStream_t st) {
  if (fits32(d.in_size()))
    VCNN_CUDA_TRY(launch_pdl(pool_fwd_kernel<IdxT, int>, dim3(grid_for(d.out_size())), dim3(kThreads), 0, st, d, x, bias, act, y, arg));
  else
    VCNN_CUDA_TRY(launch_pdl(pool_fwd_kernel<IdxT, int64_t>, dim3(grid_for(d.out_size())), dim3(kThreads), 0, st, d, x, bias, act, y,
                                                                                arg));
  VCNN_LAUNCHED();
  return VCNN_OK;
}
template int launch_pool_fwd<int32_t>(const PoolDesc&, const float*, const float*, int, float*,
                                      int32_t*, cudaStream_t);
template int launch_pool_fwd<int64_t>(const PoolDesc&, const float*, const float*, int, float*,
                                      int64_t*, cudaStream_t);

template <class IdxT>
int launch_pool_bwd(const PoolDesc& d, int bwd_mode, const float* gpre, const IdxT* arg,
                    float* dx, const float* yprev, int act_prev, cudaStream_t st) {
  if (fits32(d.in_size()))
    VCNN_CUDA_TRY(launch_pdl(pool_bwd_kernel<IdxT, int>, dim3(grid_for(d.in_size())), dim3(kThreads), 0, st, d, bwd_mode, gpre, arg,
                                                                           dx, yprev, act_prev));
  else
    VCNN_CUDA_TRY(launch_pdl(pool_bwd_kernel<IdxT, int64_t>, dim3(grid_for(d.in_size())), dim3(kThreads), 0, st, 
        d, bwd_mode, gpre, arg, dx, yprev, act_prev));
  VCNN_LAUNCHED();
  return VCNN_OK;
}
template int launch_pool_bwd<int32_t>(const PoolDesc&, int, const float*, const int32_t*, float*,
                                      const float*, int, cudaStream_t);
template int launch_pool_bwd<int64_t>(const PoolDesc&, int, const float*, const int64_t*, float*,
                                      const float*, int, cudaStream_t);

int launch_pool_bias_grad(const PoolDesc& d, const float* gpre, float* dbias, cudaStream_t st) {
  VCNN_CUDA_TRY(launch_pdl(pool_bias_grad_kernel, dim3(d.C), dim3(kThreads), 0, st, d, gpre, dbias));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int launch_act_fwd(int64_t n, int act, const float* x, float* y, cudaStream_t st) {
  VCNN_CUDA_TRY(launch_pdl(act_fwd_kernel, dim3(grid_for(n)), dim3(kThreads), 0, st, n, act, x, y));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int launch_act_bwd(int64_t n, int act, const float* y, const float* dy, float* g,
                   cudaStream_t st) {
  VCNN_CUDA_TRY(launch_pdl(act_bwd_kernel, dim3(grid_for(n)), dim3(kThreads), 0, st, n, act, y, dy, g));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int launch_loss(int kind, int B, int units, const float* pred, const int* cls,
                const float* values, float* loss, float* grad, int act_last, int* err,
                cudaStream_t st, float* ws) {
  const int64_t n = (int64_t)B * units;
  if (kind == VCNN_LOSS_MSE && ws && n >= 32768) {
    // ~16K elements per CTA, chunk a multiple of 4 so float4 runs stay aligned
    int64_t ctas = cdiv(n, 16384);
    if (ctas > kMseMaxCtas) ctas = kMseMaxCtas;
    const int64_t chunk = (cdiv(n, ctas) + 3) & ~int64_t(3);
    ctas = cdiv(n, chunk);
    const int vec = ((reinterpret_cast<uintptr_t>(pred) | reinterpret_cast<uintptr_t>(values) |
                      reinterpret_cast<uintptr_t>(grad)) & 15) == 0;
    VCNN_CUDA_TRY(launch_pdl(mse_multi_kernel, dim3((unsigned)ctas), dim3(kMseThreads), 0, st, n,
                             chunk, pred, values, loss, grad, act_last, ws, vec));
    VCNN_LAUNCHED();
    return VCNN_OK;
  }
  if (kind == VCNN_LOSS_SOFTMAX_CE) {
    VCNN_CUDA_TRY(launch_pdl(softmax_ce_kernel, dim3(1), dim3(kLossThreads), 0, st, B, units, pred, cls, loss, grad, act_last, err));
  } else {
    VCNN_CUDA_TRY(launch_pdl(mse_kernel, dim3(1), dim3(kLossThreads), 0, st, (int64_t)B * units, pred, values, loss, grad,
                                           act_last));
  }
  VCNN_LAUNCHED();
  return VCNN_OK;
}

// The network head in ONE kernel: the last full layer forward, the loss
// forward + backward, and the layer's weight / bias / data gradients
// (full_forward + loss_forward/backward + full_backward_core, layers.hpp:
// 230-267, :402-468), replacing 4 launches on the critical path.  One thread-
// block cluster: CTA r owns batch rows [r*R, (r+1)*R) for the forward, the
// loss and dx; its partial dW/db over those rows stays in its shared memory
// and, after a cluster barrier, CTA r reduces slice r of dW/db over the
// cluster's CTAs through distributed shared memory in rank order (CTA 0 also
// the loss).  fp32 throughout, every reduction in a fixed order.
constexpr int kHeadThreads = 256;
constexpr int kHeadCluster = 8;

__global__ void __launch_bounds__(kHeadThreads) head_kernel(
    int B, int in, int out, const float* __restrict__ x, const float* __restrict__ W,
    const float* __restrict__ bias, int act, float* __restrict__ y, int loss_kind,
    const int* __restrict__ cls, const float* __restrict__ values, float* __restrict__ loss,
    float* __restrict__ gpre, float* __restrict__ dW, float* __restrict__ db,
    float* __restrict__ dx, int act_prev, int* __restrict__ err) {
  PDL_ENTRY();
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks(), rank = (int)cluster.block_rank();
  const int R = (B + C - 1) / C;
  const int r0 = rank * R < B ? rank * R : B;
  const int nr = (r0 + R <= B ? R : B - r0);
  const int ld = in + 1;  // padded rows: conflict-free strided reads
  const int np = out * ld;  // dW row o = [dW[o][0..in), db[o]]
  extern __shared__ float hs[];
  float* part = hs;                  // [out][ld] partial dW | db over my rows
  float* ws = part + np;             // [out][ld]
  float* xs = ws + np;               // [R][ld]
  float* gs = xs + (size_t)R * ld;   // [R][out]: y, then the gradient
  __shared__ float red[32];
  __shared__ float loss_part;
  const int tid = threadIdx.x, nt = blockDim.x;
  const float* xg = x + (size_t)r0 * in;
  for (int i = tid; i < nr * in; i += nt) xs[i + i / in] = xg[i];
  for (int i = tid; i < out * in; i += nt) ws[i + i / in] = W[i];
  __syncthreads();
  // forward: y = act(x W^T + b)
  for (int t = tid; t < nr * out; t += nt) {
    const int bb = t / out, o = t - bb * out;
    const float* xr = xs + (size_t)bb * ld;
    const float* wr = ws + (size_t)o * ld;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int k = 0;
    for (; k + 3 < in; k += 4) {
      a0 += xr[k] * wr[k];
      a1 += xr[k + 1] * wr[k + 1];
      a2 += xr[k + 2] * wr[k + 2];
      a3 += xr[k + 3] * wr[k + 3];
    }
    for (; k < in; ++k) a0 += xr[k] * wr[k];
    const float v = act_fwd(act, ((a0 + a1) + (a2 + a3)) + bias[o]);
    gs[t] = v;
    y[(size_t)r0 * out + t] = v;
  }
  __syncthreads();
  // loss + dL/dy * act'(y): one thread per sample (softmax-CE) or element (MSE)
  float mine = 0.f;
  if (loss_kind == VCNN_LOSS_SOFTMAX_CE) {
    const float inv_b = 1.0f / (float)B;
    for (int bb = tid; bb < nr; bb += nt) {
      float* l = gs + (size_t)bb * out;
      const int c = cls[r0 + bb];
      const bool bad = c < 0 || c >= out;
      if (bad && err) atomicExch(err, 1);
      float m = l[0];
      for (int u = 1; u < out; ++u) m = fmaxf(m, l[u]);
      float sum = 0.f;
      for (int u = 0; u < out; ++u) sum += expf(l[u] - m);
      if (!bad) mine += m + logf(sum) - l[c];
      const float inv = inv_b / sum;
      for (int u = 0; u < out; ++u) {
        const float yv = l[u];
        float gv = expf(yv - m) * inv;
        if (u == c) gv -= inv_b;
        if (act != VCNN_ACT_IDENTITY) gv *= act_grad_from_out(act, yv);
        l[u] = gv;
      }
    }
  } else {
    const float scale = 2.0f / (float)(B * out);
    const float* vg = values + (size_t)r0 * out;
    for (int t = tid; t < nr * out; t += nt) {
      const float yv = gs[t], dd = yv - vg[t];
      mine += dd * dd;
      float gv = scale * dd;
      if (act != VCNN_ACT_IDENTITY) gv *= act_grad_from_out(act, yv);
      gs[t] = gv;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((tid & 31) == 0) red[tid >> 5] = mine;
  __syncthreads();
  if (tid < 32) {
    float v = tid < (nt >> 5) ? red[tid] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (tid == 0) loss_part = v;
  }
  for (int t = tid; t < nr * out; t += nt) gpre[(size_t)r0 * out + t] = gs[t];
  // partial dW[o][i] = sum_{my b} g[b][o] x[b][i]; db[o] = sum_{my b} g[b][o]
  for (int t = tid; t < np; t += nt) {
    const int o = t / ld, i = t - o * ld;
    float a0 = 0.f, a1 = 0.f;
    int bb = 0;
    if (i < in) {
      for (; bb + 1 < nr; bb += 2) {
        a0 += gs[bb * out + o] * xs[(size_t)bb * ld + i];
        a1 += gs[(bb + 1) * out + o] * xs[(size_t)(bb + 1) * ld + i];
      }
      for (; bb < nr; ++bb) a0 += gs[bb * out + o] * xs[(size_t)bb * ld + i];
    } else {
      for (; bb + 1 < nr; bb += 2) {
        a0 += gs[bb * out + o];
        a1 += gs[(bb + 1) * out + o];
      }
      for (; bb < nr; ++bb) a0 += gs[bb * out + o];
    }
    part[t] = a0 + a1;
  }
  // dx[b][i] = (sum_o g[b][o] W[o][i]) * act_prev'(x[b][i])
  if (dx) {
    float* dxg = dx + (size_t)r0 * in;
    for (int t = tid; t < nr * in; t += nt) {
      const int bb = t / in, i = t - bb * in;
      float acc = 0.f;
      for (int o = 0; o < out; ++o) acc += gs[bb * out + o] * ws[(size_t)o * ld + i];
      if (act_prev != VCNN_ACT_IDENTITY)
        acc *= act_grad_from_out(act_prev, xs[(size_t)bb * ld + i]);
      dxg[t] = acc;
    }
  }
  cluster.sync();  // every CTA's partials are visible cluster-wide
  const int per = (np + C - 1) / C;
  const int e0 = rank * per, e1 = e0 + per < np ? e0 + per : np;
  for (int e = e0 + tid; e < e1; e += nt) {
    float acc = 0.f;
    for (int c = 0; c < C; ++c) acc += *cluster.map_shared_rank(part + e, c);
    const int o = e / ld, i = e - o * ld;
    if (i < in) dW[(size_t)o * in + i] = acc;
    else db[o] = acc;
  }
  if (rank == 0 && tid == 0 && loss) {
    float v = 0.f;
    for (int c = 0; c < C; ++c) v += *cluster.map_shared_rank(&loss_part, c);
    *loss = loss_kind == VCNN_LOSS_SOFTMAX_CE ? v / (float)B : v / (float)(B * out);
  }
  cluster.sync();  // no CTA leaves while its shared memory is being read
}

static int head_cluster(int B) { return B < kHeadCluster ? (B > 0 ? B : 1) : kHeadCluster; }

size_t head_smem_floats(int B, int in, int out) {
  const int C = head_cluster(B), R = (B + C - 1) / C;
  return 2 * (size_t)out * (in + 1) + (size_t)R * (in + 1) + (size_t)R * out;
}

bool head_fusable(int B, int in, int out) {
  return head_smem_floats(B, in, out) * sizeof(float) <= 160 * 1024 &&
         (int64_t)B * in * out <= (1 << 20);
}

int launch_head(int B, int in, int out, const float* x, const float* W, const float* bias,
                int act, float* y, int loss_kind, const int* cls, const float* values,
                float* loss, float* gpre, float* dW, float* db, float* dx, int act_prev, int* err,
                cudaStream_t st) {
  const size_t smem = sizeof(float) * head_smem_floats(B, in, out);
  static size_t configured = 0;
  if (smem > configured) {
    VCNN_CUDA_TRY(cudaFuncSetAttribute(head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    configured = smem;
  }
  const int C = head_cluster(B);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kHeadThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = C;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  VCNN_CUDA_TRY(cudaLaunchKernelEx(&cfg, head_kernel, B, in, out, x, W, bias, act, y, loss_kind,
                                   cls, values, loss, gpre, dW, db, dx, act_prev, err));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

// gather_batch (network.hpp:165-176) on the device: row j of the batch =
// dataset sample order[start + j]; labels / value targets alongside
__global__ void gather_rows_kernel(int n, int64_t per, const float* __restrict__ src,
                                   const int* __restrict__ order, int start,
                                   float* __restrict__ dst, int64_t tper,
                                   const int* __restrict__ cls_src, int* __restrict__ cls_dst,
                                   const float* __restrict__ val_src, float* __restrict__ val_dst) {
  PDL_ENTRY();
  const int j = blockIdx.y;
  if (j >= n) return;
  const int64_t id = order[start + j];
  const float* s = src + id * per;
  float* d = dst + (int64_t)j * per;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < per;
       i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[i];
  if (blockIdx.x == 0) {
    if (cls_src && threadIdx.x == 0) cls_dst[j] = cls_src[id];
    if (val_src)
      for (int64_t i = threadIdx.x; i < tper; i += blockDim.x)
        val_dst[(int64_t)j * tper + i] = val_src[id * tper + i];
  }
}

int launch_gather_rows(int n, int64_t per, const float* src, const int* order, int start,
                       float* dst, int64_t tper, const int* cls_src, int* cls_dst,
                       const float* val_src, float* val_dst, cudaStream_t st) {
  int64_t bx = cdiv(per, kThreads);
  if (bx > 8) bx = 8;
  VCNN_CUDA_TRY(launch_pdl(gather_rows_kernel, dim3((unsigned)bx, (unsigned)n), dim3(kThreads), 0,
                           st, n, per, src, order, start, dst, tper, cls_src, cls_dst, val_src,
                           val_dst));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

// losses[i] = *loss (device scalar copy into the epoch's loss history)
__global__ void store_scalar_kernel(const float* __restrict__ src, float* __restrict__ dst) {
  PDL_ENTRY();
  if (threadIdx.x == 0) *dst = *src;
}

// stage a device batch into the net's input slots: the images (float4 when
// 16-byte aligned) and the targets (32-bit words) in ONE launch -- a kernel
// between two graph launches pipelines; two copy-engine memcpys did not
__global__ void stage_batch_kernel(const float* __restrict__ xs, float* __restrict__ xd, int64_t nx,
                                   const uint32_t* __restrict__ ts, uint32_t* __restrict__ td,
                                   int64_t nt, int vec) {
  PDL_ENTRY();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (vec) {
    const float4* s4 = reinterpret_cast<const float4*>(xs);
    float4* d4 = reinterpret_cast<float4*>(xd);
    for (int64_t i = i0; i < nx / 4; i += stride) d4[i] = __ldg(s4 + i);
    for (int64_t i = nx / 4 * 4 + i0; i < nx; i += stride) xd[i] = __ldg(xs + i);
  } else {
    for (int64_t i = i0; i < nx; i += stride) xd[i] = __ldg(xs + i);
  }
  for (int64_t i = i0; i < nt; i += stride) td[i] = __ldg(ts + i);
}

int launch_stage_batch(const float* xs, float* xd, int64_t nx, const void* ts, void* td,
                       int64_t nt_words, cudaStream_t st) {
  const int vec = ((reinterpret_cast<uintptr_t>(xs) | reinterpret_cast<uintptr_t>(xd)) & 15) == 0;
  int64_t blocks = cdiv(vec ? nx / 4 + 1 : nx, 256);
  if (blocks > 2 * sm_count()) blocks = 2 * sm_count();
  if (blocks < 1) blocks = 1;
  VCNN_CUDA_TRY(launch_pdl(stage_batch_kernel, dim3((unsigned)blocks), dim3(256), 0, st, xs, xd,
                           nx, static_cast<const uint32_t*>(ts), static_cast<uint32_t*>(td),
                           ts ? nt_words : (int64_t)0, vec));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

// the ring variant: the batch index is the step counter cursor[2] (mod
// nbatch), advanced by the step's update kernel (sgd_pack), so this kernel
// only reads it -- no ticket, fence or barrier between the staging blocks
__global__ void ring_stage_kernel(const float* __restrict__ xs, float* __restrict__ xd, int64_t nx,
                                  int64_t xstride, const uint32_t* __restrict__ ts,
                                  uint32_t* __restrict__ td, int64_t nt, int64_t tstride,
                                  int nbatch, const int* cursor, const float* lsrc, float* lhist,
                                  int lmask) {
  PDL_ENTRY();
  const int step = *((volatile const int*)(cursor + 2));
  const int slot = step % nbatch;
  // (host stream) the previous step's loss into its history slot
  if (lhist && blockIdx.x == 0 && threadIdx.x == 0 && step > 0)
    lhist[(step - 1) & lmask] = *lsrc;
  const float* xsrc = xs + (int64_t)slot * xstride;
  const uint32_t* tsrc = ts + (int64_t)slot * tstride;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const float4* s4 = reinterpret_cast<const float4*>(xsrc);
  float4* d4 = reinterpret_cast<float4*>(xd);
  for (int64_t i = i0; i < nx / 4; i += stride) d4[i] = __ldg(s4 + i);
  for (int64_t i = nx / 4 * 4 + i0; i < nx; i += stride) xd[i] = __ldg(xsrc + i);
  for (int64_t i = i0; i < nt; i += stride) td[i] = __ldg(tsrc + i);
}

int launch_ring_stage(const float* xs, float* xd, int64_t nx, int64_t xstride, const void* ts,
                      void* td, int64_t nt, int64_t tstride, int nbatch, const int* cursor,
                      cudaStream_t st, const float* lsrc, float* lhist, int lmask) {
  if (((reinterpret_cast<uintptr_t>(xs) | reinterpret_cast<uintptr_t>(xd)) & 15) ||
      xstride % 4)
    return fail(VCNN_ESHAPE, "batch ring: x must be 16-byte aligned, x_stride a multiple of 4");
  int64_t blocks = cdiv(nx / 4 + 1, 256);
  if (blocks > 2 * sm_count()) blocks = 2 * sm_count();
  VCNN_CUDA_TRY(launch_pdl(ring_stage_kernel, dim3((unsigned)blocks), dim3(256), 0, st, xs, xd,
                           nx, xstride, static_cast<const uint32_t*>(ts),
                           static_cast<uint32_t*>(td), nt, tstride, nbatch, cursor, lsrc,
                           lhist, lmask));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int launch_store_scalar(const float* src, float* dst, cudaStream_t st) {
  VCNN_CUDA_TRY(launch_pdl(store_scalar_kernel, dim3(1), dim3(32), 0, st, src, dst));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int launch_sgd(int64_t n, float* w, float* v, const float* g, float lr, float mom, float scale,
               cudaStream_t st) {
  const bool aligned = ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(v) |
                         reinterpret_cast<uintptr_t>(g)) & 15) == 0;
  const int64_t work = aligned ? ((n >> 2) > 0 ? (n >> 2) : 1) : n;
  unsigned grid = grid_for(work);
  if (grid > (unsigned)sm_count() * 8) grid = (unsigned)sm_count() * 8;
  VCNN_CUDA_TRY(launch_pdl(sgd_kernel, dim3(grid), dim3(kThreads), 0, st, n, w, v, g, lr, mom, scale, aligned ? 1 : 0));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int launch_accumulate(const float* values, const int64_t* source, const int64_t* target,
                      int64_t pairs, int64_t target_len, int reducer, float* out, int64_t* arg,
                      cudaStream_t st) {
  int64_t *keys_out = nullptr, *idx_in = nullptr, *idx_out = nullptr;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  const int64_t np = pairs > 0 ? pairs : 1;
  VCNN_CUDA_TRY(cudaMallocAsync(&keys_out, sizeof(int64_t) * np, st));
  VCNN_CUDA_TRY(cudaMallocAsync(&idx_in, sizeof(int64_t) * np, st));
  VCNN_CUDA_TRY(cudaMallocAsync(&idx_out, sizeof(int64_t) * np, st));
  if (pairs > 0) {
    VCNN_CUDA_TRY(launch_pdl(iota_kernel, dim3(grid_for(pairs)), dim3(kThreads), 0, st, pairs, idx_in));
    VCNN_LAUNCHED();
    // stable radix sort: equal targets keep their map order
    VCNN_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, target, keys_out, idx_in,
                                                  idx_out, pairs, 0, 64, st));
    VCNN_CUDA_TRY(cudaMallocAsync(&temp, temp_bytes, st));
    VCNN_CUDA_TRY(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, target, keys_out, idx_in,
                                                  idx_out, pairs, 0, 64, st));
  }
  VCNN_CUDA_TRY(launch_pdl(accumulate_kernel, dim3(grid_for(target_len)), dim3(kThreads), 0, st, 
      values, keys_out, idx_out, source, pairs, target_len, reducer, out, arg));
  VCNN_LAUNCHED();
  if (temp) cudaFreeAsync(temp, st);
  cudaFreeAsync(keys_out, st);
  cudaFreeAsync(idx_in, st);
  cudaFreeAsync(idx_out, st);
  return VCNN_OK;
}

namespace simt {

int conv_fwd(const ConvDesc& d, const float* x, const float* w, const float* b, int act,
             float* y, cudaStream_t st) {
  VCNN_CUDA_TRY(launch_pdl(conv_fwd_simt, dim3(grid_for(d.out_size())), dim3(kThreads), 0, st, d, x, w, b, act, y));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int conv_wgrad(const ConvDesc& d, const float* x, const float* gpre, float* dw, float* db,
               cudaStream_t st) {
  dim3 grid((unsigned)(d.kd() + 1), (unsigned)d.K);
  VCNN_CUDA_TRY(launch_pdl(conv_wgrad_simt, dim3(grid), dim3(kThreads), 0, st, d, x, gpre, dw, db));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int conv_dgrad(const ConvDesc& d, const float* gpre, const float* w, float* dx,
               const float* yprev, int act_prev, cudaStream_t st) {
  VCNN_CUDA_TRY(launch_pdl(conv_dgrad_simt, dim3(grid_for(d.in_size())), dim3(kThreads), 0, st, d, gpre, w, dx, yprev, act_prev));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

// mid-size FC forward (in the forward-only chain: CIFAR-3's dense conv3,
// 128 x 800 -> 64): one warp per output, float4 loads of the x row and the W
// row strided over the lanes, fixed shuffle-tree reduction (deterministic,
// exact fp32).  ~3 us where a split-K tensor-core GEMM + reduce takes 16 us.
__global__ void full_fwd_warp(int B, int in, int out, const float* __restrict__ x,
                              const float* __restrict__ w, const float* __restrict__ b, int act,
                              float* __restrict__ y) {
  PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (wid >= (int64_t)B * out) return;
  const int o = (int)(wid % out);
  const int64_t bb = wid / out;
  const float4* xr = reinterpret_cast<const float4*>(x + bb * in);
  const float4* wr = reinterpret_cast<const float4*>(w + (int64_t)o * in);
  float acc = 0.f;
  for (int k = lane; k < (in >> 2); k += 32) {
    const float4 a = __ldg(xr + k), c = __ldg(wr + k);
    acc = fmaf(a.x, c.x, acc);
    acc = fmaf(a.y, c.y, acc);
    acc = fmaf(a.z, c.z, acc);
    acc = fmaf(a.w, c.w, acc);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) y[wid] = act_fwd(act, acc + b[o]);
}

bool full_fwd_warp_ok(int B, int in, int out, const float* x, const float* w) {
  const int64_t macs = (int64_t)B * in * out;
  return in % 4 == 0 && in >= 64 && macs < (int64_t(1) << 24) &&
         ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) & 15) == 0;
}

int full_fwd_mid(int B, int in, int out, const float* x, const float* w, const float* b, int act,
                 float* y, cudaStream_t st) {
  const int64_t threads = (int64_t)B * out * 32;
  VCNN_CUDA_TRY(launch_pdl(full_fwd_warp, dim3((unsigned)cdiv(threads, 256)), dim3(256), 0, st, B,
                           in, out, x, w, b, act, y));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int full_fwd(int B, int in, int out, const float* x, const float* w, const float* b, int act,
             float* y, cudaStream_t st) {
  VCNN_CUDA_TRY(launch_pdl(full_fwd_simt, dim3(grid_for((int64_t)B * out)), dim3(kThreads), 0, st, B, in, out, x, w, b, act, y));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int full_wgrad(int B, int in, int out, const float* x, const float* gpre, float* dw, float* db,
               cudaStream_t st) {
  VCNN_CUDA_TRY(launch_pdl(full_wgrad_simt, dim3(grid_for((int64_t)out * (in + 1))), dim3(kThreads), 0, st, B, in, out, x, gpre,
                                                                          dw, db));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int full_dgrad(int B, int in, int out, const float* gpre, const float* w, float* dx,
               const float* yprev, int act_prev, cudaStream_t st) {
  VCNN_CUDA_TRY(launch_pdl(full_dgrad_simt, dim3(grid_for((int64_t)B * in)), dim3(kThreads), 0, st, B, in, out, gpre, w, dx,
                                                                  yprev, act_prev));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int gemm(int64_t m, int64_t n, int64_t k, const float* a, int64_t as_m, int64_t as_k,
         const float* b, int64_t bs_k, int64_t bs_n, float* c, int64_t ldc, const float* bias,
         int act, cudaStream_t st) {
  VCNN_CUDA_TRY(launch_pdl(gemm_simt, dim3(grid_for(m * n)), dim3(kThreads), 0, st, m, n, k, a, as_m, as_k, b, bs_k, bs_n, c, ldc, bias, act));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int matmul(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c,
           bool transB, cudaStream_t st) {
  VCNN_CUDA_TRY(launch_pdl(matmul_simt, dim3(grid_for(m * n)), dim3(kThreads), 0, st, m, k, n, a, b, c, transB));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

}  // namespace simt
}  // namespace vcnn_b200
