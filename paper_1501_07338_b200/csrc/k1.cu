// k1.cu -- single-output-map convolutions (K = 1: the reconstruction layer
// of the denoise / deconvolution CNNs: conv 64->1 8x8,
// conv 38->1 5x5), forward and weight gradient, exact fp32 on the SIMT pipes.
// (A direct full-correlation data gradient in the same style measured 2x
// slower than the tcgen05 implicit GEMM on denoise-16 -- 696 vs 372 us -- so
// the dgrad stays on the generic path.)
//
// conv_forward / conv_backward_core (layers.hpp:139-195) with K = 1 are
// GEMMs with N = 1: on the tensor cores the N tile (8..32) would be 8-32x
// padding, so these run as register-blocked direct convolutions instead:
//   y[b][oy][ox] = act(b0 + sum_{c,ky,kx} W[c][ky][kx] x[b][c][oy+ky][ox+kx])
//   dW[c][ky][kx] = sum_{b,oy,ox} g[b][oy][ox] x[b][c][oy+ky][ox+kx]
//   db = sum_{b,oy,ox} g[b][oy][ox]
// Each output is one fixed-order fp32 sum (deterministic, and at least as
// accurate as the TF32 path), so one kernel serves every precision mode.
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace vcnn_b200 {
namespace k1 {
namespace {

constexpr int KT = 128;     // threads
constexpr int KWMAX = 16;   // kernel width handled by the register window
constexpr int kSmem = 48 * 1024;

// ---- forward: CTA = (row band, image); thread = (row, 4 consecutive ox) ----
struct FGeo {
  int B, C, H, W, kh, kw, OH, OW;
  int colg, R, bands;  // 4-wide column groups per row, rows per CTA, bands
  int Wp, rows, CC;    // smem row stride (float4 aligned, zero padded), rows, channels/chunk
};

bool fplan(const ConvDesc& d, FGeo& g) {
  g = FGeo{};
  if (d.K != 1 || d.s != 1 || d.kw > KWMAX || d.kh > 64) return false;
  g.B = d.B, g.C = d.C, g.H = d.H, g.W = d.W, g.kh = d.kh, g.kw = d.kw, g.OH = d.OH, g.OW = d.OW;
  g.colg = (d.OW + 3) / 4;
  if (g.colg > KT) return false;
  g.R = KT / g.colg;
  if (g.R > d.OH) g.R = d.OH;
  g.bands = (d.OH + g.R - 1) / g.R;
  int need = 4 * g.colg + d.kw - 1;
  need = need > d.W ? need : d.W;
  g.Wp = (need + 3) / 4 * 4 + 4;  // + one float4 of slack for the register window
  if (g.Wp > 96) return false;    // staging covers a row in three 32-lane passes
  g.rows = g.R + d.kh - 1;
  const int per_c = 4 * (g.rows * g.Wp + d.kh * d.kw);
  g.CC = kSmem / per_c;
  if (g.CC < 1) return false;
  if (g.CC > d.C) g.CC = d.C;
  return true;
}

struct FArgs {
  FGeo g;
  const float* x;
  const float* w;
  const float* bias;
  float* y;
};

template <int ACT>
__device__ __forceinline__ float act_k1(float v) {
  if (ACT == VCNN_ACT_RELU) return v > 0.f ? v : 0.f;
  if (ACT == VCNN_ACT_SIGMOID) return 1.f / (1.f + expf(-v));
  if (ACT == VCNN_ACT_TANH) return tanhf(v);
  return v;
}

template <int ACT>
__global__ void __launch_bounds__(KT) k1_fwd_kernel(const FArgs a) {
  pdl_launch_dependents();
  const FGeo& g = a.g;
  extern __shared__ __align__(16) float sm[];
  float* sx = sm;                            // [CC][rows][Wp]
  float* sw = sm + g.CC * g.rows * g.Wp;     // [CC][kh][kw]
  const int tid = threadIdx.x;
  const int b = blockIdx.y, oy0 = blockIdx.x * g.R;
  const int r = tid / g.colg, cg = tid - r * g.colg;
  const bool active = r < g.R;
  const int hw = g.H * g.W;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  pdl_wait();
  for (int c0 = 0; c0 < g.C; c0 += g.CC) {
    const int cc = g.C - c0 < g.CC ? g.C - c0 : g.CC;
    __syncthreads();  // the previous chunk is consumed
    // stage rows [oy0, oy0+rows) of channels c0.. (zero outside the image):
    // a warp takes 4 rows x 3 column passes at a time, all loads in flight
    {
      const int warp = tid >> 5, lane = tid & 31, nrows = cc * g.rows;
      for (int rr0 = warp * 4; rr0 < nrows; rr0 += (KT / 32) * 4) {
        float v[4][3];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int rr = rr0 + u, c = rr / g.rows, iy = oy0 + rr - c * g.rows;
#pragma unroll
          for (int h = 0; h < 3; ++h) {
            const int xx = lane + 32 * h;
            v[u][h] = (rr < nrows && xx < g.W && iy < g.H)
                          ? __ldg(a.x + ((int64_t)b * g.C + c0 + c) * hw + iy * g.W + xx)
                          : 0.f;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int h = 0; h < 3; ++h) {
            const int xx = lane + 32 * h;
            if (rr0 + u < nrows && xx < g.Wp) sx[(rr0 + u) * g.Wp + xx] = v[u][h];
          }
      }
    }
    for (int i = tid; i < cc * g.kh * g.kw; i += KT)
      sw[i] = __ldg(a.w + (int64_t)c0 * g.kh * g.kw + i);
    __syncthreads();
    if (active) {
      for (int c = 0; c < cc; ++c)
        for (int ky = 0; ky < g.kh; ++ky) {
          const float* row = sx + (c * g.rows + r + ky) * g.Wp + 4 * cg;
          float v[KWMAX + 4];
#pragma unroll
          for (int q = 0; q < (KWMAX + 4) / 4; ++q)
            if (4 * q < g.kw + 3) {
              const float4 f = reinterpret_cast<const float4*>(row)[q];
              v[4 * q] = f.x;
              v[4 * q + 1] = f.y;
              v[4 * q + 2] = f.z;
              v[4 * q + 3] = f.w;
            }
          const float* wr = sw + (c * g.kh + ky) * g.kw;
#pragma unroll
          for (int kx = 0; kx < KWMAX; ++kx)
            if (kx < g.kw) {
              const float wv = wr[kx];
#pragma unroll
              for (int u = 0; u < 4; ++u) acc[u] = fmaf(wv, v[kx + u], acc[u]);
            }
        }
    }
  }
  if (!active) return;
  const int oy = oy0 + r;
  if (oy >= g.OH) return;
  const float bv = __ldg(a.bias);
  float* yr = a.y + ((int64_t)b * g.OH + oy) * g.OW;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int ox = 4 * cg + u;
    if (ox < g.OW) yr[ox] = act_k1<ACT>(acc[u] + bv);
  }
}

// ---- weight gradient: CTA = (channel group, image); thread = (channel,
//      ky, row slice) with kw accumulators over a register window ----
struct WGeo {
  int B, C, H, W, kh, kw, OH, OW;
  int CG, QS;          // channels per CTA, row slices per (channel, ky)
  int ngroups;
  int64_t part, pstride;  // per-image partial: C*kh*kw + 1 (db)
};

bool wplan(const ConvDesc& d, WGeo& g) {
  g = WGeo{};
  if (d.K != 1 || d.s != 1 || d.kw > KWMAX || d.kh > KT) return false;
  g.B = d.B, g.C = d.C, g.H = d.H, g.W = d.W, g.kh = d.kh, g.kw = d.kw, g.OH = d.OH, g.OW = d.OW;
  // channels per CTA: as many as fit 128 threads with >= 1 row slice, and smem
  int cg = KT / d.kh;
  if (cg < 1) return false;
  const int img = 4 * (d.H * d.W);
  const int gb = 4 * (d.OH * d.OW + 4);
  while (cg > 1 && (size_t)cg * img + gb > (size_t)kSmem) --cg;
  if ((size_t)cg * img + gb > (size_t)kSmem) return false;
  if (cg > d.C) cg = d.C;
  g.CG = cg;
  g.QS = KT / (cg * d.kh);
  if (g.QS > d.OH) g.QS = d.OH;
  g.ngroups = (d.C + cg - 1) / cg;
  g.part = (int64_t)d.C * d.kh * d.kw + 1;
  g.pstride = (g.part + 3) / 4 * 4;
  return true;
}

struct WArgs {
  WGeo g;
  const float* x;
  const float* gr;  // [B][1][OH][OW]
  float* part;      // [B][pstride]
};

template <int KW>  // 0: any width (one shared load per FMA); else a register window
__global__ void __launch_bounds__(KT) k1_wgrad_kernel(const WArgs a) {
  pdl_launch_dependents();
  const WGeo& g = a.g;
  extern __shared__ __align__(16) float sm[];
  const int ohw = g.OH * g.OW, hw = g.H * g.W;
  float* sg = sm;               // [OH*OW]
  float* sx = sm + ohw + 4;     // [CG][H][W]
  __shared__ float red[KT];
  const int tid = threadIdx.x;
  const int grp = blockIdx.x, b = blockIdx.y, c0 = grp * g.CG;
  const int cc = g.C - c0 < g.CG ? g.C - c0 : g.CG;
  pdl_wait();
  {
    const float* gsrc = a.gr + (int64_t)b * ohw;
    const float* xsrc = a.x + ((int64_t)b * g.C + c0) * hw;
    const int nx = cc * hw;
    for (int i0 = tid; i0 < ohw + nx; i0 += KT * 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * KT;
        v[u] = i < ohw ? __ldg(gsrc + i) : (i < ohw + nx ? __ldg(xsrc + (i - ohw)) : 0.f);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * KT;
        if (i < ohw) sg[i] = v[u];
        else if (i < ohw + nx) sx[i - ohw] = v[u];
      }
    }
  }
  __syncthreads();
  // thread -> (channel cl, ky, slice qs)
  const int per_c = g.kh * g.QS;
  const int cl = tid / per_c, rem = tid - cl * per_c, ky = rem / g.QS, qs = rem - ky * g.QS;
  float acc[KWMAX];
#pragma unroll
  for (int k = 0; k < KWMAX; ++k) acc[k] = 0.f;
  const bool active = cl < cc;
  if (active) {
    const int rs = (g.OH + g.QS - 1) / g.QS, oyb = qs * rs;
    const int oye = oyb + rs < g.OH ? oyb + rs : g.OH;
    for (int oy = oyb; oy < oye; ++oy) {
      const float* xr = sx + (cl * g.H + oy + ky) * g.W;
      const float* gr = sg + oy * g.OW;
      if (KW == 0) {
        for (int ox = 0; ox < g.OW; ++ox) {
          const float gv = gr[ox];
#pragma unroll
          for (int kx = 0; kx < KWMAX; ++kx)
            if (kx < g.kw) acc[kx] = fmaf(gv, xr[ox + kx], acc[kx]);
        }
      } else {
        float win[KW > 0 ? KW : 1];
#pragma unroll
        for (int k = 0; k < KW - 1; ++k) win[k + 1] = xr[k];
        for (int ox = 0; ox < g.OW; ++ox) {
#pragma unroll
          for (int k = 0; k < KW - 1; ++k) win[k] = win[k + 1];
          win[KW - 1] = xr[ox + KW - 1];
          const float gv = gr[ox];
#pragma unroll
          for (int kx = 0; kx < KW; ++kx) acc[kx] = fmaf(gv, win[kx], acc[kx]);
        }
      }
    }
  }
  // the row slices of (cl, ky) in slice order, through shared memory
  float* part = a.part + (int64_t)b * g.pstride;
  for (int kx = 0; kx < g.kw; ++kx) {
    red[tid] = acc[kx];
    __syncthreads();
    if (active && qs == 0) {
      float s = 0.f;
      for (int q = 0; q < g.QS; ++q) s += red[tid + q];
      part[((int64_t)(c0 + cl) * g.kh + ky) * g.kw + kx] = s;
    }
    __syncthreads();
  }
  if (grp == 0) {  // db: this image's gradient sum, fixed order
    float s = 0.f;
    for (int i = tid; i < ohw; i += KT) s += sg[i];
    red[tid] = s;
    __syncthreads();
    for (int st = KT / 2; st > 0; st >>= 1) {
      if (tid < st) red[tid] += red[tid + st];
      __syncthreads();
    }
    if (tid == 0) part[g.part - 1] = red[0];
  }
}


// out[i] = sum over images of part[b][i] in image order (8 loads in flight)
__global__ void k1_reduce_kernel(int nimg, int64_t per, int64_t stride, const float* part,
                                 float* dw, int64_t nw, float* db) {
  PDL_ENTRY();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= per) return;
  float s = 0.f;
  int b = 0;
  for (; b + 8 <= nimg; b += 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(part + (int64_t)(b + u) * stride + i);
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; b < nimg; ++b) s += __ldg(part + (int64_t)b * stride + i);
  if (i < nw) dw[i] = s;
  else if (db) *db = s;
}

}  // namespace

bool fwd_ok(const ConvDesc& d) {
  FGeo g;
  return fplan(d, g);
}

int conv_fwd(const ConvDesc& d, const float* x, const float* w, const float* bias, int act,
             float* y, cudaStream_t st) {
  FArgs a{};
  if (!fplan(d, a.g)) return fail(VCNN_ESHAPE, "k1 conv forward: geometry not supported");
  a.x = x, a.w = w, a.bias = bias, a.y = y;
  const size_t smem = sizeof(float) * ((size_t)a.g.CC * a.g.rows * a.g.Wp + a.g.CC * d.kh * d.kw);
  const dim3 grid((unsigned)a.g.bands, (unsigned)d.B);
  switch (act) {
    case VCNN_ACT_RELU:
      VCNN_CUDA_TRY(launch_pdl(k1_fwd_kernel<VCNN_ACT_RELU>, grid, dim3(KT), smem, st, a));
      break;
    case VCNN_ACT_SIGMOID:
      VCNN_CUDA_TRY(launch_pdl(k1_fwd_kernel<VCNN_ACT_SIGMOID>, grid, dim3(KT), smem, st, a));
      break;
    case VCNN_ACT_TANH:
      VCNN_CUDA_TRY(launch_pdl(k1_fwd_kernel<VCNN_ACT_TANH>, grid, dim3(KT), smem, st, a));
      break;
    default:
      VCNN_CUDA_TRY(launch_pdl(k1_fwd_kernel<VCNN_ACT_IDENTITY>, grid, dim3(KT), smem, st, a));
  }
  VCNN_LAUNCHED();
  return VCNN_OK;
}

bool wgrad_ok(const ConvDesc& d) {
  WGeo g;
  return wplan(d, g);
}

size_t wgrad_workspace(const ConvDesc& d) {
  WGeo g;
  if (!wplan(d, g)) return 0;
  return sizeof(float) * (size_t)(g.pstride * d.B);
}

int conv_wgrad(const ConvDesc& d, const float* x, const float* gpre, float* dw, float* db,
               const Workspace& ws, cudaStream_t st) {
  WArgs a{};
  if (!wplan(d, a.g)) return fail(VCNN_ESHAPE, "k1 wgrad: geometry not supported");
  if (ws.bytes < sizeof(float) * (size_t)(a.g.pstride * d.B))
    return fail(VCNN_ECONFIG, "k1 wgrad: workspace too small");
  a.x = x, a.gr = gpre, a.part = ws.ptr;
  const size_t smem = sizeof(float) * ((size_t)d.OH * d.OW + 4 + (size_t)a.g.CG * d.H * d.W);
  const dim3 grid((unsigned)a.g.ngroups, (unsigned)d.B);
  if (d.kw == 8)
    VCNN_CUDA_TRY(launch_pdl(k1_wgrad_kernel<8>, grid, dim3(KT), smem, st, a));
  else if (d.kw == 5)
    VCNN_CUDA_TRY(launch_pdl(k1_wgrad_kernel<5>, grid, dim3(KT), smem, st, a));
  else
    VCNN_CUDA_TRY(launch_pdl(k1_wgrad_kernel<0>, grid, dim3(KT), smem, st, a));
  VCNN_LAUNCHED();
  const int64_t per = a.g.part, nw = per - 1;
  VCNN_CUDA_TRY(launch_pdl(k1_reduce_kernel, dim3((unsigned)cdiv(per, 128)), dim3(128), 0, st,
                           d.B, per, a.g.pstride, (const float*)ws.ptr, dw, nw, db));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

}  // namespace k1
}  // namespace vcnn_b200
