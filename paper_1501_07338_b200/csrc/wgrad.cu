// wgrad.cu -- stride-1 convolution weight gradient as shifted-view GEMMs on
// the sm_100a tensor cores (tcgen05, TF32): conv_backward_core dW / db
// (layers.hpp:164-178: dW = G^T * im2col(x), db = column sums of G).
//
// For a kernel offset (ky,kx) the weight gradient is a GEMM over output
// positions q of one image's super-grid (row width Wg = W):
//     dW[n][c][ky][kx] = sum_q G[n][q] * x[c][q + d],   d = ky*W + kx.
// The reduction runs along positions, so the shift lands on the GEMM K axis,
// where a K-major operand moves in 16-byte (4-position) granules only.  The
// CTA therefore stages S = 128/Cp copies of the image, copy j shifted by j
// positions, stacked as the M = 128 rows (j, c) of the A operand:
//     A[(j,c)][q] = x[c][q + 4a + j]
// so ONE MMA at granule offset a yields dW for the S consecutive shifts
// d = 4a .. 4a+S-1 of all channels.  Per kernel row ky the kw shifts
// ky*W .. ky*W+kw-1 need ceil(.../S) such MMA groups; each group has its own
// TMEM accumulator (M=128 x N=K maps).  B = G staged [granule][n][4].
// Layouts are K-major, no swizzle: element (row, k) at
// (k/4)*rows*16 + row*16 + (k%4)*4 (SBO = 128 B, LBO = rows*16 B), so the
// shift is +a*LBO on the descriptor start and a K step of 8 positions is
// +2*LBO.  One CTA per image; its dW|db partial (the reference layout) goes
// to the workspace and a fixed-order reduce over images writes dW / db
// (deterministic).  The routed pool backward (GradSrc.pool) scatters dP to
// the argmax positions while G is staged.
#include "image_sum.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace vcnn_b200 {
namespace direct {

namespace {

constexpr int WT = 256;                 // threads
constexpr size_t kSmemMax = 227 * 1024;
constexpr int kMaxGroups = 32;

struct WGeo {
  int B, C, H, W, K, kh, kw, OH, OW;
  int Cp, S;          // channels per copy (8/16/32), copies (128 / Cp)
  int Kn;             // N = maps padded to 16
  int Rc, nchunk;     // output rows per position chunk, chunks per image
  int Q, ksteps;      // positions per chunk (Rc*W padded to 8), K steps of 8
  int amax, NG;       // max granule offset, staged A granules per chunk
  int ngroups;        // MMA groups (shift sets)
  int gky[kMaxGroups], ga[kMaxGroups];
  int tmem_cols;      // power of 2 >= ngroups * Kn
  int pool, POH, POW; // routed gradient (pool > 0)
  int off_a, off_g, off_raw, off_win, smem;   // bytes
  int raw_n, wsz;     // floats: image, routed windows (K*POH*POW)
  int64_t part;       // floats per image partial: K*C*kh*kw + K
  int64_t pstride;    // partial stride (multiple of 4: float4 stores)
};

bool wplan(const ConvDesc& d, const GradSrc& gs, WGeo& g) {
  g = WGeo{};
  if (d.s != 1 || d.C < 1 || d.C > 32 || d.K < 1 || d.K > 256) return false;
  g.B = d.B, g.C = d.C, g.H = d.H, g.W = d.W, g.K = d.K, g.kh = d.kh, g.kw = d.kw;
  g.OH = d.OH, g.OW = d.OW;
  g.Cp = d.C <= 8 ? 8 : d.C <= 16 ? 16 : 32;
  g.S = 128 / g.Cp;
  g.Kn = (d.K + 15) / 16 * 16;
  const int dmax = (d.kh - 1) * d.W + d.kw - 1;
  g.amax = dmax / 4;
  int ng = 0;
  for (int ky = 0; ky < d.kh; ++ky) {
    const int lo = ky * d.W, hi = ky * d.W + d.kw - 1;
    for (int a = lo / 4; 4 * a <= hi; a += g.S / 4) {
      if (ng == kMaxGroups) return false;
      g.gky[ng] = ky;
      g.ga[ng] = a;
      ++ng;
    }
  }
  g.ngroups = ng;
  int cols = 32;
  while (cols < ng * g.Kn) cols *= 2;
  if (cols > 512) return false;
  g.tmem_cols = cols;
  g.raw_n = d.C * d.H * d.W;
  if (g.raw_n % 4) return false;
  g.pool = gs.pool, g.POH = gs.POH, g.POW = gs.POW;
  g.wsz = gs.pool ? d.K * gs.POH * gs.POW : 0;
  if (gs.pool && g.wsz % 4) return false;
  // window scratch is reserved for any >= 2x2 pool whether or not this call
  // is routed, so a routed layer and its unrouted trace twin get the same
  // plan (bit-identical results)
  const int win_n = ((d.K * ((d.OH + 1) / 2) * ((d.OW + 1) / 2)) + 3) & ~3;
  if (g.wsz > win_n) return false;
  g.part = (int64_t)d.K * d.C * d.kh * d.kw + d.K;
  g.pstride = (g.part + 3) / 4 * 4;
  // per chunk: A = NG granules x 128 rows x 16 B (the dW tile reuses it at
  // the end), G = Q/4 granules x Kn rows x 16 B; per image: the input image
  // and the routed windows.  The largest chunk that fits; chunk starts must
  // be granule aligned (Rc*W % 4 == 0) and whole pool rows.
  const int dw_bytes = (int)(4 * g.part);
  // (one chunk only: chunked images lose to the slab kernel on CIFAR-3's
  // conv1 (C=3): with one A buffer build and MMA serialise (47 us vs 34 us);
  // a per-kernel-row variant without the shift halo, A/G double-buffered,
  // measured 79 us -- rebuilding 64 KB of shifted copies per 16 MMAs doubles
  // the shared-memory traffic the MMAs already saturate, and 5/8 of the rows
  // are channel padding at C=3)
  for (int Rc = d.OH; Rc >= d.OH; --Rc) {
    const int nch = (d.OH + Rc - 1) / Rc;
    if (nch > 1 && ((Rc * d.W) % 4 || (gs.pool && Rc % gs.pool))) continue;
    const int Q = (Rc * d.W + 7) / 8 * 8;
    const int NG = Q / 4 + g.amax;
    const int a_bytes = NG * 128 * 16;
    const int off_g = ((a_bytes > dw_bytes ? a_bytes : dw_bytes) + 127) & ~127;
    const int off_raw = off_g + Q / 4 * g.Kn * 16;
    const int off_win = off_raw + 4 * g.raw_n;
    const int smem = off_win + 4 * 2 * win_n + 1024;
    if ((size_t)smem + 512 > kSmemMax) continue;
    g.Rc = Rc, g.nchunk = nch, g.Q = Q, g.ksteps = Q / 8, g.NG = NG;
    g.off_a = 0, g.off_g = off_g, g.off_raw = off_raw, g.off_win = off_win, g.smem = smem;
    return true;
  }
  return false;
}

#ifdef VCNN_PHASE_TIMING
__device__ unsigned long long g_sphase[4][8];
#define SPHASE(i)                                                              \
  do {                                                                         \
    if (threadIdx.x == 0 && blockIdx.x < 4) g_sphase[blockIdx.x][i] = clock64(); \
  } while (0)
#else
#define SPHASE(i) \
  do {            \
  } while (0)
#endif

#ifdef VCNN_PHASE_TIMING
__device__ unsigned long long g_wphase[4][8];
#define WPHASE(i)                                                             \
  do {                                                                        \
    if ((threadIdx.x & 31) == 0 && blockIdx.x < 4) g_wphase[blockIdx.x][i] = clock64(); \
  } while (0)
#else
#define WPHASE(i) \
  do {            \
  } while (0)
#endif

struct WArgs {
  WGeo g;
  const float* x;       // [B][C][H][W]
  GradSrc gs;           // routed (pool) or plain g [B][K][OH][OW]
  float* part;          // [B][part]
};

__global__ void __launch_bounds__(WT, 1) wgrad_shift_kernel(const WArgs a) {
  pdl_launch_dependents();
  const WGeo& g = a.g;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  __shared__ uint64_t load_bar, done_bar;
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = blockIdx.x;
  const uint32_t sbase = ptx::smem_u32(smem);
  const uint32_t s_a = sbase + g.off_a, s_g = sbase + g.off_g, s_raw = sbase + g.off_raw,
                 s_win = sbase + g.off_win;
  const bool routed = a.gs.pool != 0;
  const int ohw = g.OH * g.OW;
  if (tid == 0) WPHASE(0);

  if (warp == 0) {
    ptx::tmem_alloc(&tmem_base_sh, g.tmem_cols);
    ptx::tmem_relinquish();
  }
  pdl_wait();
  if (tid == 0) {
    ptx::mbar_init(&load_bar, 1);
    ptx::mbar_init(&done_bar, 1);
    ptx::fence_mbar_init();
    // the image and (routed) the pooled windows; a plain gradient is read
    // chunk by chunk from global memory
    const uint32_t rb = 4u * (uint32_t)g.raw_n;
    ptx::mbar_expect_tx(&load_bar, rb);
    ptx::bulk_g2s(s_raw, a.x + (int64_t)b * g.raw_n, rb, &load_bar);
    if (routed) {
      const uint32_t gb = 4u * (uint32_t)g.wsz;
      ptx::mbar_expect_tx(&load_bar, 2 * gb);
      ptx::bulk_g2s(s_win, a.gs.dP + (int64_t)b * g.wsz, gb, &load_bar);
      ptx::bulk_g2s(s_win + gb, a.gs.parg + (int64_t)b * g.wsz, gb, &load_bar);
    }
    ptx::mbar_arrive(&load_bar);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  ptx::mbar_wait(&load_bar, 0);
  if (tid == 0) WPHASE(1);

  auto g_at = [&](int n, int q) -> uint32_t {  // G[n][q] in [granule][n][4]
    return s_g + 4u * (uint32_t)(((q >> 2) * g.Kn + n) * 4 + (q & 3));
  };
  const int hw = g.H * g.W;
  float db_acc = 0.f;  // thread n < K: this image's bias gradient, chunk by chunk
  for (int ch = 0; ch < g.nchunk; ++ch) {
    const int r0 = ch * g.Rc, nrows = r0 + g.Rc <= g.OH ? g.Rc : g.OH - r0;
    if (ch > 0) {  // the previous chunk's MMAs have read A and G
      ptx::mbar_wait(&done_bar, (uint32_t)((ch - 1) & 1));
      ptx::tc_fence_after();
      __syncthreads();
    }
    // ---- G[n][q] (q = (oy - r0)*W + ox) for this chunk, tf32 ----
    for (int i = tid; i < g.Q * g.Kn / 4; i += WT)
      ptx::sts_f32x4(s_g + 16u * i, make_float4(0.f, 0.f, 0.f, 0.f));
    __syncthreads();
    if (routed) {  // the windows of this chunk's pooled rows, dP at the argmax
      const int base = (int)((int64_t)b * g.K * ohw);
      const int prs = r0 / g.pool;
      int npr = (nrows + g.pool - 1) / g.pool;
      if (prs + npr > g.POH) npr = g.POH - prs;
      const int per_n = npr * g.POW;
      for (int i = tid; i < g.K * per_n; i += WT) {
        const int n = i / per_n, r = i - n * per_n;
        const int w = n * g.POH * g.POW + prs * g.POW + r;
        const int at = ptx::lds_s32(s_win + 4u * (uint32_t)(g.wsz + w)) - base;
        const int rr = at - n * ohw, oy = rr / g.OW, ox = rr - oy * g.OW;
        ptx::sts_f32(g_at(n, (oy - r0) * g.W + ox), ptx::to_tf32(ptx::lds_f32(s_win + 4u * w)));
      }
    } else {
      const int per_n = nrows * g.OW;
      const float* gsrc = a.gs.g + (int64_t)b * g.K * ohw + (int64_t)r0 * g.OW;
      for (int i = tid; i < g.K * per_n; i += WT) {
        const int n = i / per_n, r = i - n * per_n, oy = r / g.OW, ox = r - oy * g.OW;
        ptx::sts_f32(g_at(n, oy * g.W + ox), ptx::to_tf32(__ldg(gsrc + (int64_t)n * ohw + r)));
      }
    }
    // ---- A: S shifted copies of the image from position r0*W, rows (j, c) ----
    const int pbase = r0 * g.W;
    if (hw % 4 == 0 && g.S == 4) {
      // 32 channels, 4 copies (CIFAR-3 conv2): two items per thread in flight
      // (2 x 2 aligned float4 loads, then 2 x 4 stores) -- the one-item loop
      // below is load-latency bound here
      for (int i0 = tid; i0 < g.NG * 32; i0 += 2 * WT) {
        float4 f[2][2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int i = i0 + t * WT, gr = i >> 5, c = i & 31;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int p = pbase + 4 * gr + 4 * u;
            f[t][u] = (i < g.NG * 32 && c < g.C && p < hw)
                          ? ptx::lds_f32x4(s_raw + 4u * (uint32_t)(c * hw + p))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int i = i0 + t * WT, gr = i >> 5, c = i & 31;
          if (i >= g.NG * 32) continue;
          const float v[8] = {ptx::to_tf32(f[t][0].x), ptx::to_tf32(f[t][0].y),
                              ptx::to_tf32(f[t][0].z), ptx::to_tf32(f[t][0].w),
                              ptx::to_tf32(f[t][1].x), ptx::to_tf32(f[t][1].y),
                              ptx::to_tf32(f[t][1].z), ptx::to_tf32(f[t][1].w)};
          const uint32_t dst = s_a + 16u * (uint32_t)(gr * 128 + c);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            ptx::sts_f32x4(dst + 16u * (uint32_t)(j * 32),
                           make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
        }
      }
    } else if (hw % 4 == 0) {
      // thread -> (granule, channel): the S+3 positions from 4*gr are read as
      // aligned float4s once and written as the S copies' granule entries
      const int nq = (g.S + 6) / 4;  // float4s per item
      for (int i = tid; i < g.NG * g.Cp; i += WT) {
        const int gr = i / g.Cp, c = i - gr * g.Cp;
        float v[20];
#pragma unroll
        for (int u = 0; u < 5; ++u) {
          if (u < nq) {
            const int p = pbase + 4 * gr + 4 * u;
            float4 f = (c < g.C && p < hw) ? ptx::lds_f32x4(s_raw + 4u * (uint32_t)(c * hw + p))
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
            v[4 * u] = ptx::to_tf32(f.x);
            v[4 * u + 1] = ptx::to_tf32(f.y);
            v[4 * u + 2] = ptx::to_tf32(f.z);
            v[4 * u + 3] = ptx::to_tf32(f.w);
          }
        }
        const uint32_t dst = s_a + 16u * (uint32_t)(gr * 128 + c);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (j < g.S)
            ptx::sts_f32x4(dst + 16u * (uint32_t)(j * g.Cp),
                           make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
      }
    } else {
      for (int i = tid; i < g.NG * 128; i += WT) {
        const int gr = i >> 7, row = i & 127;
        const int j = row / g.Cp, c = row - j * g.Cp;
        const int p0 = pbase + 4 * gr + j;
        float v[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int p = p0 + t;
          v[t] = (c < g.C && p < hw) ? ptx::to_tf32(ptx::lds_f32(s_raw + 4u * (c * hw + p))) : 0.f;
        }
        ptx::sts_f32x4(s_a + 16u * i, make_float4(v[0], v[1], v[2], v[3]));
      }
    }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (tid == 0 && ch == 0) WPHASE(2);

    // ---- one elected lane of warp 0 issues ngroups x ksteps MMAs ----
    if (warp == 0) {
      if (ptx::elect_one()) {
        const uint32_t idesc = ptx::idesc_tf32(128, g.Kn);
        const uint32_t lbo_a = 128u * 16u, lbo_g = (uint32_t)g.Kn * 16u;
        const uint64_t a0 = ptx::interleave_desc(s_a, lbo_a, 128u);
        const uint64_t g0 = ptx::interleave_desc(s_g, lbo_g, 128u);
        // group-major: each accumulator's K sequence is a run of additions
        // on the descriptors (the issue loop is the MMA rate limiter)
        const uint64_t sa = (uint64_t)(2u * lbo_a >> 4), sg = (uint64_t)(2u * lbo_g >> 4);
        for (int m = 0; m < g.ngroups; ++m) {
          uint64_t ad = a0 + (uint64_t)((uint32_t)g.ga[m] * lbo_a >> 4), bd = g0;
          const uint32_t dt = tmem + (uint32_t)(m * g.Kn);
          ptx::mma_tf32(dt, ad, bd, idesc, ch > 0 ? 1u : 0u);
          for (int k = 1; k < g.ksteps; ++k) {
            ad += sa;
            bd += sg;
            ptx::mma_tf32(dt, ad, bd, idesc, 1u);
          }
        }
        ptx::mma_commit(&done_bar);
        if (ch == 0) WPHASE(3);
      }
      __syncwarp();
    }
    // this chunk's share of db (fixed order) while the MMAs run
    for (int n = tid; n < g.K; n += WT)
      for (int q = 0; q < g.Q; ++q) db_acc += ptx::lds_f32(g_at(n, q));
  }
  float* part = a.part + (int64_t)b * g.pstride;
  const int64_t nw = g.part - g.K;
  if (tid < g.K) part[nw + tid] = db_acc;
  ptx::mbar_wait(&done_bar, (uint32_t)((g.nchunk - 1) & 1));
  ptx::tc_fence_after();
  if (tid == 0) WPHASE(4);

  // ---- epilogue: TMEM rows (j, c) x cols n -> dW tile [n][c][ky][kx] in
  //      shared memory (over A, dead now), then coalesced stores ----
  const uint32_t s_dw = s_a;
  const int khw = g.kh * g.kw, ckk = g.C * khw;
  {  // warps w and w+4 share TMEM lanes 32*(w%4)..; they split the groups
    const int row = (warp & 3) * 32 + lane, j = row / g.Cp, c = row - j * g.Cp;
    const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    for (int m = warp >> 2; m < g.ngroups; m += 2) {
      const int ky = g.gky[m], kx = 4 * g.ga[m] + j - ky * g.W;
      const bool ok = c < g.C && kx >= 0 && kx < g.kw;
      for (int n0 = 0; n0 < g.Kn; n0 += 16) {
        uint32_t r[16];
        ptx::tmem_ld16(trow + (uint32_t)(m * g.Kn + n0), r);
        ptx::tmem_wait_ld();
        if (ok) {
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int n = n0 + u;
            if (n < g.K)
              ptx::sts_f32(s_dw + 4u * (uint32_t)(n * ckk + c * khw + ky * g.kw + kx),
                           __uint_as_float(r[u]));
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (tid == 0) WPHASE(5);
  for (int64_t i = tid; i < nw / 4; i += WT)
    reinterpret_cast<float4*>(part)[i] = ptx::lds_f32x4(s_dw + 16u * (uint32_t)i);
  for (int64_t i = nw / 4 * 4 + tid; i < nw; i += WT) part[i] = ptx::lds_f32(s_dw + 4u * (uint32_t)i);
  __syncthreads();
  if (tid == 0) WPHASE(6);
  if (warp == 0) ptx::tmem_dealloc(tmem, g.tmem_cols);
}


// ---------------------------------------------------------------------------
// Small-Kd weight gradient (first layers: C*kh*kw + 1 <= 96, e.g. CIFAR-3
// conv1 C=3 5x5, LeNet conv1 C=1 5x5) on mma.sync m16n8k8 TF32.
//   dW|db [n][j] = sum_q G[n][q] * P[j][q],  P[j][q] = x[c][oy+ky][ox+kx]
// for j = (c,ky,kx) < Kd, and P[Kd][q] = 1 (the bias gradient as a ones
// column).  One CTA per image; M = maps (G rows, tf32 in shared memory),
// N = Kd+1 columns gathered straight from the staged image (a column is a
// fixed offset into [c][H][W]; a position is an offset table), K = the
// image's output positions split over the 8 warps, whose partial tiles are
// summed in warp order (deterministic).  At these sizes the per-image GEMM
// (32 x 76 x 784 for conv1) is far below one tcgen05 tile's fill cost: the
// tcgen05 slab kernel spends 5/8 of its A rows on channel padding and
// serialises staging and MMA; here staging is one bulk copy + one scatter
// and the MMAs run at 512 FMA/clk/SM from registers.
constexpr int SKG = 8;   // K groups: warps w, w + 8, ... share K steps and split N
constexpr int SNH = 2;   // N parts (4 measured slower: 17 vs 15.7 us)
constexpr int ST = 32 * SKG * SNH;  // threads
constexpr int kSmallMaxCols = 96;

struct SGeo {
  int B, C, H, W, K, kh, kw, OH, OW;
  int Kd, mt, nt;        // columns, M tiles (16 maps), N tiles (8 columns)
  int ohw, Q8, Qs;       // positions, padded to 8 (K extent), G row stride
  int ksteps;
  int pool, POH, POW, wsz;
  int off_g, off_x, off_q, off_win, smem;  // bytes
  int xfl;               // floats staged for x: image + zero + ones regions
  int64_t part, pstride;
};

bool splan(const ConvDesc& d, const GradSrc& gs, SGeo& g) {
  g = SGeo{};
  if (d.s != 1 || d.K < 1 || d.K > 32) return false;
  g.B = d.B, g.C = d.C, g.H = d.H, g.W = d.W, g.K = d.K, g.kh = d.kh, g.kw = d.kw;
  g.OH = d.OH, g.OW = d.OW;
  g.Kd = d.C * d.kh * d.kw;
  if (g.Kd + 1 > kSmallMaxCols) return false;
  g.mt = (d.K + 15) / 16;
  g.nt = (g.Kd + 1 + 7) / 8;
  g.ohw = d.OH * d.OW;
  g.Q8 = (g.ohw + 7) / 8 * 8;
  g.Qs = g.Q8 + 4;  // row stride = 4 (mod 8): the A-fragment loads are conflict-free
  g.ksteps = g.Q8 / 8;
  const int hw = d.H * d.W;
  if ((d.C * hw) % 4) return false;
  g.xfl = (d.C + 2) * hw;
  g.pool = gs.pool, g.POH = gs.POH, g.POW = gs.POW;
  g.wsz = gs.pool ? d.K * gs.POH * gs.POW : 0;
  if (gs.pool && g.wsz % 4) return false;
  // windows reserved for any 2x2-or-larger pool, routed or not (same plan on
  // the fused and the trace path -> bit-identical)
  const int win_n = ((d.K * ((d.OH + 1) / 2) * ((d.OW + 1) / 2)) + 3) & ~3;
  if (g.wsz > win_n) return false;
  g.off_g = 0;
  const int gbytes = 4 * g.mt * 16 * g.Qs;
  const int ntb = g.nt <= 4 ? 4 : g.nt <= 8 ? 8 : 12;  // the kernel's NT bucket
  const int red_bytes = 4 * SKG * g.mt * 16 * (ntb * 8 + 8);  // reuses G
  g.off_x = ((gbytes > red_bytes ? gbytes : red_bytes) + 127) & ~127;
  g.off_q = (g.off_x + 4 * g.xfl + 127) & ~127;
  g.off_win = (g.off_q + 4 * g.Q8 + 127) & ~127;
  g.smem = g.off_win + 8 * win_n + 128;
  if ((size_t)g.smem > kSmemMax) return false;
  g.part = (int64_t)d.K * g.Kd + d.K;
  g.pstride = (g.part + 3) / 4 * 4;
  return true;
}

struct SArgs {
  SGeo g;
  const float* x;
  GradSrc gs;
  float* part;
};

__device__ __forceinline__ void mma_tf32_sync(float (&c)[4], uint32_t a0, uint32_t a1,
                                              uint32_t a2, uint32_t a3, uint32_t b0,
                                              uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, "
      "{%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int MT, int NT>
__global__ void __launch_bounds__(ST, 1) wgrad_small_kernel(const SArgs a) {
  pdl_launch_dependents();
  const SGeo& g = a.g;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // pointer arithmetic on the shared array (not an integer round trip) keeps
  // the accesses below LDS/STS instead of generic LD/ST
  uint8_t* smem = smem_raw + ((128u - (ptx::smem_u32(smem_raw) & 127u)) & 127u);
  __shared__ uint64_t load_bar;
  float* sg = reinterpret_cast<float*>(smem + g.off_g);
  float* sx = reinterpret_cast<float*>(smem + g.off_x);
  int* sq = reinterpret_cast<int*>(smem + g.off_q);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = blockIdx.x, hw = g.H * g.W, ohw = g.ohw;
  const bool routed = a.gs.pool != 0;
  const uint32_t s_x = ptx::smem_u32(sx), s_win = ptx::smem_u32(smem + g.off_win);
  SPHASE(0);

  if (tid == 0) {
    ptx::mbar_init(&load_bar, 1);
    ptx::fence_mbar_init();
  }
  // independent of the predecessor: zero G, the zero / ones columns, the
  // position table (q -> oy*W + ox, padding clamped to a real position)
  const int gfl = MT * 16 * g.Qs;
  for (int i = tid; i < gfl / 4; i += ST)
    reinterpret_cast<float4*>(sg)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = tid; i < 2 * hw; i += ST) sx[g.C * hw + i] = i < hw ? 0.f : 1.f;
  for (int q = tid; q < g.Q8; q += ST) {
    const int qq = q < ohw ? q : ohw - 1, oy = qq / g.OW;
    sq[q] = oy * g.W + (qq - oy * g.OW);
  }
  __syncthreads();
  SPHASE(1);
  pdl_wait();
  SPHASE(2);
  if (tid == 0) {
    const uint32_t xb = 4u * (uint32_t)(g.C * hw);
    uint32_t tx = xb;
    if (routed) tx += 8u * (uint32_t)g.wsz;
    ptx::mbar_expect_tx(&load_bar, tx);
    ptx::bulk_g2s(s_x, a.x + (int64_t)b * g.C * hw, xb, &load_bar);
    if (routed) {
      const uint32_t gb = 4u * (uint32_t)g.wsz;
      ptx::bulk_g2s(s_win, a.gs.dP + (int64_t)b * g.wsz, gb, &load_bar);
      ptx::bulk_g2s(s_win + gb, a.gs.parg + (int64_t)b * g.wsz, gb, &load_bar);
    }
    ptx::mbar_arrive(&load_bar);
  }
  if (!routed) {  // plain gradient [K][OH][OW] of this image, tf32
    const float* src = a.gs.g + (int64_t)b * g.K * ohw;
    for (int i = tid; i < g.K * ohw; i += ST) {
      const int n = i / ohw, q = i - n * ohw;
      sg[n * g.Qs + q] = ptx::to_tf32(__ldg(src + i));
    }
  }
  ptx::mbar_wait(&load_bar, 0);
  SPHASE(3);
  if (routed) {  // dP scattered to the argmax positions (global index - image base)
    const float* wv = reinterpret_cast<const float*>(smem + g.off_win);
    const int* wa = reinterpret_cast<const int*>(smem + g.off_win) + g.wsz;
    const int base = b * g.K * ohw, pw = g.POH * g.POW;
    for (int i = tid; i < g.wsz; i += ST) {
      const int n = i / pw;
      sg[n * g.Qs + (wa[i] - base - n * ohw)] = ptx::to_tf32(wv[i]);
    }
  }
  for (int i = tid; i < g.C * hw; i += ST) sx[i] = ptx::to_tf32(sx[i]);
  __syncthreads();
  SPHASE(4);

  // ---- per lane: N-tile column offsets (c,ky,kx) -> c*hw + ky*W + kx ----
  // warp -> (K group kg, N half nh): N tiles [nh*NTW, nh*NTW + NTW)
  constexpr int NTW = (NT + SNH - 1) / SNH;
  const int kg = warp % SKG, nh = warp / SKG;
  const int gq = lane >> 2, t = lane & 3;
  int coff[NTW];
#pragma unroll
  for (int jl = 0; jl < NTW; ++jl) {
    const int jt = nh * NTW + jl;
    const int j = jt * 8 + gq;
    if (j < g.Kd) {
      const int c = j / (g.kh * g.kw), r = j - c * g.kh * g.kw, ky = r / g.kw;
      coff[jl] = c * hw + ky * g.W + (r - ky * g.kw);
    } else {
      coff[jl] = (j == g.Kd ? g.C + 1 : g.C) * hw;  // ones (bias) / zero column
    }
  }
  float acc[MT][NTW][4];
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int jl = 0; jl < NTW; ++jl)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[mi][jl][u] = 0.f;
  const int nt = g.nt - nh * NTW;  // N tiles of this half
  for (int ks = kg; ks < g.ksteps; ks += SKG) {
    const int q0 = ks * 8 + t;
    uint32_t af[MT][4];
#pragma unroll
    for (int mi = 0; mi < MT; ++mi) {
      const float* r0 = sg + (mi * 16 + gq) * g.Qs + q0;
      af[mi][0] = __float_as_uint(r0[0]);
      af[mi][1] = __float_as_uint(r0[8 * g.Qs]);
      af[mi][2] = __float_as_uint(r0[4]);
      af[mi][3] = __float_as_uint(r0[8 * g.Qs + 4]);
    }
    const int p0 = sq[q0], p1 = sq[q0 + 4];
#pragma unroll
    for (int jl = 0; jl < NTW; ++jl) {
      if (jl < nt) {
        const uint32_t b0 = __float_as_uint(sx[coff[jl] + p0]);
        const uint32_t b1 = __float_as_uint(sx[coff[jl] + p1]);
#pragma unroll
        for (int mi = 0; mi < MT; ++mi)
          mma_tf32_sync(acc[mi][jl], af[mi][0], af[mi][1], af[mi][2], af[mi][3], b0, b1);
      }
    }
  }
  __syncthreads();  // G is dead: the K groups' partial tiles go over it
  SPHASE(5);
  // floats per K-group tile [m][n]; row stride NT*8 + 8 (= 8 mod 32) and
  // 8-byte stores of each fragment column pair: a warp's 32 pairs land in 32
  // distinct 8-byte slots (two wavefronts, no replays)
  constexpr int RS = NT * 8 + 8;
  const int tw = MT * 16 * RS;
  float* red = sg + kg * tw;
#pragma unroll
  for (int mi = 0; mi < MT; ++mi)
#pragma unroll
    for (int jl = 0; jl < NTW; ++jl) {
      const int jt = nh * NTW + jl;
      if (jt >= NT) continue;
      const int m = mi * 16 + gq, n = jt * 8 + 2 * t;
      *reinterpret_cast<float2*>(red + m * RS + n) = make_float2(acc[mi][jl][0], acc[mi][jl][1]);
      *reinterpret_cast<float2*>(red + (m + 8) * RS + n) =
          make_float2(acc[mi][jl][2], acc[mi][jl][3]);
    }
  __syncthreads();
  float* part = a.part + (int64_t)b * g.pstride;
  const int cols = g.Kd + 1;
  for (int i = tid; i < g.K * cols; i += ST) {
    const int m = i / cols, j = i - m * cols;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < SKG; ++w) s += sg[w * tw + m * RS + j];
    part[j < g.Kd ? m * g.Kd + j : g.K * g.Kd + m] = s;
  }
  SPHASE(6);
}

}  // namespace

// out[i] = sum over images of part[b][i] (dW then db) in a fixed order
// (image_sum.cuh).  External linkage: wgrad1d.cu launches it too.
__global__ void __launch_bounds__(32 * kRedSlices) wgrad_reduce_kernel(
    int nimg, int64_t per, int64_t stride, int64_t nw, const float* __restrict__ part,
    float* __restrict__ dw, float* __restrict__ db) {
  PDL_ENTRY();
  __shared__ float red[kRedSlices][33];
  const int64_t i = blockIdx.x * 32ll + (threadIdx.x & 31);
  const float t = image_sum(nimg, per, stride, i, part, red);
  if ((threadIdx.x >> 5) == 0 && i < per) {
    if (i < nw) dw[i] = t;
    else if (db) db[i - nw] = t;
  }
}

// the float4 variant: outputs [0, nw) to dw, [nw, per) to db (per, stride
// and nw multiples of 4, 16-byte aligned buffers); same bits as the scalar one
__global__ void __launch_bounds__(32 * kRedSlices) wgrad_reduce4_kernel(
    int nimg, int64_t per, int64_t stride, int64_t nw, const float* __restrict__ part,
    float* __restrict__ dw, float* __restrict__ db) {
  PDL_ENTRY();
  __shared__ float4 red[kRedSlices][33];
  const int64_t i4 = blockIdx.x * 32ll + (threadIdx.x & 31);
  const float4 t = image_sum4(nimg, per / 4, stride / 4, i4,
                              reinterpret_cast<const float4*>(part), red);
  if ((threadIdx.x >> 5) == 0 && 4 * i4 < per) {
    const int64_t i = 4 * i4;
    if (i < nw) *reinterpret_cast<float4*>(dw + i) = t;
    else if (db) *reinterpret_cast<float4*>(db + (i - nw)) = t;
  }
}

bool wgrad_ok(const ConvDesc& d, const GradSrc& gs) {
  WGeo g;
  return wplan(d, gs, g);
}

size_t wgrad_workspace(const ConvDesc& d) {
  WGeo g;
  GradSrc gs;
  if (!wplan(d, gs, g)) return 0;
  return sizeof(float) * (size_t)(g.pstride * d.B);
}

int conv_wgrad(const ConvDesc& d, const float* x, const GradSrc& gs, float* dw, float* db,
               const Workspace& ws, cudaStream_t st) {
  WArgs a{};
  if (!wplan(d, gs, a.g)) return fail(VCNN_ESHAPE, "direct wgrad: geometry not supported");
  const size_t need = sizeof(float) * (size_t)(a.g.pstride * d.B);
  if (ws.bytes < need) return fail(VCNN_ECONFIG, "direct wgrad: workspace too small");
  a.x = x;
  a.gs = gs;
  a.part = ws.ptr;
  const size_t smem = (size_t)a.g.smem;
  static size_t configured = 0;
  if (smem > configured) {
    VCNN_CUDA_TRY(cudaFuncSetAttribute(wgrad_shift_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  VCNN_CUDA_TRY(launch_pdl(wgrad_shift_kernel, dim3((unsigned)d.B), dim3(WT), smem, st, a));
  VCNN_LAUNCHED();
  const int64_t per = a.g.part, nw = per - d.K;
  const bool vec = per % 4 == 0 && nw % 4 == 0 && a.g.pstride % 4 == 0 &&
                   ((reinterpret_cast<uintptr_t>(ws.ptr) | reinterpret_cast<uintptr_t>(dw) |
                     reinterpret_cast<uintptr_t>(db)) & 15) == 0;
  if (vec)
    VCNN_CUDA_TRY(launch_pdl(wgrad_reduce4_kernel, dim3((unsigned)cdiv(per / 4, 32)),
                             dim3(32 * kRedSlices), 0, st, d.B, per, a.g.pstride, nw,
                             (const float*)ws.ptr, dw, db));
  else
    VCNN_CUDA_TRY(launch_pdl(wgrad_reduce_kernel, dim3((unsigned)cdiv(per, 32)),
                             dim3(32 * kRedSlices), 0, st, d.B, per, a.g.pstride, nw,
                             (const float*)ws.ptr, dw, db));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int sum_partials(int nimg, int64_t per, int64_t stride, const float* part, float* out,
                 cudaStream_t st) {
  VCNN_CUDA_TRY(launch_pdl(wgrad_reduce_kernel, dim3((unsigned)cdiv(per, 32)),
                           dim3(32 * kRedSlices), 0, st, nimg, per, stride, per, part, out,
                           (float*)nullptr));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

bool wgrad_small_ok(const ConvDesc& d, const GradSrc& gs) {
  SGeo g;
  return splan(d, gs, g);
}

size_t wgrad_small_workspace(const ConvDesc& d) {
  SGeo g;
  GradSrc gs;
  if (!splan(d, gs, g)) return 0;
  return sizeof(float) * (size_t)(g.pstride * d.B);
}

int conv_wgrad_small(const ConvDesc& d, const float* x, const GradSrc& gs, float* dw, float* db,
                     const Workspace& ws, cudaStream_t st, ImageSumFold* defer) {
  SArgs a{};
  if (!splan(d, gs, a.g)) return fail(VCNN_ESHAPE, "small wgrad: geometry not supported");
  const size_t need = sizeof(float) * (size_t)(a.g.pstride * d.B);
  if (ws.bytes < need) return fail(VCNN_ECONFIG, "small wgrad: workspace too small");
  a.x = x;
  a.gs = gs;
  a.part = ws.ptr;
  const size_t smem = (size_t)a.g.smem;
  auto go = [&](auto kern, size_t& configured) -> int {
    if (smem > configured) {
      VCNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
      configured = smem;
    }
    VCNN_CUDA_TRY(launch_pdl(kern, dim3((unsigned)d.B), dim3(ST), smem, st, a));
    VCNN_LAUNCHED();
    return VCNN_OK;
  };
  static size_t c14 = 0, c18 = 0, c112 = 0, c24 = 0, c28 = 0, c212 = 0;
  int s;
  if (a.g.mt == 1)
    s = a.g.nt <= 4 ? go(wgrad_small_kernel<1, 4>, c14)
        : a.g.nt <= 8 ? go(wgrad_small_kernel<1, 8>, c18) : go(wgrad_small_kernel<1, 12>, c112);
  else
    s = a.g.nt <= 4 ? go(wgrad_small_kernel<2, 4>, c24)
        : a.g.nt <= 8 ? go(wgrad_small_kernel<2, 8>, c28) : go(wgrad_small_kernel<2, 12>, c212);
  if (s) return s;
  const int64_t per = a.g.part, nw = per - d.K;
  if (defer) {  // the caller's update sums the per-image partials itself
    *defer = ImageSumFold{ws.ptr, d.B, per, a.g.pstride};
    return VCNN_OK;
  }
  VCNN_CUDA_TRY(launch_pdl(wgrad_reduce_kernel, dim3((unsigned)cdiv(per, 32)),
                           dim3(32 * kRedSlices), 0, st, d.B, per, a.g.pstride, nw,
                           (const float*)ws.ptr, dw, db));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

}  // namespace direct
}  // namespace vcnn_b200

#ifdef VCNN_PHASE_TIMING
extern "C" int vcnn_debug_sphases(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, vcnn_b200::direct::g_sphase, sizeof(unsigned long long) * 32) ==
                 cudaSuccess
             ? 0
             : 4;
}
extern "C" int vcnn_debug_wphases(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, vcnn_b200::direct::g_wphase, sizeof(unsigned long long) * 32) ==
                 cudaSuccess
             ? 0
             : 4;
}
#endif
