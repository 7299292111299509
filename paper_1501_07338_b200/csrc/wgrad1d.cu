// wgrad1d.cu -- weight gradient of a 1-D (kh == 1) convolution with a long
// kernel (kw up to 128, e.g. the 1x121 layer of the deconvolution net) on the
// sm_100a tensor cores: conv_backward_core dW / db (layers.hpp:164-178).
//
//     dW[n][c][kx] = sum_{b,y,x} G[b][n][y][x] * X[b][c][y][x + kx]
//
// Per input row (b, y) and channel c this is a GEMM with M = the kernel taps
// kx (<= 128 rows), N = the maps n, K = the row's output positions x.  The
// A operand A(kx, x) = X[c][y][x + kx] is a shifted view along K; K-major
// operands move in 16-byte (4-element) granules only, so the row is staged
// once as "granules" Gr[p] = (X[p], X[p+1], X[p+2], X[p+3]): then A's core
// matrices are 8 consecutive granules (SBO = 128 B) and the two 4-position
// halves of a K=8 step are 4 granules apart (LBO = 64 B) -- element
// (kx, x) sits at granule 4*(x/4) + kx, lane x%4 = X[x + kx].  B = the G row
// staged [x/4][n][4].  One TMEM accumulator (128 lanes x N) per channel of
// the CTA's channel group; the CTA accumulates a contiguous range of rows
// (double-buffered staging overlaps the previous row's MMAs), writes its
// dW | db partial in the reference layout, and a fixed-order reduce over the
// row groups finishes dW / db (deterministic).
#include "image_sum.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace vcnn_b200 {
namespace direct {

namespace {

constexpr int W1T = 256;  // threads
constexpr size_t kSmem1 = 227 * 1024;

struct W1Geo {
  int B, C, H, W, K, kw, OW;
  int Kn;       // N: maps padded to 16
  int NC;       // channels per CTA (TMEM: NC * Kn columns)
  int ncg;      // channel groups
  int xs;       // K extent: OW padded to 8
  int GN;       // granules staged per channel (>= xs + 128)
  int rows, nrg, rpg;  // rows B*H, row groups, rows per group
  int tmem_cols;
  int buf_bytes, off_gb, smem;  // per buffer: Gr [NC][GN][16 B], then Gb [xs/4][Kn][16 B]
  int64_t part, pstride;        // floats per partial (K*C*kw + K), stride
};

bool w1plan(const ConvDesc& d, W1Geo& g) {
  g = W1Geo{};
  if (d.s != 1 || d.kh != 1 || d.kw < 16 || d.kw > 128 || d.K < 1 || d.K > 128) return false;
  g.B = d.B, g.C = d.C, g.H = d.H, g.W = d.W, g.K = d.K, g.kw = d.kw, g.OW = d.OW;
  if (d.OH != d.H || d.OW % 4 || d.W % 4) return false;  // float4 row loads
  g.Kn = (d.K + 15) / 16 * 16;
  g.NC = 512 / g.Kn;
  if (g.NC > 8) g.NC = 8;
  if (g.NC > d.C) g.NC = d.C;
  g.ncg = (d.C + g.NC - 1) / g.NC;
  int cols = 32;
  while (cols < g.NC * g.Kn) cols *= 2;
  g.tmem_cols = cols;
  g.xs = (d.OW + 7) / 8 * 8;
  g.GN = g.xs + 128;
  const int gr = g.NC * g.GN * 16, gb = g.xs / 4 * g.Kn * 16;
  g.buf_bytes = (gr + gb + 127) & ~127;
  g.off_gb = gr;
  g.smem = 2 * g.buf_bytes + 1024;
  if ((size_t)g.smem > kSmem1) return false;
  g.rows = d.B * d.H;
  // ~2 CTAs per SM over all channel groups
  int want = (2 * 148 + g.ncg - 1) / g.ncg;
  if (want > g.rows) want = g.rows;
  if (want < 1) want = 1;
  g.rpg = (g.rows + want - 1) / want;
  g.nrg = (g.rows + g.rpg - 1) / g.rpg;
  g.part = (int64_t)d.K * d.C * d.kw + d.K;
  g.pstride = (g.part + 3) / 4 * 4;
  return true;
}

struct W1Args {
  W1Geo g;
  const float* x;   // [B][C][H][W]
  const float* gr;  // G [B][K][H][OW] (pre-activation gradient)
  float* part;      // [nrg][pstride]
};

__device__ __forceinline__ uint64_t kdesc(uint32_t base, uint32_t lbo) {
  return ptx::interleave_desc(base, lbo, 128u);
}

__global__ void __launch_bounds__(W1T, 1) wgrad1d_kernel(const W1Args a) {
  pdl_launch_dependents();
  const W1Geo& g = a.g;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  __shared__ uint64_t mma_done[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cgi = blockIdx.x, rg = blockIdx.y;
  const int c0 = cgi * g.NC, nc = g.C - c0 < g.NC ? g.C - c0 : g.NC;
  const int r0 = rg * g.rpg, r1 = r0 + g.rpg < g.rows ? r0 + g.rpg : g.rows;
  if (warp == 0) {
    ptx::tmem_alloc(&tmem_base_sh, (uint32_t)g.tmem_cols);
    ptx::tmem_relinquish();
  }
  if (tid == 32) {
    ptx::mbar_init(&mma_done[0], 1);
    ptx::mbar_init(&mma_done[1], 1);
    ptx::fence_mbar_init();
  }
  pdl_wait();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t sbase = ptx::smem_u32(smem);
  const int q = g.xs / 4;  // x quads
  float dbacc[3] = {0.f, 0.f, 0.f};  // db: this thread's (n, xq) entries, summed over rows

  for (int r = r0; r < r1; ++r) {
    const int i = r - r0, buf = i & 1;
    const int b = r / g.H, y = r - b * g.H;
    if (i >= 2) ptx::mbar_wait(&mma_done[buf], (uint32_t)((i - 2) >> 1) & 1u);
    uint8_t* B0 = smem + buf * g.buf_bytes;
    float* Gr = reinterpret_cast<float*>(B0);
    float* Gb = reinterpret_cast<float*>(B0 + g.off_gb);
    // granules of the NC channel rows: Gr[c][p] = X[c][y][p .. p+3] (0 past W)
    const float* xr = a.x + (((int64_t)b * g.C + c0) * g.H + y) * g.W;
    for (int t = tid; t < g.NC * g.GN; t += W1T) {
      const int c = t / g.GN, p = t - c * g.GN;
      float v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        v[e] = (c < nc && p + e < g.W) ? ptx::to_tf32(__ldg(xr + (int64_t)c * g.H * g.W + p + e))
                                       : 0.f;
      reinterpret_cast<float4*>(Gr)[t] = make_float4(v[0], v[1], v[2], v[3]);
    }
    // the G row, [x/4][n][4] (n < K, x < OW; zero padded to Kn, xs)
    const float* grow = a.gr + ((int64_t)b * g.K * g.H + y) * g.OW;
    int e = 0;
    for (int t = tid; t < q * g.Kn; t += W1T, ++e) {
      const int xq = t / g.Kn, n = t - xq * g.Kn;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (n < g.K && 4 * xq < g.OW)
        v = __ldg(reinterpret_cast<const float4*>(grow + (int64_t)n * g.H * g.OW + 4 * xq));
      if (cgi == 0 && e < 3) dbacc[e] += (v.x + v.y) + (v.z + v.w);
      v.x = ptx::to_tf32(v.x), v.y = ptx::to_tf32(v.y), v.z = ptx::to_tf32(v.z),
      v.w = ptx::to_tf32(v.w);
      reinterpret_cast<float4*>(Gb)[t] = v;
    }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0 && ptx::elect_one()) {
      const uint32_t idesc = ptx::idesc_tf32(128, g.Kn);
      const uint32_t a_base = sbase + (uint32_t)(buf * g.buf_bytes);
      const uint32_t b_base = a_base + (uint32_t)g.off_gb;
      for (int c = 0; c < nc; ++c)
        for (int ks = 0; ks < g.xs / 8; ++ks)
          ptx::mma_tf32(tmem + (uint32_t)(c * g.Kn),
                        kdesc(a_base + (uint32_t)(c * g.GN * 16 + ks * 128), 64u),
                        kdesc(b_base + (uint32_t)(ks * 2 * g.Kn * 16), (uint32_t)(g.Kn * 16)),
                        idesc, (i > 0 || ks > 0) ? 1u : 0u);
      ptx::mma_commit(&mma_done[buf]);
    }
    __syncwarp();
  }
  // drain: the last row's MMAs (the commit tracks every earlier one too)
  const int nrow = r1 - r0;
  if (nrow > 0) ptx::mbar_wait(&mma_done[(nrow - 1) & 1], (uint32_t)((nrow - 1) >> 1) & 1u);
  ptx::tc_fence_after();
  float* part = a.part + (int64_t)rg * g.pstride;
  // dW partial: thread = TMEM lane = tap kx (warps 0-3; 4-7 take the odd channels)
  {
    const int quad = warp & 3, kx = quad * 32 + lane;
    const uint32_t lrow = (uint32_t)(quad * 32) << 16;
    for (int c = warp >> 2; c < nc; c += W1T / 128) {
      for (int n0 = 0; n0 < g.Kn; n0 += 16) {
        uint32_t v[16];
        ptx::tmem_ld16(tmem + lrow + (uint32_t)(c * g.Kn + n0), v);
        ptx::tmem_wait_ld();
        if (kx < g.kw)
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int n = n0 + j;
            if (n < g.K)
              part[((int64_t)n * g.C + c0 + c) * g.kw + kx] = nrow > 0 ? __uint_as_float(v[j]) : 0.f;
          }
      }
    }
  }
  // db partial (channel group 0): the per-thread row sums of G, then per map
  // over the x quads in order
  if (cgi == 0) {
    // gather the per-thread row sums through shared memory, one slot at a time
    const int nent = q * g.Kn;
    float* dbsum = reinterpret_cast<float*>(smem);  // staging buffers are dead now
    for (int e2 = 0; e2 < 3; ++e2) {
      const int t = e2 * W1T + tid;
      if (t < nent) dbsum[t] = dbacc[e2];
    }
    __syncthreads();  // (every thread passed the dW drain: the buffers are dead)
    for (int n = tid; n < g.K; n += W1T) {
      float s = 0.f;
      for (int xq = 0; xq < q; ++xq) s += dbsum[xq * g.Kn + n];
      part[(int64_t)g.K * g.C * g.kw + n] = s;
    }
  }  // (the db slot of a row group's partial belongs to its channel group 0)
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, (uint32_t)g.tmem_cols);
}

}  // namespace

bool wgrad1d_ok(const ConvDesc& d) {
  W1Geo g;
  return w1plan(d, g) && (g.xs / 4) * g.Kn <= 3 * W1T;  // db: <= 3 row-sum slots per thread
}

size_t wgrad1d_workspace(const ConvDesc& d) {
  W1Geo g;
  if (!w1plan(d, g)) return 0;
  return sizeof(float) * (size_t)(g.pstride * g.nrg);
}

int conv_wgrad1d(const ConvDesc& d, const float* x, const float* gpre, float* dw, float* db,
                 const Workspace& ws, cudaStream_t st) {
  W1Args a{};
  if (!wgrad1d_ok(d) || !w1plan(d, a.g)) return fail(VCNN_ESHAPE, "wgrad1d: geometry not supported");
  const size_t need = sizeof(float) * (size_t)(a.g.pstride * a.g.nrg);
  if (ws.bytes < need) return fail(VCNN_ECONFIG, "wgrad1d: workspace too small");
  a.x = x;
  a.gr = gpre;
  a.part = ws.ptr;
  const size_t smem = (size_t)a.g.smem;
  static size_t configured = 0;
  if (smem > configured) {
    VCNN_CUDA_TRY(cudaFuncSetAttribute(wgrad1d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    configured = smem;
  }
  VCNN_CUDA_TRY(launch_pdl(wgrad1d_kernel, dim3((unsigned)a.g.ncg, (unsigned)a.g.nrg), dim3(W1T),
                           smem, st, a));
  VCNN_LAUNCHED();
  const int64_t per = a.g.part, nw = per - d.K;
  VCNN_CUDA_TRY(launch_pdl(wgrad_reduce_kernel, dim3((unsigned)cdiv(per, 32)),
                           dim3(32 * kRedSlices), 0, st, a.g.nrg, per, a.g.pstride, nw,
                           (const float*)ws.ptr, dw, db));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

}  // namespace direct
}  // namespace vcnn_b200
