// tc.cu -- tcgen05 implicit-GEMM engine for every GEMM-shaped op of the
// VCNN training step (conv fwd / wgrad / dgrad, FC fwd / wgrad / dgrad,
// matmul).  One CTA = 128 threads computes a 128 x BN tile of D in TMEM:
//   * all 4 warps gather operands straight from the NCHW tensors (implicit
//     im2col: no patch matrix in HBM) into 128B-swizzled K-major shared-memory
//     tiles, rounding to tf32 (or splitting hi/lo for the fp32-faithful 3xTF32
//     mode).  Index math is hoisted: every CTA first builds a shared-memory
//     table of the K-dimension offsets of its K range (im2col offsets, pixel
//     bases, ...) and every thread computes its row contexts once, so a
//     gathered element costs one table read, one add and one load.  The
//     gather is two-phase (all loads of a stage in flight, then convert +
//     st.shared) and register-prefetched one stage ahead;
//   * one elected thread issues tcgen05.mma.kind::tf32 (M=128, N=BN, K=8) and
//     tcgen05.commit's each stage back to an mbarrier (STAGES-deep ring);
//   * the epilogue reads TMEM with tcgen05.ld (thread = row) and fuses bias,
//     activation, the upstream activation derivative, or stores a split-K
//     partial that a fixed-order reduce kernel finishes with the same fused
//     epilogue -- deterministic, no float atomics.
// Small problems split K so the grid covers the 148 SMs (3 CTAs/SM).  The
// bias gradient is folded into the wgrad GEMMs as one extra K-row / N-column
// of ones.  Layers whose output is much smaller than their input (e.g. a 1x1
// output) use the explicit dgrad W^T*G -> col2im instead of the implicit one,
// which would multiply mostly zero padding.
#include <algorithm>
#include <string>

#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace vcnn_b200 {
namespace tc {

namespace {

constexpr int BM = 128;            // rows per tile == TMEM lanes
constexpr int BK = 32;             // fp32 K per stage == one 128-B swizzle row
constexpr int NT = 128;            // threads per CTA
constexpr int TAB_MAX_INTS = 4096; // per-CTA K-offset tables (16 KB)
constexpr int CTAS_PER_SM = 3;     // smem sized for 3 resident CTAs / SM

// Out-of-line activation helpers for the epilogues: the unrolled epilogue
// would otherwise inline the transcendental branches 16x per TMEM load and
// blow the instruction cache (the kernels are I$-bound when every launch is
// a different kernel).
__device__ __noinline__ float epi_act(int act, float x) { return act_fwd(act, x); }
__device__ __noinline__ float epi_dact(int act, float y) { return act_grad_from_out(act, y); }

// store 4 consecutive K values of one row into a SW128 K-major tile
template <bool SPLIT3, int ROWS>
__device__ __forceinline__ void store_chunk(uint8_t* tile, int row, int ch, const float (&v)[4]) {
  const uint32_t off = (uint32_t)row * 128u + ((uint32_t)(ch ^ (row & 7)) << 4);
  if (SPLIT3) {
    float4 hi, lo;
    hi.x = ptx::to_tf32(v[0]);
    hi.y = ptx::to_tf32(v[1]);
    hi.z = ptx::to_tf32(v[2]);
    hi.w = ptx::to_tf32(v[3]);
    lo.x = ptx::to_tf32(v[0] - hi.x);
    lo.y = ptx::to_tf32(v[1] - hi.y);
    lo.z = ptx::to_tf32(v[2] - hi.z);
    lo.w = ptx::to_tf32(v[3] - hi.w);
    *reinterpret_cast<float4*>(tile + off) = hi;
    *reinterpret_cast<float4*>(tile + ROWS * 128 + off) = lo;
  } else {
    float4 q;
    q.x = ptx::to_tf32(v[0]);
    q.y = ptx::to_tf32(v[1]);
    q.z = ptx::to_tf32(v[2]);
    q.w = ptx::to_tf32(v[3]);
    *reinterpret_cast<float4*>(tile + off) = q;
  }
}

// thread -> (row, chunk) of slot i.  rowmajor: consecutive threads take
// consecutive ROWS (rows contiguous in gmem); else consecutive 4-element K
// chunks (K contiguous in gmem).
template <int ROWS>
__device__ __forceinline__ void slot_of(int i, bool rowmajor, int& row, int& ch) {
  const int q = threadIdx.x + i * NT;
  if (rowmajor) {
    row = q % ROWS;
    ch = q / ROWS;
  } else {
    ch = q & 7;
    row = q >> 3;
  }
}

template <int BN, bool SPLIT3>
struct TileCfg {
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int NS = SPLIT3 ? 2 : 1;
  static constexpr int STAGE_BYTES = (A_BYTES + B_BYTES) * NS;
  static constexpr int STAGES_RAW = (44 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 4 ? 4 : (STAGES_RAW < 2 ? 2 : STAGES_RAW);
  static constexpr int TAB_OFF = STAGES * STAGE_BYTES;
  static constexpr int SMEM_MAX = TAB_OFF + TAB_MAX_INTS * 4 + 1024;
  static constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr int PA = BM * 8 / NT;  // A chunks per thread per stage
  static constexpr int PB = BN * 8 / NT;  // B chunks per thread per stage
};

// per-CTA K table: nk entries per sub-table (nk = this CTA's K extent)
struct Tab {
  const int* t;
  int nk;
};

// K range of a split + split-K partial output ([split][N][M], M fastest)
struct KRange {
  int kb_total = 0, kb_per = 0;
  float* part = nullptr;
  int part_m = 0, part_n = 0;
  __device__ __forceinline__ void k_range(int z, int& kb0, int& kb1) const {
    kb0 = z * kb_per;
    kb1 = kb0 + kb_per;
    if (kb1 > kb_total) kb1 = kb_total;
  }
};

// The generic kernel.  Prob supplies
//   static constexpr int TABLES                        K tables (ints per K entry)
//   void setup(int* tab, int kbase, int nk)            fill them (all threads)
//   bool a_rowmajor() / b_rowmajor()                   thread mapping of the gathers
//   ACtx a_ctx(int m) / BCtx b_ctx(int n)              per-row context, once per CTA
//   void a4(ACtx, Tab, int kt, int k, float (&v)[4])   A(m, k..k+3), kt = k - kbase
//   void b4(BCtx, Tab, int kt, int k, float (&v)[4])   B(n, k..k+3)
//   ECtx e_ctx(int m); void store(ECtx, int n, float v) final epilogue
template <class Prob, int BN, bool SPLIT3>
__global__ void __launch_bounds__(NT, 2) tc_gemm_kernel(const Prob p) {
  using C = TileCfg<BN, SPLIT3>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  __shared__ uint64_t empty_bar[C::STAGES];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  int kb0, kb1;
  p.k_range(blockIdx.z, kb0, kb1);
  const int nkb = kb1 > kb0 ? kb1 - kb0 : 0;
  const int kbase = kb0 * BK;
  const bool arm = p.a_rowmajor(), brm = p.b_rowmajor();

  if (warp == 0) {
    ptx::tmem_alloc(&tmem_base_sh, C::TMEM_COLS);
    ptx::tmem_relinquish();
  }
  if (tid == 32) {
#pragma unroll
    for (int s = 0; s < C::STAGES; ++s) ptx::mbar_init(&empty_bar[s], 1);
    ptx::mbar_init(&done_bar, 1);
    ptx::fence_mbar_init();
  }
  int* tabp = reinterpret_cast<int*>(smem + C::TAB_OFF);
  const Tab tab{tabp, nkb * BK};
  if (Prob::TABLES > 0) p.setup(tabp, kbase, nkb * BK);

  // per-thread row contexts (loop invariant)
  typename Prob::ACtx actx[C::PA];
  typename Prob::BCtx bctx[C::PB];
#pragma unroll
  for (int i = 0; i < C::PA; ++i) {
    int row, ch;
    slot_of<BM>(i, arm, row, ch);
    actx[i] = p.a_ctx(m0 + row);
  }
#pragma unroll
  for (int i = 0; i < C::PB; ++i) {
    int row, ch;
    slot_of<BN>(i, brm, row, ch);
    bctx[i] = p.b_ctx(n0 + row);
  }

  ptx::tc_fence_before();
  __syncthreads();  // TMEM address, barriers and K tables visible
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  constexpr uint32_t IDESC = ptx::idesc_tf32(BM, BN);

  // phase 1 of the gather: all loads of one stage into registers
  float va[C::PA][4], vb[C::PB][4];
  auto gather = [&](int k0) {
#pragma unroll
    for (int i = 0; i < C::PA; ++i) {
      int row, ch;
      slot_of<BM>(i, arm, row, ch);
      p.a4(actx[i], tab, k0 - kbase + ch * 4, k0 + ch * 4, va[i]);
    }
#pragma unroll
    for (int i = 0; i < C::PB; ++i) {
      int row, ch;
      slot_of<BN>(i, brm, row, ch);
      p.b4(bctx[i], tab, k0 - kbase + ch * 4, k0 + ch * 4, vb[i]);
    }
  };
  // software pipeline: iteration it stores stage it (gathered during
  // iteration it-1), then issues the loads of stage it+1 and the MMAs of
  // stage it -- one copy of the gather / store code keeps the loop small.
  for (int it = -1; it < nkb; ++it) {
    const int s = it < 0 ? 0 : it % C::STAGES;
    uint8_t* sa = smem + s * C::STAGE_BYTES;
    uint8_t* sb = sa + C::A_BYTES * C::NS;
    if (it >= 0) {
      if (it >= C::STAGES) ptx::mbar_wait(&empty_bar[s], (uint32_t)((it / C::STAGES) - 1) & 1u);
      // phase 2: convert + swizzled st.shared
#pragma unroll
      for (int i = 0; i < C::PA; ++i) {
        int row, ch;
        slot_of<BM>(i, arm, row, ch);
        store_chunk<SPLIT3, BM>(sa, row, ch, va[i]);
      }
#pragma unroll
      for (int i = 0; i < C::PB; ++i) {
        int row, ch;
        slot_of<BN>(i, brm, row, ch);
        store_chunk<SPLIT3, BN>(sb, row, ch, vb[i]);
      }
      ptx::fence_proxy_async_smem();
      __syncthreads();
    }
    if (it + 1 < nkb) gather(kbase + (it + 1) * BK);  // loads of the next stage in flight
    if (it >= 0 && tid == 0) {
      ptx::tc_fence_after();
      const uint32_t a_addr = ptx::smem_u32(sa), b_addr = ptx::smem_u32(sb);
#pragma unroll
      for (int kk = 0; kk < BK / 8; ++kk) {
        const uint64_t ad = ptx::sw128_kmajor_desc(a_addr + kk * 32);
        const uint64_t bd = ptx::sw128_kmajor_desc(b_addr + kk * 32);
        ptx::mma_tf32(tmem, ad, bd, IDESC, (it > 0 || kk > 0) ? 1u : 0u);
        if (SPLIT3) {
          const uint64_t adl = ptx::sw128_kmajor_desc(a_addr + C::A_BYTES + kk * 32);
          const uint64_t bdl = ptx::sw128_kmajor_desc(b_addr + C::B_BYTES + kk * 32);
          ptx::mma_tf32(tmem, ad, bdl, IDESC, 1u);
          ptx::mma_tf32(tmem, adl, bd, IDESC, 1u);
        }
      }
      ptx::mma_commit(&empty_bar[s]);
    }
  }
  if (tid == 0) ptx::mma_commit(&done_bar);
  ptx::mbar_wait(&done_bar, 0);
  ptx::tc_fence_after();

  // epilogue: thread owns accumulator row (warp*32 + lane)
  const int m = m0 + warp * 32 + lane;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  if (p.part) {  // split-K partial, [split][N][M]: lanes write consecutive m
    float* dst = p.part + (int64_t)blockIdx.z * p.part_n * p.part_m + m;
    const bool mok = m < p.part_m;
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      uint32_t r[16];
      ptx::tmem_ld16(trow + (uint32_t)c, r);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = n0 + c + j;
        if (mok && n < p.part_n) dst[(int64_t)n * p.part_m] = nkb > 0 ? __uint_as_float(r[j]) : 0.f;
      }
    }
  } else {
    const typename Prob::ECtx ec = p.e_ctx(m);
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      uint32_t r[16];
      ptx::tmem_ld16(trow + (uint32_t)c, r);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j) p.store(ec, n0 + c + j, nkb > 0 ? __uint_as_float(r[j]) : 0.f);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, C::TMEM_COLS);
}

// Fixed-order split-K reductions + the problem's own epilogue.
// Few splits: one thread per output, 4 independent accumulators.
template <class Prob>
__global__ void splitk_reduce_small(const Prob p, int splits) {
  const int64_t M = p.part_m, N = p.part_n, total = M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int z = 0;
    for (; z + 3 < splits; z += 4) {
      a0 += p.part[(int64_t)z * total + i];
      a1 += p.part[(int64_t)(z + 1) * total + i];
      a2 += p.part[(int64_t)(z + 2) * total + i];
      a3 += p.part[(int64_t)(z + 3) * total + i];
    }
    for (; z < splits; ++z) a0 += p.part[(int64_t)z * total + i];
    const int n = (int)(i / M), m = (int)(i - (int64_t)n * M);
    p.store(p.e_ctx(m), n, (a0 + a1) + (a2 + a3));
  }
}

// Many splits: a block owns 32 consecutive outputs; its 8 warps each sum a
// strided subset of the splits (4 accumulators), then warp-0 lanes add the 8
// partial sums in warp order -- fixed order, deterministic.
template <class Prob>
__global__ void splitk_reduce_kernel(const Prob p, int splits) {
  __shared__ float sh[8][33];
  const int64_t M = p.part_m, N = p.part_n, total = M * N;
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * 32 + lane;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  if (i < total) {
    int z = g;
    for (; z + 24 < splits; z += 32) {
      a0 += p.part[(int64_t)z * total + i];
      a1 += p.part[(int64_t)(z + 8) * total + i];
      a2 += p.part[(int64_t)(z + 16) * total + i];
      a3 += p.part[(int64_t)(z + 24) * total + i];
    }
    for (; z < splits; z += 8) a0 += p.part[(int64_t)z * total + i];
  }
  sh[g][lane] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (g == 0 && i < total) {
    float acc = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) acc += sh[w][lane];
    const int n = (int)(i / M), m = (int)(i - (int64_t)n * M);
    p.store(p.e_ctx(m), n, acc);
  }
}

// ============================================================================
// problems
// ============================================================================
// conv forward: D[m = pixel (b,oy,ox)][n = map] = sum_k x[b][c][oy*s+ky][ox*s+kx] W[n][k]
// table: im2col offset c*H*W + ky*W + kx of every k (-1 past kd)
struct ConvFwdProb : KRange {
  ConvDesc d;
  const float* x;
  const float* w;
  const float* bias;
  float* y;
  int act;
  static constexpr int TABLES = 1;
  using ACtx = int;  // pixel base offset into x, -1 past M
  using BCtx = int;  // n * kd, -1 past K
  __device__ void setup(int* tab, int kbase, int nk) const {
    const int Kd = (int)d.kd(), khw = d.kh * d.kw;
    for (int t = threadIdx.x; t < nk; t += NT) {
      const int k = kbase + t;
      int v = -1;
      if (k < Kd) {
        const int c = k / khw, rem = k - c * khw, ky = rem / d.kw, kx = rem - ky * d.kw;
        v = (c * d.H + ky) * d.W + kx;
      }
      tab[t] = v;
    }
  }
  __device__ bool a_rowmajor() const { return true; }
  __device__ bool b_rowmajor() const { return false; }
  __device__ __forceinline__ int a_ctx(int m) const {
    if (m >= (int)d.pixels()) return -1;
    const int ohw = d.OH * d.OW, b = m / ohw, r = m - b * ohw, oy = r / d.OW, ox = r - oy * d.OW;
    return b * d.C * d.H * d.W + oy * d.s * d.W + ox * d.s;
  }
  __device__ __forceinline__ int b_ctx(int n) const { return n < d.K ? n * (int)d.kd() : -1; }
  __device__ __forceinline__ void a4(int ctx, Tab tab, int kt, int, float (&v)[4]) const {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int o = tab.t[kt + e];
      v[e] = (ctx >= 0 && o >= 0) ? __ldg(x + ctx + o) : 0.f;
    }
  }
  __device__ __forceinline__ void b4(int ctx, Tab, int, int k, float (&v)[4]) const {
    const int Kd = (int)d.kd();
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = (ctx >= 0 && k + e < Kd) ? __ldg(w + ctx + k + e) : 0.f;
  }
  using ECtx = int64_t;  // offset of (b, n=0, r) in y, -1 past M
  __device__ __forceinline__ int64_t e_ctx(int m) const {
    if (m >= (int)d.pixels()) return -1;
    const int ohw = d.OH * d.OW, b = m / ohw;
    return (int64_t)b * d.K * ohw + (m - b * ohw);
  }
  __device__ __forceinline__ void store(int64_t ec, int n, float v) const {
    if (ec < 0 || n >= d.K) return;
    y[ec + (int64_t)n * d.OH * d.OW] = epi_act(act, v + bias[n]);
  }
};

// conv wgrad: D[k (patch row; k == kd -> ones = bias)][n] = sum_p P[k][p] G[n][p]
// tables (K = pixels): [0,nk) pixel base into x, [nk,2nk) pixel base into G
struct ConvWgradProb : KRange {
  ConvDesc d;
  const float* x;
  const float* g;  // pre-activation gradient [B][K][OH][OW]
  float* dw;
  float* db;
  static constexpr int TABLES = 2;
  using ACtx = int;  // im2col offset of patch row k; -2 = ones (bias row); -3 = zero row
  using BCtx = int;  // n * OH*OW, -1 past K
  __device__ void setup(int* tab, int kbase, int nk) const {
    const int P = (int)d.pixels(), ohw = d.OH * d.OW;
    for (int t = threadIdx.x; t < nk; t += NT) {
      const int p = kbase + t;
      int xb = -1, gb = -1;
      if (p < P) {
        const int b = p / ohw, r = p - b * ohw, oy = r / d.OW, ox = r - oy * d.OW;
        xb = b * d.C * d.H * d.W + oy * d.s * d.W + ox * d.s;
        gb = b * d.K * ohw + r;
      }
      tab[t] = xb;
      tab[nk + t] = gb;
    }
  }
  __device__ bool a_rowmajor() const { return false; }
  __device__ bool b_rowmajor() const { return false; }
  __device__ __forceinline__ int a_ctx(int k) const {
    const int Kd = (int)d.kd(), khw = d.kh * d.kw;
    if (k > Kd) return -3;
    if (k == Kd) return -2;
    const int c = k / khw, rem = k - c * khw, ky = rem / d.kw, kx = rem - ky * d.kw;
    return (c * d.H + ky) * d.W + kx;
  }
  __device__ __forceinline__ int b_ctx(int n) const { return n < d.K ? n * d.OH * d.OW : -1; }
  __device__ __forceinline__ void a4(int ctx, Tab tab, int pt, int, float (&v)[4]) const {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int xb = tab.t[pt + e];
      float val = 0.f;
      if (xb >= 0) val = ctx >= 0 ? __ldg(x + xb + ctx) : (ctx == -2 ? 1.f : 0.f);
      v[e] = val;
    }
  }
  __device__ __forceinline__ void b4(int ctx, Tab tab, int pt, int, float (&v)[4]) const {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int gb = tab.t[tab.nk + pt + e];
      v[e] = (ctx >= 0 && gb >= 0) ? __ldg(g + gb + ctx) : 0.f;
    }
  }
  using ECtx = int;  // patch row k
  __device__ __forceinline__ int e_ctx(int k) const { return k; }
  __device__ __forceinline__ void store(int k, int n, float v) const {
    const int Kd = (int)d.kd();
    if (k > Kd || n >= d.K) return;
    if (k < Kd) dw[(int64_t)n * Kd + k] = v;
    else db[n] = v;
  }
};

// implicit conv dgrad: D[m = input pixel (b,y,x)][c] =
//   sum_{n,ky,kx} G[b][n][(y-ky)/s][(x-kx)/s] W[n][c][ky][kx]
// tables (K = (n,ky,kx)): [0,nk) n*OH*OW (-1 past), [nk,2nk) ky<<16|kx,
// [2nk,3nk) n*kd + ky*kw + kx (W offset without the c term)
struct DgradCtx {
  int gb, y, x;
};
template <bool UNIT>
struct ConvDgradProb : KRange {
  ConvDesc d;
  const float* g;
  const float* w;
  float* dx;
  const float* yprev;
  int act_prev;
  static constexpr int TABLES = 3;
  using ACtx = DgradCtx;
  using BCtx = int;  // c * kh*kw, -1 past C
  __device__ void setup(int* tab, int kbase, int nk) const {
    const int KK = d.K * d.kh * d.kw, khw = d.kh * d.kw, ohw = d.OH * d.OW, Kd = (int)d.kd();
    for (int t = threadIdx.x; t < nk; t += NT) {
      const int k = kbase + t;
      int go = -1, kyx = 0, wo = -1;
      if (k < KK) {
        const int n = k / khw, rem = k - n * khw, ky = rem / d.kw, kx = rem - ky * d.kw;
        go = n * ohw;
        kyx = (ky << 16) | kx;
        wo = n * Kd + rem;
      }
      tab[t] = go;
      tab[nk + t] = kyx;
      tab[2 * nk + t] = wo;
    }
  }
  __device__ bool a_rowmajor() const { return true; }
  __device__ bool b_rowmajor() const { return false; }
  __device__ __forceinline__ DgradCtx a_ctx(int m) const {
    const int HW = d.H * d.W;
    if (m >= d.B * HW) return DgradCtx{-1, 0, 0};
    const int b = m / HW, r = m - b * HW, y = r / d.W;
    return DgradCtx{b * d.K * d.OH * d.OW, y, r - y * d.W};
  }
  __device__ __forceinline__ int b_ctx(int c) const { return c < d.C ? c * d.kh * d.kw : -1; }
  __device__ __forceinline__ void a4(DgradCtx ctx, Tab tab, int kt, int, float (&v)[4]) const {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int go = tab.t[kt + e];
      const int kyx = tab.t[tab.nk + kt + e];
      float val = 0.f;
      if (ctx.gb >= 0 && go >= 0) {
        int ty = ctx.y - (kyx >> 16), tx = ctx.x - (kyx & 0xFFFF);
        bool ok = ty >= 0 && tx >= 0;
        if (!UNIT && ok) {  // strided conv: only positions on the stride grid
          ok = (ty % d.s == 0) && (tx % d.s == 0);
          ty /= d.s;
          tx /= d.s;
        }
        if (ok && ty < d.OH && tx < d.OW) val = __ldg(g + ctx.gb + go + ty * d.OW + tx);
      }
      v[e] = val;
    }
  }
  __device__ __forceinline__ void b4(int ctx, Tab tab, int kt, int, float (&v)[4]) const {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int wo = tab.t[2 * tab.nk + kt + e];
      v[e] = (ctx >= 0 && wo >= 0) ? __ldg(w + wo + ctx) : 0.f;
    }
  }
  using ECtx = int64_t;  // offset of (b, c=0, y, x) in dx, -1 past M
  __device__ __forceinline__ int64_t e_ctx(int m) const {
    const int HW = d.H * d.W;
    if (m >= d.B * HW) return -1;
    const int b = m / HW;
    return (int64_t)b * d.C * HW + (m - b * HW);
  }
  __device__ __forceinline__ void store(int64_t ec, int c, float v) const {
    if (ec < 0 || c >= d.C) return;
    const int64_t i = ec + (int64_t)c * d.H * d.W;
    if (yprev) v *= epi_dact(act_prev, yprev[i]);
    dx[i] = v;
  }
};

// explicit conv dgrad GEMM: dP[k][p] = sum_n W[n][k] G[b][n][r]  (p = b*OHW + r)
struct ConvDPProb : KRange {
  ConvDesc d;
  const float* g;
  const float* w;
  float* dP;  // [kd][pixels]
  static constexpr int TABLES = 0;
  using ACtx = int;  // k, -1 past kd
  using BCtx = int;  // b*K*OHW + r, -1 past pixels
  __device__ void setup(int*, int, int) const {}
  __device__ bool a_rowmajor() const { return true; }  // A(k, n) = W[n][k]: k contiguous
  __device__ bool b_rowmajor() const { return true; }  // B(p, n) = G: p contiguous
  __device__ __forceinline__ int a_ctx(int k) const { return k < (int)d.kd() ? k : -1; }
  __device__ __forceinline__ int b_ctx(int p) const {
    if (p >= (int)d.pixels()) return -1;
    const int ohw = d.OH * d.OW, b = p / ohw;
    return b * d.K * ohw + (p - b * ohw);
  }
  __device__ __forceinline__ void a4(int ctx, Tab, int, int n, float (&v)[4]) const {
    const int Kd = (int)d.kd();
#pragma unroll
    for (int e = 0; e < 4; ++e)
      v[e] = (ctx >= 0 && n + e < d.K) ? __ldg(w + (int64_t)(n + e) * Kd + ctx) : 0.f;
  }
  __device__ __forceinline__ void b4(int ctx, Tab, int, int n, float (&v)[4]) const {
    const int ohw = d.OH * d.OW;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      v[e] = (ctx >= 0 && n + e < d.K) ? __ldg(g + ctx + (n + e) * ohw) : 0.f;
  }
  using ECtx = int64_t;  // row offset k * pixels, -1 past kd
  __device__ __forceinline__ int64_t e_ctx(int k) const {
    return k < (int)d.kd() ? (int64_t)k * d.pixels() : -1;
  }
  __device__ __forceinline__ void store(int64_t ec, int p, float v) const {
    if (ec < 0 || p >= (int)d.pixels()) return;
    dP[ec + p] = v;
  }
};

// generic dense GEMM with strided operand access:
//   A(m,k) = a[m*as_m + k*as_k], B(n,k) = b[n*bs_n + k*bs_k]   (beyond bounds: 0)
// plus an optional "ones" column at n == ones_col (bias-gradient fold).
enum { EPI_PLAIN = 0, EPI_BIAS_ACT = 1, EPI_DACT = 2, EPI_WGRAD = 3 };
struct DenseProb : KRange {
  int M, N, K;
  const float* a;
  int64_t as_m, as_k;
  const float* b;
  int64_t bs_n, bs_k;
  int ones_col;
  int epi;
  float* c;
  int64_t ldc;
  const float* bias;
  int act;
  const float* yprev;
  float* db;
  static constexpr int TABLES = 0;
  using ACtx = int64_t;  // m*as_m, -1 past M
  using BCtx = int64_t;  // n*bs_n, -1 past N, -2 ones column
  __device__ void setup(int*, int, int) const {}
  __device__ bool a_rowmajor() const { return as_m == 1; }
  __device__ bool b_rowmajor() const { return bs_n == 1; }
  __device__ __forceinline__ int64_t a_ctx(int m) const { return m < M ? m * as_m : -1; }
  __device__ __forceinline__ int64_t b_ctx(int n) const {
    return n >= N ? -1 : (n == ones_col ? -2 : n * bs_n);
  }
  __device__ __forceinline__ void a4(int64_t ctx, Tab, int, int k, float (&v)[4]) const {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      v[e] = (ctx >= 0 && k + e < K) ? __ldg(a + ctx + (int64_t)(k + e) * as_k) : 0.f;
  }
  __device__ __forceinline__ void b4(int64_t ctx, Tab, int, int k, float (&v)[4]) const {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float val = 0.f;
      if (ctx != -1 && k + e < K) val = ctx == -2 ? 1.f : __ldg(b + ctx + (int64_t)(k + e) * bs_k);
      v[e] = val;
    }
  }
  using ECtx = int;  // row m
  __device__ __forceinline__ int e_ctx(int m) const { return m; }
  __device__ __forceinline__ void store(int m, int n, float v) const {
    if (m >= M || n >= N) return;
    switch (epi) {
      case EPI_BIAS_ACT: c[m * ldc + n] = epi_act(act, v + bias[n]); break;
      case EPI_DACT: {
        const int64_t i = m * ldc + n;
        c[i] = yprev ? v * epi_dact(act, yprev[i]) : v;
        break;
      }
      case EPI_WGRAD:
        if (n == ones_col) db[m] = v;
        else c[m * ldc + n] = v;
        break;
      default: c[m * ldc + n] = v;
    }
  }
};

// ============================================================================
// planning + launch
// ============================================================================
int pick_bn(int64_t n) {
  if (n <= 16) return 16;
  if (n <= 32) return 32;
  if (n <= 64) return 64;
  if (n <= 128) return 128;
  return 256;
}

bool fits_i32(int64_t v) { return v < (int64_t(1) << 31) - 1; }

struct Plan {
  int bn = 16;
  int64_t mt = 0, nt = 0;
  int kb_total = 0, kb_per = 0, splits = 1;
  int tables = 0;
  int64_t M = 0, N = 0;
  size_t ws_bytes() const {
    return splits > 1 ? sizeof(float) * (size_t)(splits * M * N) : 0;
  }
  size_t tab_bytes() const { return sizeof(int) * (size_t)tables * kb_per * BK; }
};

// Split K so that tiles * splits covers <= 3 CTAs per SM (one wave), with >= min_kb K
// blocks per split (the partial write + reduce must pay for itself) and
// <= the K blocks whose offset tables fit in shared memory.
Plan make_plan(int64_t M, int64_t N, int64_t K, int tables, int min_kb = 2) {
  Plan p;
  p.M = M;
  p.N = N;
  p.tables = tables;
  p.bn = pick_bn(N);
  p.mt = cdiv(M, BM);
  p.nt = cdiv(N, p.bn);
  p.kb_total = (int)cdiv(K, BK);
  if (p.kb_total < 1) p.kb_total = 1;
  const int64_t tiles = p.mt * p.nt;
  const int64_t target = CTAS_PER_SM * (int64_t)sm_count();
  int64_t splits = 1;
  if (tiles < target) {
    splits = target / tiles;  // floor: never spill a near-empty extra wave
    int64_t cap = p.kb_total / min_kb;
    if (cap < 1) cap = 1;
    if (splits > cap) splits = cap;
  }
  if (tables > 0) {  // K tables must fit: kb_per * 32 * tables <= TAB_MAX_INTS
    const int64_t kb_cap = TAB_MAX_INTS / (BK * tables);
    const int64_t need = cdiv(p.kb_total, kb_cap);
    if (splits < need) splits = need;
  }
  p.kb_per = (int)cdiv(p.kb_total, splits);
  p.splits = (int)cdiv(p.kb_total, p.kb_per);
  return p;
}

template <class Prob, int BN, bool SPLIT3>
int launch_one(const Prob& p, dim3 grid, size_t tab_bytes, cudaStream_t st) {
  using C = TileCfg<BN, SPLIT3>;
  static bool configured = false;  // attribute set once per instantiation
  if (!configured) {
    VCNN_CUDA_TRY(cudaFuncSetAttribute(tc_gemm_kernel<Prob, BN, SPLIT3>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_MAX));
    configured = true;
  }
  const size_t smem = C::TAB_OFF + tab_bytes + 1024;
  tc_gemm_kernel<Prob, BN, SPLIT3><<<grid, NT, smem, st>>>(p);
  VCNN_LAUNCHED();
  return VCNN_OK;
}

template <class Prob, bool SPLIT3>
int launch_bn(const Prob& p, int bn, dim3 grid, size_t tab, cudaStream_t st) {
  switch (bn) {
    case 16: return launch_one<Prob, 16, SPLIT3>(p, grid, tab, st);
    case 32: return launch_one<Prob, 32, SPLIT3>(p, grid, tab, st);
    case 64: return launch_one<Prob, 64, SPLIT3>(p, grid, tab, st);
    case 128: return launch_one<Prob, 128, SPLIT3>(p, grid, tab, st);
    default: return launch_one<Prob, 256, SPLIT3>(p, grid, tab, st);
  }
}

// run a planned problem: GEMM (+ split-K reduce with the fused epilogue)
template <class Prob>
int run(Prob p, const Plan& pl, bool split3, const Workspace& ws, cudaStream_t st) {
  p.kb_total = pl.kb_total;
  p.kb_per = pl.kb_per;
  p.part = nullptr;
  if (pl.splits > 1) {
    if (!ws.ptr || ws.bytes < pl.ws_bytes())
      return fail(VCNN_ECUDA, "tc gemm: split-K workspace too small");
    p.part = ws.ptr;
    p.part_m = (int)pl.M;
    p.part_n = (int)pl.N;
  }
  dim3 grid((unsigned)pl.mt, (unsigned)pl.nt, (unsigned)pl.splits);
  int s = split3 ? launch_bn<Prob, true>(p, pl.bn, grid, pl.tab_bytes(), st)
                 : launch_bn<Prob, false>(p, pl.bn, grid, pl.tab_bytes(), st);
  if (s || pl.splits == 1) return s;
  if (pl.splits <= 16) {
    int64_t blocks = cdiv(pl.M * pl.N, 256);
    if (blocks > 8 * sm_count()) blocks = 8 * sm_count();
    splitk_reduce_small<Prob><<<(unsigned)blocks, 256, 0, st>>>(p, pl.splits);
  } else {
    splitk_reduce_kernel<Prob><<<(unsigned)cdiv(pl.M * pl.N, 32), 256, 0, st>>>(p, pl.splits);
  }
  VCNN_LAUNCHED();
  return VCNN_OK;
}

DenseProb dense_prob(int M, int N, int K, const float* a, int64_t as_m, int64_t as_k,
                     const float* b, int64_t bs_n, int64_t bs_k, int ones_col, int epi, float* c,
                     int64_t ldc, const float* bias, int act, const float* yprev, float* db) {
  DenseProb p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.a = a;
  p.as_m = as_m;
  p.as_k = as_k;
  p.b = b;
  p.bs_n = bs_n;
  p.bs_k = bs_k;
  p.ones_col = ones_col;
  p.epi = epi;
  p.c = c;
  p.ldc = ldc;
  p.bias = bias;
  p.act = act;
  p.yprev = yprev;
  p.db = db;
  return p;
}

bool explicit_dgrad(const ConvDesc& d) {
  // implicit dgrad multiplies H*W/(OH*OW) times the algorithmic work
  return (int64_t)d.H * d.W > 2 * (int64_t)d.OH * d.OW;
}

Plan plan_conv_fwd(const ConvDesc& d) { return make_plan(d.pixels(), d.K, d.kd(), 1); }
Plan plan_conv_wgrad(const ConvDesc& d) { return make_plan(d.kd() + 1, d.K, d.pixels(), 2, 4); }
Plan plan_conv_dgrad_implicit(const ConvDesc& d) {
  return make_plan((int64_t)d.B * d.H * d.W, d.C, (int64_t)d.K * d.kh * d.kw, 3);
}
Plan plan_conv_dP(const ConvDesc& d) { return make_plan(d.kd(), d.pixels(), d.K, 0); }
Plan plan_full_fwd(int B, int in, int out) { return make_plan(B, out, in, 0); }
Plan plan_full_wgrad(int B, int in, int out) { return make_plan(out, in + 1, B, 0); }
Plan plan_full_dgrad(int B, int in, int out) { return make_plan(B, in, out, 0); }

size_t align_up(size_t v) { return (v + 255) & ~(size_t)255; }

}  // namespace

// ============================================================================
// workspace requirements (max over the ops the engine will run)
// ============================================================================
size_t conv_workspace(const ConvDesc& d) {
  size_t w = plan_conv_fwd(d).ws_bytes();
  w = std::max(w, plan_conv_wgrad(d).ws_bytes());
  if (explicit_dgrad(d)) {
    w = std::max(w, align_up(sizeof(float) * (size_t)(d.kd() * d.pixels())) +
                        plan_conv_dP(d).ws_bytes());
  } else {
    w = std::max(w, plan_conv_dgrad_implicit(d).ws_bytes());
  }
  return w;
}

size_t full_workspace(int B, int in, int out) {
  size_t w = plan_full_fwd(B, in, out).ws_bytes();
  w = std::max(w, plan_full_wgrad(B, in, out).ws_bytes());
  w = std::max(w, plan_full_dgrad(B, in, out).ws_bytes());
  return w;
}

size_t matmul_workspace(int64_t m, int64_t k, int64_t n) {
  return make_plan(m, n, k, 0).ws_bytes();
}

// ============================================================================
// public tc:: launchers
// ============================================================================
static int check_conv(const ConvDesc& d, const char* what) {
  if (!fits_i32(d.in_size()) || !fits_i32(d.out_size()) || !fits_i32(d.kd() * d.pixels()))
    return fail(VCNN_ESHAPE, std::string(what) + ": tensor exceeds 2^31 elements");
  return VCNN_OK;
}

int conv_fwd(const ConvDesc& d, const float* x, const float* w, const float* b, int act,
             float* y, bool split3, const Workspace& ws, cudaStream_t st) {
  if (int s = check_conv(d, "conv_fwd")) return s;
  ConvFwdProb p;
  p.d = d;
  p.x = x;
  p.w = w;
  p.bias = b;
  p.y = y;
  p.act = act;
  return run(p, plan_conv_fwd(d), split3, ws, st);
}

int conv_wgrad(const ConvDesc& d, const float* x, const float* gpre, float* dw, float* db,
               bool split3, const Workspace& ws, cudaStream_t st) {
  if (int s = check_conv(d, "conv_wgrad")) return s;
  ConvWgradProb p;
  p.d = d;
  p.x = x;
  p.g = gpre;
  p.dw = dw;
  p.db = db;
  return run(p, plan_conv_wgrad(d), split3, ws, st);
}

int conv_dgrad(const ConvDesc& d, const float* gpre, const float* w, float* dx,
               const float* yprev, int act_prev, bool split3, const Workspace& ws,
               cudaStream_t st) {
  if (int s = check_conv(d, "conv_dgrad")) return s;
  if (explicit_dgrad(d)) {
    // dP = W^T G (exactly the algorithmic MACs), then col2im gather (+ act')
    const size_t dp_bytes = align_up(sizeof(float) * (size_t)(d.kd() * d.pixels()));
    if (!ws.ptr || ws.bytes < dp_bytes) return fail(VCNN_ECUDA, "conv_dgrad: workspace too small");
    ConvDPProb p;
    p.d = d;
    p.g = gpre;
    p.w = w;
    p.dP = ws.ptr;
    Workspace rest{reinterpret_cast<float*>(reinterpret_cast<char*>(ws.ptr) + dp_bytes),
                   ws.bytes - dp_bytes};
    if (int s = run(p, plan_conv_dP(d), split3, rest, st)) return s;
    return launch_col2im(d, ws.ptr, dx, st, yprev, act_prev);
  }
  auto go = [&](auto p) {
    p.d = d;
    p.g = gpre;
    p.w = w;
    p.dx = dx;
    p.yprev = yprev;
    p.act_prev = act_prev;
    return run(p, plan_conv_dgrad_implicit(d), split3, ws, st);
  };
  return d.s == 1 ? go(ConvDgradProb<true>{}) : go(ConvDgradProb<false>{});
}

// FC forward: y[b][o] = act(sum_i x[b][i] W[o][i] + bias[o])
int full_fwd(int B, int in, int out, const float* x, const float* w, const float* b, int act,
             float* y, bool split3, const Workspace& ws, cudaStream_t st) {
  return run(dense_prob(B, out, in, x, in, 1, w, in, 1, -1, EPI_BIAS_ACT, y, out, b, act, nullptr,
                        nullptr),
             plan_full_fwd(B, in, out), split3, ws, st);
}

// FC wgrad: dW[o][i] = sum_b G[b][o] x[b][i]; ones column i == in -> db[o]
int full_wgrad(int B, int in, int out, const float* x, const float* gpre, float* dw, float* db,
               bool split3, const Workspace& ws, cudaStream_t st) {
  return run(dense_prob(out, in + 1, B, gpre, 1, out, x, 1, in, in, EPI_WGRAD, dw, in, nullptr, 0,
                        nullptr, db),
             plan_full_wgrad(B, in, out), split3, ws, st);
}

// FC dgrad: dx[b][i] = (sum_o G[b][o] W[o][i]) * act_prev'(yprev[b][i])
int full_dgrad(int B, int in, int out, const float* gpre, const float* w, float* dx,
               const float* yprev, int act_prev, bool split3, const Workspace& ws,
               cudaStream_t st) {
  return run(dense_prob(B, in, out, gpre, out, 1, w, 1, in, -1, EPI_DACT, dx, in, nullptr,
                        act_prev, yprev, nullptr),
             plan_full_dgrad(B, in, out), split3, ws, st);
}

int matmul(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c,
           bool transB, bool split3, const Workspace& ws, cudaStream_t st) {
  if (!fits_i32(m) || !fits_i32(n) || !fits_i32(k))
    return fail(VCNN_ESHAPE, "matmul: extent exceeds 2^31");
  const Plan pl = make_plan(m, n, k, 0);
  if (transB)
    return run(dense_prob((int)m, (int)n, (int)k, a, k, 1, b, k, 1, -1, EPI_PLAIN, c, n, nullptr,
                          0, nullptr, nullptr),
               pl, split3, ws, st);
  return run(dense_prob((int)m, (int)n, (int)k, a, k, 1, b, 1, n, -1, EPI_PLAIN, c, n, nullptr, 0,
                        nullptr, nullptr),
             pl, split3, ws, st);
}

}  // namespace tc
}  // namespace vcnn_b200
