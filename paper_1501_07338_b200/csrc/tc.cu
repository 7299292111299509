// tc.cu -- tcgen05 implicit-GEMM engine for every GEMM-shaped op of the
// VCNN training step (conv fwd / wgrad / dgrad, FC fwd / wgrad / dgrad,
// matmul).  One CTA = 128 threads computes a 128 x BN tile of D in TMEM:
//   * all 4 warps gather operands straight from the NCHW tensors (implicit
//     im2col / col2im: no patch matrix ever touches HBM) into 128B-swizzled
//     K-major shared-memory tiles, rounding to tf32 (or splitting hi/lo for
//     the fp32-faithful 3xTF32 mode);
//   * one elected thread issues tcgen05.mma.kind::tf32 (M=128, N=BN, K=8) and
//     tcgen05.commit's the stage back to an mbarrier, so the gather of stage
//     s+1 overlaps the MMAs of stage s (STAGES-deep ring);
//   * the epilogue reads TMEM with tcgen05.ld (thread = row) and fuses bias,
//     activation, the upstream activation derivative, or the split-K
//     partial store.
// The bias gradient is folded into the wgrad GEMMs as one extra K-row /
// N-column of ones, so dB costs no extra pass.  Deterministic: split-K
// partials are reduced in a fixed order by a second kernel.
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace vcnn_b200 {
namespace tc {

namespace {

constexpr int BM = 128;      // rows per tile == TMEM lanes
constexpr int BK = 32;       // fp32 K per stage == one 128-B swizzle row
constexpr int NT = 128;      // threads per CTA

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

// consecutive threads -> consecutive ROWS (use when rows are contiguous in gmem)
template <int ROWS, bool SPLIT3, class F>
__device__ __forceinline__ void fill_rowmajor(uint8_t* tile, F&& f) {
  constexpr int PER = ROWS * 8 / NT;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int q = threadIdx.x + i * NT;
    const int row = q % ROWS, ch = q / ROWS;
    float v[4];
    f(row, ch, v);
    store_chunk<SPLIT3, ROWS>(tile, row, ch, v);
  }
}

// consecutive threads -> consecutive 4-element K chunks (K contiguous in gmem)
template <int ROWS, bool SPLIT3, class F>
__device__ __forceinline__ void fill_kcontig(uint8_t* tile, F&& f) {
  constexpr int PER = ROWS * 8 / NT;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int q = threadIdx.x + i * NT;
    const int ch = q & 7, row = q >> 3;
    float v[4];
    f(row, ch, v);
    store_chunk<SPLIT3, ROWS>(tile, row, ch, v);
  }
}

template <int BN, bool SPLIT3>
struct TileCfg {
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int NS = SPLIT3 ? 2 : 1;
  static constexpr int STAGE_BYTES = (A_BYTES + B_BYTES) * NS;
  static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 4 ? 4 : (STAGES_RAW < 2 ? 2 : STAGES_RAW);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024;
  static constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
};

// The generic kernel.  Prob supplies:
//   void k_range(int z, int& kb0, int& kb1)        -- K blocks of split z
//   void fill_a<SPLIT3>(uint8_t*, int m0, int k0)   -- 128 x 32 tile
//   void fill_b<BN,SPLIT3>(uint8_t*, int n0, int k0)-- BN x 32 tile
//   void store(int m, int n, float v, int z)         -- epilogue, per element
template <class Prob, int BN, bool SPLIT3>
__global__ void __launch_bounds__(NT, 1) tc_gemm_kernel(const Prob p) {
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
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  constexpr uint32_t IDESC = ptx::idesc_tf32(BM, BN);

  for (int it = 0; it < nkb; ++it) {
    const int s = it % C::STAGES;
    if (it >= C::STAGES) ptx::mbar_wait(&empty_bar[s], (uint32_t)((it / C::STAGES) - 1) & 1u);
    uint8_t* sa = smem + s * C::STAGE_BYTES;
    uint8_t* sb = sa + C::A_BYTES * C::NS;
    const int k0 = (kb0 + it) * BK;
    p.template fill_a<SPLIT3>(sa, m0, k0);
    p.template fill_b<BN, SPLIT3>(sb, n0, k0);
    ptx::fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
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
#pragma unroll 1
  for (int c = 0; c < BN; c += 16) {
    uint32_t r[16];
    ptx::tmem_ld16(trow + (uint32_t)c, r);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 16; ++j)
      p.store(m, n0 + c + j, nkb > 0 ? __uint_as_float(r[j]) : 0.f, (int)blockIdx.z);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, C::TMEM_COLS);
}

// ============================================================================
// problems
// ============================================================================
struct KRange {
  int kb_total = 0, kb_per = 0;
  __device__ __forceinline__ void k_range(int z, int& kb0, int& kb1) const {
    kb0 = z * kb_per;
    kb1 = kb0 + kb_per;
    if (kb1 > kb_total) kb1 = kb_total;
  }
};

// conv forward: D[m = pixel (b,oy,ox)][n = map] = sum_k x[b][c][oy*s+ky][ox*s+kx] W[n][k]
struct ConvFwdProb : KRange {
  ConvDesc d;
  const float* x;
  const float* w;
  const float* bias;
  float* y;
  int act;

  template <bool SPLIT3>
  __device__ __forceinline__ void fill_a(uint8_t* t, int m0, int k0) const {
    const int M = (int)d.pixels(), Kd = (int)d.kd(), khw = d.kh * d.kw;
    const int ohw = d.OH * d.OW, HW = d.H * d.W, CHW = d.C * HW;
    fill_rowmajor<BM, SPLIT3>(t, [&](int row, int ch, float (&v)[4]) {
      const int m = m0 + row;
      int kk = k0 + ch * 4;
      if (m >= M) {
        v[0] = v[1] = v[2] = v[3] = 0.f;
        return;
      }
      const int b = m / ohw, r = m - b * ohw;
      const int oy = r / d.OW, ox = r - oy * d.OW;
      const float* xb = x + (int64_t)b * CHW + oy * d.s * d.W + ox * d.s;
      int c = kk / khw, rem = kk - c * khw;
      int ky = rem / d.kw, kx = rem - ky * d.kw;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        v[e] = (kk + e < Kd) ? __ldg(xb + c * HW + ky * d.W + kx) : 0.f;
        if (++kx == d.kw) {
          kx = 0;
          if (++ky == d.kh) {
            ky = 0;
            ++c;
          }
        }
      }
    });
  }
  template <int BN, bool SPLIT3>
  __device__ __forceinline__ void fill_b(uint8_t* t, int n0, int k0) const {
    const int Kd = (int)d.kd();
    fill_kcontig<BN, SPLIT3>(t, [&](int row, int ch, float (&v)[4]) {
      const int n = n0 + row, kk = k0 + ch * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        v[e] = (n < d.K && kk + e < Kd) ? __ldg(w + (int64_t)n * Kd + kk + e) : 0.f;
    });
  }
  __device__ __forceinline__ void store(int m, int n, float v, int) const {
    if (m >= (int)d.pixels() || n >= d.K) return;
    const int ohw = d.OH * d.OW;
    const int b = m / ohw, r = m - b * ohw;
    y[((int64_t)b * d.K + n) * ohw + r] = act_fwd(act, v + bias[n]);
  }
};

// conv wgrad: D[k (patch row; k==kd -> ones = bias)][n] = sum_pixels P[k][p] G[n][p]
struct ConvWgradProb : KRange {
  ConvDesc d;
  const float* x;
  const float* g;  // pre-activation gradient [B][K][OH][OW]
  float* part;     // [splits][K][kd+1]

  template <bool SPLIT3>
  __device__ __forceinline__ void fill_a(uint8_t* t, int m0, int k0) const {
    const int P = (int)d.pixels(), Kd = (int)d.kd(), khw = d.kh * d.kw;
    const int ohw = d.OH * d.OW, HW = d.H * d.W, CHW = d.C * HW;
    // this thread's 4 pixels (fixed chunk ch = tid & 7)
    const int ch = threadIdx.x & 7;
    int base[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int p = k0 + ch * 4 + e;
      if (p < P) {
        const int b = p / ohw, r = p - b * ohw;
        const int oy = r / d.OW, ox = r - oy * d.OW;
        base[e] = b * CHW + oy * d.s * d.W + ox * d.s;
      } else {
        base[e] = -1;
      }
    }
    fill_kcontig<BM, SPLIT3>(t, [&](int row, int, float (&v)[4]) {
      const int k = m0 + row;
      if (k < Kd) {
        const int c = k / khw, rem = k - c * khw;
        const int ky = rem / d.kw, kx = rem - ky * d.kw;
        const int off = c * HW + ky * d.W + kx;
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = base[e] >= 0 ? __ldg(x + base[e] + off) : 0.f;
      } else {
        const float one = (k == Kd) ? 1.f : 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = base[e] >= 0 ? one : 0.f;
      }
    });
  }
  template <int BN, bool SPLIT3>
  __device__ __forceinline__ void fill_b(uint8_t* t, int n0, int k0) const {
    const int P = (int)d.pixels(), ohw = d.OH * d.OW;
    const int ch = threadIdx.x & 7;
    int gb[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int p = k0 + ch * 4 + e;
      if (p < P) {
        const int b = p / ohw, r = p - b * ohw;
        gb[e] = b * d.K * ohw + r;
      } else {
        gb[e] = -1;
      }
    }
    fill_kcontig<BN, SPLIT3>(t, [&](int row, int, float (&v)[4]) {
      const int n = n0 + row;
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = (n < d.K && gb[e] >= 0) ? __ldg(g + gb[e] + n * ohw) : 0.f;
    });
  }
  __device__ __forceinline__ void store(int m, int n, float v, int z) const {
    const int Kd1 = (int)d.kd() + 1;
    if (m >= Kd1 || n >= d.K) return;
    part[((int64_t)z * d.K + n) * Kd1 + m] = v;
  }
};

// conv dgrad: D[m = input pixel (b,y,x)][c] = sum_{n,ky,kx} G[b][n][(y-ky)/s][(x-kx)/s] W[n][c][ky][kx]
struct ConvDgradProb : KRange {
  ConvDesc d;
  const float* g;
  const float* w;
  float* dx;
  const float* yprev;
  int act_prev;

  template <bool SPLIT3>
  __device__ __forceinline__ void fill_a(uint8_t* t, int m0, int k0) const {
    const int M = (int)d.in_size() / d.C;  // B*H*W
    const int KK = d.K * d.kh * d.kw, khw = d.kh * d.kw;
    const int HW = d.H * d.W, ohw = d.OH * d.OW;
    fill_rowmajor<BM, SPLIT3>(t, [&](int row, int ch, float (&v)[4]) {
      const int m = m0 + row;
      int kk = k0 + ch * 4;
      if (m >= M) {
        v[0] = v[1] = v[2] = v[3] = 0.f;
        return;
      }
      const int b = m / HW, r = m - b * HW;
      const int y = r / d.W, xx = r - y * d.W;
      const float* gb = g + (int64_t)b * d.K * ohw;
      int n = kk / khw, rem = kk - n * khw;
      int ky = rem / d.kw, kx = rem - ky * d.kw;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float val = 0.f;
        if (kk + e < KK) {
          const int ty = y - ky, tx = xx - kx;
          if (ty >= 0 && tx >= 0) {
            const int oy = ty / d.s, ox = tx / d.s;
            if (oy * d.s == ty && ox * d.s == tx && oy < d.OH && ox < d.OW)
              val = __ldg(gb + n * ohw + oy * d.OW + ox);
          }
        }
        v[e] = val;
        if (++kx == d.kw) {
          kx = 0;
          if (++ky == d.kh) {
            ky = 0;
            ++n;
          }
        }
      }
    });
  }
  template <int BN, bool SPLIT3>
  __device__ __forceinline__ void fill_b(uint8_t* t, int n0, int k0) const {
    const int KK = d.K * d.kh * d.kw, khw = d.kh * d.kw, Kd = (int)d.kd();
    fill_kcontig<BN, SPLIT3>(t, [&](int row, int ch, float (&v)[4]) {
      const int c = n0 + row;
      int kk = k0 + ch * 4;
      int n = kk / khw, rem = kk - n * khw;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        v[e] = (c < d.C && kk + e < KK) ? __ldg(w + (int64_t)n * Kd + c * khw + rem) : 0.f;
        if (++rem == khw) {
          rem = 0;
          ++n;
        }
      }
    });
  }
  __device__ __forceinline__ void store(int m, int c, float v, int) const {
    const int HW = d.H * d.W;
    if (m >= d.B * HW || c >= d.C) return;
    const int b = m / HW, r = m - b * HW;
    const int64_t i = ((int64_t)b * d.C + c) * HW + r;
    if (yprev) v *= act_grad_from_out(act_prev, yprev[i]);
    dx[i] = v;
  }
};

// generic dense GEMM with strided operand access:
//   A(m,k) = a[m*as_m + k*as_k], B(n,k) = b[n*bs_n + k*bs_k]   (beyond bounds: 0)
// plus an optional "ones" column at n == N1 (bias-gradient fold).
// Epilogue modes: plain store, bias+act (FC fwd), act'-scaled (FC dgrad),
// wgrad split (dw / db).
enum { EPI_PLAIN = 0, EPI_BIAS_ACT = 1, EPI_DACT = 2, EPI_WGRAD = 3 };
struct DenseProb : KRange {
  int M, N, K;          // logical extents (N includes a ones column if ones_col >= 0)
  const float* a;
  int64_t as_m, as_k;
  const float* b;
  int64_t bs_n, bs_k;
  int ones_col;         // B(ones_col, k) = 1 for k < K
  bool a_rows_contig;   // as_m == 1 -> use row-major thread mapping
  bool b_rows_contig;
  int epi;
  float* c;
  int64_t ldc;
  const float* bias;    // EPI_BIAS_ACT
  int act;
  const float* yprev;   // EPI_DACT
  float* db;            // EPI_WGRAD: column ones_col goes to db[m]

  template <bool SPLIT3>
  __device__ __forceinline__ void fill_a(uint8_t* t, int m0, int k0) const {
    auto f = [&](int row, int ch, float (&v)[4]) {
      const int mm = m0 + row, kk = k0 + ch * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        v[e] = (mm < M && kk + e < K) ? __ldg(a + mm * as_m + (int64_t)(kk + e) * as_k) : 0.f;
    };
    if (a_rows_contig) fill_rowmajor<BM, SPLIT3>(t, f);
    else fill_kcontig<BM, SPLIT3>(t, f);
  }
  template <int BN, bool SPLIT3>
  __device__ __forceinline__ void fill_b(uint8_t* t, int n0, int k0) const {
    auto f = [&](int row, int ch, float (&v)[4]) {
      const int nn = n0 + row, kk = k0 + ch * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float val = 0.f;
        if (nn < N && kk + e < K)
          val = (nn == ones_col) ? 1.f : __ldg(b + nn * bs_n + (int64_t)(kk + e) * bs_k);
        v[e] = val;
      }
    };
    if (b_rows_contig) fill_rowmajor<BN, SPLIT3>(t, f);
    else fill_kcontig<BN, SPLIT3>(t, f);
  }
  __device__ __forceinline__ void store(int m, int n, float v, int) const {
    if (m >= M || n >= N) return;
    switch (epi) {
      case EPI_BIAS_ACT: c[m * ldc + n] = act_fwd(act, v + bias[n]); break;
      case EPI_DACT: {
        const int64_t i = m * ldc + n;
        c[i] = yprev ? v * act_grad_from_out(act, yprev[i]) : v;
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

// deterministic split-K reduction for conv wgrad: dw[n][k] = sum_z part[z][n][k]
__global__ void wgrad_reduce_kernel(int splits, int K, int Kd, const float* __restrict__ part,
                                    float* __restrict__ dw, float* __restrict__ db) {
  const int Kd1 = Kd + 1;
  const int64_t total = (int64_t)K * Kd1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int z = 0; z < splits; ++z) acc += part[(int64_t)z * total + i];
    const int n = (int)(i / Kd1), k = (int)(i - (int64_t)n * Kd1);
    if (k < Kd) dw[(int64_t)n * Kd + k] = acc;
    else db[n] = acc;
  }
}

template <class Prob, int BN, bool SPLIT3>
int launch_one(const Prob& p, dim3 grid, cudaStream_t st) {
  using C = TileCfg<BN, SPLIT3>;
  static bool configured = false;  // attribute set once per instantiation
  if (!configured) {
    VCNN_CUDA_TRY(cudaFuncSetAttribute(tc_gemm_kernel<Prob, BN, SPLIT3>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    configured = true;
  }
  tc_gemm_kernel<Prob, BN, SPLIT3><<<grid, NT, C::SMEM, st>>>(p);
  VCNN_LAUNCHED();
  return VCNN_OK;
}

template <class Prob, bool SPLIT3>
int launch_bn(const Prob& p, int bn, dim3 grid, cudaStream_t st) {
  switch (bn) {
    case 16: return launch_one<Prob, 16, SPLIT3>(p, grid, st);
    case 32: return launch_one<Prob, 32, SPLIT3>(p, grid, st);
    case 64: return launch_one<Prob, 64, SPLIT3>(p, grid, st);
    case 128: return launch_one<Prob, 128, SPLIT3>(p, grid, st);
    default: return launch_one<Prob, 256, SPLIT3>(p, grid, st);
  }
}

template <class Prob>
int launch(const Prob& p, int bn, dim3 grid, bool split3, cudaStream_t st) {
  return split3 ? launch_bn<Prob, true>(p, bn, grid, st) : launch_bn<Prob, false>(p, bn, grid, st);
}

int pick_bn(int n) {
  if (n <= 16) return 16;
  if (n <= 32) return 32;
  if (n <= 64) return 64;
  if (n <= 128) return 128;
  return 256;
}

bool fits_i32(int64_t v) { return v < (int64_t(1) << 31) - 1; }

void set_k(KRange& kr, int64_t K, int splits) {
  kr.kb_total = (int)cdiv(K, BK);
  if (splits < 1) splits = 1;
  kr.kb_per = (int)cdiv(kr.kb_total, splits);
  if (kr.kb_per < 1) kr.kb_per = 1;
}

int dense(int M, int N, int K, const float* a, int64_t as_m, int64_t as_k, const float* b,
          int64_t bs_n, int64_t bs_k, int ones_col, int epi, float* c, int64_t ldc,
          const float* bias, int act, const float* yprev, float* db, bool split3,
          cudaStream_t st) {
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
  p.a_rows_contig = (as_m == 1);
  p.b_rows_contig = (bs_n == 1);
  p.epi = epi;
  p.c = c;
  p.ldc = ldc;
  p.bias = bias;
  p.act = act;
  p.yprev = yprev;
  p.db = db;
  set_k(p, K, 1);
  const int bn = pick_bn(N);
  dim3 grid((unsigned)cdiv(M, BM), (unsigned)cdiv(N, bn), 1);
  return launch(p, bn, grid, split3, st);
}

}  // namespace

// ============================================================================
// public tc:: launchers
// ============================================================================
int conv_fwd(const ConvDesc& d, const float* x, const float* w, const float* b, int act,
             float* y, bool split3, cudaStream_t st) {
  if (!fits_i32(d.in_size()) || !fits_i32(d.out_size()))
    return fail(VCNN_ESHAPE, "conv_fwd: tensor exceeds 2^31 elements");
  ConvFwdProb p;
  p.d = d;
  p.x = x;
  p.w = w;
  p.bias = b;
  p.y = y;
  p.act = act;
  set_k(p, d.kd(), 1);
  const int bn = pick_bn(d.K);
  dim3 grid((unsigned)cdiv(d.pixels(), BM), (unsigned)cdiv(d.K, bn), 1);
  return launch(p, bn, grid, split3, st);
}

size_t conv_wgrad_workspace(const ConvDesc& d) {
  const int64_t mt = cdiv(d.kd() + 1, BM);
  const int bn = pick_bn(d.K);
  const int64_t nt = cdiv(d.K, bn);
  const int64_t kb_total = cdiv(d.pixels(), BK);
  int64_t splits = (2 * sm_count()) / (mt * nt);
  if (splits < 1) splits = 1;
  if (splits > kb_total) splits = kb_total;
  const int64_t per = cdiv(kb_total, splits);
  splits = cdiv(kb_total, per);
  return sizeof(float) * (size_t)(splits * d.K * (d.kd() + 1));
}

int conv_wgrad(const ConvDesc& d, const float* x, const float* gpre, float* dw, float* db,
               bool split3, const Workspace& ws, cudaStream_t st) {
  if (!fits_i32(d.in_size()) || !fits_i32(d.out_size()))
    return fail(VCNN_ESHAPE, "conv_wgrad: tensor exceeds 2^31 elements");
  ConvWgradProb p;
  p.d = d;
  p.x = x;
  p.g = gpre;
  const int64_t mt = cdiv(d.kd() + 1, BM);
  const int bn = pick_bn(d.K);
  const int64_t nt = cdiv(d.K, bn);
  const int64_t kb_total = cdiv(d.pixels(), BK);
  int64_t splits = (2 * sm_count()) / (mt * nt);
  if (splits < 1) splits = 1;
  if (splits > kb_total) splits = kb_total;
  const int64_t per = cdiv(kb_total, splits);
  splits = cdiv(kb_total, per);
  const size_t need = sizeof(float) * (size_t)(splits * d.K * (d.kd() + 1));
  if (ws.bytes < need || !ws.ptr) return fail(VCNN_ECUDA, "conv_wgrad: workspace too small");
  p.part = ws.ptr;
  p.kb_total = (int)kb_total;
  p.kb_per = (int)per;
  dim3 grid((unsigned)mt, (unsigned)nt, (unsigned)splits);
  int s = launch(p, bn, grid, split3, st);
  if (s) return s;
  const int64_t total = (int64_t)d.K * (d.kd() + 1);
  wgrad_reduce_kernel<<<(unsigned)cdiv(total, 256), 256, 0, st>>>((int)splits, d.K, (int)d.kd(),
                                                                  ws.ptr, dw, db);
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int conv_dgrad(const ConvDesc& d, const float* gpre, const float* w, float* dx,
               const float* yprev, int act_prev, bool split3, cudaStream_t st) {
  if (!fits_i32(d.in_size()) || !fits_i32(d.out_size()))
    return fail(VCNN_ESHAPE, "conv_dgrad: tensor exceeds 2^31 elements");
  ConvDgradProb p;
  p.d = d;
  p.g = gpre;
  p.w = w;
  p.dx = dx;
  p.yprev = yprev;
  p.act_prev = act_prev;
  set_k(p, (int64_t)d.K * d.kh * d.kw, 1);
  const int bn = pick_bn(d.C);
  const int64_t M = (int64_t)d.B * d.H * d.W;
  dim3 grid((unsigned)cdiv(M, BM), (unsigned)cdiv(d.C, bn), 1);
  return launch(p, bn, grid, split3, st);
}

// FC forward: y[b][o] = act(sum_i x[b][i] W[o][i] + bias[o])
int full_fwd(int B, int in, int out, const float* x, const float* w, const float* b, int act,
             float* y, bool split3, cudaStream_t st) {
  return dense(B, out, in, x, in, 1, w, in, 1, -1, EPI_BIAS_ACT, y, out, b, act, nullptr,
               nullptr, split3, st);
}

// FC wgrad: dW[o][i] = sum_b G[b][o] x[b][i]; ones column i == in -> db[o]
int full_wgrad(int B, int in, int out, const float* x, const float* gpre, float* dw, float* db,
               bool split3, cudaStream_t st) {
  return dense(out, in + 1, B, gpre, 1, out, x, 1, in, in, EPI_WGRAD, dw, in, nullptr, 0,
               nullptr, db, split3, st);
}

// FC dgrad: dx[b][i] = (sum_o G[b][o] W[o][i]) * act_prev'(yprev[b][i])
int full_dgrad(int B, int in, int out, const float* gpre, const float* w, float* dx,
               const float* yprev, int act_prev, bool split3, cudaStream_t st) {
  return dense(B, in, out, gpre, out, 1, w, 1, in, -1, EPI_DACT, dx, in, nullptr, act_prev,
               yprev, nullptr, split3, st);
}

int matmul(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c,
           bool transB, bool split3, cudaStream_t st) {
  if (!fits_i32(m) || !fits_i32(n) || !fits_i32(k))
    return fail(VCNN_ESHAPE, "matmul: extent exceeds 2^31");
  if (transB)
    return dense((int)m, (int)n, (int)k, a, k, 1, b, k, 1, -1, EPI_PLAIN, c, n, nullptr, 0,
                 nullptr, nullptr, split3, st);
  return dense((int)m, (int)n, (int)k, a, k, 1, b, 1, n, -1, EPI_PLAIN, c, n, nullptr, 0,
               nullptr, nullptr, split3, st);
}

}  // namespace tc
}  // namespace vcnn_b200
