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
#include <type_traits>

#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace vcnn_b200 {
namespace tc {

#ifdef VCNN_PHASE_TIMING
// clock64 stamps of the first 8 CTAs of the last tc_gemm launch (debug build)
__device__ unsigned long long g_phase[8][16];
#define PHASE(i)                                                             \
  do {                                                                       \
    if (blockIdx.x + blockIdx.y + blockIdx.z < 8 && (threadIdx.x & 31) == 0) \
      g_phase[blockIdx.x + blockIdx.y + blockIdx.z][(i)] = clock64();        \
  } while (0)
#define PHASE_ACC_DECL unsigned long long _acc0 = 0, _acc1 = 0, _t0 = 0;
#define PHASE_T0() _t0 = clock64()
#define PHASE_ACC(a) a += clock64() - _t0
#define PHASE_PUT(i, a)                                                      \
  do {                                                                       \
    if (blockIdx.x + blockIdx.y + blockIdx.z < 8)                            \
      g_phase[blockIdx.x + blockIdx.y + blockIdx.z][(i)] = (a);              \
  } while (0)
#else
#define PHASE_ACC_DECL
#define PHASE_T0()
#define PHASE_ACC(a)
#define PHASE_PUT(i, a)
#define PHASE(i) \
  do {           \
  } while (0)
#endif

namespace {

constexpr int BM = 128;            // rows per tile == TMEM lanes
constexpr int BK = 32;             // fp32 K per stage == one 128-B swizzle row
constexpr int NT = 128;            // producer / epilogue threads (4 warps, one per TMEM lane quarter)
constexpr int NTH = NT + 32;       // + 1 MMA-issuer warp = threads per CTA
constexpr int MAX_STAGES = 8;
constexpr int TAB_MAX_INTS = 4096; // per-CTA K-offset tables (16 KB)
constexpr int CTAS_PER_SM = 3;     // smem sized for 3 resident CTAs / SM
constexpr size_t kSmemOptin = 227 * 1024;

// Out-of-line activation helpers for the epilogues: the unrolled epilogue
// would otherwise inline the transcendental branches 16x per TMEM load and
// blow the instruction cache (the kernels are I$-bound when every launch is
// a different kernel).
__device__ __noinline__ float epi_act(int act, float x) { return act_fwd(act, x); }
__device__ __noinline__ float epi_dact(int act, float y) { return act_grad_from_out(act, y); }

// store 4 consecutive K values of one row into a SW128 K-major tile
// (CVT = false: the values are already tf32-rounded, e.g. staged in a slab)
template <bool SPLIT3, int ROWS, bool CVT = true>
__device__ __forceinline__ void store_chunk(uint8_t* tile, int row, int ch, const float (&v)[4]) {
  const uint32_t off = (uint32_t)row * 128u + ((uint32_t)(ch ^ (row & 7)) << 4);
  if (!SPLIT3 && !CVT) {
    *reinterpret_cast<float4*>(tile + off) = make_float4(v[0], v[1], v[2], v[3]);
  } else if (SPLIT3) {
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
  // 3xTF32: the main (hi*hi) products rotate over R TMEM accumulators per
  // K block and the two correction products (hi*lo, lo*hi) go to a separate
  // one, so no accumulator sees more than 1/R of the main MMAs and the small
  // terms are never added into a large accumulator (the tensor core's fp32
  // accumulation truncates; this keeps the fp32-faithful path within 1e-5
  // at K ~ 3e4).  Slots are summed in a fixed order in the epilogue.
  static constexpr int R = !SPLIT3 ? 1 : (BN >= 256 ? 1 : BN == 128 ? 3 : 7);
  static constexpr uint32_t ACC_COLS = BN < 16 ? 16 : BN;
  static constexpr uint32_t TMEM_NEED = SPLIT3 ? (uint32_t)(R + 1) * ACC_COLS : ACC_COLS;
  static constexpr uint32_t TMEM_COLS = TMEM_NEED <= 32    ? 32
                                        : TMEM_NEED <= 64  ? 64
                                        : TMEM_NEED <= 128 ? 128
                                        : TMEM_NEED <= 256 ? 256
                                                           : 512;
  static constexpr int PA = BM * 8 / NT;  // A chunks per thread per stage
  static constexpr int PB = BN * 8 / NT;  // B chunks per thread per stage
};

// per-CTA K table: nk entries per sub-table (nk = this CTA's K extent), and
// the CTA's shared-memory slab (problems that stage their inputs)
struct Tab {
  const int* t;
  int nk;
  uint32_t ta;  // shared address of t
  uint32_t sa;  // shared address of the slab
  __device__ __forceinline__ int t1(int i) const { return ptx::lds_s32(ta + 4u * (uint32_t)i); }
  __device__ __forceinline__ int4 t4(int i) const { return ptx::lds_s32x4(ta + 4u * (uint32_t)i); }
  __device__ __forceinline__ float s1(int i) const { return ptx::lds_f32(sa + 4u * (uint32_t)i); }
  __device__ __forceinline__ float4 s4(int i) const { return ptx::lds_f32x4(sa + 4u * (uint32_t)i); }
};

// K range of a split + split-K partial output ([split][N][M], M fastest).
// Also the defaults of the optional problem hooks:
//   SLAB      stage(float* slab, int tile, int n0, int z, uint64_t* bar): all threads copy the
//             CTA's input window into shared memory once (coalesced, fused
//             routing / tf32 rounding); a4/b4 then gather from Tab::s.
//   PRE_ROUNDED  a4/b4 return tf32-rounded values (no cvt at the tile store).
//   SMEM_EPI  the accumulator tile goes to shared memory ([n][128], raw) and
//             smem_epilogue(ep, tile, n0, bn) finishes it with all threads
//             (cross-row epilogues such as a fused max-pool).
struct KRange {
  static constexpr bool SLAB = false;
  static constexpr bool PRE_ROUNDED = false;
  static constexpr bool SMEM_EPI = false;
  // TWO_PHASE: a4/b4 take their chunk's K-table entries (int4) loaded in a
  // first pass (ta4/tb4), so all table loads of a stage are in flight before
  // the dependent operand loads
  static constexpr bool TWO_PHASE = false;
  // A_ZERO_ROWS: a_zero(ctx) marks A rows that are identically zero (M
  // padding); once every ring slot holds them they are not rewritten
  static constexpr bool A_ZERO_ROWS = false;
  int kb_total = 0, kb_per = 0;
  float* part = nullptr;
  int part_m = 0, part_n = 0;
  int nst = 2;       // ring depth (stages), set at launch from the free shared memory
  int slab_off = 0;  // bytes from the table area to the slab (set by run())
  __device__ __forceinline__ void k_range(int z, int& kb0, int& kb1) const {
    kb0 = z * kb_per;
    kb1 = kb0 + kb_per;
    if (kb1 > kb_total) kb1 = kb_total;
  }
};

// The generic kernel.  Prob supplies
//   static constexpr int TABLES                        K tables (ints per K entry)
//   void setup(int* tab, int kbase, int nk)            fill them (all NTH threads)
//   bool a_rowmajor() / b_rowmajor()                   thread mapping of the gathers
//   ACtx a_ctx(int m) / BCtx b_ctx(int n)              per-row context, once per CTA
//   void a4(ACtx, Tab, int kt, int k, float (&v)[4])   A(m, k..k+3), kt = k - kbase
//   void b4(BCtx, Tab, int kt, int k, float (&v)[4])   B(n, k..k+3)
//   ECtx e_ctx(int m); void store(ECtx, int n, float v) final epilogue
// Warp-specialised pipeline: warps 0-3 produce stages (gather -> swizzled
// st.shared, software-pipelined one stage ahead in registers) into a ring of
// p.nst stages and arrive on full[s]; warp 4 (one elected lane) waits full[s],
// issues the tcgen05.mma's and commits them to empty[s].  No CTA-wide barrier
// inside the K loop.  Epilogue: warps 0-3, thread = TMEM lane = row.
template <class Prob, int BN, bool SPLIT3>
__global__ void __launch_bounds__(NTH, 1) tc_gemm_kernel(const Prob p) {
  pdl_launch_dependents();
  using C = TileCfg<BN, SPLIT3>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  __shared__ uint64_t full_bar[MAX_STAGES];
  __shared__ uint64_t empty_bar[MAX_STAGES];
  __shared__ uint64_t done_bar;
  __shared__ uint64_t stage_bar;
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int S = p.nst;
  if (tid == 0) PHASE(0);
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
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full_bar[s], 4);  // one arrive per producer warp
      ptx::mbar_init(&empty_bar[s], 1);
    }
    ptx::mbar_init(&done_bar, 1);
    ptx::fence_mbar_init();
  }
  pdl_wait();  // TMEM / barrier setup above overlapped the previous kernel
  const int tab_off = S * C::STAGE_BYTES;
  int* tabp = reinterpret_cast<int*>(smem + tab_off);
  float* slab = reinterpret_cast<float*>(smem + tab_off + p.slab_off);
  const Tab tab{tabp, nkb * BK, ptx::smem_u32(tabp), ptx::smem_u32(slab)};
  if (Prob::TABLES > 0) p.setup(tabp, kbase, nkb * BK);
  if (tid == 0) PHASE(1);
  if constexpr (Prob::SLAB) p.stage(slab, blockIdx.x, n0, blockIdx.z, &stage_bar);

  ptx::tc_fence_before();
  __syncthreads();  // TMEM address, barriers, K tables and slab visible
  ptx::tc_fence_after();
  if (tid == 0) PHASE(2);
  const uint32_t tmem = tmem_base_sh;
  constexpr uint32_t IDESC = ptx::idesc_tf32(BM, BN);

  if (warp == 4) {
    // ---------------- MMA issuer (one elected lane of a converged warp, so
    // the tcgen05 issue stays on the uniform datapath) ----------------
    if (ptx::elect_one()) {
      PHASE_ACC_DECL
      for (int it = 0; it < nkb; ++it) {
        const int s = it % S;
        PHASE_T0();
        ptx::mbar_wait(&full_bar[s], (uint32_t)(it / S) & 1u);
        PHASE_ACC(_acc0);
        ptx::tc_fence_after();
        uint8_t* sa = smem + s * C::STAGE_BYTES;
        uint8_t* sb = sa + C::A_BYTES * C::NS;
        const uint32_t a_addr = ptx::smem_u32(sa), b_addr = ptx::smem_u32(sb);
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          const uint64_t ad = ptx::sw128_kmajor_desc(a_addr + kk * 32);
          const uint64_t bd = ptx::sw128_kmajor_desc(b_addr + kk * 32);
          if constexpr (!SPLIT3) {
            ptx::mma_tf32(tmem, ad, bd, IDESC, (it > 0 || kk > 0) ? 1u : 0u);
          } else {
            const uint32_t tm = tmem + (uint32_t)((it % C::R) * C::ACC_COLS);
            const uint32_t tc = tmem + (uint32_t)(C::R * C::ACC_COLS);
            const uint64_t adl = ptx::sw128_kmajor_desc(a_addr + C::A_BYTES + kk * 32);
            const uint64_t bdl = ptx::sw128_kmajor_desc(b_addr + C::B_BYTES + kk * 32);
            ptx::mma_tf32(tm, ad, bd, IDESC, (it >= C::R || kk > 0) ? 1u : 0u);
            ptx::mma_tf32(tc, ad, bdl, IDESC, (it > 0 || kk > 0) ? 1u : 0u);
            ptx::mma_tf32(tc, adl, bd, IDESC, 1u);
          }
        }
        ptx::mma_commit(&empty_bar[s]);
      }
      ptx::mma_commit(&done_bar);
      PHASE(4);
      PHASE_PUT(13, _acc0);
    }
    __syncwarp();
  } else {
    // ---------------- producers (warps 0-3) ----------------
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
    float va[C::PA][4], vb[C::PB][4];
    auto gather = [&](int k0) {
      if constexpr (Prob::TWO_PHASE) {
        int4 ta[C::PA], tb[C::PB];
#pragma unroll
        for (int i = 0; i < C::PA; ++i) {
          int row, ch;
          slot_of<BM>(i, arm, row, ch);
          ta[i] = p.ta4(tab, k0 - kbase + ch * 4);
        }
#pragma unroll
        for (int i = 0; i < C::PB; ++i) {
          int row, ch;
          slot_of<BN>(i, brm, row, ch);
          tb[i] = p.tb4(tab, k0 - kbase + ch * 4);
        }
#pragma unroll
        for (int i = 0; i < C::PA; ++i) {
          int row, ch;
          slot_of<BM>(i, arm, row, ch);
          p.a4(actx[i], tab, ta[i], k0 + ch * 4, va[i]);
        }
#pragma unroll
        for (int i = 0; i < C::PB; ++i) {
          int row, ch;
          slot_of<BN>(i, brm, row, ch);
          p.b4(bctx[i], tab, tb[i], k0 + ch * 4, vb[i]);
        }
      } else {
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
      }
    };
    PHASE_ACC_DECL
    if (nkb > 0) gather(kbase);
    for (int it = 0; it < nkb; ++it) {
      const int s = it % S;
      uint8_t* sa = smem + s * C::STAGE_BYTES;
      uint8_t* sb = sa + C::A_BYTES * C::NS;
      PHASE_T0();
      if (it >= S) ptx::mbar_wait(&empty_bar[s], (uint32_t)((it / S) - 1) & 1u);
      PHASE_ACC(_acc0);
#pragma unroll
      for (int i = 0; i < C::PA; ++i) {
        int row, ch;
        slot_of<BM>(i, arm, row, ch);
        if constexpr (Prob::A_ZERO_ROWS)
          if (it >= S && p.a_zero(actx[i])) continue;  // still zero from the first pass
        store_chunk<SPLIT3, BM, !Prob::PRE_ROUNDED>(sa, row, ch, va[i]);
      }
#pragma unroll
      for (int i = 0; i < C::PB; ++i) {
        int row, ch;
        slot_of<BN>(i, brm, row, ch);
        store_chunk<SPLIT3, BN, !Prob::PRE_ROUNDED>(sb, row, ch, vb[i]);
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&full_bar[s]);
      PHASE_T0();
      if (it + 1 < nkb) gather(kbase + (it + 1) * BK);  // next stage's loads in flight
      PHASE_ACC(_acc1);
    }
    if (tid == 0) PHASE(3);
    if (tid == 0) PHASE_PUT(12, _acc0);
    if (tid == 0) PHASE_PUT(14, _acc1);
    if (tid == 0) PHASE_PUT(15, (unsigned long long)S);
  }
  ptx::mbar_wait(&done_bar, 0);
  ptx::tc_fence_after();
  if (tid == 0) PHASE(5);

  // epilogue: warps 0-3, thread owns accumulator row (warp*32 + lane)
  const int m = m0 + (warp & 3) * 32 + lane;
  const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  // 16 accumulator columns of this row (3xTF32: main slots in order, then the
  // corrections; slots beyond nkb were never written)
  auto acc16 = [&](int c, uint32_t (&r)[16]) {
    ptx::tmem_ld16(trow + (uint32_t)c, r);
    ptx::tmem_wait_ld();
    if constexpr (SPLIT3) {
      const int slots = nkb < C::R ? nkb : C::R;
      for (int j = 1; j <= slots; ++j) {
        uint32_t q[16];
        const int col = j < slots ? j * (int)C::ACC_COLS : C::R * (int)C::ACC_COLS;
        ptx::tmem_ld16(trow + (uint32_t)(col + c), q);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int t = 0; t < 16; ++t)
          r[t] = __float_as_uint(__uint_as_float(r[t]) + __uint_as_float(q[t]));
      }
    }
  };
  if constexpr (Prob::SMEM_EPI) {
    // raw accumulators -> shared memory [n][BM] (the stage ring is idle now:
    // every stage was consumed by the MMAs done_bar tracked; the CTA barrier
    // also orders the producers' last stage writes for tools that do not
    // follow mbarrier / tcgen05.commit ordering, e.g. racecheck)
    __syncthreads();
    float* ep = reinterpret_cast<float*>(smem);
    if (warp < 4) {
      const uint32_t eb = ptx::smem_u32(ep);
      const int row = warp * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        uint32_t r[16];
        acc16(c, r);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          ptx::sts_f32(eb + 4u * ((c + j) * BM + row), nkb > 0 ? __uint_as_float(r[j]) : 0.f);
      }
    }
    __syncthreads();
    p.smem_epilogue(ep, blockIdx.x, n0, BN);
  } else if (warp < 4) {
    if (p.part) {  // split-K partial, [split][N][M]: lanes write consecutive m
      float* dst = p.part + (int64_t)blockIdx.z * p.part_n * p.part_m + m;
      const bool mok = m < p.part_m;
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        uint32_t r[16];
        acc16(c, r);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int n = n0 + c + j;
          if (mok && n < p.part_n)
            dst[(int64_t)n * p.part_m] = nkb > 0 ? __uint_as_float(r[j]) : 0.f;
        }
      }
    } else {
      const typename Prob::ECtx ec = p.e_ctx(m);
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        uint32_t r[16];
        acc16(c, r);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          p.store(ec, n0 + c + j, nkb > 0 ? __uint_as_float(r[j]) : 0.f);
      }
    }
  }
  if (tid == 0) PHASE(6);
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, C::TMEM_COLS);
  if (tid == 0) PHASE(7);
}

// Fixed-order split-K reductions + the problem's own epilogue.
// Few splits: one thread per output, 4 independent accumulators.
template <class Prob>
__global__ void splitk_reduce_small(const Prob p, int splits) {
  PDL_ENTRY();
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
  PDL_ENTRY();
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
    for (int t = threadIdx.x; t < nk; t += NTH) {
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
      const int o = tab.t1(kt + e);
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
    for (int t = threadIdx.x; t < nk; t += NTH) {
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
      const int xb = tab.t1(pt + e);
      float val = 0.f;
      if (xb >= 0) val = ctx >= 0 ? __ldg(x + xb + ctx) : (ctx == -2 ? 1.f : 0.f);
      v[e] = val;
    }
  }
  __device__ __forceinline__ void b4(int ctx, Tab tab, int pt, int, float (&v)[4]) const {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int gb = tab.t1(tab.nk + pt + e);
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
    for (int t = threadIdx.x; t < nk; t += NTH) {
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
      const int go = tab.t1(kt + e);
      const int kyx = tab.t1(tab.nk + kt + e);
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
      const int wo = tab.t1(2 * tab.nk + kt + e);
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
    if (yprev) v *= epi_dact(act_prev, __ldg(yprev + i));
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

// ============================================================================
// slab problems (stride-1 convolutions, TF32): every CTA first stages the
// input window its tile needs into shared memory with coalesced loads (tf32-
// rounded once, pool routing fused), then the implicit-GEMM gathers of the
// pipeline read shared memory instead of L2/HBM.
// ============================================================================

// ---- staging helpers (all threads) ----------------------------------------
// Staging context: TMA bulk copies for 16-byte-aligned contiguous chunks,
// each issued by the thread `issuer` (spread the issues over threads: one
// thread issues serially), which also registers its transaction bytes on the
// stage mbarrier; ragged chunks fall back to cp.async by all threads.
// finish() = every copy landed and is visible to every thread.
struct Stager {
  uint64_t* bar;
  __device__ explicit Stager(uint64_t* b) : bar(b) {
    if (threadIdx.x == 0) {
      ptx::mbar_init(bar, 1);
      ptx::fence_mbar_init();
    }
    __syncthreads();
  }
  // n floats; every thread calls with the same arguments
  __device__ __forceinline__ void copy(uint32_t dst, const void* src, int n, int issuer = 0) {
    if (n <= 0) return;
    const uint32_t nb = 4u * (uint32_t)n;
    if (((((uintptr_t)src) | dst | nb) & 15) == 0) {
      if (threadIdx.x == issuer % NTH) {
        ptx::mbar_expect_tx(bar, nb);
        ptx::bulk_g2s(dst, src, nb, bar);
      }
    } else {
      const char* sp = static_cast<const char*>(src);
      for (int i = threadIdx.x; i < n; i += NTH) ptx::cp_async4(dst + 4u * i, sp + 4 * i);
    }
  }
  __device__ __forceinline__ void finish() {
    ptx::cp_async_wait_all();
    __syncthreads();  // every expect_tx registered, every cp.async landed
    if (threadIdx.x == 0) ptx::mbar_arrive(bar);
    ptx::mbar_wait(bar, 0);
  }
};

__device__ __forceinline__ void fill_zero(uint32_t dst, int n) {
  for (int i = threadIdx.x; i < n; i += NTH) ptx::sts_f32(dst + 4u * i, 0.f);
}
// in-place tf32 rounding of n floats (dst 16-byte aligned)
__device__ __forceinline__ void round_tf32(uint32_t dst, int n) {
  const int n4 = n >> 2;
  for (int i = threadIdx.x; i < n4; i += NTH) {
    float4 v = ptx::lds_f32x4(dst + 16u * i);
    v.x = ptx::to_tf32(v.x);
    v.y = ptx::to_tf32(v.y);
    v.z = ptx::to_tf32(v.z);
    v.w = ptx::to_tf32(v.w);
    ptx::sts_f32x4(dst + 16u * i, v);
  }
  for (int i = (n4 << 2) + threadIdx.x; i < n; i += NTH)
    ptx::sts_f32(dst + 4u * i, ptx::to_tf32(ptx::lds_f32(dst + 4u * i)));
}
__host__ __device__ __forceinline__ int round4(int v) { return (v + 3) & ~3; }

// activation applied to a run of smem values (epilogues): the act switch is
// hoisted out of the element loops
template <int ACT>
__device__ __forceinline__ float actf(float x) {
  if (ACT == VCNN_ACT_RELU) return x > 0.f ? x : 0.f;
  if (ACT == VCNN_ACT_SIGMOID) return 1.f / (1.f + expf(-x));
  if (ACT == VCNN_ACT_TANH) return tanhf(x);
  return x;
}
template <class F>
__device__ __forceinline__ void with_act(int act, F&& f) {
  switch (act) {
    case VCNN_ACT_RELU: f(std::integral_constant<int, VCNN_ACT_RELU>{}); break;
    case VCNN_ACT_SIGMOID: f(std::integral_constant<int, VCNN_ACT_SIGMOID>{}); break;
    case VCNN_ACT_TANH: f(std::integral_constant<int, VCNN_ACT_TANH>{}); break;
    default: f(std::integral_constant<int, VCNN_ACT_IDENTITY>{});
  }
}

// conv forward over row-block tiles: CTA = (image b, output rows [r0, r0+R)),
// M = R*OW pixels (<= 128).  Slab = input rows [r0, r0+R+kh-1) x W per
// channel (stride cstride, tf32-rounded in place), one zero plane (the K
// padding gathers from it), then the CTA's prepared weight rows [n0, n0+bn)
// x kd4 (tf32, zero-padded; prep_weights).  Rows past the tile gather real
// (ignored) pixels, so the gather has no predicates.
// Epilogue in shared memory: bias + act, NCHW store of the conv output
// (optional), and an optional fused non-overlapping max pool (window ==
// stride == pool; strict >, ties -> lowest index, int32 global argmax --
// pool_forward + accumulate_max_arg, vectorize.hpp:197-210, tensor.hpp:271-289).
struct SlabFwdProb : KRange {
  static constexpr bool SLAB = true, PRE_ROUNDED = true, SMEM_EPI = true, TWO_PHASE = true;
  static constexpr int TABLES = 1;
  ConvDesc d;
  const float* x;
  const float* wf;  // prepared weights [K][kd4]
  const float* bias;
  int act;
  float* y;  // conv output (nullable when pooled)
  int R, rows, tpi, cstride;
  int w_off = 0, kd4 = 0, bn = 0;
  int pool = 0, POH = 0, POW = 0;
  float* py = nullptr;
  int32_t* parg = nullptr;
  __device__ void setup(int* tab, int kbase, int nk) const {
    const int Kd = (int)d.kd(), khw = d.kh * d.kw;
    for (int t = threadIdx.x; t < nk; t += NTH) {
      const int k = kbase + t;
      int v = d.C * cstride;  // the zero plane
      if (k < Kd) {
        const int c = k / khw, rem = k - c * khw, ky = rem / d.kw, kx = rem - ky * d.kw;
        v = c * cstride + ky * d.W + kx;
      }
      tab[t] = v;
    }
  }
  __device__ void stage(float* slab, int tile, int n0, int, uint64_t* bar) const {
    const uint32_t sb = ptx::smem_u32(slab);
    Stager sg(bar);
    const int b = tile / tpi, r0 = (tile - b * tpi) * R;
    const int vn = (d.H - r0 < rows ? d.H - r0 : rows) * d.W;
    if (r0 == 0 && vn == d.H * d.W && cstride == vn) {  // the window is the whole image
      sg.copy(sb, x + (int64_t)b * d.C * d.H * d.W, d.C * vn);
    } else {
      for (int c = 0; c < d.C; ++c) {
        sg.copy(sb + 4u * (c * cstride), x + (((int64_t)b * d.C + c) * d.H + r0) * d.W, vn,
                (c + 1) * 32);
        fill_zero(sb + 4u * (c * cstride + vn), cstride - vn);
      }
    }
    fill_zero(sb + 4u * (d.C * cstride), cstride);
    if (threadIdx.x == 0) PHASE(8);
    const int nrow = d.K - n0 < bn ? d.K - n0 : bn;
    sg.copy(sb + 4u * w_off, wf + (int64_t)n0 * kd4, nrow * kd4);
    fill_zero(sb + 4u * (w_off + nrow * kd4), (bn - nrow) * kd4);
    if (threadIdx.x == 0) PHASE(9);
    sg.finish();
    if (threadIdx.x == 0) PHASE(10);
    round_tf32(sb, d.C * cstride);
    if (threadIdx.x == 0) PHASE(11);
  }
  __device__ bool a_rowmajor() const { return true; }
  __device__ bool b_rowmajor() const { return false; }
  using ACtx = int;  // slab offset of the pixel (0 for rows past the tile: ignored)
  __device__ __forceinline__ int a_ctx(int m) const {
    const int l = m & 127, r = l / d.OW, ox = l - r * d.OW;
    if (r >= R) return 0;
    return r * d.W + ox;
  }
  using BCtx = int;  // slab offset of the weight row, -1 past K
  __device__ __forceinline__ int b_ctx(int n) const {
    return n < d.K ? w_off + (n % bn) * kd4 : -1;
  }
  __device__ __forceinline__ int4 ta4(const Tab& tab, int kt) const { return tab.t4(kt); }
  __device__ __forceinline__ int4 tb4(const Tab&, int) const { return int4{}; }
  __device__ __forceinline__ void a4(int ctx, const Tab& tab, int4 o, int, float (&v)[4]) const {
    v[0] = tab.s1(ctx + o.x);
    v[1] = tab.s1(ctx + o.y);
    v[2] = tab.s1(ctx + o.z);
    v[3] = tab.s1(ctx + o.w);
  }
  __device__ __forceinline__ void b4(int ctx, const Tab& tab, int4, int k, float (&v)[4]) const {
    float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ctx >= 0 && k < kd4) q = tab.s4(ctx + k);
    v[0] = q.x;
    v[1] = q.y;
    v[2] = q.z;
    v[3] = q.w;
  }
  using ECtx = int;
  __device__ __forceinline__ int e_ctx(int m) const { return m; }
  __device__ __forceinline__ void store(int, int, float) const {}
  __device__ void smem_epilogue(const float* ep, int tile, int n0, int bnt) const {
    const int b = tile / tpi, r0 = (tile - b * tpi) * R;
    const int nr = d.OH - r0 < R ? d.OH - r0 : R;
    const int npix = nr * d.OW;
    const int nmaps = d.K - n0 < bnt ? d.K - n0 : bnt;
    const int ohw = d.OH * d.OW;
    const uint32_t eb = ptx::smem_u32(ep);
    with_act(act, [&](auto A) {
      constexpr int ACT = decltype(A)::value;
      if (y) {
        for (int i = threadIdx.x; i < nmaps * npix; i += NTH) {
          const int n = i / npix, l = i - n * npix;
          y[((int64_t)b * d.K + n0 + n) * ohw + (int64_t)r0 * d.OW + l] =
              actf<ACT>(ptx::lds_f32(eb + 4u * (n * BM + l)) + __ldg(bias + n0 + n));
        }
      }
      if (pool) {
        const int p = pool;
        int nwr = (r0 + nr) / p - r0 / p;  // complete window rows of this tile
        if (r0 / p + nwr > POH) nwr = POH - r0 / p;
        const int nwin = nwr * POW;
        for (int i = threadIdx.x; i < nmaps * nwin; i += NTH) {
          const int n = i / nwin, rem = i - n * nwin, wr = rem / POW, wc = rem - wr * POW;
          const float bn_ = __ldg(bias + n0 + n);
          const int l0 = wr * p * d.OW + wc * p;  // tile-local top-left
          float best = actf<ACT>(ptx::lds_f32(eb + 4u * (n * BM + l0)) + bn_);
          int bl = l0;
          for (int a = 0; a < p; ++a)
            for (int c = 0; c < p; ++c) {
              const int l = l0 + a * d.OW + c;
              const float v = actf<ACT>(ptx::lds_f32(eb + 4u * (n * BM + l)) + bn_);
              if (v > best) {
                best = v;
                bl = l;
              }
            }
          const int64_t plane0 = ((int64_t)b * d.K + n0 + n);
          const int64_t o = (plane0 * POH + r0 / p + wr) * POW + wc;
          py[o] = best;
          parg[o] = (int32_t)(plane0 * ohw + (int64_t)r0 * d.OW + bl);
        }
      }
    });
  }
};

// conv wgrad: D[k = (c,ky,kx) | ones row for the bias][n] = sum_pixels P G,
// K = pixels of `imgs` whole images per split (blockIdx.z).  Slab = those
// images' input planes [img][C][H][W] and G planes [img][K][OH][OW] (one
// bulk copy each), plus, for a fused pool, the window gradients / argmaxes
// scattered into zeroed G planes (the argmax is a global [B][K][OH][OW]
// index, so its offset from image b0 IS the slab offset).  With OH*OW % 4 ==
// 0 four consecutive pixels are one aligned 16-byte G load (vecg).
// Deterministic split-K reduce.
struct SlabWgradProb : KRange {
  static constexpr bool SLAB = true, PRE_ROUNDED = true, TWO_PHASE = true, A_ZERO_ROWS = true;
  static constexpr int TABLES = 2;
  ConvDesc d;
  const float* x;
  GradSrc gs;
  float* dw;
  float* db;
  int imgs, vecg;
  int g_off, sc_off, sc_n;  // slab offsets (floats): G planes, window scratch (+ its size)
  __device__ void setup(int* tab, int kbase, int nk) const {
    const int z = kbase / (kb_per * BK), b0 = z * imgs;
    int nimg = d.B - b0 < imgs ? d.B - b0 : imgs;
    const int ohw = d.OH * d.OW, npix = nimg * ohw;
    for (int t = threadIdx.x; t < nk; t += NTH) {
      int xo = 0, go = -1;  // past the images: any finite pixel, zero G
      if (t < npix) {
        const int im = t / ohw, r = t - im * ohw, oy = r / d.OW, ox = r - oy * d.OW;
        xo = im * d.C * d.H * d.W + oy * d.W + ox;
        go = g_off + im * d.K * ohw + r;
      }
      tab[t] = xo;
      tab[nk + t] = go;
    }
  }
  __device__ void stage(float* slab, int, int, int z, uint64_t* bar) const {
    const uint32_t sb = ptx::smem_u32(slab);
    Stager sg(bar);
    const int b0 = z * imgs;
    const int nimg = d.B - b0 < imgs ? d.B - b0 : imgs;
    const int xs = d.C * d.H * d.W, gsz = d.K * d.OH * d.OW;
    sg.copy(sb, x + (int64_t)b0 * xs, nimg * xs);
    if (gs.pool == 0) {
      sg.copy(sb + 4u * g_off, gs.g + (int64_t)b0 * gsz, nimg * gsz, 32);
      sg.finish();
      round_tf32(sb, nimg * xs);
      round_tf32(sb + 4u * g_off, nimg * gsz);
      return;
    }
    const int wsz = d.K * gs.POH * gs.POW, nw = nimg * wsz;
    sg.copy(sb + 4u * sc_off, gs.dP + (int64_t)b0 * wsz, nw, 32);
    sg.copy(sb + 4u * (sc_off + sc_n), gs.parg + (int64_t)b0 * wsz, nw, 64);
    fill_zero(sb + 4u * g_off, nimg * gsz);
    sg.finish();
    const int base = (int)((int64_t)b0 * gsz);
    for (int i = threadIdx.x; i < nw; i += NTH) {
      const int a = ptx::lds_s32(sb + 4u * (sc_off + sc_n + i)) - base;
      ptx::sts_f32(sb + 4u * (g_off + a), ptx::to_tf32(ptx::lds_f32(sb + 4u * (sc_off + i))));
    }
    round_tf32(sb, nimg * xs);
  }
  __device__ bool a_rowmajor() const { return false; }
  __device__ bool b_rowmajor() const { return false; }
  using ACtx = int;  // im2col offset of patch row k; -2 = ones (bias row); -3 = zero row
  __device__ __forceinline__ int a_ctx(int k) const {
    const int Kd = (int)d.kd(), khw = d.kh * d.kw;
    if (k > Kd) return -3;
    if (k == Kd) return -2;
    const int c = k / khw, rem = k - c * khw, ky = rem / d.kw, kx = rem - ky * d.kw;
    return (c * d.H + ky) * d.W + kx;
  }
  __device__ __forceinline__ bool a_zero(int ctx) const { return ctx == -3; }
  using BCtx = int;  // n * OH*OW, -1 past K
  __device__ __forceinline__ int b_ctx(int n) const { return n < d.K ? n * d.OH * d.OW : -1; }
  __device__ __forceinline__ int4 ta4(const Tab& tab, int pt) const { return tab.t4(pt); }
  __device__ __forceinline__ int4 tb4(const Tab& tab, int pt) const {
    return vecg ? int4{tab.t1(tab.nk + pt), 0, 0, 0} : tab.t4(tab.nk + pt);
  }
  __device__ __forceinline__ void a4(int ctx, const Tab& tab, int4 o, int, float (&v)[4]) const {
    if (ctx >= 0) {
      v[0] = tab.s1(o.x + ctx);
      v[1] = tab.s1(o.y + ctx);
      v[2] = tab.s1(o.z + ctx);
      v[3] = tab.s1(o.w + ctx);
    } else {
      const float one = ctx == -2 ? 1.f : 0.f;
      v[0] = v[1] = v[2] = v[3] = one;
    }
  }
  __device__ __forceinline__ void b4(int ctx, const Tab& tab, int4 o, int, float (&v)[4]) const {
    if (vecg) {  // 4 pixels of one image, contiguous and aligned (or all past the images)
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ctx >= 0 && o.x >= 0) q = tab.s4(o.x + ctx);
      v[0] = q.x;
      v[1] = q.y;
      v[2] = q.z;
      v[3] = q.w;
      return;
    }
    v[0] = (ctx >= 0 && o.x >= 0) ? tab.s1(o.x + ctx) : 0.f;
    v[1] = (ctx >= 0 && o.y >= 0) ? tab.s1(o.y + ctx) : 0.f;
    v[2] = (ctx >= 0 && o.z >= 0) ? tab.s1(o.z + ctx) : 0.f;
    v[3] = (ctx >= 0 && o.w >= 0) ? tab.s1(o.w + ctx) : 0.f;
  }
  using ECtx = int;
  __device__ __forceinline__ int e_ctx(int k) const { return k; }
  __device__ __forceinline__ void store(int k, int n, float v) const {
    const int Kd = (int)d.kd();
    if (k > Kd || n >= d.K) return;
    if (k < Kd) dw[(int64_t)n * Kd + k] = v;
    else db[n] = v;
  }
};

// implicit conv dgrad over row-block tiles of dX: CTA = (image b, input rows
// [r0, r0+R)), M = R*W pixels; K = (n,ky,kx); N = C.  Slab = G rows
// [r0-kh+1, r0+R) zero-padded to width W+kw-1 (routed from a fused pool when
// gs.pool): A(m,k) = Gpad[n][y+kh-1-ky][x+kw-1-kx]; a zero plane (K
// padding); then the prepared transposed weights of the CTA's channels
// [c - n0][n][ky][kx] (tf32).  Epilogue: dX * act'(yprev).
struct SlabDgradProb : KRange {
  static constexpr bool SLAB = true, PRE_ROUNDED = true, TWO_PHASE = true;
  static constexpr int TABLES = 2;
  ConvDesc d;
  GradSrc gs;
  const float* wt;  // prepared transposed weights [C][K*kh*kw]
  float* dx;
  const float* yprev;
  int act_prev;
  int R, srows, scols, tpi;
  int w_off = 0, bn = 0, sc_off = 0, sc_n = 0;
  __device__ void setup(int* tab, int kbase, int nk) const {
    const int KK = d.K * d.kh * d.kw, khw = d.kh * d.kw;
    for (int t = threadIdx.x; t < nk; t += NTH) {
      const int k = kbase + t;
      int go = d.K * srows * scols, wo = -1;  // the zero plane
      if (k < KK) {
        const int n = k / khw, rem = k - n * khw, ky = rem / d.kw, kx = rem - ky * d.kw;
        go = (n * srows + (d.kh - 1 - ky)) * scols + (d.kw - 1 - kx);
        wo = k;
      }
      tab[t] = go;
      tab[nk + t] = wo;
    }
  }
  __device__ void stage(float* slab, int tile, int n0, int, uint64_t* bar) const {
    const uint32_t sb = ptx::smem_u32(slab);
    Stager sg(bar);
    const int b = tile / tpi, r0 = (tile - b * tpi) * R;
    const int gr0 = r0 - (d.kh - 1);  // conv-output row of slab row 0
    const int plane = srows * scols;
    const int KK = d.K * d.kh * d.kw;
    const int nch = d.C - n0 < bn ? d.C - n0 : bn;
    const int ohw = d.OH * d.OW;
    // the whole image's G (or window gradients + argmaxes) -> scratch, one
    // bulk copy each; the weights of the CTA's channels; zero slab
    if (gs.pool == 0) {
      sg.copy(sb + 4u * sc_off, gs.g + (int64_t)b * d.K * ohw, d.K * ohw, 32);
    } else {
      const int wsz = d.K * gs.POH * gs.POW;
      sg.copy(sb + 4u * sc_off, gs.dP + (int64_t)b * wsz, wsz, 32);
      sg.copy(sb + 4u * (sc_off + sc_n), gs.parg + (int64_t)b * wsz, wsz, 64);
    }
    sg.copy(sb + 4u * w_off, wt + (int64_t)n0 * KK, nch * KK);
    fill_zero(sb, (d.K + 1) * plane);
    fill_zero(sb + 4u * (w_off + nch * KK), (bn - nch) * KK);
    sg.finish();
    const int lo = gr0 > 0 ? gr0 : 0;
    const int hi = gr0 + srows < d.OH ? gr0 + srows : d.OH;  // conv-output rows [lo, hi)
    if (gs.pool == 0) {  // expand rows [lo, hi) into the zero-padded slab
      const int per = (hi - lo) * d.OW;
      for (int i = threadIdx.x; i < d.K * per; i += NTH) {
        const int n = i / per, rem = i - n * per, r = rem / d.OW, c = rem - r * d.OW;
        const float v = ptx::lds_f32(sb + 4u * (sc_off + n * ohw + (lo + r) * d.OW + c));
        ptx::sts_f32(sb + 4u * ((n * srows + lo - gr0 + r) * scols + c + d.kw - 1),
                     ptx::to_tf32(v));
      }
      return;
    }
    // routed: scatter the windows whose argmax lies in rows [lo, hi)
    const int wsz = d.K * gs.POH * gs.POW;
    const int base = (int)((int64_t)b * d.K * ohw);
    for (int i = threadIdx.x; i < wsz; i += NTH) {
      const int a = ptx::lds_s32(sb + 4u * (sc_off + sc_n + i)) - base;  // [n][oy][ox]
      const int n = a / ohw, rem = a - n * ohw, oy = rem / d.OW, ox = rem - oy * d.OW;
      if (oy < lo || oy >= hi) continue;
      ptx::sts_f32(sb + 4u * ((n * srows + oy - gr0) * scols + ox + d.kw - 1),
                   ptx::to_tf32(ptx::lds_f32(sb + 4u * (sc_off + i))));
    }
  }
  __device__ bool a_rowmajor() const { return true; }
  __device__ bool b_rowmajor() const { return false; }
  using ACtx = int;  // (0 for rows past the tile: ignored)
  __device__ __forceinline__ int a_ctx(int m) const {
    const int l = m & 127, r = l / d.W, x = l - r * d.W;
    if (r >= R) return 0;
    return r * scols + x;
  }
  using BCtx = int;  // slab offset of the channel's weight row, -1 past C
  __device__ __forceinline__ int b_ctx(int c) const {
    return c < d.C ? w_off + (c % bn) * d.K * d.kh * d.kw : -1;
  }
  __device__ __forceinline__ int4 ta4(const Tab& tab, int kt) const { return tab.t4(kt); }
  __device__ __forceinline__ int4 tb4(const Tab& tab, int kt) const { return tab.t4(tab.nk + kt); }
  __device__ __forceinline__ void a4(int ctx, const Tab& tab, int4 o, int, float (&v)[4]) const {
    v[0] = tab.s1(ctx + o.x);
    v[1] = tab.s1(ctx + o.y);
    v[2] = tab.s1(ctx + o.z);
    v[3] = tab.s1(ctx + o.w);
  }
  __device__ __forceinline__ void b4(int ctx, const Tab& tab, int4 o, int, float (&v)[4]) const {
    v[0] = (ctx >= 0 && o.x >= 0) ? tab.s1(o.x + ctx) : 0.f;
    v[1] = (ctx >= 0 && o.y >= 0) ? tab.s1(o.y + ctx) : 0.f;
    v[2] = (ctx >= 0 && o.z >= 0) ? tab.s1(o.z + ctx) : 0.f;
    v[3] = (ctx >= 0 && o.w >= 0) ? tab.s1(o.w + ctx) : 0.f;
  }
  using ECtx = int64_t;  // offset of (b, c=0, y, x) in dx, -1 past the tile
  __device__ __forceinline__ int64_t e_ctx(int m) const {
    const int tile = m >> 7, l = m & 127, r = l / d.W, x = l - r * d.W;
    const int b = tile / tpi, r0 = (tile - b * tpi) * R;
    if (r >= R || r0 + r >= d.H) return -1;
    return (int64_t)b * d.C * d.H * d.W + (int64_t)(r0 + r) * d.W + x;
  }
  __device__ __forceinline__ void store(int64_t ec, int c, float v) const {
    if (ec < 0 || c >= d.C) return;
    const int64_t i = ec + (int64_t)c * d.H * d.W;
    if (yprev) v *= epi_dact(act_prev, __ldg(yprev + i));
    dx[i] = v;
  }
};

// weight preparation for the slab kernels (once per parameter update):
// wf[n][kd4] = tf32(W[n][k]) zero-padded, wt[c][(n,ky,kx)] = tf32(W[n][c][ky][kx])
__global__ void prep_weights_kernel(ConvDesc d, const float* __restrict__ w,
                                    float* __restrict__ wf, float* __restrict__ wt) {
  PDL_ENTRY();
  const int Kd = (int)d.kd(), kd4 = round4(Kd), khw = d.kh * d.kw;
  const int nf = d.K * kd4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += gridDim.x * blockDim.x) {
    const int n = i / kd4, k = i - n * kd4;
    const float v = k < Kd ? ptx::to_tf32(w[(int64_t)n * Kd + k]) : 0.f;
    wf[i] = v;
    if (wt && k < Kd) {
      const int c = k / khw, rem = k - c * khw;
      wt[((int64_t)c * d.K + n) * khw + rem] = v;
    }
  }
}

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
      case EPI_BIAS_ACT: c[m * ldc + n] = epi_act(act, bias ? v + bias[n] : v); break;
      case EPI_DACT: {
        const int64_t i = m * ldc + n;
        c[i] = yprev ? v * epi_dact(act, __ldg(yprev + i)) : v;
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
  // few M tiles and a wide N: narrower N tiles spread the work over more
  // CTAs (a BN=256 tile is 4x the gather work of one SM at BN=64)
  while (p.bn > 32 && cdiv(M, BM) * cdiv(N, p.bn) < sm_count() / 2) p.bn /= 2;
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
int launch_one(const Prob& p0, dim3 grid, size_t tab_bytes, size_t slab_bytes, cudaStream_t st) {
  using C = TileCfg<BN, SPLIT3>;
  (void)tab_bytes;
  Prob p = p0;
  const size_t rest = (size_t)p.slab_off + slab_bytes + 1024;
  // ring depth: slab problems take what the slab leaves (1 CTA / SM);
  // gather problems ~88 KB of ring so two CTAs share an SM
  const size_t budget = Prob::SLAB ? kSmemOptin - 2048 - rest : (size_t)88 * 1024;
  int nst = (int)(budget / C::STAGE_BYTES);
  if (nst > (Prob::SLAB ? MAX_STAGES : 6)) nst = Prob::SLAB ? MAX_STAGES : 6;
  if (nst > p.kb_per) nst = p.kb_per;  // no deeper than the K loop
  if (nst < 2) nst = 2;
  p.nst = nst;
  const size_t smem = (size_t)nst * C::STAGE_BYTES + rest;
  if (smem > kSmemOptin) return fail(VCNN_ESHAPE, "tc gemm: shared-memory plan exceeds 227 KB");
  static size_t configured = 0;  // attribute raised per instantiation as needed
  if (smem > configured) {
    VCNN_CUDA_TRY(cudaFuncSetAttribute(tc_gemm_kernel<Prob, BN, SPLIT3>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  VCNN_CUDA_TRY(launch_pdl(tc_gemm_kernel<Prob, BN, SPLIT3>, dim3(grid), dim3(NTH), smem, st, p));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

template <class Prob, bool SPLIT3>
int launch_bn(const Prob& p, int bn, dim3 grid, size_t tab, size_t slab, cudaStream_t st) {
  switch (bn) {
    case 16: return launch_one<Prob, 16, SPLIT3>(p, grid, tab, slab, st);
    case 32: return launch_one<Prob, 32, SPLIT3>(p, grid, tab, slab, st);
    case 64: return launch_one<Prob, 64, SPLIT3>(p, grid, tab, slab, st);
    case 128: return launch_one<Prob, 128, SPLIT3>(p, grid, tab, slab, st);
    default:
      if constexpr (Prob::SMEM_EPI) return fail(VCNN_ESHAPE, "smem epilogue needs N <= 128");
      else return launch_one<Prob, 256, SPLIT3>(p, grid, tab, slab, st);
  }
}

// run a planned problem: GEMM (+ split-K reduce with the fused epilogue).
// Slab problems: grid.x = tiles (pl.mt), slab_bytes of staged input per CTA,
// TF32 only.
template <class Prob>
int run(Prob p, const Plan& pl, bool split3, const Workspace& ws, cudaStream_t st,
        size_t slab_bytes = 0) {
  p.kb_total = pl.kb_total;
  p.kb_per = pl.kb_per;
  p.part = nullptr;
  p.slab_off = (int)((pl.tab_bytes() + 15) & ~(size_t)15);
  if (pl.splits > 1) {
    if (!ws.ptr || ws.bytes < pl.ws_bytes())
      return fail(VCNN_ECUDA, "tc gemm: split-K workspace too small");
    p.part = ws.ptr;
    p.part_m = (int)pl.M;
    p.part_n = (int)pl.N;
  }
  dim3 grid((unsigned)pl.mt, (unsigned)pl.nt, (unsigned)pl.splits);
  int s;
  if constexpr (Prob::SLAB) {
    if (split3) return fail(VCNN_ECONFIG, "slab kernels are TF32-only");
    s = launch_bn<Prob, false>(p, pl.bn, grid, pl.tab_bytes(), slab_bytes, st);
  } else {
    s = split3 ? launch_bn<Prob, true>(p, pl.bn, grid, pl.tab_bytes(), 0, st)
               : launch_bn<Prob, false>(p, pl.bn, grid, pl.tab_bytes(), 0, st);
  }
  if (s || pl.splits == 1) return s;
  if (pl.splits <= 16) {
    int64_t blocks = cdiv(pl.M * pl.N, 256);
    if (blocks > 8 * sm_count()) blocks = 8 * sm_count();
    VCNN_CUDA_TRY(launch_pdl(splitk_reduce_small<Prob>, dim3((unsigned)blocks), dim3(256), 0, st, p, pl.splits));
  } else {
    VCNN_CUDA_TRY(launch_pdl(splitk_reduce_kernel<Prob>, dim3((unsigned)cdiv(pl.M * pl.N, 32)), dim3(256), 0, st, p, pl.splits));
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
  // implicit dgrad multiplies H*W/(OH*OW) times the algorithmic work; the
  // explicit one writes and re-reads the kd x pixels dP matrix (1.2 GB for
  // deconv-121's 1x121 layer: 2.0 ms GEMM + 1.4 ms col2im)
  return (int64_t)d.H * d.W > 4 * (int64_t)d.OH * d.OW && fits_i32(d.kd() * d.pixels());
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
  w = std::max(w, slab_wgrad_workspace(d));
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
// the implicit GEMMs index x, G / y and W with 32-bit offsets (no patch
// matrix is materialised, so its size is not a limit); the explicit dgrad's
// dP buffer is checked where it is used
static int check_conv(const ConvDesc& d, const char* what) {
  if (!fits_i32(d.in_size()) || !fits_i32(d.out_size()) || !fits_i32(d.pixels()) ||
      !fits_i32((int64_t)d.B * d.H * d.W) || !fits_i32(d.kd() * d.K))
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
    if (!fits_i32(d.kd() * d.pixels()))
      return fail(VCNN_ESHAPE, "conv_dgrad: patch gradient exceeds 2^31 elements");
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

// ---------------------------------------------------------------------------
// slab kernels: planning.  Shared memory per CTA = stage ring + K tables +
// slab; the slab budget keeps the total under the 227 KB opt-in.
// ---------------------------------------------------------------------------
namespace {
template <int BN>
size_t ring_bytes() {
  return 2 * (size_t)TileCfg<BN, false>::STAGE_BYTES;  // minimum ring
}
size_t ring_for(int bn) {
  switch (bn) {
    case 16: return ring_bytes<16>();
    case 32: return ring_bytes<32>();
    case 64: return ring_bytes<64>();
    case 128: return ring_bytes<128>();
    default: return ring_bytes<256>();
  }
}
bool fits_smem(const Plan& p, size_t slab) {
  return ring_for(p.bn) + ((p.tab_bytes() + 15) & ~(size_t)15) + slab + 1024 + 2048 <=
         kSmemOptin;
}

struct SlabFwdPlan {
  bool ok = false;
  int R = 0, rows = 0, tpi = 0, bn = 0, kd4 = 0, w_off = 0, cstride = 0;
  size_t slab = 0;
  Plan pl;
};
SlabFwdPlan plan_slab_fwd(const ConvDesc& d, int pool) {
  SlabFwdPlan s;
  if (d.s != 1 || d.OW > BM || d.OW < 1 || d.kd() > 8192) return s;
  int R = BM / d.OW;
  if (R > d.OH) R = d.OH;
  if (pool) R = (R / pool) * pool;
  if (R < 1) return s;
  s.R = R;
  s.rows = R + d.kh - 1;
  s.cstride = round4(s.rows * d.W);
  s.tpi = (int)cdiv(d.OH, R);
  s.bn = pick_bn(d.K) > 128 ? 128 : pick_bn(d.K);
  s.kd4 = round4((int)d.kd());
  s.w_off = (d.C + 1) * s.cstride;  // + the zero plane
  s.slab = sizeof(float) * ((size_t)s.w_off + (size_t)s.bn * s.kd4);
  Plan& p = s.pl;
  p.M = (int64_t)d.B * s.tpi * BM;
  p.N = d.K;
  p.tables = 1;
  p.bn = s.bn;
  p.mt = (int64_t)d.B * s.tpi;
  p.nt = cdiv(d.K, s.bn);
  p.kb_total = (int)cdiv(d.kd(), BK);
  p.kb_per = p.kb_total;
  p.splits = 1;
  s.ok = p.mt < (1 << 24) && fits_smem(p, s.slab);
  return s;
}

struct SlabWgradPlan {
  bool ok = false;
  int imgs = 0, g_off = 0, sc_off = 0, sc_n = 0, vecg = 0;
  size_t slab = 0;
  Plan pl;
};
SlabWgradPlan plan_slab_wgrad(const ConvDesc& d, int pool, int POH, int POW) {
  SlabWgradPlan s;
  if (d.s != 1) return s;
  const int xs = d.C * d.H * d.W, gsz = d.K * d.OH * d.OW, wsz = d.K * POH * POW;
  auto bytes = [&](int im) {  // X planes + G planes (+ window scratch)
    size_t f = (size_t)round4(im * xs) + round4(im * gsz);
    if (pool) f += 2 * (size_t)round4(im * wsz);
    return sizeof(float) * f;
  };
  Plan& p = s.pl;
  p.M = d.kd() + 1;
  p.N = d.K;
  p.tables = 2;
  p.bn = pick_bn(d.K);
  p.mt = cdiv(d.kd() + 1, BM);
  p.nt = cdiv(d.K, p.bn);
  auto plan_for = [&](int im) {
    p.kb_per = (int)cdiv((int64_t)im * d.OH * d.OW, BK);
    p.splits = (int)cdiv(d.B, im);
    p.kb_total = p.kb_per * p.splits;
  };
  // more images per CTA while the slab fits and the grid still covers the SMs
  int imgs = 1;
  while (imgs < d.B && p.mt * cdiv(d.B, imgs + 1) >= sm_count()) {
    plan_for(imgs + 1);
    if (!fits_smem(p, bytes(imgs + 1))) break;
    ++imgs;
  }
  plan_for(imgs);
  if (!fits_smem(p, bytes(imgs)) || (int64_t)imgs * d.OH * d.OW > 8192) return s;
  s.imgs = imgs;
  s.g_off = round4(imgs * xs);
  s.sc_off = s.g_off + round4(imgs * gsz);
  s.sc_n = pool ? round4(imgs * wsz) : 0;
  s.vecg = (d.OH * d.OW) % 4 == 0;
  s.slab = bytes(imgs);
  s.ok = true;
  return s;
}

struct SlabDgradPlan {
  bool ok = false;
  int R = 0, srows = 0, scols = 0, tpi = 0, w_off = 0, sc_off = 0, sc_n = 0;
  size_t slab = 0;
  Plan pl;
};
SlabDgradPlan plan_slab_dgrad(const ConvDesc& d, int pool, int POW) {
  SlabDgradPlan s;
  if (d.s != 1 || d.W > BM) return s;
  int R = BM / d.W;
  if (R > d.H) R = d.H;
  R = (int)cdiv(d.H, cdiv(d.H, R));  // balanced row blocks
  s.R = R;
  s.srows = R + d.kh - 1;
  s.scols = d.W + d.kw - 1;
  s.tpi = (int)cdiv(d.H, R);
  const int64_t KK = (int64_t)d.K * d.kh * d.kw;
  if (KK > 4096) return s;
  Plan& p = s.pl;
  p.M = (int64_t)d.B * s.tpi * BM;
  p.N = d.C;
  p.tables = 2;
  p.bn = pick_bn(d.C);
  p.mt = (int64_t)d.B * s.tpi;
  p.nt = cdiv(d.C, p.bn);
  p.kb_total = (int)cdiv(KK, BK);
  p.kb_per = p.kb_total;
  p.splits = 1;
  s.w_off = round4((d.K + 1) * s.srows * s.scols);  // + the zero plane
  s.sc_off = s.w_off + round4((int)(p.bn * KK));
  // scratch: the image's G planes, or its window gradients + argmaxes
  s.sc_n = pool ? round4(d.K * (d.OH / pool) * POW) : round4(d.K * d.OH * d.OW);
  s.slab = sizeof(float) * ((size_t)s.sc_off + (pool ? 2 : 1) * (size_t)s.sc_n);
  s.ok = p.mt < (1 << 24) && fits_smem(p, s.slab);
  return s;
}
}  // namespace

bool slab_fwd_ok(const ConvDesc& d, int pool) { return plan_slab_fwd(d, pool).ok; }
bool slab_wgrad_ok(const ConvDesc& d, int pool, int POH, int POW) {
  return plan_slab_wgrad(d, pool, POH, POW).ok;
}
bool slab_dgrad_ok(const ConvDesc& d, int pool, int POW) {
  return plan_slab_dgrad(d, pool, POW).ok;
}
size_t slab_wgrad_workspace(const ConvDesc& d) {
  // the unrouted plan has the fewest images per CTA, i.e. the most partials
  const SlabWgradPlan s = plan_slab_wgrad(d, 0, 0, 0);
  size_t w = s.ok ? s.pl.ws_bytes() : 0;
  const SlabWgradPlan r = plan_slab_wgrad(d, 2, d.OH / 2, d.OW / 2);
  if (r.ok && r.pl.ws_bytes() > w) w = r.pl.ws_bytes();
  return w;
}
size_t prep_floats_f(const ConvDesc& d) { return (size_t)d.K * round4((int)d.kd()); }
size_t prep_floats_t(const ConvDesc& d) { return (size_t)d.K * d.kd(); }

int prep_weights(const ConvDesc& d, const float* w, float* wf, float* wt, cudaStream_t st) {
  const int64_t n = (int64_t)prep_floats_f(d);
  int64_t blocks = cdiv(n, 256);
  if (blocks > 4 * sm_count()) blocks = 4 * sm_count();
  VCNN_CUDA_TRY(launch_pdl(prep_weights_kernel, dim3((unsigned)blocks), dim3(256), 0, st, d, w, wf, wt));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int slab_conv_fwd(const ConvDesc& d, const float* x, const float* wf, const float* b, int act,
                  float* y, const PoolFuse& pf, cudaStream_t st) {
  const SlabFwdPlan s = plan_slab_fwd(d, pf.pool);
  if (!s.ok) return fail(VCNN_ESHAPE, "slab_conv_fwd: geometry not supported");
  SlabFwdProb p;
  p.d = d;
  p.x = x;
  p.wf = wf;
  p.bias = b;
  p.act = act;
  p.y = y;
  p.R = s.R;
  p.rows = s.rows;
  p.tpi = s.tpi;
  p.cstride = s.cstride;
  p.w_off = s.w_off;
  p.kd4 = s.kd4;
  p.bn = s.bn;
  p.pool = pf.pool;
  p.POH = pf.POH;
  p.POW = pf.POW;
  p.py = pf.y;
  p.parg = pf.arg;
  return run(p, s.pl, false, Workspace{}, st, s.slab);
}

int slab_conv_wgrad(const ConvDesc& d, const float* x, const GradSrc& gs, float* dw, float* db,
                    const Workspace& ws, cudaStream_t st) {
  const SlabWgradPlan s = plan_slab_wgrad(d, gs.pool, gs.POH, gs.POW);
  if (!s.ok) return fail(VCNN_ESHAPE, "slab_conv_wgrad: geometry not supported");
  SlabWgradProb p;
  p.d = d;
  p.x = x;
  p.gs = gs;
  p.dw = dw;
  p.db = db;
  p.imgs = s.imgs;
  p.g_off = s.g_off;
  p.sc_off = s.sc_off;
  p.sc_n = s.sc_n;
  p.vecg = s.vecg;
  return run(p, s.pl, false, ws, st, s.slab);
}

int slab_conv_dgrad(const ConvDesc& d, const GradSrc& gs, const float* wt, float* dx,
                    const float* yprev, int act_prev, cudaStream_t st) {
  const SlabDgradPlan s = plan_slab_dgrad(d, gs.pool, gs.POW);
  if (!s.ok) return fail(VCNN_ESHAPE, "slab_conv_dgrad: geometry not supported");
  SlabDgradProb p;
  p.d = d;
  p.gs = gs;
  p.wt = wt;
  p.dx = dx;
  p.yprev = yprev;
  p.act_prev = act_prev;
  p.R = s.R;
  p.srows = s.srows;
  p.scols = s.scols;
  p.tpi = s.tpi;
  p.w_off = s.w_off;
  p.bn = s.pl.bn;
  p.sc_off = s.sc_off;
  p.sc_n = s.sc_n;
  return run(p, s.pl, false, Workspace{}, st, s.slab);
}

// C[m][n] (ldc) = act(sum_k A(m,k) B(k,n) + bias[n]); A(m,k) = a[m*as_m + k*as_k],
// B(k,n) = b[k*bs_k + n*bs_n]
int gemm(int64_t m, int64_t n, int64_t k, const float* a, int64_t as_m, int64_t as_k,
         const float* b, int64_t bs_k, int64_t bs_n, float* c, int64_t ldc, const float* bias,
         int act, bool split3, const Workspace& ws, cudaStream_t st) {
  if (!fits_i32(m) || !fits_i32(n) || !fits_i32(k))
    return fail(VCNN_ESHAPE, "gemm: extent exceeds 2^31");
  return run(dense_prob((int)m, (int)n, (int)k, a, as_m, as_k, b, bs_n, bs_k, -1, EPI_BIAS_ACT, c,
                        ldc, bias, act, nullptr, nullptr),
             make_plan(m, n, k, 0), split3, ws, st);
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

#ifdef VCNN_PHASE_TIMING
extern "C" int vcnn_debug_phases(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, vcnn_b200::tc::g_phase, sizeof(unsigned long long) * 128) ==
                 cudaSuccess
             ? 0
             : 4;
}
#endif
