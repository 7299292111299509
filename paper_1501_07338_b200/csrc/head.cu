// The two-layer network tail in ONE kernel (training steps): a small full
// layer H (a full layer, or a conv whose kernel covers its input -- the
// engine's "dense" conv) followed by the last full layer O, the loss, and
// both layers' backward:
//   h  = act_H(x W_H^T + b_H)            full_forward / conv_forward (layers.hpp:230-247)
//   y  = act_O(h W_O^T + b_O)            full_forward
//   L, gO = dL/dy * act_O'(y)            loss_forward / loss_backward (layers.hpp:402-468)
//   gH = (gO W_O) * act_H'(h)            full_backward_core (layers.hpp:249-267)
//   dW_O, db_O, dW_H, db_H, dx = (gH W_H) * act_prev'(x)
// One thread-block cluster of kC CTAs.  CTA r owns input columns
// [r*Kc, (r+1)*Kc) of x / W_H (a K-split of the first GEMM and an N-split of
// the dW_H and dx GEMMs) and batch rows [r*R, (r+1)*R) (the small second
// layer and the loss).  Exchanges go through distributed shared memory:
// K-split partials of x W_H^T are reduced by the row owner in rank order,
// the rows of gH are all-gathered, dW_O partials are reduced slice-wise in
// rank order.  The three contractions run on the tcgen05 tensor cores (TF32,
// fp32 accumulators in TMEM, one elected thread issuing): every operand is
// staged (tf32-rounded) in the K-major no-swizzle layout [k/4][rows][4]
// (8-row x 16-byte core matrices, LBO = rows*16, SBO = 128 B), M = 128 rows
// (the batch, or the CTA's input columns), results read back with
// tcgen05.ld by all 16 warps (4 lane quadrants x 4 column groups).  Every
// reduction in a fixed order (deterministic).  Replaces 6-8 launches on the
// critical path.
#include <cooperative_groups.h>

#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace vcnn_b200 {

namespace {

namespace cg = cooperative_groups;

constexpr int kC = 16;        // cluster size (non-portable; B200 supports 16)
constexpr int kThreadsM = 512;

struct Dims {
  int B, in, h, out;
  int R, Kc;                  // batch rows / input columns per CTA (Kc % 4 == 0)
  int Kp, Hp, Np, Bk;         // GEMM extents: K of x W_H^T (Kc to 8), hidden (to 16),
                              // dx N (Kc to 16), K of dW_H (B to 8)
  int sH;                     // row stride of the hidden rows: multiple of 4, odd in 16B units
  int per5;                   // dW_O | db_O elements reduced per CTA
  // smem offsets (floats); operand tiles in the K-major [k/4][rows][4] layout
  int oA1, oB1;               // x[:, mine] [Kp/4][128][4], W_H[:, mine] [Kp/4][Hp][4]
  int oA2;                    // gH [Hp/4][128][4]   (over A1/B1 once x W_H^T is done)
  int oB2;                    // W_H[:, mine]^T [Hp/4][Np][4]
  int oXT;                    // x[:, mine]^T [Bk/4][128][4]
  int oGT;                    // gH^T [Bk/4][Hp][4]
  int oPs, oW5, ohs, og5, ogl, op5, odb, obH, obO, oy5, otg;
  int total;
};

__host__ __device__ inline int up4(int v) { return (v + 3) & ~3; }
__host__ __device__ inline int up8(int v) { return (v + 7) & ~7; }
__host__ __device__ inline int up16(int v) { return (v + 15) & ~15; }
// a row stride of v floats (v % 4 == 0) whose 16-byte units are odd: float4
// accesses of 8 consecutive rows hit distinct banks
__host__ __device__ inline int odd16(int v) { return (v >> 2) & 1 ? v : v + 4; }
// offset (floats) of element (row, k) of a K-major [k/4][rows][4] tile
__host__ __device__ inline int kmaj(int row, int k, int rows) {
  return ((k >> 2) * rows + row) * 4 + (k & 3);
}

__host__ __device__ inline Dims dims_of(int B, int in, int h, int out) {
  Dims d;
  d.B = B; d.in = in; d.h = h; d.out = out;
  d.R = (B + kC - 1) / kC;
  d.Kc = up4((in + kC - 1) / kC);
  d.Kp = up8(d.Kc); d.Hp = up16(h); d.Np = up16(d.Kc); d.Bk = up8(B);
  d.sH = odd16(d.Hp);
  d.per5 = (out * (h + 1) + kC - 1) / kC;
  int o = 0;
  const int a1b1 = 128 * d.Kp + d.Hp * d.Kp, a2 = 128 * d.Hp;
  d.oA1 = o; d.oB1 = o + 128 * d.Kp; d.oA2 = o;
  o += a1b1 > a2 ? a1b1 : a2;
  d.oB2 = o; o += d.Hp * d.Np;
  d.oXT = o; o += 128 * d.Bk;
  d.oGT = o; o += d.Hp * d.Bk;
  d.oPs = o; o += kC * d.R * d.sH;    // pushed partials of my rows [src rank][R][sH]
  d.oW5 = o; o += out * (h + 1);      // W_O [out][h+1]
  d.ohs = o; o += d.R * (h + 1);      // h rows [R][h+1]
  d.og5 = o; o += d.R * out;          // y / gO rows [R][out]
  o = up4(o);
  d.ogl = o; o += d.R * d.sH;         // my gH rows [R][sH] (fp32)
  d.op5 = o; o += kC * d.per5;        // pushed dW_O | db_O partials [src rank][per5]
  d.odb = o; o += kC * d.Hp;          // pushed db_H partials [src rank][Hp] (rank 0)
  d.obH = o; o += h;                  // b_H
  d.obO = o; o += out;                // b_O
  d.oy5 = o; o += d.R * out;          // y rows (stored after the exchange)
  d.otg = o; o += d.R * out;          // my rows' targets (class ids or values)
  d.total = o;
  return d;
}

struct MlpArgs {
  int B, in, h, out;
  const float* x;             // [B][in] (the layer below's output)
  const float* WH; const float* bH; int actH;
  const float* WO; const float* bO; int actO;
  float* yH; float* yO;       // layer outputs (trace / inference reads)
  int loss_kind; const int* cls; const float* values; float* loss; int* err;
  float* gH; float* gO;       // dL/d(pre-activation) of each layer
  float* dWH; float* dbH; float* dWO; float* dbO;
  float* dx; int act_prev;    // dx * act_prev'(x); null for the first layer
  int vec;                    // x / W_H rows 16B aligned: float4 staging
};

#ifdef VCNN_PHASE_TIMING
__device__ unsigned long long g_hphase[kC][16];
#define HPHASE(i)                                                   \
  do {                                                              \
    if (threadIdx.x == 0) g_hphase[blockIdx.x % kC][i] = clock64(); \
  } while (0)
#else
#define HPHASE(i) \
  do {            \
  } while (0)
#endif

__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// out-of-line activation helpers (one copy of the switch, not one per use)
__device__ __noinline__ float actf(int act, float x) { return act_fwd(act, x); }
__device__ __noinline__ float actg(int act, float y) { return act_grad_from_out(act, y); }

__device__ __forceinline__ float rtf32(float f) { return ptx::to_tf32(f); }

// one K-major [k/4][rows][4] descriptor per K step of 8 (two 4-column halves
// LBO = rows*16 apart, 8-row core matrices SBO = 128 B apart)
__device__ __forceinline__ uint64_t kdesc(uint32_t base, int rows, int kstep) {
  return ptx::interleave_desc(base + (uint32_t)(kstep * 2 * rows * 16), (uint32_t)(rows * 16),
                              128u);
}

__global__ void __launch_bounds__(kThreadsM) mlp_head_kernel(MlpArgs a) {
  HPHASE(0);
  // every CTA of the cluster has started before anyone writes into its smem
  cluster_arrive_relaxed();
  const Dims d = dims_of(a.B, a.in, a.h, a.out);
  const int B = a.B, in = a.in, h = a.h, out = a.out;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = nt >> 5;
  extern __shared__ __align__(128) float sm[];
  __shared__ uint64_t mma_bar[2];
  __shared__ uint32_t tmem_base_sh;
  if (warp == 0) {  // accumulators: x W_H^T [0, Hp), dx [64, 64+Np), dW_H^T after
    ptx::tmem_alloc(&tmem_base_sh, 256);
    ptx::tmem_relinquish();
  }
  if (tid == 32) {
    ptx::mbar_init(&mma_bar[0], 1);
    ptx::mbar_init(&mma_bar[1], 1);
    ptx::fence_mbar_init();
  }
  // zero the operand tiles (padding rows / columns; independent of the
  // predecessor): A1, B1, B2, XT, GT (peers push gH^T into GT only after the
  // first cluster barrier)
  for (int i = tid; i < (d.oGT + d.Hp * d.Bk - d.oA1) / 4; i += nt)
    reinterpret_cast<float4*>(sm + d.oA1)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  PDL_ENTRY();
  HPHASE(1);
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  float* A1 = sm + d.oA1;
  float* B1 = sm + d.oB1;
  float* B2 = sm + d.oB2;
  float* XT = sm + d.oXT;
  float* Ps = sm + d.oPs;
  float* W5 = sm + d.oW5;
  float* hs = sm + d.ohs;
  float* g5 = sm + d.og5;
  float* gl = sm + d.ogl;
  float* p5 = sm + d.op5;
  float* pdb = sm + d.odb;
  float* sbH = sm + d.obH;
  float* sbO = sm + d.obO;
  float* y5 = sm + d.oy5;
  float* tg = sm + d.otg;
  __shared__ float lossp[kC];
  __shared__ float rowloss[kThreadsM / 32];
  const int lh = h + 1, sH = d.sH;
  const uint32_t s_base = ptx::smem_u32(sm);

  // ---- stage my input columns of x and W_H as MMA operands (tf32), all of W_O ----
  const int k0 = rank * d.Kc < in ? rank * d.Kc : in;
  const int nc = k0 + d.Kc <= in ? d.Kc : in - k0;
  // the small operands phase 2 reads (W_O, b_H, b_O, my rows' targets) are
  // loaded into registers first so their latency overlaps the x / W_H staging
  const int r0 = rank * d.R < B ? rank * d.R : B;
  const int nr = r0 + d.R <= B ? d.R : B - r0;
  const bool ce = a.loss_kind == VCNN_LOSS_SOFTMAX_CE;
  const int nw5 = out * h, ntg = ce ? nr : nr * out;
  const int nsmall = nw5 + h + out + ntg;
  auto small_src = [&](int i) -> float {
    if (i < nw5) return __ldg(a.WO + i);
    i -= nw5;
    if (i < h) return __ldg(a.bH + i);
    i -= h;
    if (i < out) return __ldg(a.bO + i);
    i -= out;
    return ce ? __int_as_float(__ldg(a.cls + r0 + i)) : __ldg(a.values + (size_t)r0 * out + i);
  };
  auto small_dst = [&](int i) -> float* {
    if (i < nw5) return W5 + (i / h) * lh + (i - (i / h) * h);
    i -= nw5;
    if (i < h) return sbH + i;
    i -= h;
    if (i < out) return sbO + i;
    return tg + (i - out);
  };
  const float sv0 = tid < nsmall ? small_src(tid) : 0.f;
  const float sv1 = tid + nt < nsmall ? small_src(tid + nt) : 0.f;
  __syncthreads();  // the zero fill is complete before the data lands
  {
    // x rows b, columns c: A1 (b, c) and XT (c, b); W_H rows o: B1 (o, c) and
    // B2 (c, o).  4 columns per item (float4 when the rows allow it).
    const int q = (nc + 3) >> 2, nx = B * q, nw = h * q;
#pragma unroll 1
    for (int i = tid; i < nx + nw; i += nt) {
      const bool isx = i < nx;
      const int ii = isx ? i : i - nx, r = ii / q, c = 4 * (ii - r * q);
      const float* src = (isx ? a.x + (size_t)r * in : a.WH + (size_t)r * in) + k0 + c;
      float v[4];
      if (a.vec && c + 4 <= nc) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(src));
        v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = c + u < nc ? __ldg(src + u) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = rtf32(v[u]);
      if (isx) {
        *reinterpret_cast<float4*>(A1 + kmaj(r, c, 128)) = make_float4(v[0], v[1], v[2], v[3]);
#pragma unroll
        for (int u = 0; u < 4; ++u) XT[kmaj(c + u, r, 128)] = v[u];
      } else {
        *reinterpret_cast<float4*>(B1 + kmaj(r, c, d.Hp)) = make_float4(v[0], v[1], v[2], v[3]);
#pragma unroll
        for (int u = 0; u < 4; ++u) B2[kmaj(c + u, r, d.Np)] = v[u];
      }
    }
  }
  if (tid < nsmall) *small_dst(tid) = sv0;
  if (tid + nt < nsmall) *small_dst(tid + nt) = sv1;
#pragma unroll 1
  for (int i = tid + 2 * nt; i < nsmall; i += nt) *small_dst(i) = small_src(i);
  if (tid < kThreadsM / 32) rowloss[tid] = 0.f;
  ptx::fence_proxy_async_smem();  // generic stores -> the MMAs' async proxy
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t tH = tmem, tX = tmem + 64, tW = tmem + 64 + (uint32_t)d.Np;
  HPHASE(2);

  // ---- 1: partial x[:, mine] W_H[:, mine]^T on the tensor cores (M = the
  //         128 batch rows, N = Hp hidden units, K = my columns), pushed to the
  //         row owner's slot [rank] ----
  if (warp == 0 && ptx::elect_one()) {
    const uint32_t idesc = ptx::idesc_tf32(128, d.Hp);
    for (int ks = 0; ks < (d.Kp >> 3); ++ks)
      ptx::mma_tf32(tH, kdesc(s_base + 4u * d.oA1, 128, ks), kdesc(s_base + 4u * d.oB1, d.Hp, ks),
                    idesc, ks > 0 ? 1u : 0u);
    ptx::mma_commit(&mma_bar[0]);
  }
  __syncwarp();
  cluster_wait();
  ptx::mbar_wait(&mma_bar[0], 0);
  ptx::tc_fence_after();
  {
    const int qd = warp & 3, cgp = warp >> 2;  // lane quadrant, 16-column group
    const int b = qd * 32 + lane;
    for (int c0 = cgp * 16; c0 < d.Hp; c0 += (nwarps >> 2) * 16) {
      uint32_t r[16];
      ptx::tmem_ld16(tH + ((uint32_t)(qd * 32) << 16) + (uint32_t)c0, r);
      ptx::tmem_wait_ld();
      if (b < B) {
        const int owner = b / d.R;
        float* dst = cluster.map_shared_rank(Ps, owner) + (rank * d.R + (b - owner * d.R)) * sH + c0;
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(dst + j) =
              make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                          __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
      }
    }
  }
  HPHASE(3);
  cluster_arrive();
  cluster_wait();
  HPHASE(4);

  // ---- 2: my rows: h = act(sum over ranks, in order + b); the last layer,
  //         the loss, dW_O partials, gH rows ----
#pragma unroll 1
  for (int e = tid; e < nr * h; e += nt) {
    const int b = e / h, o = e - b * h;
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < kC; ++c) acc += Ps[(c * d.R + b) * sH + o];
    hs[b * lh + o] = actf(a.actH, acc + sbH[o]);
  }
  __syncthreads();
  HPHASE(10);
#pragma unroll 1
  for (int e = tid; e < nr * out; e += nt) {
    const int b = e / out, o = e - b * out;
    const float* hr = hs + b * lh;
    const float* wo = W5 + o * lh;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int k = 0;
#pragma unroll 1
    for (; k + 3 < h; k += 4) {
      a0 += hr[k] * wo[k];
      a1 += hr[k + 1] * wo[k + 1];
      a2 += hr[k + 2] * wo[k + 2];
      a3 += hr[k + 3] * wo[k + 3];
    }
#pragma unroll 1
    for (; k < h; ++k) a0 += hr[k] * wo[k];
    const float v = actf(a.actO, ((a0 + a1) + (a2 + a3)) + sbO[o]);
    g5[e] = v;
    y5[e] = v;
  }
  __syncthreads();
  HPHASE(11);
  // loss + dL/dy * act'(y).  softmax-CE: one warp per sample, lanes over
  // the classes (shuffle-tree max / sum); MSE: one thread per element.  The
  // partial loss: per-warp values summed by thread 0 in warp order.
  if (ce) {
    const float inv_b = 1.0f / (float)B;
#pragma unroll 1
    for (int b = warp; b < nr; b += nwarps) {
      float* l = g5 + b * out;
      const int c = __float_as_int(tg[b]);
      const bool bad = c < 0 || c >= out;
      if (bad && a.err && lane == 0) atomicExch(a.err, 1);
      float m = -INFINITY;
#pragma unroll 1
      for (int u = lane; u < out; u += 32) m = fmaxf(m, l[u]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      float sum = 0.f;
#pragma unroll 1
      for (int u = lane; u < out; u += 32) sum += expf(l[u] - m);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane == 0 && !bad) rowloss[warp] += m + logf(sum) - l[c];
      __syncwarp();
      const float inv = inv_b / sum;
#pragma unroll 1
      for (int u = lane; u < out; u += 32) {
        const float yv = l[u];
        float gv = expf(yv - m) * inv;
        if (u == c) gv -= inv_b;
        if (a.actO != VCNN_ACT_IDENTITY) gv *= actg(a.actO, yv);
        l[u] = gv;
      }
    }
  } else {
    const float scale = 2.0f / (float)(B * out);
    float mine = 0.f;
#pragma unroll 1
    for (int t = tid; t < nr * out; t += nt) {
      const float yv = g5[t], dd = yv - tg[t];
      mine += dd * dd;
      float gv = scale * dd;
      if (a.actO != VCNN_ACT_IDENTITY) gv *= actg(a.actO, yv);
      g5[t] = gv;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if (lane == 0) rowloss[warp] += mine;
  }
  __syncthreads();
  if (tid == 0) {
    float v = 0.f;
#pragma unroll 1
    for (int w = 0; w < nwarps; ++w) v += rowloss[w];
    *cluster.map_shared_rank(lossp + rank, 0) = v;
  }
  HPHASE(12);
  // dW_O | db_O partials over my rows, pushed to the slice owner's slot [rank]
#pragma unroll 1
  for (int t = tid; t < out * lh; t += nt) {
    const int o = t / lh, i = t - o * lh;
    float acc = 0.f;
    if (i < h)
#pragma unroll 1
      for (int b = 0; b < nr; ++b) acc += g5[b * out + o] * hs[b * lh + i];
    else
#pragma unroll 1
      for (int b = 0; b < nr; ++b) acc += g5[b * out + o];
    const int c = t / d.per5;
    *cluster.map_shared_rank(p5 + rank * d.per5 + (t - c * d.per5), c) = acc;
  }
  // gH rows = (gO W_O) * act_H'(h), zero padded to Hp
#pragma unroll 1
  for (int t = tid; t < d.R * d.Hp; t += nt) {
    const int b = t / d.Hp, i = t - b * d.Hp;
    float acc = 0.f;
    if (b < nr && i < h) {
#pragma unroll 1
      for (int o = 0; o < out; ++o) acc += g5[b * out + o] * W5[o * lh + i];
      if (a.actH != VCNN_ACT_IDENTITY) acc *= actg(a.actH, hs[b * lh + i]);
    }
    gl[b * sH + i] = acc;
  }
  __syncthreads();
  HPHASE(13);
  // db_H partial of my rows -> rank 0's slot [rank]; my gH rows (tf32) into
  // every CTA's gH (A2) and gH^T (GT) operand tiles
  for (int i = tid; i < d.Hp; i += nt) {
    float acc = 0.f;
#pragma unroll 1
    for (int b = 0; b < nr; ++b) acc += gl[b * sH + i];
    *cluster.map_shared_rank(pdb + rank * d.Hp + i, 0) = acc;
  }
  {
    const int q = d.Hp >> 2, na2 = nr * q;  // A2: float4 over 4 hidden units
    const int nb4 = (nr + 3) >> 2, ngt = d.Hp * nb4;  // GT: float4 over 4 batch rows
    const int per = na2 + ngt;
#pragma unroll 1
    for (int t = tid; t < per * kC; t += nt) {
      const int c = t / per, u = t - c * per;
      if (u < na2) {
        const int b = u / q, k = 4 * (u - b * q);
        const float* g = gl + b * sH + k;
        *reinterpret_cast<float4*>(cluster.map_shared_rank(sm + d.oA2, c) +
                                   kmaj(r0 + b, k, 128)) =
            make_float4(rtf32(g[0]), rtf32(g[1]), rtf32(g[2]), rtf32(g[3]));
      } else {
        const int v = u - na2, o = v / nb4, bq = 4 * (v - o * nb4);
        float f[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) f[e] = bq + e < nr ? rtf32(gl[(bq + e) * sH + o]) : 0.f;
        float* gt = cluster.map_shared_rank(sm + d.oGT, c);
        if ((d.R & 3) == 0) {  // my rows are whole 4-row groups: one 16-byte store
          *reinterpret_cast<float4*>(gt + kmaj(o, r0 + bq, d.Hp)) =
              make_float4(f[0], f[1], f[2], f[3]);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (bq + e < nr) gt[kmaj(o, r0 + bq + e, d.Hp)] = f[e];
        }
      }
    }
  }
  asm volatile("fence.proxy.async;" ::: "memory");  // my pushes -> peers' MMAs
  HPHASE(5);
  cluster_arrive();
  cluster_wait();
  HPHASE(6);
  // ---- 4 (issued now, drained below): on the tensor cores
  //         dx[:, mine]     = gH W_H[:, mine]     (M = batch, N = my columns, K = hidden)
  //         dW_H[:, mine]^T = x[:, mine]^T gH     (M = my columns, N = hidden, K = batch) ----
  if (warp == 0 && ptx::elect_one()) {
    ptx::fence_proxy_async_smem();  // the pushed gH tiles -> the async proxy
    const uint32_t idx = ptx::idesc_tf32(128, d.Np), idw = ptx::idesc_tf32(128, d.Hp);
    for (int ks = 0; ks < (d.Hp >> 3); ++ks)
      ptx::mma_tf32(tX, kdesc(s_base + 4u * d.oA2, 128, ks), kdesc(s_base + 4u * d.oB2, d.Np, ks),
                    idx, ks > 0 ? 1u : 0u);
    for (int ks = 0; ks < (d.Bk >> 3); ++ks)
      ptx::mma_tf32(tW, kdesc(s_base + 4u * d.oXT, 128, ks), kdesc(s_base + 4u * d.oGT, d.Hp, ks),
                    idw, ks > 0 ? 1u : 0u);
    ptx::mma_commit(&mma_bar[1]);
  }
  __syncwarp();
  // my rows' layer outputs and gradients (stored after the exchange: the
  // cluster barrier's release would otherwise wait for them)
#pragma unroll 1
  for (int e = tid; e < nr * h; e += nt) {
    const int b = e / h, o = e - b * h;
    a.yH[(size_t)r0 * h + e] = hs[b * lh + o];
    a.gH[(size_t)r0 * h + e] = gl[b * sH + o];
  }
#pragma unroll 1
  for (int e = tid; e < nr * out; e += nt) {
    a.yO[(size_t)r0 * out + e] = y5[e];
    a.gO[(size_t)r0 * out + e] = g5[e];
  }

  // ---- 3: my slice of dW_O | db_O, (rank 0) the loss and db_H, summed in rank order ----
  {
    const int np = out * lh, e0 = rank * d.per5;
    const int e1 = e0 + d.per5 < np ? e0 + d.per5 : np;
#pragma unroll 1
    for (int e = e0 + tid; e < e1; e += nt) {
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < kC; ++c) acc += p5[c * d.per5 + (e - e0)];
      const int o = e / lh, i = e - o * lh;
      if (i < h) a.dWO[(size_t)o * h + i] = acc;
      else a.dbO[o] = acc;
    }
  }
  if (rank == 0 && tid == 0 && a.loss) {
    float v = 0.f;
#pragma unroll 1
    for (int c = 0; c < kC; ++c) v += lossp[c];
    *a.loss = a.loss_kind == VCNN_LOSS_SOFTMAX_CE ? v / (float)B : v / (float)(B * out);
  }
  if (rank == 0)
#pragma unroll 1
    for (int o = tid; o < h; o += nt) {
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < kC; ++c) acc += pdb[c * d.Hp + o];
      a.dbH[o] = acc;
    }
  HPHASE(7);

  // ---- 4 (drain): 4 lane quadrants x 4 column groups; dx *= act_prev'(x) ----
  ptx::mbar_wait(&mma_bar[1], 0);
  ptx::tc_fence_after();
  {
    const int qd = warp & 3, cgp = warp >> 2, step = (nwarps >> 2) * 16;
    const int row = qd * 32 + lane;  // dx: batch row b; dW^T: my column
    const uint32_t lrow = (uint32_t)(qd * 32) << 16;
    if (a.dx)
      for (int c0 = cgp * 16; c0 < d.Np; c0 += step) {
        uint32_t r[16];
        ptx::tmem_ld16(tX + lrow + (uint32_t)c0, r);
        ptx::tmem_wait_ld();
        if (row < B) {
          const float* xs = a.x + (size_t)row * in + k0;
          float* p = a.dx + (size_t)row * in + k0;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int col = c0 + j;
            if (col >= nc) break;
            float v = __uint_as_float(r[j]);
            if (a.act_prev == VCNN_ACT_RELU) v *= __ldg(xs + col) > 0.f ? 1.f : 0.f;
            else if (a.act_prev != VCNN_ACT_IDENTITY) v *= actg(a.act_prev, __ldg(xs + col));
            p[col] = v;
          }
        }
      }
    for (int c0 = cgp * 16; c0 < d.Hp; c0 += step) {
      uint32_t r[16];
      ptx::tmem_ld16(tW + lrow + (uint32_t)c0, r);
      ptx::tmem_wait_ld();
      if (row < nc)
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (c0 + j < h) a.dWH[(size_t)(c0 + j) * in + k0 + row] = __uint_as_float(r[j]);
    }
  }
  HPHASE(8);
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 256);
  HPHASE(9);
}

}  // namespace

#ifdef VCNN_PHASE_TIMING
extern "C" int vcnn_debug_hphases(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_hphase, sizeof(unsigned long long) * kC * 16) ==
                 cudaSuccess
             ? 0
             : 4;
}
#endif

size_t mlp_head_smem(int B, int in, int h, int out) {
  return sizeof(float) * (size_t)dims_of(B, in, h, out).total;
}

// cluster of kC CTAs with this kernel's shared memory schedulable? (cached)
static bool cluster_ok(size_t smem) {
  static size_t ok_upto = 0, bad_from = ~(size_t)0;
  if (smem <= ok_upto) return true;
  if (smem >= bad_from) return false;
  bool ok = cudaFuncSetAttribute(mlp_head_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed,
                                 1) == cudaSuccess &&
            cudaFuncSetAttribute(mlp_head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) == cudaSuccess;
  if (ok) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kC);
    cfg.blockDim = dim3(kThreadsM);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kC;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    ok = cudaOccupancyMaxActiveClusters(&nclusters, mlp_head_kernel, &cfg) == cudaSuccess &&
         nclusters > 0;
  }
  cudaGetLastError();
  if (ok) ok_upto = smem;
  else bad_from = smem;
  return ok;
}

bool mlp_head_fusable(int B, int in, int h, int out) {
  // M = 128 batch rows / input columns per CTA; the dx accumulator sits at
  // TMEM column 64 (Np <= 128) and dW_H^T after it (Hp <= 64): 256 columns
  if (B < 1 || B > 128 || h < 1 || h > 64 || out < 1 || out > 64 || in < kC || in > 128 * kC)
    return false;
  const size_t smem = mlp_head_smem(B, in, h, out);
  return smem + 1024 <= 227 * 1024 && cluster_ok(smem);
}

int launch_mlp_head(int B, int in, int h, int out, const float* x, const float* WH,
                    const float* bH, int actH, const float* WO, const float* bO, int actO,
                    float* yH, float* yO, int loss_kind, const int* cls, const float* values,
                    float* loss, int* err, float* gH, float* gO, float* dWH, float* dbH,
                    float* dWO, float* dbO, float* dx, int act_prev, cudaStream_t st) {
  const size_t smem = mlp_head_smem(B, in, h, out);
  if (!cluster_ok(smem)) return fail(VCNN_ECUDA, "mlp head: cluster not schedulable");
  const bool vec = in % 4 == 0 && ((reinterpret_cast<uintptr_t>(x) |
                                    reinterpret_cast<uintptr_t>(WH)) & 15) == 0;
  MlpArgs a{B, in, h, out, x, WH, bH, actH, WO, bO, actO, yH, yO, loss_kind, cls, values,
            loss, err, gH, gO, dWH, dbH, dWO, dbO, dx, act_prev, vec ? 1 : 0};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kC);
  cfg.blockDim = dim3(kThreadsM);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = kC;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  VCNN_CUDA_TRY(cudaLaunchKernelEx(&cfg, mlp_head_kernel, a));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

}  // namespace vcnn_b200
