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
// rank order.  fp32 SIMT with 4x4 register tiles; every reduction in a fixed
// order (deterministic).  Replaces 6-8 launches on the critical path.
#include <cooperative_groups.h>

#include "kernels.cuh"

namespace vcnn_b200 {

namespace {

namespace cg = cooperative_groups;

constexpr int kC = 16;        // cluster size (non-portable; B200 supports 16)
constexpr int kThreadsM = 512;

struct Dims {
  int B, in, h, out;
  int R, Kc;                  // batch rows / input columns per CTA (Kc % 4 == 0)
  int Bp, Hp, Kp;             // padded: Bp, Hp to 16 (mma M), Kp to 8 (mma K / N)
  int sK, sH;                 // row strides: multiples of 4 floats, odd in 16B units
  int per5;                   // dW_O | db_O elements reduced per CTA
  // smem offsets (floats)
  int oxr, owr, oPs, oG, oW5, ohs, og5, ogl, op5, obH, obO, oy5, otg;
  int total;
};

__host__ __device__ inline int up4(int v) { return (v + 3) & ~3; }
__host__ __device__ inline int up8(int v) { return (v + 7) & ~7; }
__host__ __device__ inline int up16(int v) { return (v + 15) & ~15; }
// a row stride of v floats (v % 4 == 0) rounded up to 8 (mod 32): the mma
// fragment loads hit 32 distinct banks both row-major (bank g*s + t) and
// transposed (bank g + t*s) -- the dW GEMM reads x and gH transposed; an odd
// number of 16-byte units (the previous rule) left those 2-way conflicted
__host__ __device__ inline int pad8of32(int v) { return v + ((8 - v % 32) + 32) % 32; }

__host__ __device__ inline Dims dims_of(int B, int in, int h, int out) {
  Dims d;
  d.B = B; d.in = in; d.h = h; d.out = out;
  d.R = (B + kC - 1) / kC;
  d.Kc = up4((in + kC - 1) / kC);
  d.Bp = up16(B); d.Hp = up16(h); d.Kp = up8(d.Kc);
  d.sK = pad8of32(d.Kp);
  d.sH = pad8of32(d.Hp);
  d.per5 = (out * (h + 1) + kC - 1) / kC;
  int o = 0;
  d.oxr = o; o += d.Bp * d.sK;        // x[:, mine]   [Bp][sK]
  d.owr = o; o += d.Hp * d.sK;        // W_H[:, mine] [Hp][sK]
  d.oPs = o; o += kC * d.R * d.sH;    // pushed partials of my rows [src rank][R][sH]
  d.oG = o;  o += d.Bp * d.sH;        // gH, all rows (pushed by the row owners) [Bp][sH]
  d.oW5 = o; o += out * (h + 1);      // W_O [out][h+1]
  d.ohs = o; o += d.R * (h + 1);      // h rows [R][h+1]
  d.og5 = o; o += d.R * out;          // y / gO rows [R][out]
  o = up4(o);
  d.ogl = o; o += d.R * d.sH;         // my gH rows [R][sH] (float4 pushes)
  d.op5 = o; o += kC * d.per5;        // pushed dW_O | db_O partials [src rank][per5]
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
  // batch slices: cluster c owns rows [c*B, (c+1)*B) of the Bg-row batch; with
  // more than one cluster the dW/db of each slice go to part + c*per (param
  // order W_H | b_H | W_O | b_O; the caller sums the slices in order) and the
  // loss partials are summed by the last cluster to finish (ticket)
  int Bg, ncl;
  float* part; float* lpart; unsigned* ticket;
};

#ifdef VCNN_PHASE_TIMING
__device__ unsigned long long g_hphase[kC][16];
#define HPHASE(i)                                                   \
  do {                                                              \
    if (threadIdx.x == 0 && blockIdx.x < kC) g_hphase[blockIdx.x][i] = clock64(); \
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

__device__ __forceinline__ uint32_t tf32(float f) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(f));
  return r;
}

// One warp's m16 x (NG x n8) tile of C += A B over ksteps k8 steps with
// mma.sync TF32 (the tensor-core path for these small per-CTA GEMMs; fp32
// accumulate).  A(m, k) = A[m*am + k*ak], B(k, n) = Bm[n*bn + k*bk]; the
// fragment layouts are the PTX m16n8k8 .row.col ones: lane = 4g + t,
// a = {(g,t), (g+8,t), (g,t+4), (g+8,t+4)}, b = {(t,g), (t+4,g)},
// c = {(g,2t), (g,2t+1), (g+8,2t), (g+8,2t+1)}.
template <int NG, bool B_TF32 = false>  // B_TF32: B already rounded in smem
__device__ __forceinline__ void warp_mma(float (&c)[NG][4], const float* A, int am, int ak,
                                         const float* Bm, int bn, int bk, int m0, int n0,
                                         int nvalid, int ksteps, int lane) {
  const int g = lane >> 2, t = lane & 3;
  const float* pa = A + (m0 + g) * am + t * ak;
  const float* pb = Bm + (n0 + g) * bn + t * bk;
  for (int ks = 0; ks < ksteps; ++ks) {
    const int k = ks * 8;
    const uint32_t a0 = tf32(pa[k * ak]), a1 = tf32(pa[8 * am + k * ak]);
    const uint32_t a2 = tf32(pa[(k + 4) * ak]), a3 = tf32(pa[8 * am + (k + 4) * ak]);
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      if (j < nvalid) {
        const float f0 = pb[j * 8 * bn + k * bk], f1 = pb[j * 8 * bn + (k + 4) * bk];
        const uint32_t b0 = B_TF32 ? __float_as_uint(f0) : tf32(f0);
        const uint32_t b1 = B_TF32 ? __float_as_uint(f1) : tf32(f1);
        asm volatile(
            "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, "
            "{%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      }
    }
  }
}

// stage rows [0, nrows) x columns [k0, k0+nc) of a row-major [*][ld] matrix
// into smem [Rp][s] (zero padded to Rp rows and Kp columns)
__device__ __forceinline__ void stage_cols(float* dst, int s, const float* src, int ld, int nrows,
                                           int Rp, int k0, int nc, int Kp, bool vec, int tid,
                                           int nt, bool round = false) {
  if (vec) {  // float4: Kp, k0, ld multiples of 4, src 16B aligned
    const int q = Kp >> 2, n = Rp * q;
    constexpr int kU = 4;
    for (int base = 0; base < n; base += kU * nt) {
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = base + u * nt + tid, r = i / q, k = 4 * (i - r * q);
        v[u] = (r < nrows && k < nc)
                   ? __ldg(reinterpret_cast<const float4*>(src + (size_t)r * ld + k0 + k))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = base + u * nt + tid, r = i / q, k = 4 * (i - r * q);
        float4 w = v[u];
        if (round) {
          w.x = __uint_as_float(tf32(w.x));
          w.y = __uint_as_float(tf32(w.y));
          w.z = __uint_as_float(tf32(w.z));
          w.w = __uint_as_float(tf32(w.w));
        }
        if (i < n) *reinterpret_cast<float4*>(dst + r * s + k) = w;
      }
    }
  } else {
    const int n = Rp * Kp;
#pragma unroll 1
    for (int i = tid; i < n; i += nt) {
      const int r = i / Kp, k = i - r * Kp;
      const float v = (r < nrows && k < nc) ? __ldg(src + (size_t)r * ld + k0 + k) : 0.f;
      dst[r * s + k] = round ? __uint_as_float(tf32(v)) : v;
    }
  }
}

// TB/TIN/TH/TOUT: compile-time dims for the common shape (CIFAR-3's tail:
// every index division and loop bound folds), 0 = read from the arguments
// (LOSS, AH, AO, AP: compile-time loss kind and activations of layer H,
// layer O and the layer below, -1 = read from the arguments -- the
// specialised kernel carries only its own loss / activation code)
template <int TB, int TIN, int TH, int TOUT, int LOSS = -1, int AH = -1, int AO = -1, int AP = -1>
__global__ void __launch_bounds__(kThreadsM) mlp_head_kernel(MlpArgs a) {
  HPHASE(0);
  // every CTA of the cluster has started before anyone writes into its smem
  cluster_arrive_relaxed();
  PDL_ENTRY();
  HPHASE(1);
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int B = TB ? TB : a.B, in = TIN ? TIN : a.in, h = TH ? TH : a.h,
            out = TOUT ? TOUT : a.out;
  const int loss_kind = LOSS >= 0 ? LOSS : a.loss_kind;
  const int actH = AH >= 0 ? AH : a.actH, actO = AO >= 0 ? AO : a.actO;
  const int act_prev = AP >= 0 ? AP : a.act_prev;
  // this cluster's batch slice (rows rb .. rb + B of the Bg-row batch)
  const int cid = (int)(blockIdx.x / kC), Bg = a.Bg;
  const size_t rb = (size_t)cid * B;
  const float* x_ = a.x + rb * in;
  const int* cls_ = a.cls ? a.cls + rb : nullptr;
  const float* vals_ = a.values ? a.values + rb * out : nullptr;
  float* yH_ = a.yH + rb * h;
  float* gH_ = a.gH + rb * h;
  float* yO_ = a.yO + rb * out;
  float* gO_ = a.gO + rb * out;
  float* dx_ = a.dx ? a.dx + rb * in : nullptr;
  const size_t per = (size_t)h * in + h + (size_t)out * h + out;
  float* sl = a.ncl > 1 ? a.part + cid * per : nullptr;
  float* dWH_ = sl ? sl : a.dWH;
  float* dbH_ = sl ? sl + (size_t)h * in : a.dbH;
  float* dWO_ = sl ? sl + (size_t)h * in + h : a.dWO;
  float* dbO_ = sl ? sl + (size_t)h * in + h + (size_t)out * h : a.dbO;
  const Dims d = dims_of(B, in, h, out);
  const int tid = threadIdx.x, nt = kThreadsM, lane = tid & 31, warp = tid >> 5;
  const int nwarps = nt >> 5;
  extern __shared__ __align__(16) float sm[];
  float* xr = sm + d.oxr;
  float* wr = sm + d.owr;
  float* Ps = sm + d.oPs;
  float* G = sm + d.oG;
  float* W5 = sm + d.oW5;
  float* hs = sm + d.ohs;
  float* g5 = sm + d.og5;
  float* gl = sm + d.ogl;
  float* p5 = sm + d.op5;
  float* sbH = sm + d.obH;
  float* sbO = sm + d.obO;
  float* y5 = sm + d.oy5;
  float* tg = sm + d.otg;
  __shared__ float lossp[kC];
  __shared__ float rowloss[kThreadsM / 32];
  const int lh = h + 1, sK = d.sK, sH = d.sH;

  // ---- stage my input columns of x and W_H (zero padded), all of W_O ----
  const int k0 = rank * d.Kc < in ? rank * d.Kc : in;
  const int nc = k0 + d.Kc <= in ? d.Kc : in - k0;
  // the small operands phase 2 reads (W_O, b_H, b_O, my rows' targets) are
  // loaded into registers first so their latency overlaps the x / W_H staging
  const int r0 = rank * d.R < B ? rank * d.R : B;
  const int nr = r0 + d.R <= B ? d.R : B - r0;
  const bool ce = loss_kind == VCNN_LOSS_SOFTMAX_CE;
  const int nw5 = out * h, ntg = ce ? nr : nr * out;
  const int nsmall = nw5 + h + out + ntg;
  auto small_src = [&](int i) -> float {
    if (i < nw5) return __ldg(a.WO + i);
    i -= nw5;
    if (i < h) return __ldg(a.bH + i);
    i -= h;
    if (i < out) return __ldg(a.bO + i);
    i -= out;
    return ce ? __int_as_float(__ldg(cls_ + r0 + i)) : __ldg(vals_ + (size_t)r0 * out + i);
  };
  auto small_dst = [&](int i) -> float* {
    if (i < nw5) return W5 + (i / h) * lh + (i - (i / h) * h);
    i -= nw5;
    if (i < h) return sbH + i;
    i -= h;
    if (i < out) return sbO + i;
    return tg + (i - out);
  };
  // (one straight-line copy each: this kernel runs once per step, so its
  // instruction footprint is fetched cold -- code size is latency here)
  const float sv0 = tid < nsmall ? small_src(tid) : 0.f;
  const float sv1 = tid + nt < nsmall ? small_src(tid + nt) : 0.f;
  stage_cols(xr, sK, x_, in, B, d.Bp, k0, nc, d.Kp, a.vec, tid, nt);
  stage_cols(wr, sK, a.WH, in, h, d.Hp, k0, nc, d.Kp, a.vec, tid, nt, true);  // MMA-only: tf32
  if (tid < nsmall) *small_dst(tid) = sv0;
  if (tid + nt < nsmall) *small_dst(tid + nt) = sv1;
#pragma unroll 1
  for (int i = tid + 2 * nt; i < nsmall; i += nt) *small_dst(i) = small_src(i);
  for (int i = tid; i < (d.Bp - B) * sH; i += nt) G[B * sH + i] = 0.f;  // pad rows
  if (tid < kThreadsM / 32) rowloss[tid] = 0.f;
  __syncthreads();
  HPHASE(2);

  // ---- 1: partial x[:, mine] W_H[:, mine]^T on the tensor cores (m16 = 16
  //         batch rows, n = 4 x n8 hidden units per warp tile), pushed to the
  //         row owner's slot [rank] ----
  cluster_wait();
  {
    const int mt = d.Bp >> 4, nN = d.Hp >> 3, ngr = (nN + 3) >> 2;
    for (int tile = warp; tile < mt * ngr; tile += nwarps) {
      const int im = tile / ngr, ig = tile - im * ngr;
      const int m0 = im * 16, n0 = ig * 32;
      const int nv = nN - ig * 4 < 4 ? nN - ig * 4 : 4;
      float c[4][4] = {};
      warp_mma<4, true>(c, xr, sK, 1, wr, sK, 1, m0, n0, nv, d.Kp >> 3, lane);
      const int g = lane >> 2, t = lane & 3;
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const int b = m0 + g + 8 * hf;
        if (b >= B) continue;
        const int owner = b / d.R;
        float* dst = cluster.map_shared_rank(Ps, owner) + (rank * d.R + (b - owner * d.R)) * sH;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int o = n0 + j * 8 + 2 * t;
          if (j < nv && o < h)  // o even, h may be odd: o + 1 < Hp always
            *reinterpret_cast<float2*>(dst + o) = make_float2(c[j][2 * hf], c[j][2 * hf + 1]);
        }
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
    hs[b * lh + o] = AH >= 0 ? act_fwd(AH, acc + sbH[o]) : actf(actH, acc + sbH[o]);
  }
  __syncthreads();
  HPHASE(10);
  // y = act(h W_O^T + b): 4 lanes per output (strided k, independent loads),
  // fixed xor tree; warp-uniform loop so every lane reaches the shuffles
#pragma unroll 1
  for (int base = warp * 32; base < nr * out * 4; base += nt) {
    const int e = (base + lane) >> 2, part = lane & 3;
    const bool ok = e < nr * out;
    const int b = ok ? e / out : 0, o = ok ? e - b * out : 0;
    const float* hr = hs + b * lh;
    const float* wo = W5 + o * lh;
    float acc = 0.f;
    if (ok)
#pragma unroll 4
      for (int k = part; k < h; k += 4) acc += hr[k] * wo[k];
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (ok && part == 0) {
      const float v = AO >= 0 ? act_fwd(AO, acc + sbO[o]) : actf(actO, acc + sbO[o]);
      g5[e] = v;
      y5[e] = v;
    }
  }
  __syncthreads();
  HPHASE(11);
  // loss + dL/dy * act'(y).  softmax-CE: one warp per sample, lanes over
  // the classes (shuffle-tree max / sum); MSE: one thread per element.  The
  // partial loss: per-warp values summed by thread 0 in warp order.
  if (ce) {
    const float inv_b = 1.0f / (float)Bg;
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
        if (actO != VCNN_ACT_IDENTITY)
          gv *= AO >= 0 ? act_grad_from_out(AO, yv) : actg(actO, yv);
        l[u] = gv;
      }
    }
  } else {
    const float scale = 2.0f / (float)(Bg * out);
    float mine = 0.f;
#pragma unroll 1
    for (int t = tid; t < nr * out; t += nt) {
      const float yv = g5[t], dd = yv - tg[t];
      mine += dd * dd;
      float gv = scale * dd;
      if (actO != VCNN_ACT_IDENTITY)
        gv *= AO >= 0 ? act_grad_from_out(AO, yv) : actg(actO, yv);
      g5[t] = gv;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if (lane == 0) rowloss[warp] += mine;
  }
  __syncthreads();
  if (warp == 0) {  // the per-warp partial losses, fixed xor tree (16 warps)
    float v = lane < nwarps ? rowloss[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) *cluster.map_shared_rank(lossp + rank, 0) = v;
  }
  HPHASE(12);
  // dW_O | db_O partials over my rows, pushed to the slice owner's slot [rank]
#pragma unroll 1
  for (int t = tid; t < out * lh; t += nt) {
    const int o = t / lh, i = t - o * lh;
    float acc = 0.f;
    const float* hc = i < h ? hs + i : nullptr;
#pragma unroll
    for (int b = 0; b < 8; ++b)  // nr <= R <= 8 (B <= 128 over 16 CTAs)
      if (b < nr) acc += g5[b * out + o] * (hc ? hc[b * lh] : 1.f);
    const int c = t / d.per5;
    *cluster.map_shared_rank(p5 + rank * d.per5 + (t - c * d.per5), c) = acc;
  }
  // gH rows = (gO W_O) * act_H'(h), zero padded to Hp
#pragma unroll 1
  for (int t = tid; t < d.R * d.Hp; t += nt) {
    const int b = t / d.Hp, i = t - b * d.Hp;
    float acc = 0.f;
    if (b < nr && i < h) {
#pragma unroll 4
      for (int o = 0; o < out; ++o) acc += g5[b * out + o] * W5[o * lh + i];
      if (actH != VCNN_ACT_IDENTITY)
        acc *= AH >= 0 ? act_grad_from_out(AH, hs[b * lh + i]) : actg(actH, hs[b * lh + i]);
    }
    gl[b * sH + i] = acc;
  }
  __syncthreads();
  HPHASE(13);
  // push my gH rows into every CTA's G (float4)
  {
    const int q = d.Hp >> 2, n = nr * q * kC;
#pragma unroll 1
    for (int t = tid; t < n; t += nt) {
      const int c = t / (nr * q), u = t - c * (nr * q), b = u / q, k = 4 * (u - b * q);
      *reinterpret_cast<float4*>(cluster.map_shared_rank(G, c) + (r0 + b) * sH + k) =
          *reinterpret_cast<const float4*>(gl + b * sH + k);
    }
  }
  HPHASE(5);
  cluster_arrive();
  cluster_wait();
  HPHASE(6);
  // my rows' layer outputs and gradients (stored after the exchange: the
  // cluster barrier's release would otherwise wait for them)
#pragma unroll 1
  for (int e = tid; e < nr * h; e += nt) {
    const int b = e / h, o = e - b * h;
    yH_[(size_t)r0 * h + e] = hs[b * lh + o];
    gH_[(size_t)r0 * h + e] = gl[b * sH + o];
  }
#pragma unroll 1
  for (int e = tid; e < nr * out; e += nt) {
    yO_[(size_t)r0 * out + e] = y5[e];
    gO_[(size_t)r0 * out + e] = g5[e];
  }

  // ---- 3: my slice of dW_O | db_O and (rank 0) the loss, summed in rank order ----
  {
    const int np = out * lh, e0 = rank * d.per5;
    const int e1 = e0 + d.per5 < np ? e0 + d.per5 : np;
#pragma unroll 1
    for (int e = e0 + tid; e < e1; e += nt) {
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < kC; ++c) acc += p5[c * d.per5 + (e - e0)];
      const int o = e / lh, i = e - o * lh;
      if (i < h) dWO_[(size_t)o * h + i] = acc;
      else dbO_[o] = acc;
    }
  }
  if (rank == 0 && tid == 0 && a.loss) {
    float v = 0.f;
#pragma unroll 1
    for (int c = 0; c < kC; ++c) v += lossp[c];
    const float norm = loss_kind == VCNN_LOSS_SOFTMAX_CE ? (float)Bg : (float)(Bg * out);
    if (a.ncl == 1) {
      *a.loss = v / norm;
    } else {  // the last slice to finish sums the partials in slice order
      a.lpart[cid] = v;
      __threadfence();
      if (atomicAdd(a.ticket, 1u) == (unsigned)a.ncl - 1) {
        __threadfence();
        float t = 0.f;
        for (int c = 0; c < a.ncl; ++c) t += *(volatile float*)(a.lpart + c);
        *a.loss = t / norm;
        *a.ticket = 0u;
      }
    }
  }
  if (rank == 0) {
    // db_H = column sums of gH: 8 lanes per unit, each over a contiguous
    // run of rows (independent loads), then a fixed xor tree (h <= 64 = nt/8)
    const int o = tid >> 3, part = tid & 7, per = (B + 7) >> 3;
    const int b0 = part * per, b1 = b0 + per < B ? b0 + per : B;
    float acc = 0.f;
    if (o < h)
#pragma unroll 4
      for (int b = b0; b < b1; ++b) acc += G[b * sH + o];
    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (o < h && part == 0) dbH_[o] = acc;
  }
  HPHASE(7);

  // ---- 4: on the tensor cores, one tile pool:
  //         dW_H[:, mine] = gH^T x[:, mine]   (m16 hidden units x 2 n8 columns, K = batch)
  //         dx[:, mine] = gH W_H[:, mine]      (m16 batch rows x 4 n8 columns, K = hidden)
  //         dx *= act_prev'(x) ----
  {
    const int nN = d.Kp >> 3;
    const int ga = (nN + 1) >> 1, na = (d.Hp >> 4) * ga;
    const int gb = (nN + 3) >> 2, nb = dx_ ? (d.Bp >> 4) * gb : 0;
    const int g = lane >> 2, t = lane & 3;
    for (int tile = warp; tile < na + nb; tile += nwarps) {
      if (tile < na) {
        const int im = tile / ga, ig = tile - im * ga;
        const int m0 = im * 16, n0 = ig * 16;
        const int nv = nN - ig * 2 < 2 ? nN - ig * 2 : 2;
        float c[2][4] = {};
        warp_mma<2>(c, G, 1, sH, xr, 1, sK, m0, n0, nv, d.Bp >> 3, lane);
        // column pairs (2t, 2t+1) are adjacent: one 8-byte store when both
        // are in range and the address is 8-byte aligned
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const int o = m0 + g + 8 * hf;
          if (o >= h) continue;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int col = n0 + j * 8 + 2 * t;
            if (j >= nv || col >= nc) continue;
            float* p = dWH_ + (size_t)o * in + k0 + col;
            if (col + 1 < nc && (reinterpret_cast<uintptr_t>(p) & 7) == 0) {
              *reinterpret_cast<float2*>(p) = make_float2(c[j][2 * hf], c[j][2 * hf + 1]);
            } else {
              p[0] = c[j][2 * hf];
              if (col + 1 < nc) p[1] = c[j][2 * hf + 1];
            }
          }
        }
      } else {
        const int u = tile - na, im = u / gb, ig = u - im * gb;
        const int m0 = im * 16, n0 = ig * 32;
        const int nv = nN - ig * 4 < 4 ? nN - ig * 4 : 4;
        float c[4][4] = {};
        warp_mma<4, true>(c, G, sH, 1, wr, 1, sK, m0, n0, nv, d.Hp >> 3, lane);
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const int b = m0 + g + 8 * hf;
          if (b >= B) continue;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int col = n0 + j * 8 + 2 * t;
            if (j >= nv || col >= nc) continue;
            float v0 = c[j][2 * hf], v1 = c[j][2 * hf + 1];
            if (act_prev == VCNN_ACT_RELU) {  // the common case inline
              v0 *= xr[b * sK + col] > 0.f ? 1.f : 0.f;
              v1 *= xr[b * sK + col + 1] > 0.f ? 1.f : 0.f;
            } else if (act_prev != VCNN_ACT_IDENTITY) {
              v0 *= actg(act_prev, xr[b * sK + col]);
              if (col + 1 < nc) v1 *= actg(act_prev, xr[b * sK + col + 1]);
            }
            float* p = dx_ + (size_t)b * in + k0 + col;
            if (col + 1 < nc && (reinterpret_cast<uintptr_t>(p) & 7) == 0) {
              *reinterpret_cast<float2*>(p) = make_float2(v0, v1);
            } else {
              p[0] = v0;
              if (col + 1 < nc) p[1] = v1;
            }
          }
        }
      }
    }
  }
  HPHASE(8);
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

using HeadFn = void (*)(MlpArgs);
// the specialised shape (CIFAR-3: B 128, 5*5*32 -> 64 -> 10) or the generic kernel
static HeadFn head_fn(int B, int in, int h, int out, int loss = -1, int actH = -1, int actO = -1,
                      int act_prev = -1) {
  const bool cifar = in == 800 && h == 64 && out == 10;
  // CIFAR-3's tail: softmax-CE, relu dense conv, identity fc10, relu below
  const bool prof = loss == VCNN_LOSS_SOFTMAX_CE && actH == VCNN_ACT_RELU &&
                    actO == VCNN_ACT_IDENTITY && act_prev == VCNN_ACT_RELU;
  constexpr int CE = VCNN_LOSS_SOFTMAX_CE, RL = VCNN_ACT_RELU, ID = VCNN_ACT_IDENTITY;
  if (cifar && prof && B == 16) return mlp_head_kernel<16, 800, 64, 10, CE, RL, ID, RL>;
  if (cifar && prof && B == 32) return mlp_head_kernel<32, 800, 64, 10, CE, RL, ID, RL>;
  if (cifar && B == 128) return mlp_head_kernel<128, 800, 64, 10>;
  if (cifar && B == 64) return mlp_head_kernel<64, 800, 64, 10>;
  if (cifar && B == 32) return mlp_head_kernel<32, 800, 64, 10>;
  if (cifar && B == 16) return mlp_head_kernel<16, 800, 64, 10>;
  return mlp_head_kernel<0, 0, 0, 0>;
}

// cluster of kC CTAs with this kernel's shared memory schedulable? (cached per kernel)
static bool cluster_ok(HeadFn fn, size_t smem) {
  struct Cache { HeadFn fn; size_t ok_upto, bad_from; };
  static Cache cache[8] = {{nullptr, 0, ~(size_t)0}, {nullptr, 0, ~(size_t)0},
                           {nullptr, 0, ~(size_t)0}, {nullptr, 0, ~(size_t)0},
                           {nullptr, 0, ~(size_t)0}, {nullptr, 0, ~(size_t)0},
                           {nullptr, 0, ~(size_t)0}, {nullptr, 0, ~(size_t)0}};
  Cache* c = &cache[7];
  for (Cache& e : cache)
    if (e.fn == fn || e.fn == nullptr) {
      c = &e;
      break;
    }
  c->fn = fn;
  if (smem <= c->ok_upto) return true;
  if (smem >= c->bad_from) return false;
  bool ok = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                cudaSuccess &&
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) ==
                cudaSuccess;
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
    ok = cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) == cudaSuccess && nclusters > 0;
  }
  cudaGetLastError();
  if (ok) c->ok_upto = smem;
  else c->bad_from = smem;
  return ok;
}

bool mlp_head_fusable(int B, int in, int h, int out) {
  if (B < 1 || B > 128 || h < 1 || h > 64 || out < 1 || out > 64 || in < kC || in > 128 * kC)
    return false;
  const size_t smem = mlp_head_smem(B, in, h, out);
  return smem <= 200 * 1024 && cluster_ok(head_fn(B, in, h, out), smem);
}

int mlp_head_slices(int B, int in, int h, int out) {
  // batch slices (one 16-CTA cluster each) while every slice keeps >= 16
  // rows: each per-row phase shrinks with the slice.  CIFAR-3 b128 (graph
  // replay): 1 slice 19.7 us / 1.22M img/s, 2: 15.5 us / 1.24M, 4: 13.6 us /
  // 1.27M, 8 (16 rows, 128 SMs): 13.4 us / 1.30M
  static const int want = getenv("VCNN_TAIL_SLICES") ? atoi(getenv("VCNN_TAIL_SLICES")) : 8;
  for (int ncl = want < kMaxSlices ? want : kMaxSlices; ncl > 1; ncl /= 2)
    if (B >= 16 * ncl && B % ncl == 0 && mlp_head_fusable(B / ncl, in, h, out)) return ncl;
  return 1;
}

size_t mlp_head_part_floats(int B, int in, int h, int out) {
  const int ncl = mlp_head_slices(B, in, h, out);
  return ncl > 1 ? (size_t)ncl * ((size_t)h * in + h + (size_t)out * h + out) : 0;
}

int launch_mlp_head(int B, int in, int h, int out, const float* x, const float* WH,
                    const float* bH, int actH, const float* WO, const float* bO, int actO,
                    float* yH, float* yO, int loss_kind, const int* cls, const float* values,
                    float* loss, int* err, float* gH, float* gO, float* dWH, float* dbH,
                    float* dWO, float* dbO, float* dx, int act_prev, cudaStream_t st,
                    int ncl, float* part, float* lpart, unsigned* ticket) {
  if (ncl < 1 || B % ncl || (ncl > 1 && (!part || !lpart || !ticket)))
    return fail(VCNN_ECONFIG, "mlp head: bad batch slicing");
  const int Bc = B / ncl;
  const size_t smem = mlp_head_smem(Bc, in, h, out);
  const HeadFn fn = head_fn(Bc, in, h, out, loss_kind, actH, actO, act_prev);
  if (!cluster_ok(fn, smem)) return fail(VCNN_ECUDA, "mlp head: cluster not schedulable");
  const bool vec = in % 4 == 0 && ((reinterpret_cast<uintptr_t>(x) |
                                    reinterpret_cast<uintptr_t>(WH)) & 15) == 0;
  MlpArgs a{Bc, in, h, out, x, WH, bH, actH, WO, bO, actO, yH, yO, loss_kind, cls, values,
            loss, err, gH, gO, dWH, dbH, dWO, dbO, dx, act_prev, vec ? 1 : 0,
            B, ncl, part, lpart, ticket};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kC * ncl);
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
  VCNN_CUDA_TRY(cudaLaunchKernelEx(&cfg, fn, a));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

}  // namespace vcnn_b200
