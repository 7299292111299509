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
  int R, Kc;                  // rows / input columns per CTA
  int Bp, Hp, Kp;             // padded to multiples of 4
  int sB, sK;                 // strides of the [k][b] / [b][k] tiles
  // smem offsets (floats)
  int oxT, owT, oxr, owr, oP, ogT, oW5, ohs, og5, ogl, op5;
  int total;
};

__host__ __device__ inline int up4(int v) { return (v + 3) & ~3; }

__host__ __device__ inline Dims dims_of(int B, int in, int h, int out) {
  Dims d;
  d.B = B; d.in = in; d.h = h; d.out = out;
  d.R = (B + kC - 1) / kC;
  d.Kc = (in + kC - 1) / kC;
  d.Bp = up4(B); d.Hp = up4(h); d.Kp = up4(d.Kc);
  d.sB = d.Bp + 4;            // 16B-aligned rows, staggered banks
  d.sK = d.Kp + 4;
  int o = 0;
  d.oxT = o; o += d.Kp * d.sB;        // x^T  [Kp][sB]
  d.owT = o; o += d.Kp * (d.Hp + 4);  // W_H^T [Kp][Hp+4]
  d.oxr = o; o += d.Bp * d.sK;        // x    [Bp][sK]
  d.owr = o; o += d.Hp * d.sK;        // W_H  [Hp][sK]
  d.oP = o;  o += d.Bp * d.Hp;        // partial x W_H^T [Bp][Hp]; later gH [Bp][Hp]
  d.ogT = o; o += d.Hp * d.sB;        // gH^T [Hp][sB]
  d.oW5 = o; o += out * (h + 1);      // W_O  [out][h+1]
  d.ohs = o; o += d.R * (h + 1);      // h rows [R][h+1]
  d.og5 = o; o += d.R * out;          // y / gO rows [R][out]
  d.ogl = o; o += d.R * d.Hp;         // gH rows [R][Hp] (all-gathered by the cluster)
  d.op5 = o; o += out * (h + 1);      // partial dW_O | db_O [out][h+1]
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
};

__global__ void __launch_bounds__(kThreadsM) mlp_head_kernel(MlpArgs a) {
  PDL_ENTRY();
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const Dims d = dims_of(a.B, a.in, a.h, a.out);
  const int B = a.B, in = a.in, h = a.h, out = a.out;
  const int tid = threadIdx.x, nt = blockDim.x;
  extern __shared__ __align__(16) float sm[];
  float* xT = sm + d.oxT;
  float* wT = sm + d.owT;
  float* xr = sm + d.oxr;
  float* wr = sm + d.owr;
  float* P = sm + d.oP;
  float* gT = sm + d.ogT;
  float* W5 = sm + d.oW5;
  float* hs = sm + d.ohs;
  float* g5 = sm + d.og5;
  float* gl = sm + d.ogl;
  float* p5 = sm + d.op5;
  __shared__ float red[32];
  __shared__ float loss_part;
  const int sW = d.Hp + 4, lh = h + 1;

  // ---- stage: my input columns of x and W_H (zero padded), all of W_O ----
  const int k0 = rank * d.Kc < in ? rank * d.Kc : in;
  const int nc = k0 + d.Kc <= in ? d.Kc : in - k0;
  for (int i = tid; i < d.Bp * d.Kp; i += nt) {
    const int b = i / d.Kp, k = i - b * d.Kp;
    const float v = (b < B && k < nc) ? __ldg(a.x + (size_t)b * in + k0 + k) : 0.f;
    xr[b * d.sK + k] = v;
    xT[k * d.sB + b] = v;
  }
  for (int i = tid; i < d.Hp * d.Kp; i += nt) {
    const int o = i / d.Kp, k = i - o * d.Kp;
    const float v = (o < h && k < nc) ? __ldg(a.WH + (size_t)o * in + k0 + k) : 0.f;
    wr[o * d.sK + k] = v;
    wT[k * sW + o] = v;
  }
  for (int i = tid; i < out * h; i += nt) {
    const int o = i / h, k = i - o * h;
    W5[o * lh + k] = __ldg(a.WO + i);
  }
  __syncthreads();

  // ---- 1: partial P = x[:, mine] W_H[:, mine]^T  ([Bp][Hp], 4x4 tiles) ----
  {
    const int th = d.Hp >> 2, nt1 = (d.Bp >> 2) * th;
    for (int t = tid; t < nt1; t += nt) {
      const int tb = t / th, to = t - tb * th;
      float acc[4][4] = {};
      for (int k = 0; k < d.Kp; ++k) {
        const float4 xv = *reinterpret_cast<const float4*>(xT + k * d.sB + 4 * tb);
        const float4 wv = *reinterpret_cast<const float4*>(wT + k * sW + 4 * to);
        const float xa[4] = {xv.x, xv.y, xv.z, xv.w}, wa[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(xa[i], wa[j], acc[i][j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        *reinterpret_cast<float4*>(P + (4 * tb + i) * d.Hp + 4 * to) =
            make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    }
  }
  cluster.sync();

  // ---- 2: my rows: h = act(sum_c P_c + b), then the last layer + loss ----
  const int r0 = rank * d.R < B ? rank * d.R : B;
  const int nr = r0 + d.R <= B ? d.R : B - r0;
  for (int e = tid; e < nr * h; e += nt) {
    const int b = e / h, o = e - b * h;
    const float* src = P + (r0 + b) * d.Hp + o;
    float acc = 0.f;
    for (int c = 0; c < kC; ++c) acc += *cluster.map_shared_rank(src, c);
    const float v = act_fwd(a.actH, acc + __ldg(a.bH + o));
    hs[b * lh + o] = v;
    a.yH[(size_t)(r0 + b) * h + o] = v;
  }
  __syncthreads();
  for (int e = tid; e < nr * out; e += nt) {
    const int b = e / out, o = e - b * out;
    const float* hr = hs + b * lh;
    const float* wo = W5 + o * lh;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int k = 0;
    for (; k + 3 < h; k += 4) {
      a0 += hr[k] * wo[k];
      a1 += hr[k + 1] * wo[k + 1];
      a2 += hr[k + 2] * wo[k + 2];
      a3 += hr[k + 3] * wo[k + 3];
    }
    for (; k < h; ++k) a0 += hr[k] * wo[k];
    const float v = act_fwd(a.actO, ((a0 + a1) + (a2 + a3)) + __ldg(a.bO + o));
    g5[e] = v;
    a.yO[(size_t)r0 * out + e] = v;
  }
  __syncthreads();
  float mine = 0.f;
  if (a.loss_kind == VCNN_LOSS_SOFTMAX_CE) {
    const float inv_b = 1.0f / (float)B;
    for (int b = tid; b < nr; b += nt) {
      float* l = g5 + b * out;
      const int c = a.cls[r0 + b];
      const bool bad = c < 0 || c >= out;
      if (bad && a.err) atomicExch(a.err, 1);
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
        if (a.actO != VCNN_ACT_IDENTITY) gv *= act_grad_from_out(a.actO, yv);
        l[u] = gv;
      }
    }
  } else {
    const float scale = 2.0f / (float)(B * out);
    const float* vg = a.values + (size_t)r0 * out;
    for (int t = tid; t < nr * out; t += nt) {
      const float yv = g5[t], dd = yv - vg[t];
      mine += dd * dd;
      float gv = scale * dd;
      if (a.actO != VCNN_ACT_IDENTITY) gv *= act_grad_from_out(a.actO, yv);
      g5[t] = gv;
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
  for (int t = tid; t < nr * out; t += nt) a.gO[(size_t)r0 * out + t] = g5[t];
  // partial dW_O | db_O over my rows
  for (int t = tid; t < out * lh; t += nt) {
    const int o = t / lh, i = t - o * lh;
    float acc = 0.f;
    if (i < h)
      for (int b = 0; b < nr; ++b) acc += g5[b * out + o] * hs[b * lh + i];
    else
      for (int b = 0; b < nr; ++b) acc += g5[b * out + o];
    p5[t] = acc;
  }
  // gH rows = (gO W_O) * act_H'(h), zero padded to Hp
  for (int t = tid; t < d.R * d.Hp; t += nt) {
    const int b = t / d.Hp, i = t - b * d.Hp;
    float acc = 0.f;
    if (b < nr && i < h) {
      for (int o = 0; o < out; ++o) acc += g5[b * out + o] * W5[o * lh + i];
      if (a.actH != VCNN_ACT_IDENTITY) acc *= act_grad_from_out(a.actH, hs[b * lh + i]);
      a.gH[(size_t)(r0 + b) * h + i] = acc;
    }
    gl[t] = acc;
  }
  cluster.sync();

  // ---- 3: all-gather gH ([Bp][Hp] into P's space and transposed), reduce
  //         my slice of dW_O | db_O and (rank 0) the loss, in rank order ----
  float* G = P;
  for (int e = tid; e < d.Bp * d.Hp; e += nt) {
    const int b = e / d.Hp, o = e - b * d.Hp;
    float v = 0.f;
    if (b < B) {
      const int c = b / d.R;
      v = *cluster.map_shared_rank(gl + (b - c * d.R) * d.Hp + o, c);
    }
    G[e] = v;
    gT[o * d.sB + b] = v;
  }
  {
    const int np = out * lh, per = (np + kC - 1) / kC;
    const int e0 = rank * per, e1 = e0 + per < np ? e0 + per : np;
    for (int e = e0 + tid; e < e1; e += nt) {
      float acc = 0.f;
      for (int c = 0; c < kC; ++c) acc += *cluster.map_shared_rank(p5 + e, c);
      const int o = e / lh, i = e - o * lh;
      if (i < h) a.dWO[(size_t)o * h + i] = acc;
      else a.dbO[o] = acc;
    }
  }
  if (rank == 0 && tid == 0 && a.loss) {
    float v = 0.f;
    for (int c = 0; c < kC; ++c) v += *cluster.map_shared_rank(&loss_part, c);
    *a.loss = a.loss_kind == VCNN_LOSS_SOFTMAX_CE ? v / (float)B : v / (float)(B * out);
  }
  __syncthreads();

  // ---- 4a: dW_H[:, mine] = gH^T x[:, mine]  ([Hp][Kp]); db_H on rank 0 ----
  {
    const int tk = d.Kp >> 2, nt4 = (d.Hp >> 2) * tk;
    for (int t = tid; t < nt4; t += nt) {
      const int to = t / tk, tc = t - to * tk;
      float acc[4][4] = {};
      for (int b = 0; b < d.Bp; ++b) {
        const float4 gv = *reinterpret_cast<const float4*>(G + b * d.Hp + 4 * to);
        const float4 xv = *reinterpret_cast<const float4*>(xr + b * d.sK + 4 * tc);
        const float ga[4] = {gv.x, gv.y, gv.z, gv.w}, xa[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(ga[i], xa[j], acc[i][j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int o = 4 * to + i;
        if (o >= h) break;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (4 * tc + j < nc) a.dWH[(size_t)o * in + k0 + 4 * tc + j] = acc[i][j];
      }
    }
    if (rank == 0)
      for (int o = tid; o < h; o += nt) {
        float acc = 0.f;
        for (int b = 0; b < B; ++b) acc += G[b * d.Hp + o];
        a.dbH[o] = acc;
      }
  }
  // ---- 4b: dx[:, mine] = (gH W_H[:, mine]) * act_prev'(x)  ([Bp][Kp]) ----
  if (a.dx) {
    const int tk = d.Kp >> 2, nt4 = (d.Bp >> 2) * tk;
    for (int t = tid; t < nt4; t += nt) {
      const int tb = t / tk, tc = t - tb * tk;
      float acc[4][4] = {};
      for (int o = 0; o < d.Hp; ++o) {
        const float4 gv = *reinterpret_cast<const float4*>(gT + o * d.sB + 4 * tb);
        const float4 wv = *reinterpret_cast<const float4*>(wr + o * d.sK + 4 * tc);
        const float ga[4] = {gv.x, gv.y, gv.z, gv.w}, wa[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(ga[i], wa[j], acc[i][j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int b = 4 * tb + i;
        if (b >= B) break;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = 4 * tc + j;
          if (c >= nc) continue;
          float v = acc[i][j];
          if (a.act_prev != VCNN_ACT_IDENTITY)
            v *= act_grad_from_out(a.act_prev, xr[b * d.sK + c]);
          a.dx[(size_t)b * in + k0 + c] = v;
        }
      }
    }
  }
  cluster.sync();  // no CTA leaves while its shared memory is being read
}

}  // namespace

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
  if (B < 1 || B > 128 || h < 1 || h > 64 || out < 1 || out > 64 || in < kC || in > 64 * kC)
    return false;
  const size_t smem = mlp_head_smem(B, in, h, out);
  return smem <= 200 * 1024 && cluster_ok(smem);
}

int launch_mlp_head(int B, int in, int h, int out, const float* x, const float* WH,
                    const float* bH, int actH, const float* WO, const float* bO, int actO,
                    float* yH, float* yO, int loss_kind, const int* cls, const float* values,
                    float* loss, int* err, float* gH, float* gO, float* dWH, float* dbH,
                    float* dWO, float* dbO, float* dx, int act_prev, cudaStream_t st) {
  const size_t smem = mlp_head_smem(B, in, h, out);
  if (!cluster_ok(smem)) return fail(VCNN_ECUDA, "mlp head: cluster not schedulable");
  MlpArgs a{B, in, h, out, x, WH, bH, actH, WO, bO, actO, yH, yO, loss_kind, cls, values,
            loss, err, gH, gO, dWH, dbH, dWO, dbO, dx, act_prev};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kC);
  cfg.blockDim = dim3(kThreadsM);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
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
