// direct.cu -- stride-1 convolution forward and data-gradient as "shifted
// view" implicit GEMMs on the sm_100a tensor cores (tcgen05, TF32).
//
// Output positions of a tile are R rows of a super-grid of width Wg (the
// input width for the forward, W+kw-1 for dgrad), i.e. 128 consecutive
// linear positions q.  For a kernel offset (ky,kx) the A operand of the
// GEMM -- A[q][c] = in[c][q + ky*Wg + kx] -- is the staged input slab
// itself: the slab is laid out [channel group of 8][half][position][4
// channels], 16 bytes per position, and read through a no-swizzle K-major
// descriptor whose 8-row core matrices are 8 consecutive positions (SBO =
// 128 B) and whose two K halves are LBO apart.  A shift of the view by
// ky*Wg+kx positions is just +16 bytes per position on the start address.
// B (weights, K-major, 8 channels per MMA) arrives prepacked in exactly its
// shared-memory image (pack_weights) with one TMA bulk copy.  No im2col is
// ever built: after staging, ONE thread issues kh*kw*ceil(C/8) MMAs
// (M=128, N=BN, K=8) back to back into a TMEM accumulator.
//
// Positions whose column is past the valid output width (x >= OW) are
// computed and discarded -- the price of a uniform descriptor stride.
//
// Forward epilogue: bias + activation, NCHW store, optional fused
// non-overlapping max pool (window == stride; strict >, ties -> lowest
// index; int32 global argmax) -- conv_forward + pool_forward,
// layers.hpp:139-149, vectorize.hpp:197-210, tensor.hpp:271-289.
// dgrad: dX = conv(Gpad, flip(W)^T) over the zero-padded gradient; the
// gradient may be routed on the fly from a fused pool (GradSrc), epilogue
// multiplies the upstream activation derivative -- conv_backward_core dX
// (layers.hpp:179) + apply_activation_grad (layers.hpp:57-61).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "image_sum.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace vcnn_b200 {
namespace direct {

namespace {

constexpr int NT = 256;  // 8 warps: warp w drains TMEM lane quadrant w % 4, column half w / 4
constexpr int BM = 128;
constexpr int EPS = BM + 1;  // epilogue tile row stride (floats): conflict-free per-map reads
constexpr size_t kSmemOptin = 227 * 1024;

struct Geo {
  int mode;                // 0 forward, 1 dgrad
  int B;
  int Cin, Hin, Win;       // staged planes: fwd x [B][C][H][W]; dgrad G [B][K][OH][OW]
  int Cout;                // GEMM N: fwd K maps; dgrad C channels
  int kh, kw;
  int Wg;                  // super-grid row width
  int Hout, Wout;          // valid outputs per image
  int pad_y, pad_x;        // input origin inside the super-grid
  int R, tpi;              // output rows per tile, tiles per image
  int CG, NP;              // channel groups of 8; staged positions
  int BN, nblk;            // N tile, N blocks
  int off_b, off_raw, off_win, off_a, smem;  // shared-memory layout (bytes)
  int off_yp;              // dgrad: the image's yprev planes (act' in the epilogue), -1: none
  int raw_n, win_n;        // floats: raw input image, window scratch (routed dgrad)
  int tma;                 // 1: the slab arrives by ONE tensor TMA from a tf32 NHWC copy
  int rows;                // tma: staged super-grid rows (NP = rows * Wg)
  int wchunk, nbuf;        // weights streamed in chunks of SC shifts: bytes per chunk, ring depth
  int SC, nchunk;          // shifts (ky,kx) per chunk, chunks
  int seg, nseg, segw;     // 1-D row segments (kh == 1, rows wider than a tile): segments
                           // per output row, outputs per segment
  int ts, T, ngx, NM;      // tap-stacked tile (Cout <= 32): the MMA's M rows are T taps x 32
                           // maps of one kernel row (ngx groups per row), N = NM positions
  int ns;                  // N-stacked 1-D segments: the MMA's N = T taps x Cout maps
  int gbuild;              // 2-D tile slab built straight from global (image too big to stage)
  int rf, kh0;             // row fold (single-channel forward): MMA channel j = input row
                           // offset j of an 8-row kernel band; kh0 = the unfolded kernel height
  int eps, off_ep;         // epilogue staging: row stride (floats), offset (bytes)
  int bsx;                 // stacked: bytes between the staged tap blocks (incl. the +1 shift)
};

// kernel "shifts" the MMA loop walks: taps, or tap groups in the stacked mode
__host__ __device__ inline int nshift(const Geo& g) {
  return g.ts || g.ns ? g.kh * g.ngx : g.kh * g.kw;
}

// the tap-stacked mode can be switched off (VCNN_TAPSTACK=0) for A/B runs
inline bool tapstack_enabled() {
  static const bool on = [] {
    const char* e = getenv("VCNN_TAPSTACK");
    return !(e && e[0] == '0');
  }();
  return on;
}

// pack layout per N block: [s = ky*kw+kx][cg][BN/8][2][8][4] (K-major
// no-swizzle core matrices: LBO = 128 B between the two 4-channel halves,
// SBO = 256 B between 8-row groups)
__host__ __device__ inline int64_t pack_floats_per_block(const Geo& g) {
  return (int64_t)nshift(g) * g.CG * g.BN * 8;
}

// bytes of pack chunk c (the last chunk may hold fewer shifts)
__host__ __device__ inline uint32_t chunk_bytes(const Geo& g, int c) {
  const int s1 = (c + 1) * g.SC < nshift(g) ? (c + 1) * g.SC : nshift(g);
  return (uint32_t)((s1 - c * g.SC) * g.CG * g.BN * 32);
}

// tap-stacked plan (see plan()): g.Cin/Hin/.../Wg already set
bool plan_ts(const ConvDesc& d, int mode, int pool, int POH, int POW, Geo& g, int tma) {
  if (tma) return false;  // (the stacked tile builds its own slab)
  constexpr int kMaxN = 256;
  g.ts = 1;
  g.T = 4;
  g.ngx = (int)cdiv(g.kw, g.T);
  int R = (kMaxN - (g.T - 1)) / g.Wg;  // positions R*Wg + T-1 <= 256 (one MMA N)
  if (R > g.Hout) R = g.Hout;
  // at least two row tiles per image with a 2-deep weight ring, so two CTAs
  // share an SM and one's MMAs overlap the other's staging / epilogue
  // (CIFAR-3 conv2 fwd b128: 12.6 us vs 13.2 us for one whole-image tile
  // with a 3-deep ring and 14.5 us unstacked)
  if (g.Hout >= 4) {
    int half = (g.Hout + 1) / 2;
    if (pool && mode == 0) half = (int)cdiv(half, pool) * pool;  // whole pool windows
    if (R > half) R = half;
  }
  const int nt = (int)cdiv(g.Hout, R);
  if (pool && mode == 0) {
    R = (R / pool) * pool;
    if (R < 1) return false;
    R = pool * (int)cdiv(cdiv(g.Hout, pool), cdiv(g.Hout, R));
  } else {
    R = (int)cdiv(g.Hout, nt);
  }
  g.R = R;
  g.tpi = (int)cdiv(g.Hout, R);
  g.CG = (int)cdiv(g.Cin, 8);
  g.NM = (int)cdiv(R * g.Wg + g.T - 1, 16) * 16;
  if (g.NM > kMaxN) return false;
  const int maxsh = (g.kh - 1) * g.Wg + (g.ngx - 1) * g.T;
  g.NP = (int)cdiv(maxsh + g.NM, 8) * 8;
  if ((g.Cin * g.Hin * g.Win) % 4 != 0) return false;
  if (pool && mode == 1 && (d.K * POH * POW) % 4 != 0) return false;
  g.raw_n = g.Cin * g.Hin * g.Win;
  if (mode == 1) g.win_n = ((d.K * ((d.OH + 1) / 2) * ((d.OW + 1) / 2)) + 3) & ~3;
  const int a_bytes = g.CG * 2 * g.NP * 16 + 4 * g.NP;
  const int raw_bytes = 4 * g.raw_n;
  const int win_bytes = 2 * 4 * g.win_n;
  if (raw_bytes > 96 * 1024) return false;
  g.BN = BM;  // pack rows: T taps x 32 maps
  g.nblk = 1;
  g.SC = g.ngx;  // one kernel row of tap groups per chunk
  g.nchunk = g.kh;
  g.wchunk = g.ngx * g.CG * g.BN * 32;
  g.eps = g.NM + 1;  // odd: conflict-free per-lane rows
  g.bsx = 4 * (32 * g.eps + 1);
  const int ep_bytes = 4 * 32 * g.eps * 4;
  const int yp_floats = mode == 1 ? g.Cout * g.Hout * g.Wout : 0;
  const int yp_bytes = (yp_floats % 4 == 0 && 4 * yp_floats <= 48 * 1024) ? 4 * yp_floats : 0;
  for (int nbuf = g.nchunk >= 2 ? 2 : g.nchunk; nbuf >= 1; --nbuf) {
    const int b_bytes = nbuf * g.wchunk;
    const int body = b_bytes + raw_bytes + win_bytes + a_bytes;
    int total = (body > ep_bytes ? body : ep_bytes) + 1024;
    const bool stage_yp = yp_bytes && (size_t)(total + yp_bytes) + 512 <= kSmemOptin;
    const int off_yp = total - 1024;
    if (stage_yp) total += yp_bytes;
    if ((size_t)total + 512 > kSmemOptin) continue;
    g.nbuf = nbuf;
    g.off_b = 0;
    g.off_raw = b_bytes;
    g.off_win = g.off_raw + raw_bytes;
    g.off_a = g.off_win + win_bytes;
    g.off_ep = 0;  // over the ring, raw, windows and slab (all dead by then)
    g.off_yp = stage_yp ? off_yp : -1;
    g.smem = total;
    return (int64_t)g.B * g.tpi < (1 << 24);
  }
  return false;
}

// N-stacked 1-D row segments (deconv-121's 1x121 layer): the MMA's N rows
// are T consecutive taps x Cout maps (the pack, T*Cout <= 256), M = the 128
// positions of a row segment (the slab, viewed at the group's first tap).
// Accumulator column block j at row p holds tap gi*T+j's products for output
// p - j, so a segment yields 128 - (T-1) outputs and the epilogue reads
// out[n][o] = sum_j S[j*Cout + n][o + j] in j order.  Per MMA: 4 KB of slab +
// T*Cout*32 B of weights for T*Cout*128*8 MACs, vs T MMAs of N = Cout each
// issued one at a time (the single-thread issue loop, ~50 cycles per MMA,
// bounds the unstacked 1-D kernel)
bool plan_ns(const ConvDesc& d, int mode, Geo& g) {
  int T = 256 / g.Cout;
  if (T > 8) T = 8;
  if (T > g.kw) T = g.kw;
  if (T < 2) return false;
  g.ns = 1;
  g.T = T;
  g.ngx = (int)cdiv(g.kw, T);
  const int NB = (int)cdiv(T * g.Cout, 16) * 16;
  g.R = 1;
  g.nseg = (int)cdiv(g.Wout, BM - (T - 1));
  g.segw = (int)cdiv(g.Wout, g.nseg);
  g.tpi = g.Hout * g.nseg;
  g.CG = (int)cdiv(g.Cin, 8);
  g.NP = (int)cdiv((g.ngx - 1) * T + BM, 8) * 8;
  g.raw_n = g.Cin * g.Hin * g.Win;
  const int a_bytes = g.CG * 2 * g.NP * 16;
  g.BN = NB;
  g.nblk = 1;
  g.eps = EPS;
  g.bsx = 4 * (g.Cout * EPS + 1);
  const int shift_bytes = g.CG * NB * 32;  // one tap group
  g.SC = (int)std::max<int64_t>(1, (40 * 1024) / shift_bytes);
  if (g.SC > g.ngx) g.SC = g.ngx;
  g.nchunk = (int)cdiv(g.ngx, g.SC);
  g.wchunk = g.SC * shift_bytes;
  const int ep_bytes = NB * EPS * 4;
  for (int nbuf = g.nchunk >= 3 ? 3 : g.nchunk; nbuf >= 1; --nbuf) {
    const int b_bytes = nbuf * g.wchunk;
    const int body = b_bytes + a_bytes;
    const int total = (body > ep_bytes ? body : ep_bytes) + 1024;
    if ((size_t)total + 512 > kSmemOptin) continue;
    g.nbuf = nbuf;
    g.off_b = 0;
    g.off_raw = b_bytes;
    g.off_win = b_bytes;
    g.off_a = b_bytes;
    g.off_ep = 0;  // over the ring and the slab (dead by then)
    g.off_yp = -1;
    g.smem = total;
    return (int64_t)g.B * g.tpi < (1 << 24);
  }
  return false;
}

bool plan(const ConvDesc& d, int mode, int pool, int POH, int POW, Geo& g, int tma = 0) {
  g = Geo{};
  if (d.s != 1) return false;
  g.mode = mode;
  g.B = d.B;
  g.kh = d.kh;
  g.kw = d.kw;
  if (mode == 0) {
    g.Cin = d.C, g.Hin = d.H, g.Win = d.W, g.Cout = d.K;
    g.Wg = d.W, g.Hout = d.OH, g.Wout = d.OW, g.pad_y = 0, g.pad_x = 0;
  } else {
    g.Cin = d.K, g.Hin = d.OH, g.Win = d.OW, g.Cout = d.C;
    g.Wg = d.W + d.kw - 1, g.Hout = d.H, g.Wout = d.W, g.pad_y = d.kh - 1, g.pad_x = d.kw - 1;
  }
  if (g.Hout < 1) return false;
  if (g.Wg > BM) {
    // rows wider than a tile: a 1-D kernel (kh == 1, e.g. the 1x121 layer of
    // the deconvolution net) tiles each output row into segments of <= 128
    // positions; the slab is the row segment plus the kw-1 halo, staged
    // straight from global memory
    if (d.kh != 1 || pool || tma || g.Wg > 4096) return false;
    g.seg = 1;
    if (tapstack_enabled() && g.Cout <= 128 && g.kw >= 8 && (mode == 1 || g.Cin >= 4) &&
        plan_ns(d, mode, g))
      return true;
    g = Geo{g.mode, g.B, g.Cin, g.Hin, g.Win, g.Cout, g.kh, g.kw, g.Wg, g.Hout, g.Wout,
            g.pad_y, g.pad_x};
    g.seg = 1;
  }
  g.kh0 = g.kh;
  // single-channel forward with a tall kernel (denoise-16's 16x16 first
  // layer): fold 8 kernel rows into the MMA's 8 channels -- channel j of slab
  // position (y, x) is the image at (y + j, x), a folded tap (ky', kx) sits
  // 8*ky' rows down -- so K = 8 carries 8 real products instead of 1
  if (mode == 0 && g.Cin == 1 && g.kh >= 8 && !g.seg && !tma) {
    g.rf = 8;
    g.Cin = 8;
    g.kh = (int)cdiv(g.kh0, 8);
  }
  // a forward view with < 4 input channels pads the MMA K (8 channels) by 2x
  // or more; those layers go to the small-Kd kernel or the generic implicit GEMM
  if (mode == 0 && g.Cin < 4) return false;
  // tap-stacked tiles (a function of the conv alone, so every variant of a
  // layer -- pooled, routed, packed -- agrees on the pack layout): when the
  // output has <= 32 maps an M=128 MMA over positions x maps reads 4 KB of A
  // for 32 columns of N; instead the M rows are 4 taps x 32 maps (weights)
  // and N = up to 256 positions (the slab), ~4x less operand traffic per MAC
  // (scripts/micro/mma_issue.cu: an M=128 K=8 tf32 MMA costs ~32 + N/4
  // cycles -- its shared-memory operand reads)
  if (tapstack_enabled() && mode == 0 && !g.seg && !g.rf && g.Cout <= 32 && g.kw >= 3 &&
      g.Wg <= 63 && d.kd() >= 32)
    return plan_ts(d, mode, pool, POH, POW, g, tma);
  g.eps = EPS;
  int R = g.seg ? 1 : BM / g.Wg;
  if (R > g.Hout) R = g.Hout;
  if (g.seg) {
    g.nseg = (int)cdiv(g.Wout, BM);
    g.segw = (int)cdiv(g.Wout, g.nseg);
  } else if (pool && mode == 0) {  // the forward epilogue pools whole windows of its tile
    R = (R / pool) * pool;
    if (R < 1) return false;
    // balanced: as few tiles as before, window rows spread evenly over them
    const int nt = (int)cdiv(g.Hout, R);
    R = pool * (int)cdiv(cdiv(g.Hout, pool), nt);
  } else {  // (a routed dgrad stages the whole gradient image: any row tiling)
    R = (int)cdiv(g.Hout, cdiv(g.Hout, R));  // balanced row blocks
  }
  g.R = R;
  g.tpi = (int)cdiv(g.Hout, R) * (g.seg ? g.nseg : 1);
  g.CG = (int)cdiv(g.Cin, 8);
  const int ystep = g.rf ? g.rf : 1;  // image rows per (folded) kernel row
  const int maxsh = g.seg ? g.kw - 1 : (g.kh - 1) * ystep * g.Wg + g.kw - 1;
  g.NP = (int)cdiv(maxsh + BM, 8) * 8;
  if (tma) {
    // the tensor map box [2*CG quads][rows][Wg][4 channels] is the slab itself
    // (positions P = row * Wg + x, out-of-image positions zero-filled by TMA)
    if (mode == 1 && pool) return false;  // a routed gradient is scattered in smem
    if (g.Cin % 4 || g.Wg > 256 || 2 * g.CG > 256) return false;
    g.tma = 1;
    g.rows = (int)cdiv(maxsh + BM, g.Wg);
    if (g.rows > 256) return false;
    g.NP = g.rows * g.Wg;
  }
  g.raw_n = (g.rf ? 1 : g.Cin) * g.Hin * g.Win;
  // an image too big to stage whole (e.g. denoise-16's 64 x 49 x 49 maps):
  // each tile builds its slab straight from global memory (not for a routed
  // data gradient, which scatters into the staged image)
  if (!g.tma && !g.seg && 4 * g.raw_n > 96 * 1024) {
    if ((mode == 1 && pool) || g.rf) return false;
    g.gbuild = 1;
  }
  // the input image and the window arrays go in with single bulk copies
  if (!g.seg && !g.gbuild && g.raw_n % 4 != 0) return false;
  if (pool && mode == 1 && (d.K * POH * POW) % 4 != 0) return false;
  // dgrad always reserves window scratch for a >= 2x2 pool, so the routed
  // and unrouted plans (and the weight pack) share one BN
  if (mode == 1 && !g.seg && !g.gbuild) g.win_n = ((d.K * ((d.OH + 1) / 2) * ((d.OW + 1) / 2)) + 3) & ~3;
  const bool staged = !(g.tma || g.seg || g.gbuild);
  const int a_bytes = g.CG * 2 * g.NP * 16 + (staged ? (g.rf ? 8 : 4) * g.NP : 0);  // slab + table(s)
  const int raw_bytes = staged ? 4 * g.raw_n : 0;
  const int win_bytes = 2 * 4 * g.win_n;
  if (raw_bytes > 96 * 1024) return false;
  // dgrad: stage the whole image's yprev (C x H x W) with one bulk copy so
  // the epilogue's activation derivative reads shared memory
  const int yp_floats = mode == 1 && !g.seg ? g.Cout * g.Hout * g.Wout : 0;
  const int yp_bytes = (yp_floats % 4 == 0 && 4 * yp_floats <= 48 * 1024) ? 4 * yp_floats : 0;
  for (int bn = g.Cout > 128 ? 128 : (int)((g.Cout + 15) / 16 * 16); bn >= 16; bn -= 16) {
    // the pack streams through a 2-deep ring of kernel rows (ky) instead of
    // being staged whole: the CTA fits 2-3 times per SM, so one CTA's MMAs
    // overlap the others' staging and epilogues
    const int shift_bytes = g.CG * bn * 32;
    int SC = g.kw;  // one kernel row per chunk, or for a huge 1-D kernel ~30 KB
    if (g.seg) SC = (int)std::max<int64_t>(1, (30 * 1024) / shift_bytes);
    if (SC > g.kh * g.kw) SC = g.kh * g.kw;
    const int nchunk = (int)cdiv(g.kh * g.kw, SC);
    const int wchunk = SC * shift_bytes;
    const int nbuf = nchunk >= 2 ? 2 : 1;  // (a 3-deep ring: dgrad drops to 1 CTA/SM, 19.5 -> 33 us)
    const int b_bytes = nbuf * wchunk;
    // the epilogue tile [bn][128] reuses raw + window + A (all dead by then)
    const int ep_bytes = bn * EPS * 4;
    const int tail = raw_bytes + win_bytes + a_bytes > ep_bytes ? raw_bytes + win_bytes + a_bytes
                                                                : ep_bytes;
    int total = b_bytes + tail + 1024;
    const bool stage_yp = yp_bytes && (size_t)(total + yp_bytes) + 512 <= kSmemOptin;
    if (stage_yp) total += yp_bytes;
    if ((size_t)total + 512 <= kSmemOptin) {
      g.BN = bn;
      g.wchunk = wchunk;
      g.nbuf = nbuf;
      g.SC = SC;
      g.nchunk = nchunk;
      g.nblk = (int)cdiv(g.Cout, bn);
      g.off_b = 0;
      g.off_raw = b_bytes;
      g.off_win = g.off_raw + raw_bytes;
      g.off_a = g.off_win + win_bytes;  // (tma: == off_raw, the epilogue tile reuses the slab)
      g.off_ep = g.off_raw;
      g.off_yp = stage_yp ? b_bytes + tail : -1;
      g.smem = total;
      return (int64_t)g.B * g.tpi < (1 << 24);
    }
  }
  return false;
}

__global__ void pack_kernel(Geo g, int mode, const float* __restrict__ w, float* __restrict__ pk) {
  PDL_ENTRY();
  // w: [K][C][kh][kw] (conv weights).  fwd rows = maps n, channels = c;
  // dgrad rows = channels c, channels = maps n, kernel flipped.
  const int64_t per = pack_floats_per_block(g), total = per * g.nblk;
  const int Cch = mode == 0 ? g.Cin : g.Cout;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int nb = (int)(i / per);
    int64_t r = i - nb * per;
    const int k4 = (int)(r & 3), r8 = (int)((r >> 2) & 7), kh2 = (int)((r >> 5) & 1);
    r >>= 6;
    const int rg = (int)(r % (g.BN / 8));
    r /= (g.BN / 8);
    const int cg = (int)(r % g.CG);
    const int s = (int)(r / g.CG);
    const int row = nb * g.BN + rg * 8 + r8;  // GEMM N index
    const int ch = cg * 8 + kh2 * 4 + k4;     // GEMM K index (input channel of the view)
    float v = 0.f;
    // tap-stacked: pack row = j * 32 + map (ts) or j * Cout + map (ns),
    // shift = ky * ngx + gx, tap kx = gx * T + j
    const int jb = g.ts ? (row >> 5) : g.ns ? row / g.Cout : 0;
    const int prow = g.ts ? (row & 31) : g.ns ? row - jb * g.Cout : row;
    const int ky = g.ts || g.ns ? s / g.ngx : s / g.kw;
    const int kx = g.ts || g.ns ? (s - ky * g.ngx) * g.T + jb : s - ky * g.kw;
    if (prow < g.Cout && ch < g.Cin && kx < g.kw && jb < (g.ns ? g.T : 4)) {
      const int row = prow;
      if (g.rf) {  // folded: channel ch = row offset inside the 8-row band ky
        const int wy = ky * g.rf + ch;
        if (wy < g.kh0) v = ptx::to_tf32(w[((int64_t)row * g.kh0 + wy) * g.kw + kx]);
      } else {
        const int n = mode == 0 ? row : ch, c = mode == 0 ? ch : row;
        const int wy = mode == 0 ? ky : g.kh - 1 - ky, wx = mode == 0 ? kx : g.kw - 1 - kx;
        v = ptx::to_tf32(w[(((int64_t)n * Cch + c) * g.kh + wy) * g.kw + wx]);
      }
    }
    pk[i] = v;
  }
}

template <int ACT>
__device__ __forceinline__ float actf(float x) {
  if (ACT == VCNN_ACT_RELU) return x > 0.f ? x : 0.f;
  if (ACT == VCNN_ACT_SIGMOID) return 1.f / (1.f + expf(-x));
  if (ACT == VCNN_ACT_TANH) return tanhf(x);
  return x;
}

struct FwdEpi {
  const float* bias;
  int act;
  float* y;  // nullable when pooled
  int pool, POH, POW;
  float* py;
  int32_t* parg;
};
struct BwdEpi {
  float* dx;
  const float* yprev;
  int act_prev;
};

struct alignas(64) Args {
  CUtensorMap tmap;    // tma mode: the NHWC tf32 input, dims (4, W, H, C/4, B)
  Geo g;
  const float* in;     // x (fwd) or materialised G (dgrad), NCHW
  GradSrc gs;          // dgrad: routed gradient (gs.pool)
  const float* pack;   // prepacked B
  FwdEpi fe;
  BwdEpi be;
};

// one accumulator value at staging address e: plain, or (tap-stacked, ts /
// ns) the sum of the T tap blocks, block j one column further -- fixed order
template <bool TS>
__device__ __forceinline__ float epv(uint32_t e, const Geo& g) {
  if constexpr (!TS) {
    return ptx::lds_f32(e);
  } else {
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      v[j] = j < g.T ? ptx::lds_f32(e + (uint32_t)j * (uint32_t)g.bsx) : 0.f;
    float s = v[0];
#pragma unroll
    for (int j = 1; j < 8; ++j)
      if (j < g.T) s += v[j];
    return s;
  }
}

// Epilogues read the accumulator tile ep[n][128] (position m = r*Wg + x) from
// shared memory.  Work is spread warp = output row, lane = column, loop =
// map, so no thread divides by a runtime extent; stores along a row are
// coalesced.
template <int ACT, bool TS>
__device__ void fwd_epilogue(const Args& a, uint32_t eb, int b, int r0, int n0, int x0) {
  const Geo& g = a.g;
  const FwdEpi& e = a.fe;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nr = g.Hout - r0 < g.R ? g.Hout - r0 : g.R;
  const int nmaps = g.Cout - n0 < g.BN ? g.Cout - n0 : g.BN;
  const int64_t ohw = (int64_t)g.Hout * g.Wout;
  const int64_t plane0 = (int64_t)b * g.Cout + n0;
  // output columns [x0, x1) of the tile; accumulator row = r * Wg + x - x0
  const int x1 = g.seg ? (x0 + g.segw < g.Wout ? x0 + g.segw : g.Wout) : g.Wout;
  if (e.y) {
    for (int r = warp; r < nr; r += NT / 32)
      for (int x = x0 + lane; x < x1; x += 32) {
        float* yp = e.y + plane0 * ohw + (int64_t)(r0 + r) * g.Wout + x;
        const uint32_t ep = eb + 4u * (r * g.Wg + x - x0);
#pragma unroll 4
        for (int n = 0; n < nmaps; ++n)
          yp[n * ohw] = actf<ACT>(epv<TS>(ep + 4u * (n * g.eps), g) + __ldg(e.bias + n0 + n));
      }
  }
  if (e.pool) {
    const int p = e.pool;
    int nwr = (r0 + nr) / p - r0 / p;  // complete window rows of this tile
    if (r0 / p + nwr > e.POH) nwr = e.POH - r0 / p;
    const int64_t pplane = (int64_t)e.POH * e.POW;
    // lane = map (window loop per warp): all lanes busy for narrow pools
    const int nwin = nwr * e.POW;
    for (int n = lane; n < nmaps; n += 32) {
      const float bn_ = __ldg(e.bias + n0 + n);
      const uint32_t en = eb + 4u * (n * g.eps);
      int wr = 0, wc = warp;
      while (wc >= e.POW) {
        wc -= e.POW;
        ++wr;
      }
      for (int w = warp; w < nwin; w += NT / 32) {
        {
          const int ry = wr * p, cx = wc * p;
          const int64_t o0 = plane0 * pplane + (int64_t)(r0 / p + wr) * e.POW + wc;
          float best = actf<ACT>(epv<TS>(en + 4u * (ry * g.Wg + cx), g) + bn_);
          int by = 0, bx = 0;
          for (int u = 0; u < p; ++u)
            for (int v = 0; v < p; ++v) {
              const float val = actf<ACT>(epv<TS>(en + 4u * ((ry + u) * g.Wg + cx + v), g) + bn_);
              if (val > best) {
                best = val;
                by = u;
                bx = v;
              }
            }
          e.py[o0 + n * pplane] = best;
          e.parg[o0 + n * pplane] =
              (int32_t)((plane0 + n) * ohw + (int64_t)(r0 + ry + by) * g.Wout + cx + bx);
        }
        wc += NT / 32;  // next window of this warp (row-major over the tile's windows)
        while (wc >= e.POW) {
          wc -= e.POW;
          ++wr;
        }
      }
    }
  }
}

// dgrad epilogue: lane = output position of the tile (coalesced along x),
// warp = channel slice; the yprev loads of 16 (position, channel) pairs are
// in flight together (read-only path).
template <int ACT, bool TS>
__device__ void bwd_epilogue(const Args& a, uint32_t eb, int b, int r0, int n0, int x0) {
  const Geo& g = a.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nr = g.Hout - r0 < g.R ? g.Hout - r0 : g.R;
  const int nch = g.Cout - n0 < g.BN ? g.Cout - n0 : g.BN;
  const int x1 = g.seg ? (x0 + g.segw < g.Wout ? x0 + g.segw : g.Wout) : g.Wout;
  const int wid = x1 - x0;  // output columns of the tile
  const int npix = nr * wid;
  const int64_t hw = (int64_t)g.Hout * g.Wout;
  const int64_t plane0 = (int64_t)b * g.Cout + n0;
  const float* yp = a.be.yprev;
  // yprev staged in shared memory (whole image) when the plan had room
  const bool ys = yp && g.off_yp >= 0;
  const uint32_t s_yp = eb - (uint32_t)g.off_ep + (uint32_t)(g.off_yp < 0 ? 0 : g.off_yp);
  for (int p = lane; p < npix; p += 32) {
    const int r = p / wid, x = x0 + (p - r * wid);
    const int64_t o = plane0 * hw + (int64_t)(r0 + r) * g.Wout + x;
    const uint32_t ep = eb + 4u * (r * g.Wg + x - x0);
    const int lo = (r0 + r) * g.Wout + x;  // offset inside one channel plane
    for (int c0 = warp; c0 < nch; c0 += (NT / 32) * 16) {
      float yv[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int c = c0 + (NT / 32) * u;
        yv[u] = (yp && c < nch)
                    ? (ys ? ptx::lds_f32(s_yp + 4u * (uint32_t)((n0 + c) * (int)hw + lo))
                          : __ldg(yp + o + c * hw))
                    : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int c = c0 + (NT / 32) * u;
        if (c >= nch) break;
        float v = epv<TS>(ep + 4u * (c * g.eps), g);
        if (yp) {
          if (ACT == VCNN_ACT_RELU) v *= yv[u] > 0.f ? 1.f : 0.f;
          else if (ACT == VCNN_ACT_SIGMOID) v *= yv[u] * (1.f - yv[u]);
          else if (ACT == VCNN_ACT_TANH) v *= 1.f - yv[u] * yv[u];
        }
        a.be.dx[o + c * hw] = v;
      }
    }
  }
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

#ifdef VCNN_PHASE_TIMING
__device__ float g_dump[4][256];
__device__ unsigned long long g_dphase[8][8];
#define DPHASE(i)                                                                        \
  do {                                                                                   \
    if (threadIdx.x == 0 && blockIdx.x + blockIdx.y < 8) g_dphase[blockIdx.x + blockIdx.y][i] = clock64(); \
  } while (0)
#else
#define DPHASE(i) \
  do {            \
  } while (0)
#endif

__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, int c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "r"(ptx::smem_u32(bar))
      : "memory");
}

// MODE (0 forward, 1 data gradient) and the epilogue's activation are
// template parameters so each instantiation carries only its own staging /
// MMA / epilogue code (the kernel's instruction footprint is fetched cold once
// per CTA)
template <int TMEM_COLS, int MODE, int ACT>
__global__ void __launch_bounds__(NT, MODE == 1 ? 3 : 1)  // (dgrad: <= 85 registers, 3 CTAs/SM)
    direct_conv_kernel(const __grid_constant__ Args a) {
  pdl_launch_dependents();
  const Geo& g = a.g;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  __shared__ uint64_t load_bar, done_bar, wfull[3], wempty[3];  // ring depth <= 3
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tile = blockIdx.x, nb = blockIdx.y;
  const int b = tile / g.tpi, tt = tile - b * g.tpi;
  const int ry = g.seg ? tt / g.nseg : tt, r0 = ry * g.R;
  const int x0 = g.seg ? (tt - ry * g.nseg) * g.segw : 0;
  const int n0 = nb * g.BN;
  const uint32_t sbase = ptx::smem_u32(smem);
  const uint32_t s_b = sbase + g.off_b, s_raw = sbase + g.off_raw, s_win = sbase + g.off_win,
                 s_a = sbase + g.off_a;
  DPHASE(0);

  if (warp == 0) {
    ptx::tmem_alloc(&tmem_base_sh, TMEM_COLS);
    ptx::tmem_relinquish();
  }
  pdl_wait();  // TMEM allocation above overlapped the previous kernel
  // ---- TMA bulk loads: prepacked B, the input image (or routed windows) ----
  const int64_t pk_per = pack_floats_per_block(g);
  const bool routed = MODE == 1 && a.gs.pool;
  const int wsz = routed ? a.gs.POH * a.gs.POW * g.Cin : 0;
  const float* pack = a.pack + nb * pk_per;
  // the shifts that can touch a valid output of this tile: a 1-D dgrad tile
  // skips the kernel taps whose view of the zero-padded gradient is empty
  // for every valid position (they would add exact zeros) -- 121 -> 92 taps
  // per tile on deconv-121's 1x121 layer; their pack chunks are not loaded
  int s_lo = 0, s_hi = nshift(g) - 1;
  if (g.seg && MODE == 1) {
    const int wid = (x0 + g.segw < g.Wout ? x0 + g.segw : g.Wout) - x0;
    const int lo = g.pad_x - x0 - (wid - 1), hi = g.pad_x - x0 + g.Win - 1;
    s_lo = lo > 0 ? lo : 0;
    s_hi = hi < g.kw - 1 ? hi : g.kw - 1;
    if (s_lo > s_hi) s_lo = s_hi = 0;  // (no tap: one zero MMA keeps the accumulator defined)
    if (g.ns) {  // tap range -> tap-group range
      s_lo /= g.T;
      s_hi /= g.T;
    }
  }
  const int c_lo = s_lo / g.SC, nloc = s_hi / g.SC - c_lo + 1;
  const int nring = nloc < g.nbuf ? nloc : g.nbuf;
  if (tid == 0) {
    ptx::mbar_init(&load_bar, 1);
    ptx::mbar_init(&done_bar, 1);
    for (int i = 0; i < g.nbuf; ++i) {
      ptx::mbar_init(&wfull[i], 1);
      ptx::mbar_init(&wempty[i], 1);
    }
    ptx::fence_mbar_init();
    // the tile's first pack chunks into the ring
    for (int lc = 0; lc < nring; ++lc) {
      const int c = c_lo + lc;
      const uint32_t bytes = chunk_bytes(g, c);
      ptx::mbar_arrive_expect_tx(&wfull[lc], bytes);
      ptx::bulk_g2s(s_b + (uint32_t)(lc * g.wchunk), pack + (int64_t)c * (g.wchunk / 4), bytes,
                    &wfull[lc]);
    }
    if (g.off_yp >= 0 && a.be.yprev) {
      const uint32_t yb = 4u * (uint32_t)(g.Cout * g.Hout * g.Wout);
      ptx::mbar_expect_tx(&load_bar, yb);
      ptx::bulk_g2s(sbase + g.off_yp, a.be.yprev + (int64_t)b * g.Cout * g.Hout * g.Wout, yb,
                    &load_bar);
    }
    if (g.tma) {  // the whole slab, one tensor copy (zero fill outside the image)
      const uint32_t ab = 16u * (uint32_t)(2 * g.CG * g.NP);
      ptx::mbar_expect_tx(&load_bar, ab);
      tma_load_5d(s_a, &a.tmap, 0, -g.pad_x, r0 - g.pad_y, 0, b, &load_bar);
    } else if (g.seg || g.gbuild) {
      // (the row segment / tile is built from global by all threads below)
    } else if (!routed) {
      const uint32_t rb = 4u * (uint32_t)g.raw_n;
      ptx::mbar_expect_tx(&load_bar, rb);
      ptx::bulk_g2s(s_raw, a.in + (int64_t)b * g.raw_n, rb, &load_bar);
    } else {
      const uint32_t wb = 4u * (uint32_t)wsz;
      ptx::mbar_expect_tx(&load_bar, 2 * wb);
      ptx::bulk_g2s(s_win, a.gs.dP + (int64_t)b * wsz, wb, &load_bar);
      ptx::bulk_g2s(s_win + 4u * g.win_n, a.gs.parg + (int64_t)b * wsz, wb, &load_bar);
    }
    ptx::mbar_arrive(&load_bar);
  }
  __syncthreads();
  DPHASE(1);
  if (routed) {  // zero the gradient image while the windows land
    for (int i = tid; i < g.raw_n; i += NT) ptx::sts_f32(s_raw + 4u * i, 0.f);
  }
  ptx::mbar_wait(&load_bar, 0);
  DPHASE(2);
  if (routed) {  // scatter dP (already * act') to the argmax positions
    __syncthreads();
    const int hw = g.Hin * g.Win;
    const int base = (int)((int64_t)b * g.Cin * hw);
    for (int i = tid; i < wsz; i += NT) {
      const int at = ptx::lds_s32(s_win + 4u * (g.win_n + i)) - base;
      ptx::sts_f32(s_raw + 4u * at, ptx::lds_f32(s_win + 4u * i));
    }
    __syncthreads();
  }
  // ---- build the tf32-rounded [cg][half][position][4] slab ----
  // position -> offset in the staged image (-1 outside it), one division per
  // position; then thread -> (position, channel%4), 8 positions x 16 B per
  // 128-byte warp store (conflict-free)
  if (g.seg) {
    // slab position P = input column x0 + P - pad_x of row r0 - pad_y (zero
    // outside the image); thread -> (channel quad, P): 4 coalesced row loads,
    // one 16-byte store
    const int yy = r0 - g.pad_y;
    const int64_t plane = (int64_t)g.Hin * g.Win;
    const float* src = a.in + (int64_t)b * g.Cin * plane + (int64_t)yy * g.Win;
    const bool row_ok = yy >= 0 && yy < g.Hin;
    for (int j = tid; j < 2 * g.CG * g.NP; j += NT) {
      const int cq = j / g.NP, P = j - cq * g.NP;
      const int xx = x0 + P - g.pad_x;
      const bool ok = row_ok && xx >= 0 && xx < g.Win;
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = cq * 4 + u;
        v[u] = (ok && c < g.Cin) ? ptx::to_tf32(__ldg(src + c * plane + xx)) : 0.f;
      }
      ptx::sts_f32x4(s_a + 16u * (uint32_t)j, make_float4(v[0], v[1], v[2], v[3]));
    }
  } else if (g.gbuild) {
    // slab position P = (row r0 + P / Wg - pad_y, column P % Wg - pad_x) of
    // the image in global memory; thread -> (channel quad, P), 4 coalesced
    // loads, one 16-byte store
    const int64_t plane = (int64_t)g.Hin * g.Win;
    const float* src = a.in + (int64_t)b * g.Cin * plane;
    for (int j = tid; j < 2 * g.CG * g.NP; j += NT) {
      const int cq = j / g.NP, P = j - cq * g.NP;
      const int pr = P / g.Wg;
      const int yy = r0 + pr - g.pad_y, xx = P - pr * g.Wg - g.pad_x;
      const bool ok = yy >= 0 && yy < g.Hin && xx >= 0 && xx < g.Win;
      const int64_t off = (int64_t)yy * g.Win + xx;
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = cq * 4 + u;
        v[u] = (ok && c < g.Cin) ? ptx::to_tf32(__ldg(src + c * plane + off)) : 0.f;
      }
      ptx::sts_f32x4(s_a + 16u * (uint32_t)j, make_float4(v[0], v[1], v[2], v[3]));
    }
  } else if (!g.tma) {
    int* pos_off = reinterpret_cast<int*>(smem + g.off_a) + g.CG * 2 * g.NP * 4;
    int* rows_left = pos_off + g.NP;  // (row fold: image rows from the position's row on)
    for (int P = tid; P < g.NP; P += NT) {
      const int yy = r0 + P / g.Wg - g.pad_y, xx = P % g.Wg - g.pad_x;
      pos_off[P] = (yy >= 0 && yy < g.Hin && xx >= 0 && xx < g.Win) ? yy * g.Win + xx : -1;
      if (g.rf) rows_left[P] = g.Hin - yy;
    }
    __syncthreads();
    const uint32_t s_pos = ptx::smem_u32(pos_off);
    // channel stride in the staged image: a plane, or (row fold) one image row
    const int hw = g.rf ? g.Win : g.Hin * g.Win;
    const uint32_t hstride = (uint32_t)g.NP * 16u;  // bytes per (cg, half) block
    // j = (position, channel%4); the channel-group loop inside keeps 4
    // independent loads in flight per thread
    for (int j = tid; j < 4 * g.NP; j += NT) {
      const int off = ptx::lds_s32(s_pos + 4u * (j >> 2));
      const int cmax = g.rf ? ptx::lds_s32(s_pos + 4u * (g.NP + (j >> 2))) : g.Cin;
      const int c4 = j & 3;
      const uint32_t dst = s_a + 4u * j;
      int ch = 0;
      for (; ch + 3 < 2 * g.CG; ch += 4) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = (ch + u) * 4 + c4;
          v[u] = (c < g.Cin && c < cmax && off >= 0) ? ptx::lds_f32(s_raw + 4u * (c * hw + off))
                                                     : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) ptx::sts_f32(dst + (uint32_t)(ch + u) * hstride, ptx::to_tf32(v[u]));
      }
      for (; ch < 2 * g.CG; ++ch) {
        const int c = ch * 4 + c4;
        const float v = (c < g.Cin && c < cmax && off >= 0)
                            ? ptx::lds_f32(s_raw + 4u * (c * hw + off))
                            : 0.f;
        ptx::sts_f32(dst + (uint32_t)ch * hstride, ptx::to_tf32(v));
      }
    }
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
#ifdef VCNN_PHASE_TIMING
  if (blockIdx.x == 0 && blockIdx.y == 0) {
    for (int i = tid; i < 256; i += NT) {
      g_dump[0][i] = ptx::lds_f32(s_raw + 4u * i);
      g_dump[1][i] = ptx::lds_f32(s_a + 4u * i);
      g_dump[2][i] = ptx::lds_f32(s_b + 4u * i);
    }
  }
#endif

  DPHASE(3);
  // ---- one elected lane of warp 0 issues every MMA (converged warp: the
  // tcgen05 issue stays on the uniform datapath) ----
  if (MODE == 0 && g.ts && warp == 0 && ptx::elect_one()) {
    // stacked: A = the pack block of (kernel row ky, tap group gx, channel
    // group) -- 128 rows = 4 taps x 32 maps; B = the slab viewed at the
    // group's first tap (ky * Wg + gx * T), N = NM positions.  Row block j of
    // the accumulator at column n holds tap gx*T+j's products for output
    // position n - j (summed in the epilogue)
    const uint32_t idesc = ptx::idesc_tf32(BM, g.NM);
    const uint32_t half = (uint32_t)g.NP * 16u;
    const uint64_t b0 = ptx::interleave_desc(s_a, half, 128u);
    const uint64_t b_cg = (uint64_t)(2u * half >> 4), a_blk = (uint64_t)(BM * 32 >> 4);
    uint32_t acc = 0;
    for (int lc = 0; lc < nloc; ++lc) {
      const int ky = c_lo + lc, buf = lc % g.nbuf;
      ptx::mbar_wait(&wfull[buf], (uint32_t)(lc / g.nbuf) & 1u);
      ptx::tc_fence_after();
      uint64_t ad = ptx::interleave_desc(s_b + (uint32_t)(buf * g.wchunk), 128u, 256u);
      for (int gx = 0; gx < g.ngx; ++gx) {
        uint64_t bd = b0 + (uint64_t)(ky * g.Wg + gx * g.T);
        for (int cg = 0; cg < g.CG; ++cg) {
          ptx::mma_tf32(tmem, ad, bd, idesc, acc);
          acc = 1;
          ad += a_blk;
          bd += b_cg;
        }
      }
      ptx::mma_commit(&wempty[buf]);
    }
    ptx::mma_commit(&done_bar);
  } else if (g.ns && warp == 0 && ptx::elect_one()) {
    // N-stacked segments: A = the slab at the group's first tap gi*T, B = the
    // pack block of group gi (T taps x Cout maps), one MMA per channel group
    const uint32_t idesc = ptx::idesc_tf32(BM, g.BN);
    const uint32_t half = (uint32_t)g.NP * 16u;
    const uint64_t a0 = ptx::interleave_desc(s_a, half, 128u);
    const uint64_t a_cg = (uint64_t)(2u * half >> 4), b_blk = (uint64_t)(g.BN * 32 >> 4);
    uint32_t acc = 0;
    for (int lc = 0; lc < nloc; ++lc) {
      const int c = c_lo + lc, buf = lc % g.nbuf;
      ptx::mbar_wait(&wfull[buf], (uint32_t)(lc / g.nbuf) & 1u);
      ptx::tc_fence_after();
      const int g0 = c * g.SC > s_lo ? c * g.SC : s_lo;
      const int g1 = (c + 1) * g.SC - 1 < s_hi ? (c + 1) * g.SC - 1 : s_hi;
      uint64_t bd = ptx::interleave_desc(s_b + (uint32_t)(buf * g.wchunk), 128u, 256u) +
                    (uint64_t)(g0 - c * g.SC) * g.CG * b_blk;
      for (int gi = g0; gi <= g1; ++gi) {
        uint64_t ad = a0 + (uint64_t)(gi * g.T);
        for (int cg = 0; cg < g.CG; ++cg) {
          ptx::mma_tf32(tmem, ad, bd, idesc, acc);
          acc = 1;
          ad += a_cg;
          bd += b_blk;
        }
      }
      ptx::mma_commit(&wempty[buf]);
    }
    ptx::mma_commit(&done_bar);
  } else if (!(MODE == 0 && g.ts) && !g.ns && warp == 0 && ptx::elect_one()) {
    const uint32_t idesc = ptx::idesc_tf32(BM, g.BN);  // both operands K-major
    const uint32_t half = (uint32_t)g.NP * 16u;          // LBO: the two 4-channel halves
    // descriptors advance by plain additions on the start-address field
    // (16-byte units): A by the shift and the channel group, B by its block
    const uint64_t a0 = ptx::interleave_desc(s_a, half, 128u);
    const uint64_t a_cg = (uint64_t)(2u * half >> 4), b_blk = (uint64_t)(g.BN * 32 >> 4);
    uint32_t acc = 0;
    int ky = s_lo / g.kw, kx = s_lo - ky * g.kw;  // shift s = ky * kw + kx, incremental
    for (int lc = 0; lc < nloc; ++lc) {
      const int c = c_lo + lc, buf = lc % g.nbuf;
      ptx::mbar_wait(&wfull[buf], (uint32_t)(lc / g.nbuf) & 1u);
      ptx::tc_fence_after();
      const int s0 = c * g.SC > s_lo ? c * g.SC : s_lo;
      const int s1 = (c + 1) * g.SC - 1 < s_hi ? (c + 1) * g.SC - 1 : s_hi;
      uint64_t bd = ptx::interleave_desc(s_b + (uint32_t)(buf * g.wchunk), 128u, 256u) +
                    (uint64_t)(s0 - c * g.SC) * g.CG * b_blk;
      for (int sft = s0; sft <= s1; ++sft) {
        uint64_t ad = a0 + (uint64_t)(ky * (g.rf ? g.rf : 1) * g.Wg + kx);
        for (int cg = 0; cg < g.CG; ++cg) {
          ptx::mma_tf32(tmem, ad, bd, idesc, acc);
          acc = 1;
          ad += a_cg;
          bd += b_blk;
        }
        if (++kx == g.kw) {
          kx = 0;
          ++ky;
        }
      }
      ptx::mma_commit(&wempty[buf]);  // this chunk's pack slot is free once read
    }
    ptx::mma_commit(&done_bar);
  } else if (warp == 1 && ptx::elect_one()) {
    // refill the ring: chunk lc once chunk lc - nbuf's MMAs have read its slot
    for (int lc = g.nbuf; lc < nloc; ++lc) {
      const int c = c_lo + lc, buf = lc % g.nbuf;
      ptx::mbar_wait(&wempty[buf], (uint32_t)((lc - g.nbuf) / g.nbuf) & 1u);
      const uint32_t bytes = chunk_bytes(g, c);
      ptx::mbar_arrive_expect_tx(&wfull[buf], bytes);
      ptx::bulk_g2s(s_b + (uint32_t)(buf * g.wchunk), pack + (int64_t)c * (g.wchunk / 4), bytes,
                    &wfull[buf]);
    }
  }
  __syncwarp();
  if (warp == 0) ptx::mbar_wait(&done_bar, 0);  // the other warps park at the barrier
  __syncthreads();
  ptx::tc_fence_after();
  DPHASE(4);

  // ---- epilogue: TMEM -> smem [n][128] (over raw / window / slab) -> stores ----
  const uint32_t s_ep = sbase + (uint32_t)g.off_ep;
  if (MODE == 0 && g.ts) {
    // warp j holds row block j (tap offset j): stage all four; the epilogue
    // reads out[m][p] = ((S0[m][p] + S1[m][p+1]) + S2[m][p+2]) + S3[m][p+3]
    const int quad = warp & 3;
    const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16);
    const uint32_t srow = s_ep + 4u * (uint32_t)((quad * 32 + lane) * g.eps);
    // the two warps of a lane quadrant take alternate 16-column slices; four
    // loads in flight per wait (the load latency bounds this loop)
    for (int c = 16 * (warp >> 2); c < g.NM; c += 128) {
      uint32_t r[4][16];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (c + 32 * q < g.NM) ptx::tmem_ld16(trow + (uint32_t)(c + 32 * q), r[q]);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (c + 32 * q < g.NM)
#pragma unroll
          for (int jj = 0; jj < 16; ++jj)
            ptx::sts_f32(srow + 4u * (c + 32 * q + jj), __uint_as_float(r[q][jj]));
    }
    ptx::tc_fence_before();
    __syncthreads();
    DPHASE(7);
  } else {
    const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const int row = (warp & 3) * 32 + lane;
    for (int c = 16 * (warp >> 2); c < g.BN; c += 32) {
      uint32_t r[16];
      ptx::tmem_ld16(trow + (uint32_t)c, r);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int jj = 0; jj < 16; ++jj)
        ptx::sts_f32(s_ep + 4u * ((c + jj) * EPS + row), __uint_as_float(r[jj]));
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
#ifdef VCNN_PHASE_TIMING
  if (blockIdx.x == 0 && blockIdx.y == 0)
    for (int i = tid; i < 256; i += NT) g_dump[3][i] = ptx::lds_f32(s_raw + 4u * i);
#endif
  if constexpr (MODE == 0) {
    if (g.ts || g.ns) fwd_epilogue<ACT, true>(a, s_ep, b, r0, n0, x0);
    else fwd_epilogue<ACT, false>(a, s_ep, b, r0, n0, x0);
  } else {
    if (g.ns) bwd_epilogue<ACT, true>(a, s_ep, b, r0, n0, x0);
    else bwd_epilogue<ACT, false>(a, s_ep, b, r0, n0, x0);
  }
  DPHASE(5);
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, TMEM_COLS);
  DPHASE(6);
}

int launch(const Args& a, cudaStream_t st) {
  const Geo& g = a.g;
  dim3 grid((unsigned)(g.B * g.tpi), (unsigned)g.nblk);
  const size_t smem = (size_t)g.smem;
  auto go = [&](auto kern, size_t& configured) -> int {
    if (smem > configured) {
      VCNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
      configured = smem;
    }
    VCNN_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(NT), smem, st, a));
    VCNN_LAUNCHED();
    return VCNN_OK;
  };
  static size_t cfg[2][4][4] = {};  // configured smem per instantiation
  (void)cfg;
  const int act = g.mode == 0 ? a.fe.act : a.be.act_prev;
  auto pick = [&](auto M, auto A) -> int {
    constexpr int MD = decltype(M)::value, AC = decltype(A)::value;
    const int ai = AC == VCNN_ACT_RELU ? 0 : AC == VCNN_ACT_SIGMOID ? 1 : AC == VCNN_ACT_TANH ? 2 : 3;
    if (MD == 0 && g.ts) return go(direct_conv_kernel<256, MD, AC>, cfg[MD][3][ai]);
    if (g.BN <= 32) return go(direct_conv_kernel<32, MD, AC>, cfg[MD][0][ai]);
    if (g.BN <= 64) return go(direct_conv_kernel<64, MD, AC>, cfg[MD][1][ai]);
    if (g.BN <= 128) return go(direct_conv_kernel<128, MD, AC>, cfg[MD][2][ai]);
    return go(direct_conv_kernel<256, MD, AC>, cfg[MD][3][ai]);
  };
  auto by_act = [&](auto M) -> int {
    switch (act) {
      case VCNN_ACT_RELU: return pick(M, std::integral_constant<int, VCNN_ACT_RELU>{});
      case VCNN_ACT_SIGMOID: return pick(M, std::integral_constant<int, VCNN_ACT_SIGMOID>{});
      case VCNN_ACT_TANH: return pick(M, std::integral_constant<int, VCNN_ACT_TANH>{});
      default: return pick(M, std::integral_constant<int, VCNN_ACT_IDENTITY>{});
    }
  };
  return g.mode == 0 ? by_act(std::integral_constant<int, 0>{})
                     : by_act(std::integral_constant<int, 1>{});
}

}  // namespace

bool fwd_ok(const ConvDesc& d, int pool) {
  Geo g;
  return plan(d, 0, pool, 0, 0, g);
}
bool dgrad_ok(const ConvDesc& d, int pool, int POH, int POW) {
  Geo g;
  return plan(d, 1, pool, POH, POW, g);
}
size_t pack_floats(const ConvDesc& d, int mode) {
  Geo g;
  if (!plan(d, mode, 0, 0, 0, g)) return 0;
  return (size_t)(pack_floats_per_block(g) * g.nblk);
}

int pack_weights(const ConvDesc& d, int mode, const float* w, float* pk, cudaStream_t st) {
  Geo g;
  if (!plan(d, mode, 0, 0, 0, g)) return fail(VCNN_ESHAPE, "direct conv: geometry not supported");
  const int64_t n = pack_floats_per_block(g) * g.nblk;
  int64_t blocks = cdiv(n, 256);
  if (blocks > 2 * sm_count()) blocks = 2 * sm_count();
  VCNN_CUDA_TRY(launch_pdl(pack_kernel, dim3((unsigned)blocks), dim3(256), 0, st, g, mode, w, pk));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

// ---- fused SGD + weight packing: one launch per update ---------------------
namespace {
struct PackLayer {
  int64_t w_off, w_len;  // the layer's weight range in the flat params
  Geo gf, gd;            // fwd / dgrad pack geometry (BN, CG, nblk, ...)
  float* pf;
  float* pd;
  float* ps;  // small-Kd forward image [n][wst]
  int wst;
  int K, C, kh, kw;
};
struct PackTable {
  int n;
  PackLayer L[kMaxPackLayers];
};

// offset of (row = GEMM N index, ch = GEMM K index, s = ky*kw+kx) in a pack
__device__ __forceinline__ int64_t pack_index(const Geo& g, int row, int ch, int s) {
  if (g.ts || g.ns) {  // stacked: row (j = kx % T) * (32 | Cout) + row, shift ky * ngx + kx / T
    const int ky = s / g.kw, kx = s - ky * g.kw;
    row += (kx % g.T) * (g.ts ? 32 : g.Cout);
    s = ky * g.ngx + kx / g.T;
  } else if (g.rf) {  // row-folded: channel = ky % 8, folded row ky / 8
    const int ky = s / g.kw, kx = s - ky * g.kw;
    ch = ky % g.rf;
    s = (ky / g.rf) * g.kw + kx;
  }
  const int nb = row / g.BN, r = row - nb * g.BN, cg = ch >> 3, kk = ch & 7;
  return ((((int64_t)nb * nshift(g) + s) * g.CG + cg) * (g.BN / 8) + (r >> 3)) * 64 +
         (kk >> 2) * 32 + (r & 7) * 4 + (kk & 3);
}

// one element of sgd_step with the (already scaled) gradient gi, plus the
// conv weight packs that element feeds
__device__ __forceinline__ void update_pack(int64_t i, float gi, float* __restrict__ w,
                                            float* __restrict__ v, float lr, float mom,
                                            const PackTable& t) {
  const float vi = mom * v[i] + gi;
  const float wi = w[i] - lr * vi;
  v[i] = vi;
  w[i] = wi;
  for (int l = 0; l < t.n; ++l) {
    const PackLayer& L = t.L[l];
    const int64_t k = i - L.w_off;
    if (k < 0 || k >= L.w_len) continue;
    const int khw = L.kh * L.kw, kd = L.C * khw;
    const int k32 = (int)k;  // w_len < 2^31 (checked on the host): 32-bit divisions
    const int nn = k32 / kd, rem = k32 - nn * kd;
    const int c = rem / khw, s = rem - c * khw;
    const float q = ptx::to_tf32(wi);
    if (L.ps) L.ps[nn * L.wst + rem] = q;
    if (L.pf) L.pf[pack_index(L.gf, nn, c, s)] = q;
    if (L.pd) L.pd[pack_index(L.gd, c, nn, khw - 1 - s)] = q;
  }
}

// sgd_step (network.hpp:242-273): v = mom*v + scale*g; w -= lr*v; and the
// updated conv weights are written straight into the direct kernels' packs
// (fwd: row n, channel c, s = ky*kw+kx; dgrad: row c, channel n, flipped s)
__global__ void __launch_bounds__(32 * kRedSlices) sgd_pack_kernel(
    int64_t n, float* __restrict__ w, float* __restrict__ v, float* __restrict__ g, float lr,
    float mom, float scale, const PackTable t, const float* __restrict__ loss,
    int* __restrict__ guard, const ImageSumFold fold, int64_t fold_off, const ImageSumFold fold2,
    int64_t fold2_off, int* __restrict__ ring_step) {
  PDL_ENTRY();
  // the step's batch ring advances (its staging kernel only reads the count)
  if (ring_step && blockIdx.x == 0 && threadIdx.x == 0) *ring_step += 1;
  // Trainer::fit's non-finite stop (training.hpp:77-80): while the guard is
  // armed, a non-finite batch loss skips this update and every later one, so
  // the weights stay those the offending batch ran on
  if (guard && guard[0]) {
    if (guard[1] || !isfinite(*loss)) {
      if (blockIdx.x == 0 && threadIdx.x == 0) guard[1] = 1;
      return;
    }
  }
  // the first folded range (many partials): blocks [0, nfold) sum them
  // exactly as wgrad_reduce_kernel does (same bits), store the gradient,
  // update.  The second (at most kRedSlices partials, e.g. the tail's batch
  // slices) is summed inline by the update loop: with one partial per slice
  // image_sum is the plain in-order sum, so the bits are the same
  const int nfold = fold.part ? (int)cdiv(fold.per, 32) : 0;
  if ((int)blockIdx.x < nfold) {
    __shared__ float red[kRedSlices][33];
    const int64_t j = blockIdx.x * 32ll + (threadIdx.x & 31);
    const float s = image_sum(fold.nimg, fold.per, fold.stride, j, fold.part, red);
    if ((threadIdx.x >> 5) == 0 && j < fold.per) {
      g[fold_off + j] = s;
      update_pack(fold_off + j, scale * s, w, v, lr, mom, t);
    }
    return;
  }
  const int64_t f0 = nfold ? fold_off : n, f1 = nfold ? fold_off + fold.per : n;
  const int64_t h0 = fold2.part ? fold2_off : n, h1 = fold2.part ? fold2_off + fold2.per : n;
  for (int64_t i = (blockIdx.x - nfold) * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)(gridDim.x - nfold) * blockDim.x) {
    if (i >= f0 && i < f1) continue;
    float gi;
    if (i >= h0 && i < h1) {
      const float* p = fold2.part + (i - h0);
      gi = 0.f;
      for (int k = 0; k < fold2.nimg; ++k) gi += __ldg(p + k * fold2.stride);
      g[i] = gi;
    } else {
      gi = g[i];
    }
    update_pack(i, scale * gi, w, v, lr, mom, t);
  }
}

// ---- data parallelism: one-shot peer reduce + SGD + packs -----------------
// Trainer::fit's exchange point (training.hpp:76-81) for W replicas, one
// kernel per replica: every block owns one contiguous slice of the flat
// gradient; it (1) signals every peer's block b that this replica's
// gradient is final (its backward finished before this launch) and waits for
// all peers' signals, (2) reads the slice from every replica's gradient
// buffer -- peers through NVLink P2P mappings -- and sums it in RANK ORDER
// (each term weighted by B_p / B_global), so all replicas compute the same
// bits, (3) applies momentum SGD + the conv weight packs to its own
// parameters, and (4) signals "done reading" and waits for every peer's, so
// no replica overwrites its gradient (next backward) while a peer reads it.
// Signals are monotonically increasing epochs; a barrier that waits longer
// than the timeout sets *err and gives up (the host reports VCNN_ENCCL)
// instead of hanging the device.
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// warp 0, lane p < world: signal peer p's slot [phase][rank][b], wait for
// peer p's signal in my slot [phase][p][b]
__device__ __forceinline__ void dp_barrier(const DpPeers& P, int phase, uint32_t e) {
  const int lane = threadIdx.x;
  if (lane < P.world) {
    const int64_t row = (int64_t)P.nslot * P.world;
    st_release_sys(P.sig[lane] + phase * row + (int64_t)P.rank * P.nslot + blockIdx.x, e);
    const uint32_t* mine = P.my_sig + phase * row + (int64_t)lane * P.nslot + blockIdx.x;
    const uint64_t t0 = globaltimer_ns();
    while ((int32_t)(ld_acquire_sys(mine) - e) < 0) {
      if (globaltimer_ns() - t0 > (uint64_t)P.timeout_ns) {
        atomicExch(P.err, 1);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncwarp();
}

__global__ void dp_sgd_pack_kernel(int64_t n, int64_t chunk, float* __restrict__ w,
                                   float* __restrict__ v, float lr, float mom, const PackTable t,
                                   const DpPeers P, int* __restrict__ ring_step) {
  PDL_ENTRY();
  if (ring_step && blockIdx.x == 0 && threadIdx.x == 0) *ring_step += 1;
  uint32_t e = 0;
  if (P.barrier) {
    if (threadIdx.x < 32) {
      e = P.epoch[blockIdx.x] + 1;
      dp_barrier(P, 0, e);
    }
    __syncthreads();
  }
  const int64_t lo = blockIdx.x * chunk, hi = lo + chunk < n ? lo + chunk : n;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    float sum = P.scale[0] * P.g[0][i];
    for (int p = 1; p < P.world; ++p) sum = fmaf(P.scale[p], P.g[p][i], sum);
    update_pack(i, sum, w, v, lr, mom, t);
  }
  if (P.barrier) {
    __syncthreads();  // every read of the peers' slice is done
    if (threadIdx.x < 32) {
      dp_barrier(P, 1, e);
      if (threadIdx.x == 0) P.epoch[blockIdx.x] = e;
    }
  }
}
}  // namespace

namespace {
int pack_table(const std::vector<PackSpec>& layers, PackTable& t) {
  t = PackTable{};
  for (const PackSpec& p : layers) {
    if (!p.pf && !p.pd && !p.ps) continue;
    if (t.n == kMaxPackLayers) return fail(VCNN_ECONFIG, "sgd_pack: too many conv layers");
    PackLayer& L = t.L[t.n++];
    L.w_off = p.w_off;
    L.w_len = p.d.kd() * p.d.K;
    if (L.w_len >= (int64_t(1) << 31)) return fail(VCNN_ESHAPE, "sgd_pack: layer too large");
    L.pf = p.pf;
    L.pd = p.pd;
    L.ps = p.ps;
    if (p.ps) {
      L.wst = small_fwd_wst(p.d);
      if (!L.wst) return fail(VCNN_ESHAPE, "sgd_pack: small plan");
    }
    L.K = p.d.K, L.C = p.d.C, L.kh = p.d.kh, L.kw = p.d.kw;
    if (p.pf && !plan(p.d, 0, 0, 0, 0, L.gf)) return fail(VCNN_ESHAPE, "sgd_pack: fwd plan");
    if (p.pd && !plan(p.d, 1, 0, 0, 0, L.gd)) return fail(VCNN_ESHAPE, "sgd_pack: dgrad plan");
  }
  return VCNN_OK;
}
}  // namespace

int sgd_pack(int64_t n, float* w, float* v, float* g, float lr, float mom, float scale,
             const std::vector<PackSpec>& layers, cudaStream_t st, const float* loss,
             int* guard, const ImageSumFold* fold, int64_t fold_off, const ImageSumFold* fold2,
             int64_t fold2_off, int* ring_step) {
  PackTable t;
  if (int s = pack_table(layers, t)) return s;
  constexpr int kT = 32 * kRedSlices;
  int64_t blocks = cdiv(n, kT);
  if (blocks > 2 * sm_count()) blocks = 2 * sm_count();
  if (blocks < 1) blocks = 1;
  ImageSumFold f{}, f2{};
  if (fold && fold->part) {
    if (fold_off < 0 || fold_off + fold->per > n) return fail(VCNN_ESHAPE, "sgd_pack: fold range");
    f = *fold;
    blocks += cdiv(f.per, 32);
  }
  if (fold2 && fold2->part) {
    if (fold2_off < 0 || fold2_off + fold2->per > n || fold2->nimg > kRedSlices ||
        (f.part && fold2_off < fold_off + f.per && fold_off < fold2_off + fold2->per))
      return fail(VCNN_ESHAPE, "sgd_pack: fold range");
    f2 = *fold2;
  }
  VCNN_CUDA_TRY(launch_pdl(sgd_pack_kernel, dim3((unsigned)blocks), dim3(kT), 0, st, n, w, v, g, lr, mom, scale, t, loss, guard, f, fold_off, f2, fold2_off, ring_step));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int dp_blocks(int64_t n) {
  int64_t b = cdiv(n, 2048);
  if (b > kMaxDpSlots) b = kMaxDpSlots;
  if (b > sm_count()) b = sm_count();
  return b < 1 ? 1 : (int)b;
}

int dp_sgd_pack(int64_t n, float* w, float* v, float lr, float mom,
                const std::vector<PackSpec>& layers, const DpPeers& peers, cudaStream_t st,
                int* ring_step) {
  PackTable t;
  if (int s = pack_table(layers, t)) return s;
  if (peers.world < 1 || peers.world > kMaxWorld) return fail(VCNN_ECONFIG, "dp: world size");
  const int blocks = peers.nslot;
  if (blocks < 1 || blocks > kMaxDpSlots) return fail(VCNN_ECONFIG, "dp: block count");
  const int64_t chunk = cdiv(n, blocks);
  VCNN_CUDA_TRY(launch_pdl(dp_sgd_pack_kernel, dim3((unsigned)blocks), dim3(256), 0, st, n, chunk, w, v, lr, mom, t, peers, ring_step));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

namespace {
// ---------------------------------------------------------------------------
// Small-Kd forward (first layers: C*kh*kw <= 96, K <= 32; CIFAR-3 conv1 is
// 3x5x5 -> 32) on mma.sync m16n8k8 TF32, one CTA per image.
//   y[n][q] = act(sum_j W[n][j] * x[c][oy+ky][ox+kx] + b[n]),  j = (c,ky,kx)
// M = output positions (16 per tile), N = maps (W fragments live in
// registers for the whole CTA), K = Kd (a column j is a fixed offset into the
// staged image, a row a position offset).  When OH and OW are even the 16
// rows of a tile are four 2x2 windows, element-major (row = 4e + w), so a lane
// and its lane^16 partner hold all four elements of a window for two maps and
// the fused max pool + argmax is one shuffle; the trace path (no pool) uses
// the same row mapping, so fused and unfused runs are bit-identical.  The
// output of the image is staged in shared memory and written as one
// contiguous block.  At 2 FLOP/B the layer is HBM/latency-bound; the tcgen05
// direct kernel pays 5/8 channel padding (C=3 of 8) and a TMEM round trip.
constexpr int FT = 256;   // 8 warps
constexpr int kTilesPerWarp = 2;
constexpr int kTilesPerCta = (FT / 32) * kTilesPerWarp;
// row stride (floats) of the CTA's pooled [map][window] stage, = 4 (mod 32):
// the epilogue's fragment stores (lanes: 8 maps x 4 windows) hit 32 distinct
// banks (stride 65 made them 3-4-way conflicted), the [map][window] (NCHW)
// reads stay conflict-free (the NHWC reads of the TMA path are 4-way)
constexpr int kSoStride = kTilesPerCta * 4 + 4;
struct FGeo {
  int B, C, H, W, K, kh, kw, OH, OW;
  int Kd, nks, nnt;   // columns, K steps (8), N tiles (8 maps)
  int wst;            // W row stride in smem (4 mod 8: conflict-free B fragments)
  int win;            // 1: rows are 2x2 windows (OH, OW even)
  int POH, POW, nmt;  // pooled extents, M tiles per image
  int S;              // CTAs per image (kTilesPerCta M tiles each)
  int off_w, off_o, smem;  // bytes
  int pool;
  int jo[96];         // column j = (c,ky,kx) -> c*H*W + ky*W + kx (no device divisions)
};

bool fplan_small(const ConvDesc& d, int pool, FGeo& g) {
  g = FGeo{};
  if (d.s != 1 || d.K < 1 || d.K > 32) return false;
  g.B = d.B, g.C = d.C, g.H = d.H, g.W = d.W, g.K = d.K, g.kh = d.kh, g.kw = d.kw;
  g.OH = d.OH, g.OW = d.OW;
  g.Kd = d.C * d.kh * d.kw;
  if (g.Kd > 96) return false;
  g.nks = (g.Kd + 7) / 8;
  g.nnt = (d.K + 7) / 8;
  const int hw = d.H * d.W, ohw = d.OH * d.OW;
  g.wst = (g.nks <= 4 ? 32 : 96) + 4;  // the kernel's KS*8 staged columns + 4
  for (int j = 0; j < 96; ++j) {
    if (j < g.Kd) {
      const int c = j / (d.kh * d.kw), r = j - c * d.kh * d.kw, ky = r / d.kw;
      g.jo[j] = c * hw + ky * d.W + (r - ky * d.kw);
    } else {
      g.jo[j] = d.C * hw;  // the zero column
    }
  }
  if ((d.C * hw) % 4) return false;
  g.win = (d.OH % 2 == 0 && d.OW % 2 == 0) ? 1 : 0;
  if (pool && (pool != 2 || !g.win)) return false;
  g.pool = pool;
  g.POH = d.OH / 2, g.POW = d.OW / 2;
  g.nmt = g.win ? (g.POH * g.POW + 3) / 4 : (ohw + 15) / 16;
  g.S = (g.nmt + kTilesPerCta - 1) / kTilesPerCta;
  g.off_w = (4 * (d.C + 1) * hw + 127) & ~127;
  g.off_o = (g.off_w + 4 * g.nnt * 8 * g.wst + 127) & ~127;
  const int ob = 8 * d.K * kSoStride;  // pooled values + args of the CTA's windows
  g.smem = g.off_o + ob + 128;
  if (g.smem > 227 * 1024) return false;
  return true;
}

struct FSArgs {
  FGeo g;
  const float* x;
  const float* ps;  // prepacked tf32 weight image [nnt*8][wst] (or null: stage from w)
  const float* w;  // [K][Kd] (params, rounded to tf32 when staged)
  const float* bias;
  float* y;        // [B][K][OH][OW] (unpooled)
  float* py;       // [B][K][POH][POW] (pooled)
  int32_t* parg;
  float* pyn;      // nullable: [B][POH*POW][K] pooled, tf32 (the next direct conv's TMA input)
};

__device__ __forceinline__ void mma_tf32_m16n8k8(float (&c)[4], uint32_t a0, uint32_t a1,
                                                 uint32_t a2, uint32_t a3, uint32_t b0,
                                                 uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, "
      "{%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

#ifdef VCNN_PHASE_TIMING
__device__ unsigned long long g_fphase[4][8];
#define FPHASE(i)                                                              \
  do {                                                                         \
    if (threadIdx.x == 0 && blockIdx.x < 4) g_fphase[blockIdx.x][i] = clock64(); \
  } while (0)
#else
#define FPHASE(i) \
  do {            \
  } while (0)
#endif

// CTA (b, s) computes M tiles [s*kTilesPerCta, ...) of image b; warp w the
// pair 2w, 2w+1 of them (two independent accumulator sets per K step)
template <int KS, int ACT>
__global__ void __launch_bounds__(FT, 4) conv_small_fwd_kernel(const FSArgs a) {
  pdl_launch_dependents();
  FPHASE(0);
  const FGeo& g = a.g;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (ptx::smem_u32(smem_raw) & 127u)) & 127u);
  __shared__ uint64_t load_bar;
  float* sx = reinterpret_cast<float*>(smem);
  float* sw = reinterpret_cast<float*>(smem + g.off_w);
  float* so = reinterpret_cast<float*>(smem + g.off_o);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, t = lane & 3;
  const int b = blockIdx.x / g.S, sidx = blockIdx.x - b * g.S;
  const int hw = g.H * g.W, ohw = g.OH * g.OW, PP = g.POH * g.POW;
  if (tid == 0) {
    ptx::mbar_init(&load_bar, 1);
    ptx::fence_mbar_init();
  }
  for (int i = tid; i < hw; i += FT) sx[g.C * hw + i] = 0.f;  // zero column
  int coff[KS][2];  // A column offsets of this lane's two K slots per step
#pragma unroll
  for (int ks = 0; ks < KS; ++ks)
#pragma unroll
    for (int h = 0; h < 2; ++h) coff[ks][h] = g.jo[ks * 8 + t + 4 * h];
  __syncthreads();
  pdl_wait();
  FPHASE(1);
  constexpr int wcols = KS * 8;
  const int wrows = g.nnt * 8;
  if (tid == 0) {
    const uint32_t xb = 4u * (uint32_t)(g.C * hw);
    const uint32_t wb = a.ps ? 4u * (uint32_t)(wrows * g.wst) : 0u;
    ptx::mbar_expect_tx(&load_bar, xb + wb);
    ptx::bulk_g2s(ptx::smem_u32(sx), a.x + (int64_t)b * g.C * hw, xb, &load_bar);
    if (a.ps) ptx::bulk_g2s(ptx::smem_u32(sw), a.ps, wb, &load_bar);  // prepacked tf32 image
    ptx::mbar_arrive(&load_bar);
  }
  if (!a.ps) {
    // W -> smem [n][wst], tf32, zero padded (rows to nnt*8, columns to KS*8)
    // (cp.async: every element's load in flight at once; rounded after the wait)
    for (int i = tid; i < wrows * wcols; i += FT) {
      const int n = i / wcols, j = i - n * wcols;
      if (n < g.K && j < g.Kd)
        ptx::cp_async4(ptx::smem_u32(sw + n * g.wst + j), a.w + n * g.Kd + j);
      else
        sw[n * g.wst + j] = 0.f;
    }
    ptx::cp_async_wait_all();
    for (int i = tid; i < wrows * wcols; i += FT) {
      const int n = i / wcols, j = i - n * wcols;
      sw[n * g.wst + j] = ptx::to_tf32(sw[n * g.wst + j]);
    }
  }
  ptx::mbar_wait(&load_bar, 0);
  FPHASE(2);
  for (int i = tid; i < g.C * hw; i += FT) sx[i] = ptx::to_tf32(sx[i]);
  __syncthreads();
  FPHASE(3);

  const int mbase = sidx * kTilesPerCta;
  float acc[kTilesPerWarp][4][4];
  int qi[kTilesPerWarp][2], po[kTilesPerWarp][2];
  bool ok[kTilesPerWarp][2];
#pragma unroll
  for (int p = 0; p < kTilesPerWarp; ++p) {
    const int mt = mbase + warp * kTilesPerWarp + p;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = gq + 8 * h;
      int oy, ox;
      if (g.win) {
        int wi = mt * 4 + (r & 3);
        ok[p][h] = wi < PP;
        wi = ok[p][h] ? wi : PP - 1;
        const int e = r >> 2, py = wi / g.POW, px = wi - py * g.POW;
        oy = 2 * py + (e >> 1);
        ox = 2 * px + (e & 1);
      } else {
        int m = mt * 16 + r;
        ok[p][h] = m < ohw;
        m = ok[p][h] ? m : ohw - 1;
        oy = m / g.OW;
        ox = m - oy * g.OW;
      }
      qi[p][h] = oy * g.OW + ox;
      po[p][h] = oy * g.W + ox;
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[p][nt][u] = 0.f;
  }
  const float* wrow = sw + gq * g.wst + t;
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    if (ks < g.nks) {
      uint32_t bf[4][2];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
        if (nt < g.nnt) {
          bf[nt][0] = __float_as_uint(wrow[nt * 8 * g.wst + ks * 8]);
          bf[nt][1] = __float_as_uint(wrow[nt * 8 * g.wst + ks * 8 + 4]);
        }
#pragma unroll
      for (int p = 0; p < kTilesPerWarp; ++p) {
        const uint32_t a0 = __float_as_uint(sx[coff[ks][0] + po[p][0]]);
        const uint32_t a1 = __float_as_uint(sx[coff[ks][0] + po[p][1]]);
        const uint32_t a2 = __float_as_uint(sx[coff[ks][1] + po[p][0]]);
        const uint32_t a3 = __float_as_uint(sx[coff[ks][1] + po[p][1]]);
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
          if (nt < g.nnt) mma_tf32_m16n8k8(acc[p][nt], a0, a1, a2, a3, bf[nt][0], bf[nt][1]);
      }
    }
  }
  FPHASE(4);
  // epilogue: c = {(gq, 2t), (gq, 2t+1), (gq+8, 2t), (gq+8, 2t+1)}
  float bb[4][2];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int nc = nt * 8 + 2 * t + h;
      bb[nt][h] = nc < g.K ? __ldg(a.bias + nc) : 0.f;
    }
  const int wloc0 = warp * kTilesPerWarp * 4;  // first window of this warp in the CTA
#pragma unroll
  for (int p = 0; p < kTilesPerWarp; ++p) {
    const int mt = mbase + warp * kTilesPerWarp + p;
    const int wi = mt * 4 + (gq & 3);
    const int wpy = wi / g.POW, wpx = wi - wpy * g.POW;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = actf<ACT>(acc[p][nt][u] + bb[nt][u & 1]);
      if (!g.pool) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int n = nt * 8 + 2 * t + (u & 1), h = u >> 1;
          if (ok[p][h] && n < g.K && mt < g.nmt)
            a.y[((int64_t)b * g.K + n) * ohw + qi[p][h]] = v[u];
        }
      } else {
        // lane gq<4 holds elements e=0 (row gq), e=2 (row gq+8) of window
        // w=gq; its partner lane^16 holds e=1, e=3.  The low lane pools map
        // 2t, the high lane map 2t+1; window order e = 0,1,2,3, strict >.
        float pv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) pv[u] = __shfl_xor_sync(0xffffffffu, v[u], 16);
        const bool lo = gq < 4;
        float e[4];
        e[0] = lo ? v[0] : pv[1];
        e[1] = lo ? pv[0] : v[1];
        e[2] = lo ? v[2] : pv[3];
        e[3] = lo ? pv[2] : v[3];
        float best = e[0];
        int bi = 0;
#pragma unroll
        for (int k = 1; k < 4; ++k)
          if (e[k] > best) {
            best = e[k];
            bi = k;
          }
        const int n = nt * 8 + 2 * t + (lo ? 0 : 1);
        if (wi < PP && n < g.K) {
          const int q = (2 * wpy + (bi >> 1)) * g.OW + 2 * wpx + (bi & 1);
          const int wl = wloc0 + p * 4 + (gq & 3);
          so[n * kSoStride + wl] = best;
          reinterpret_cast<int32_t*>(so)[(g.K + n) * kSoStride + wl] = (b * g.K + n) * ohw + q;
        }
      }
    }
  }
  if (g.pool) {  // the CTA's windows [w0, w0+nw) of every map: row segments
    __syncthreads();
    FPHASE(5);
    constexpr int CW = kTilesPerCta * 4;
    const int w0 = mbase * 4;
    const int nw = PP - w0 < CW ? PP - w0 : CW;
    for (int i = tid; i < g.K * CW; i += FT) {
      const int n = i / CW, r = i - n * CW;
      if (r >= nw) continue;
      const int64_t o = ((int64_t)b * g.K + n) * PP + w0 + r;
      a.py[o] = so[n * kSoStride + r];
      a.parg[o] = reinterpret_cast<const int32_t*>(so)[(g.K + n) * kSoStride + r];
    }
    if (a.pyn)  // channels innermost: one contiguous run of K per window
      for (int i = tid; i < g.K * nw; i += FT) {
        const int r = i / g.K, n = i - r * g.K;
        a.pyn[((int64_t)b * PP + w0 + r) * g.K + n] = ptx::to_tf32(so[n * kSoStride + r]);
      }
  }
  FPHASE(6);
}

template <int ACT>
int launch_small_fwd(const FSArgs& a, cudaStream_t st) {
  const size_t smem = (size_t)a.g.smem;
  auto go = [&](auto kern, size_t& configured) -> int {
    if (smem > configured) {
      VCNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
      configured = smem;
    }
    VCNN_CUDA_TRY(launch_pdl(kern, dim3((unsigned)(a.g.B * a.g.S)), dim3(FT), smem, st, a));
    VCNN_LAUNCHED();
    return VCNN_OK;
  };
  static size_t c4 = 0, c12 = 0;
  if (a.g.nks <= 4) return go(conv_small_fwd_kernel<4, ACT>, c4);
  return go(conv_small_fwd_kernel<12, ACT>, c12);
}

}  // namespace

bool small_fwd_ok(const ConvDesc& d, int pool) {
  FGeo g;
  return fplan_small(d, pool, g);
}

int small_fwd_wst(const ConvDesc& d) {
  FGeo g;
  return fplan_small(d, 0, g) ? g.wst : 0;
}

size_t small_fwd_pack_floats(const ConvDesc& d) {
  FGeo g;
  if (!fplan_small(d, 0, g)) return 0;
  return (size_t)g.nnt * 8 * g.wst;
}

namespace {
__global__ void small_pack_kernel(int K, int Kd, int rows, int wst, const float* __restrict__ w,
                                  float* __restrict__ ps) {
  PDL_ENTRY();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows * wst; i += gridDim.x * blockDim.x) {
    const int n = i / wst, j = i - n * wst;
    ps[i] = (n < K && j < Kd) ? ptx::to_tf32(w[n * Kd + j]) : 0.f;
  }
}
}  // namespace

int small_fwd_pack(const ConvDesc& d, const float* w, float* ps, cudaStream_t st) {
  FGeo g;
  if (!fplan_small(d, 0, g)) return fail(VCNN_ESHAPE, "small pack: geometry not supported");
  const int rows = g.nnt * 8;
  VCNN_CUDA_TRY(launch_pdl(small_pack_kernel, dim3((unsigned)cdiv(rows * g.wst, 256)), dim3(256), 0,
                           st, d.K, g.Kd, rows, g.wst, w, ps));
  VCNN_LAUNCHED();
  return VCNN_OK;
}

int conv_fwd_small(const ConvDesc& d, const float* x, const float* w, const float* bias, int act,
                   float* y, const PoolFuse& pf, cudaStream_t st, const float* ps) {
  FSArgs a{};
  if (!fplan_small(d, pf.pool, a.g))
    return fail(VCNN_ESHAPE, "small conv forward: geometry not supported");
  a.ps = ps;
  a.x = x;
  a.w = w;
  a.bias = bias;
  a.y = y;
  a.py = pf.y;
  a.parg = pf.arg;
  a.pyn = pf.y_nhwc;
  switch (act) {
    case VCNN_ACT_RELU: return launch_small_fwd<VCNN_ACT_RELU>(a, st);
    case VCNN_ACT_SIGMOID: return launch_small_fwd<VCNN_ACT_SIGMOID>(a, st);
    case VCNN_ACT_TANH: return launch_small_fwd<VCNN_ACT_TANH>(a, st);
    default: return launch_small_fwd<VCNN_ACT_IDENTITY>(a, st);
  }
}

// ---- tf32 NHWC inputs for the tensor-TMA slab ----------------------------
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}
}  // namespace

bool fwd_tma_ok(const ConvDesc& d, int pool) {
  Geo g;
  return plan(d, 0, pool, 0, 0, g, 1);
}

size_t nhwc_map_bytes() { return sizeof(CUtensorMap); }

// the forward slab's tensor map over x_nhwc [B][H][W][C] (tf32 values):
// dims (4 channels, W, H, C/4, B), box (4, Wg, rows, 2*CG, 1)
int make_nhwc_map(const ConvDesc& d, const float* x_nhwc, void* map) {
  Geo g;
  if (!plan(d, 0, 0, 0, 0, g, 1)) return fail(VCNN_ESHAPE, "nhwc map: geometry not supported");
  auto enc = encode_fn();
  if (!enc) return fail(VCNN_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[5] = {4, (cuuint64_t)d.W, (cuuint64_t)d.H, (cuuint64_t)(d.C / 4),
                              (cuuint64_t)d.B};
  const cuuint64_t strides[4] = {(cuuint64_t)d.C * 4, (cuuint64_t)d.W * d.C * 4, 16,
                                 (cuuint64_t)d.H * d.W * d.C * 4};
  const cuuint32_t box[5] = {4, (cuuint32_t)g.Wg, (cuuint32_t)g.rows, (cuuint32_t)(2 * g.CG), 1};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(static_cast<CUtensorMap*>(map), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5,
                   const_cast<float*>(x_nhwc), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(VCNN_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return VCNN_OK;
}

int conv_fwd(const ConvDesc& d, const float* x, const float* pk, const float* bias, int act,
             float* y, const PoolFuse& pf, cudaStream_t st, const void* nhwc_map) {
  Args a{};
  if (nhwc_map && plan(d, 0, pf.pool, pf.POH, pf.POW, a.g, 1)) {
    std::memcpy(&a.tmap, nhwc_map, sizeof(CUtensorMap));
  } else if (!plan(d, 0, pf.pool, pf.POH, pf.POW, a.g)) {
    return fail(VCNN_ESHAPE, "direct conv forward: geometry not supported");
  }
  a.in = x;
  a.pack = pk;
  a.fe.bias = bias;
  a.fe.act = act;
  a.fe.y = y;
  a.fe.pool = pf.pool;
  a.fe.POH = pf.POH;
  a.fe.POW = pf.POW;
  a.fe.py = pf.y;
  a.fe.parg = pf.arg;
  return launch(a, st);
}

int conv_dgrad(const ConvDesc& d, const GradSrc& gs, const float* pk, float* dx,
               const float* yprev, int act_prev, cudaStream_t st) {
  Args a{};
  if (!plan(d, 1, gs.pool, gs.POH, gs.POW, a.g))
    return fail(VCNN_ESHAPE, "direct conv dgrad: geometry not supported");
  a.in = gs.g;
  a.gs = gs;
  a.pack = pk;
  a.be.dx = dx;
  a.be.yprev = yprev;
  a.be.act_prev = act_prev;
  return launch(a, st);
}

}  // namespace direct
}  // namespace vcnn_b200

#ifdef VCNN_PHASE_TIMING
extern "C" int vcnn_debug_fphases(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, vcnn_b200::direct::g_fphase, sizeof(unsigned long long) * 32) ==
                 cudaSuccess
             ? 0
             : 4;
}
extern "C" int vcnn_debug_dphases(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, vcnn_b200::direct::g_dphase, sizeof(unsigned long long) * 64) ==
                 cudaSuccess
             ? 0
             : 4;
}
extern "C" int vcnn_debug_dump(float* out) {
  return cudaMemcpyFromSymbol(out, vcnn_b200::direct::g_dump, sizeof(float) * 1024) ==
                 cudaSuccess
             ? 0
             : 4;
}
#endif
