/*
 * vcnn_oracle.c -- CPU restatement of the reference VCNN Imp-6 path.
 *
 * TEST INFRASTRUCTURE ONLY (see vcnn_oracle.h).  Never linked into or called
 * by the product.  Reference paths are relative to /root/reference/proj.
 */
#include "vcnn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ===================================================================== */
/* Rng: common.hpp:51-96 (std::mt19937_64, portable uniform extraction)   */
/* ===================================================================== */
#define MT_N 312
#define MT_M 156

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_N;
  r->spare = 0.0;
  r->have_spare = 0;
}

static void mt_twist(orc_rng* r) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  for (int i = 0; i < MT_N; ++i) {
    uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % MT_N] & LM);
    uint64_t y = x >> 1;
    if (x & 1ULL) y ^= A;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ y;
  }
  r->idx = 0;
}

uint64_t orc_rng_next_u64(orc_rng* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* common.hpp:58 */
double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53; }
/* common.hpp:60.  The reference build (gnu++20 => -ffp-contract=fast, with
 * -march=native on any FMA machine) contracts lo + (hi-lo)*u into one fused
 * multiply-add; restate it with fma() so initial weights are bit-identical. */
double orc_rng_uniform_range(orc_rng* r, double lo, double hi) {
  return fma(hi - lo, orc_rng_uniform(r), lo);
}
/* common.hpp:63-66 */
int orc_rng_uniform_int(orc_rng* r, int n) {
  int v = (int)(orc_rng_uniform(r) * n);
  return v < n ? v : n - 1;
}
void orc_rng_fill_uniform(orc_rng* r, double* out, int64_t n, double lo, double hi) {
  for (int64_t i = 0; i < n; ++i) out[i] = orc_rng_uniform_range(r, lo, hi);
}

/* ===================================================================== */
/* tensor.hpp:131-174                                                      */
/* ===================================================================== */
/* matmul, i-k-j axpy order, ascending k (tensor.hpp:131-150) */
void orc_matmul(int64_t m, int64_t kk, int64_t n, const double* a, const double* b, double* c) {
  memset(c, 0, sizeof(double) * (size_t)(m * n));
  for (int64_t i = 0; i < m; ++i) {
    double* crow = c + i * n;
    for (int64_t k = 0; k < kk; ++k) {
      const double aik = a[i * kk + k];
      const double* brow = b + k * n;
      for (int64_t j = 0; j < n; ++j) crow[j] += aik * brow[j];
    }
  }
}

/* matmul_transB, dot-product form, ascending k (tensor.hpp:154-174) */
void orc_matmul_transB(int64_t m, int64_t kk, int64_t n, const double* a, const double* b,
                       double* c) {
  for (int64_t i = 0; i < m; ++i) {
    const double* arow = a + i * kk;
    for (int64_t j = 0; j < n; ++j) {
      const double* brow = b + j * kk;
      double acc = 0.0;
      for (int64_t k = 0; k < kk; ++k) acc += arow[k] * brow[k];
      c[i * n + j] = acc;
    }
  }
}

/* ===================================================================== */
/* vectorize.hpp                                                           */
/* ===================================================================== */
/* ConvGeometry ctor (vectorize.hpp:19-29) */
int orc_conv_geometry(int h, int w, int c, int n, int kh, int kw, int stride, int* out_h,
                      int* out_w) {
  if (h < 1 || w < 1 || c < 1 || n < 1) return ORC_ESHAPE;
  if (kh < 1 || kw < 1) return ORC_EGEOMETRY;
  if (stride < 1) return ORC_EGEOMETRY;
  if (kh > h || kw > w) return ORC_EGEOMETRY;
  if (out_h) *out_h = (h - kh) / stride + 1;
  if (out_w) *out_w = (w - kw) / stride + 1;
  return ORC_OK;
}

/* PoolGeometry ctor (vectorize.hpp:141-151) */
int orc_pool_geometry(int h, int w, int c, int n, int ph, int pw, int stride, int* out_h,
                      int* out_w) {
  if (h < 1 || w < 1 || c < 1 || n < 1) return ORC_ESHAPE;
  if (ph < 1 || pw < 1) return ORC_EGEOMETRY;
  if (stride < 1) return ORC_EGEOMETRY;
  if (ph > h || pw > w) return ORC_EGEOMETRY;
  if (out_h) *out_h = (h - ph) / stride + 1;
  if (out_w) *out_w = (w - pw) / stride + 1;
  return ORC_OK;
}

/* im2col (vectorize.hpp:54-79): P[(c*kh+ky)*kw+kx][b*OHW + oy*OW + ox] */
int orc_im2col(int B, int C, int H, int W, int kh, int kw, int s, const double* x, double* P) {
  int OH, OW;
  int st = orc_conv_geometry(H, W, C, B, kh, kw, s, &OH, &OW);
  if (st) return st;
  const int64_t plane = (int64_t)H * W, ohw = (int64_t)OH * OW, cols = ohw * B;
  for (int c = 0; c < C; ++c)
    for (int ky = 0; ky < kh; ++ky)
      for (int kx = 0; kx < kw; ++kx) {
        const int64_t row = ((int64_t)c * kh + ky) * kw + kx;
        double* drow = P + row * cols;
        for (int b = 0; b < B; ++b) {
          const double* cplane = x + ((int64_t)b * C + c) * plane;
          for (int oy = 0; oy < OH; ++oy) {
            const double* srow = cplane + (int64_t)(oy * s + ky) * W + kx;
            double* d = drow + b * ohw + (int64_t)oy * OW;
            for (int ox = 0; ox < OW; ++ox) d[ox] = srow[(int64_t)ox * s];
          }
        }
      }
  return ORC_OK;
}

/* build_col2im_map (vectorize.hpp:84-106): pairs enumerate (c,ky,kx,b,oy,ox) */
int orc_col2im_map(int B, int C, int H, int W, int kh, int kw, int s, int64_t* src,
                   int64_t* tgt) {
  int OH, OW;
  int st = orc_conv_geometry(H, W, C, B, kh, kw, s, &OH, &OW);
  if (st) return st;
  const int64_t plane = (int64_t)H * W, ohw = (int64_t)OH * OW, cols = ohw * B;
  int64_t k = 0;
  for (int c = 0; c < C; ++c)
    for (int ky = 0; ky < kh; ++ky)
      for (int kx = 0; kx < kw; ++kx) {
        const int64_t row = ((int64_t)c * kh + ky) * kw + kx;
        for (int b = 0; b < B; ++b) {
          const int64_t cbase = ((int64_t)b * C + c) * plane;
          for (int oy = 0; oy < OH; ++oy)
            for (int ox = 0; ox < OW; ++ox) {
              src[k] = row * cols + b * ohw + (int64_t)oy * OW + ox;
              tgt[k] = cbase + (int64_t)(oy * s + ky) * W + ((int64_t)ox * s + kx);
              ++k;
            }
        }
      }
  return ORC_OK;
}

/* col2im = accumulate_by_index(sum) over the col2im map, in pair order
 * (vectorize.hpp:111-120, tensor.hpp:228-239). */
int orc_col2im(int B, int C, int H, int W, int kh, int kw, int s, const double* dP, double* dX) {
  int OH, OW;
  int st = orc_conv_geometry(H, W, C, B, kh, kw, s, &OH, &OW);
  if (st) return st;
  const int64_t plane = (int64_t)H * W, ohw = (int64_t)OH * OW, cols = ohw * B;
  memset(dX, 0, sizeof(double) * (size_t)(plane * C * B));
  for (int c = 0; c < C; ++c)
    for (int ky = 0; ky < kh; ++ky)
      for (int kx = 0; kx < kw; ++kx) {
        const int64_t row = ((int64_t)c * kh + ky) * kw + kx;
        for (int b = 0; b < B; ++b) {
          const int64_t cbase = ((int64_t)b * C + c) * plane;
          for (int oy = 0; oy < OH; ++oy)
            for (int ox = 0; ox < OW; ++ox)
              dX[cbase + (int64_t)(oy * s + ky) * W + ((int64_t)ox * s + kx)] +=
                  dP[row * cols + b * ohw + (int64_t)oy * OW + ox];
        }
      }
  return ORC_OK;
}

/* build_pool_map (vectorize.hpp:167-191): pairs enumerate (b,c,oy,ox,py,px) */
int orc_pool_map(int B, int C, int H, int W, int ph, int pw, int s, int64_t* src, int64_t* tgt) {
  int OH, OW;
  int st = orc_pool_geometry(H, W, C, B, ph, pw, s, &OH, &OW);
  if (st) return st;
  const int64_t plane = (int64_t)H * W, oplane = (int64_t)OH * OW;
  int64_t k = 0;
  for (int b = 0; b < B; ++b)
    for (int c = 0; c < C; ++c) {
      const int64_t ibase = ((int64_t)b * C + c) * plane;
      const int64_t obase = ((int64_t)b * C + c) * oplane;
      for (int oy = 0; oy < OH; ++oy)
        for (int ox = 0; ox < OW; ++ox) {
          const int64_t t = obase + (int64_t)oy * OW + ox;
          for (int py = 0; py < ph; ++py)
            for (int px = 0; px < pw; ++px) {
              src[k] = ibase + (int64_t)(oy * s + py) * W + ((int64_t)ox * s + px);
              tgt[k] = t;
              ++k;
            }
        }
    }
  return ORC_OK;
}

/* pool_forward (vectorize.hpp:197-210): max -> accumulate_max_arg
 * (tensor.hpp:271-289; ties -> lowest source), avg -> accumulate_by_index
 * mean (tensor.hpp:240-248; sum in pair order then / count). */
int orc_pool_forward(int B, int C, int H, int W, int ph, int pw, int s, int mode,
                     const double* x, double* y, int64_t* arg) {
  int OH, OW;
  int st = orc_pool_geometry(H, W, C, B, ph, pw, s, &OH, &OW);
  if (st) return st;
  const int64_t plane = (int64_t)H * W, oplane = (int64_t)OH * OW;
  for (int b = 0; b < B; ++b)
    for (int c = 0; c < C; ++c) {
      const int64_t ibase = ((int64_t)b * C + c) * plane;
      const int64_t obase = ((int64_t)b * C + c) * oplane;
      for (int oy = 0; oy < OH; ++oy)
        for (int ox = 0; ox < OW; ++ox) {
          const int64_t t = obase + (int64_t)oy * OW + ox;
          if (mode == ORC_POOL_MAX) {
            double best = 0.0;
            int64_t a = -1;
            for (int py = 0; py < ph; ++py)
              for (int px = 0; px < pw; ++px) {
                const int64_t srci = ibase + (int64_t)(oy * s + py) * W + ((int64_t)ox * s + px);
                const double v = x[srci];
                if (a < 0 || v > best || (v == best && srci < a)) {
                  best = v;
                  a = srci;
                }
              }
            y[t] = best;
            if (arg) arg[t] = a;
          } else {
            double acc = 0.0;
            for (int py = 0; py < ph; ++py)
              for (int px = 0; px < pw; ++px)
                acc += x[ibase + (int64_t)(oy * s + py) * W + ((int64_t)ox * s + px)];
            y[t] = acc / (double)(ph * pw);
            if (arg) arg[t] = -1;
          }
        }
    }
  return ORC_OK;
}

/* pool_backward (vectorize.hpp:224-249) */
int orc_pool_backward(int B, int C, int H, int W, int ph, int pw, int s, int mode, int bwd_mode,
                      const double* dy, const int64_t* arg, double* dx) {
  int OH, OW;
  int st = orc_pool_geometry(H, W, C, B, ph, pw, s, &OH, &OW);
  if (st) return st;
  const int64_t plane = (int64_t)H * W, oplane = (int64_t)OH * OW;
  const int64_t in_size = plane * C * B, out_size = oplane * C * B;
  memset(dx, 0, sizeof(double) * (size_t)in_size);
  if (bwd_mode == ORC_POOLBWD_EXACT && mode == ORC_POOL_MAX) {
    for (int64_t t = 0; t < out_size; ++t)
      if (arg[t] >= 0) dx[arg[t]] += dy[t];
    return ORC_OK;
  }
  const double scale = (bwd_mode == ORC_POOLBWD_PAPER_NN) ? 1.0 : 1.0 / (double)(ph * pw);
  for (int b = 0; b < B; ++b)
    for (int c = 0; c < C; ++c) {
      const int64_t ibase = ((int64_t)b * C + c) * plane;
      const int64_t obase = ((int64_t)b * C + c) * oplane;
      for (int oy = 0; oy < OH; ++oy)
        for (int ox = 0; ox < OW; ++ox) {
          const int64_t t = obase + (int64_t)oy * OW + ox;
          for (int py = 0; py < ph; ++py)
            for (int px = 0; px < pw; ++px) {
              const int64_t srci = ibase + (int64_t)(oy * s + py) * W + ((int64_t)ox * s + px);
              if (bwd_mode == ORC_POOLBWD_PAPER_NN)
                dx[srci] += dy[t];
              else
                dx[srci] += dy[t] * scale;
            }
        }
    }
  return ORC_OK;
}

/* ===================================================================== */
/* layers.hpp                                                              */
/* ===================================================================== */
/* activate (layers.hpp:25-34) */
double orc_activate(int act, double x) {
  switch (act) {
    case ORC_ACT_RELU: return x > 0.0 ? x : 0.0;
    case ORC_ACT_SIGMOID: return 1.0 / (1.0 + exp(-x));
    case ORC_ACT_TANH: return tanh(x);
    default: return x;
  }
}

/* activation_grad_from_output (layers.hpp:39-48) */
double orc_activation_grad_from_output(int act, double y) {
  switch (act) {
    case ORC_ACT_RELU: return y > 0.0 ? 1.0 : 0.0;
    case ORC_ACT_SIGMOID: return y * (1.0 - y);
    case ORC_ACT_TANH: return 1.0 - y * y;
    default: return 1.0;
  }
}

static void apply_activation(int act, double* d, int64_t n) {
  if (act == ORC_ACT_IDENTITY) return;
  for (int64_t i = 0; i < n; ++i) d[i] = orc_activate(act, d[i]);
}

static void apply_activation_grad(int act, const double* y, double* g, int64_t n) {
  if (act == ORC_ACT_IDENTITY) return;
  for (int64_t i = 0; i < n; ++i) g[i] *= orc_activation_grad_from_output(act, y[i]);
}

/* conv_forward (layers.hpp:139-149) = im2col + conv_affine (matmul + bias,
 * :99-109) + matrix_to_featmap (:113-123) + apply_activation */
int orc_conv_forward(int B, int C, int H, int W, int K, int kh, int kw, int s, int act,
                     const double* x, const double* w, const double* b, double* y) {
  int OH, OW;
  int st = orc_conv_geometry(H, W, C, B, kh, kw, s, &OH, &OW);
  if (st) return st;
  if (K < 1) return ORC_ESHAPE;
  const int64_t kd = (int64_t)C * kh * kw, ohw = (int64_t)OH * OW, cols = ohw * B;
  double* P = (double*)malloc(sizeof(double) * (size_t)(kd * cols));
  double* Z = (double*)malloc(sizeof(double) * (size_t)(K * cols));
  orc_im2col(B, C, H, W, kh, kw, s, x, P);
  orc_matmul(K, kd, cols, w, P, Z);
  for (int k = 0; k < K; ++k)
    for (int64_t j = 0; j < cols; ++j) Z[k * cols + j] += b[k];
  for (int k = 0; k < K; ++k)
    for (int bb = 0; bb < B; ++bb)
      memcpy(y + ((int64_t)bb * K + k) * ohw, Z + k * cols + bb * ohw, sizeof(double) * ohw);
  apply_activation(act, y, (int64_t)K * cols);
  free(P);
  free(Z);
  return ORC_OK;
}

/* conv_backward (layers.hpp:183-189) -> apply_activation_grad + conv_backward_core
 * (:161-181): G = featmap_to_matrix(gpre); dW = matmul_transB(G, P);
 * db = rowsum(G); dX = col2im(matmul(transpose(W), G)). */
int orc_conv_backward(int B, int C, int H, int W, int K, int kh, int kw, int s, int act,
                      const double* x, const double* w, const double* y, const double* dy,
                      double* dw, double* db, double* dx) {
  int OH, OW;
  int st = orc_conv_geometry(H, W, C, B, kh, kw, s, &OH, &OW);
  if (st) return st;
  const int64_t kd = (int64_t)C * kh * kw, ohw = (int64_t)OH * OW, cols = ohw * B;
  const int64_t ysz = (int64_t)K * cols;
  double* gpre = (double*)malloc(sizeof(double) * (size_t)ysz);
  memcpy(gpre, dy, sizeof(double) * (size_t)ysz);
  apply_activation_grad(act, y, gpre, ysz);
  double* G = (double*)malloc(sizeof(double) * (size_t)ysz);
  for (int k = 0; k < K; ++k)
    for (int bb = 0; bb < B; ++bb)
      memcpy(G + k * cols + bb * ohw, gpre + ((int64_t)bb * K + k) * ohw, sizeof(double) * ohw);
  double* P = (double*)malloc(sizeof(double) * (size_t)(kd * cols));
  orc_im2col(B, C, H, W, kh, kw, s, x, P);
  orc_matmul_transB(K, cols, kd, G, P, dw);
  for (int k = 0; k < K; ++k) {
    double acc = 0.0;
    for (int64_t j = 0; j < cols; ++j) acc += G[k * cols + j];
    db[k] = acc;
  }
  if (dx) {
    double* Wt = (double*)malloc(sizeof(double) * (size_t)(kd * K));
    for (int k = 0; k < K; ++k)
      for (int64_t j = 0; j < kd; ++j) Wt[j * K + k] = w[k * kd + j];
    double* dP = (double*)malloc(sizeof(double) * (size_t)(kd * cols));
    orc_matmul(kd, K, cols, Wt, G, dP);
    orc_col2im(B, C, H, W, kh, kw, s, dP, dx);
    free(Wt);
    free(dP);
  }
  free(gpre);
  free(G);
  free(P);
  return ORC_OK;
}

/* full_forward (layers.hpp:230-247): Z = flatten_to_rows(x) * W^T + b */
int orc_full_forward(int B, int in, int out, int act, const double* x, const double* w,
                     const double* b, double* y) {
  if (B < 1 || in < 1 || out < 1) return ORC_ESHAPE;
  orc_matmul_transB(B, in, out, x, w, y);
  for (int bb = 0; bb < B; ++bb)
    for (int o = 0; o < out; ++o) y[(int64_t)bb * out + o] += b[o];
  apply_activation(act, y, (int64_t)B * out);
  return ORC_OK;
}

/* full_backward (layers.hpp:270-278) -> full_backward_core (:256-267):
 * dW = matmul(transpose(G), in); db = colsum(G); dX = matmul(G, W). */
int orc_full_backward(int B, int in, int out, int act, const double* x, const double* w,
                      const double* y, const double* dy, double* dw, double* db, double* dx) {
  if (B < 1 || in < 1 || out < 1) return ORC_ESHAPE;
  const int64_t n = (int64_t)B * out;
  double* g = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(g, dy, sizeof(double) * (size_t)n);
  apply_activation_grad(act, y, g, n);
  double* gt = (double*)malloc(sizeof(double) * (size_t)n);
  for (int bb = 0; bb < B; ++bb)
    for (int o = 0; o < out; ++o) gt[(int64_t)o * B + bb] = g[(int64_t)bb * out + o];
  orc_matmul(out, B, in, gt, x, dw);
  for (int o = 0; o < out; ++o) db[o] = 0.0;
  for (int bb = 0; bb < B; ++bb)
    for (int o = 0; o < out; ++o) db[o] += g[(int64_t)bb * out + o];
  if (dx) orc_matmul(B, out, in, g, w, dx);
  free(g);
  free(gt);
  return ORC_OK;
}

/* loss_forward (layers.hpp:402-434) */
int orc_loss_forward(int kind, int B, int units, const double* pred, const int* cls,
                     const double* values, double* loss) {
  if (kind == ORC_LOSS_SOFTMAX_CE) {
    double total = 0.0;
    for (int b = 0; b < B; ++b) {
      const int c = cls[b];
      if (c < 0 || c >= units) return ORC_EBOUNDS;
      const double* l = pred + (int64_t)b * units;
      double m = l[0];
      for (int u = 1; u < units; ++u) m = (m < l[u]) ? l[u] : m; /* std::max */
      double lse = 0.0;
      for (int u = 0; u < units; ++u) lse += exp(l[u] - m);
      total += m + log(lse) - l[c];
    }
    *loss = total / (double)B;
    return ORC_OK;
  }
  const int64_t n = (int64_t)B * units;
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double d = pred[i] - values[i];
    total += d * d;
  }
  *loss = total / (double)n;
  return ORC_OK;
}

/* loss_backward (layers.hpp:436-468) */
int orc_loss_backward(int kind, int B, int units, const double* pred, const int* cls,
                      const double* values, double* grad) {
  if (kind == ORC_LOSS_SOFTMAX_CE) {
    const double inv_b = 1.0 / (double)B;
    for (int b = 0; b < B; ++b) {
      const int c = cls[b];
      if (c < 0 || c >= units) return ORC_EBOUNDS;
      const double* l = pred + (int64_t)b * units;
      double* g = grad + (int64_t)b * units;
      double m = l[0];
      for (int u = 1; u < units; ++u) m = (m < l[u]) ? l[u] : m;
      double lse = 0.0;
      for (int u = 0; u < units; ++u) lse += exp(l[u] - m);
      for (int u = 0; u < units; ++u) g[u] = exp(l[u] - m) / lse * inv_b;
      g[c] -= inv_b;
    }
    return ORC_OK;
  }
  const int64_t n = (int64_t)B * units;
  const double scale = 2.0 / (double)n;
  for (int64_t i = 0; i < n; ++i) grad[i] = scale * (pred[i] - values[i]);
  return ORC_OK;
}

/* ===================================================================== */
/* network.hpp / variants.hpp                                              */
/* ===================================================================== */
/* NetworkSpec::chain (network.hpp:45-67) */
int orc_net_chain(const orc_net* net, int* shapes) {
  int h = net->in_h, w = net->in_w, c = net->in_c;
  if (h < 1 || w < 1 || c < 1) return ORC_ESHAPE;
  for (int i = 0; i < net->nlayers; ++i) {
    const orc_layer* L = &net->layers[i];
    int oh, ow;
    if (L->kind == ORC_LAYER_CONV) {
      if (L->units < 1) return ORC_ESHAPE;
      if (orc_conv_geometry(h, w, c, 1, L->kh, L->kw, L->stride, &oh, &ow)) return ORC_ESHAPE;
      h = oh;
      w = ow;
      c = L->units;
    } else if (L->kind == ORC_LAYER_POOL) {
      if (orc_pool_geometry(h, w, c, 1, L->kh, L->kw, L->stride, &oh, &ow)) return ORC_ESHAPE;
      h = oh;
      w = ow;
    } else if (L->kind == ORC_LAYER_FULL) {
      if (L->units < 1) return ORC_ESHAPE;
      h = 1;
      w = 1;
      c = L->units;
    } else {
      return ORC_ECONFIG;
    }
    if (shapes) {
      shapes[3 * i] = h;
      shapes[3 * i + 1] = w;
      shapes[3 * i + 2] = c;
    }
  }
  return ORC_OK;
}

static void layer_in_shape(const orc_net* net, const int* shapes, int i, int* h, int* w, int* c) {
  if (i == 0) {
    *h = net->in_h;
    *w = net->in_w;
    *c = net->in_c;
  } else {
    *h = shapes[3 * (i - 1)];
    *w = shapes[3 * (i - 1) + 1];
    *c = shapes[3 * (i - 1) + 2];
  }
}

int orc_net_param_layout(const orc_net* net, int64_t* w_off, int64_t* w_len, int64_t* b_off,
                         int64_t* b_len) {
  int* shapes = (int*)malloc(sizeof(int) * 3 * (size_t)(net->nlayers > 0 ? net->nlayers : 1));
  int st = orc_net_chain(net, shapes);
  if (st) {
    free(shapes);
    return st;
  }
  int64_t off = 0;
  for (int i = 0; i < net->nlayers; ++i) {
    const orc_layer* L = &net->layers[i];
    int h, w, c;
    layer_in_shape(net, shapes, i, &h, &w, &c);
    int64_t wl = 0, bl = 0;
    if (L->kind == ORC_LAYER_CONV) {
      wl = (int64_t)L->units * L->kh * L->kw * c;
      bl = L->units;
    } else if (L->kind == ORC_LAYER_POOL) {
      bl = L->pool_bias ? c : 0;
    } else {
      wl = (int64_t)L->units * h * w * c;
      bl = L->units;
    }
    w_off[i] = off;
    w_len[i] = wl;
    off += wl;
    b_off[i] = off;
    b_len[i] = bl;
    off += bl;
  }
  free(shapes);
  return ORC_OK;
}

int64_t orc_net_num_params(const orc_net* net) {
  const int n = net->nlayers > 0 ? net->nlayers : 1;
  int64_t* a = (int64_t*)malloc(sizeof(int64_t) * 4 * (size_t)n);
  if (orc_net_param_layout(net, a, a + n, a + 2 * n, a + 3 * n)) {
    free(a);
    return -1;
  }
  int64_t total = 0;
  for (int i = 0; i < net->nlayers; ++i) total += a[n + i] + a[3 * n + i];
  free(a);
  return total;
}

/* build_network (network.hpp:102-130) + make_conv_layer / make_full_layer
 * (layers.hpp:473-501): one Rng(seed) stream, weights row-major, biases 0. */
int orc_net_init(const orc_net* net, double* params) {
  int* shapes = (int*)malloc(sizeof(int) * 3 * (size_t)(net->nlayers > 0 ? net->nlayers : 1));
  int st = orc_net_chain(net, shapes);
  if (st) {
    free(shapes);
    return st;
  }
  orc_rng rng;
  orc_rng_seed(&rng, net->seed);
  int64_t off = 0;
  for (int i = 0; i < net->nlayers; ++i) {
    const orc_layer* L = &net->layers[i];
    int h, w, c;
    layer_in_shape(net, shapes, i, &h, &w, &c);
    if (L->kind == ORC_LAYER_CONV) {
      const int64_t patch = (int64_t)L->kh * L->kw * c;
      const double fan_in = (double)patch;
      const double fan_out = (double)L->kh * L->kw * L->units;
      const double a = sqrt(6.0 / (fan_in + fan_out));
      const int64_t n = (int64_t)L->units * patch;
      for (int64_t k = 0; k < n; ++k) params[off + k] = orc_rng_uniform_range(&rng, -a, a);
      off += n;
      for (int k = 0; k < L->units; ++k) params[off + k] = 0.0;
      off += L->units;
    } else if (L->kind == ORC_LAYER_POOL) {
      if (L->pool_bias) {
        for (int k = 0; k < c; ++k) params[off + k] = 0.0;
        off += c;
      }
    } else {
      const int in_units = h * w * c;
      const double a = sqrt(6.0 / (double)(in_units + L->units));
      const int64_t n = (int64_t)L->units * in_units;
      for (int64_t k = 0; k < n; ++k) params[off + k] = orc_rng_uniform_range(&rng, -a, a);
      off += n;
      for (int k = 0; k < L->units; ++k) params[off + k] = 0.0;
      off += L->units;
    }
  }
  free(shapes);
  return ORC_OK;
}

int64_t orc_net_trace_size(const orc_net* net, int B) {
  int* shapes = (int*)malloc(sizeof(int) * 3 * (size_t)(net->nlayers > 0 ? net->nlayers : 1));
  if (orc_net_chain(net, shapes)) {
    free(shapes);
    return -1;
  }
  int64_t total = 0;
  for (int i = 0; i < net->nlayers; ++i)
    total += (int64_t)shapes[3 * i] * shapes[3 * i + 1] * shapes[3 * i + 2] * B;
  free(shapes);
  return total;
}

/* Executor<T>::run_assembled (variants.hpp:366-376) with forward_pass
 * (:484-502), conv/pool/full layer forwards (:504-596) and backward_pass
 * (:603-668). */
int orc_net_run_batch(const orc_net* net, int B, const double* params, const double* x,
                      const int* cls, const double* values, int pool_bwd_mode,
                      int compute_grads, double* out, double* loss, double* grads,
                      double* trace, int64_t* args) {
  const int L = net->nlayers;
  if (B < 1) return ORC_ESHAPE;
  if (L < 1) return ORC_ESHAPE;
  int* shapes = (int*)malloc(sizeof(int) * 3 * (size_t)L);
  int st = orc_net_chain(net, shapes);
  if (st) {
    free(shapes);
    return st;
  }
  int64_t* lay = (int64_t*)malloc(sizeof(int64_t) * 4 * (size_t)L);
  orc_net_param_layout(net, lay, lay + L, lay + 2 * L, lay + 3 * L);
  double** acts = (double**)calloc((size_t)L, sizeof(double*));
  int64_t** pargs = (int64_t**)calloc((size_t)L, sizeof(int64_t*));
  int64_t* asz = (int64_t*)calloc((size_t)L, sizeof(int64_t));

  /* ---- forward ---- */
  const double* a = x;
  for (int i = 0; i < L; ++i) {
    const orc_layer* Ly = &net->layers[i];
    int h, w, c;
    layer_in_shape(net, shapes, i, &h, &w, &c);
    const int oh = shapes[3 * i], ow = shapes[3 * i + 1], oc = shapes[3 * i + 2];
    asz[i] = (int64_t)oh * ow * oc * B;
    acts[i] = (double*)malloc(sizeof(double) * (size_t)asz[i]);
    const double* W = params + lay[i];
    const double* bias = params + lay[2 * L + i];
    if (Ly->kind == ORC_LAYER_CONV) {
      orc_conv_forward(B, c, h, w, Ly->units, Ly->kh, Ly->kw, Ly->stride, Ly->act, a, W, bias,
                       acts[i]);
    } else if (Ly->kind == ORC_LAYER_POOL) {
      pargs[i] = (int64_t*)malloc(sizeof(int64_t) * (size_t)asz[i]);
      orc_pool_forward(B, c, h, w, Ly->kh, Ly->kw, Ly->stride, Ly->pool_mode, a, acts[i],
                       pargs[i]);
      if (Ly->pool_bias) {
        const int64_t plane = (int64_t)oh * ow;
        for (int bb = 0; bb < B; ++bb)
          for (int ch = 0; ch < c; ++ch) {
            double* p = acts[i] + ((int64_t)bb * c + ch) * plane;
            for (int64_t k = 0; k < plane; ++k) p[k] += bias[ch];
          }
      }
      apply_activation(Ly->act, acts[i], asz[i]);
    } else {
      orc_full_forward(B, h * w * c, Ly->units, Ly->act, a, W, bias, acts[i]);
    }
    a = acts[i];
  }
  const int64_t out_n = asz[L - 1];
  const int units = (int)(out_n / B);
  if (out) memcpy(out, acts[L - 1], sizeof(double) * (size_t)out_n);
  if (trace) {
    int64_t off = 0;
    for (int i = 0; i < L; ++i) {
      memcpy(trace + off, acts[i], sizeof(double) * (size_t)asz[i]);
      off += asz[i];
    }
  }
  if (args) {
    int64_t off = 0;
    for (int i = 0; i < L; ++i)
      if (net->layers[i].kind == ORC_LAYER_POOL) {
        memcpy(args + off, pargs[i], sizeof(int64_t) * (size_t)asz[i]);
        off += asz[i];
      }
  }

  /* ---- loss + backward ---- */
  if (compute_grads) {
    st = orc_loss_forward(net->loss, B, units, acts[L - 1], cls, values, loss);
    double* grad = NULL;
    if (!st) {
      grad = (double*)malloc(sizeof(double) * (size_t)out_n);
      st = orc_loss_backward(net->loss, B, units, acts[L - 1], cls, values, grad);
    }
    for (int i = L - 1; i >= 0 && !st; --i) {
      const orc_layer* Ly = &net->layers[i];
      int h, w, c;
      layer_in_shape(net, shapes, i, &h, &w, &c);
      const double* in = (i == 0) ? x : acts[i - 1];
      const int64_t in_n = (int64_t)h * w * c * B;
      double* gin = (i > 0) ? (double*)malloc(sizeof(double) * (size_t)in_n) : NULL;
      const double* W = params + lay[i];
      double* gW = grads + lay[i];
      double* gB = grads + lay[2 * L + i];
      if (Ly->kind == ORC_LAYER_CONV) {
        orc_conv_backward(B, c, h, w, Ly->units, Ly->kh, Ly->kw, Ly->stride, Ly->act, in, W,
                          acts[i], grad, gW, gB, gin);
      } else if (Ly->kind == ORC_LAYER_POOL) {
        const int oh = shapes[3 * i], ow = shapes[3 * i + 1];
        apply_activation_grad(Ly->act, acts[i], grad, asz[i]);
        if (Ly->pool_bias) {
          const int64_t plane = (int64_t)oh * ow;
          for (int ch = 0; ch < c; ++ch) gB[ch] = 0.0;
          for (int bb = 0; bb < B; ++bb)
            for (int ch = 0; ch < c; ++ch) {
              const double* p = grad + ((int64_t)bb * c + ch) * plane;
              double acc = 0.0;
              for (int64_t k = 0; k < plane; ++k) acc += p[k];
              gB[ch] += acc;
            }
        }
        if (gin)
          orc_pool_backward(B, c, h, w, Ly->kh, Ly->kw, Ly->stride, Ly->pool_mode, pool_bwd_mode,
                            grad, pargs[i], gin);
      } else {
        orc_full_backward(B, h * w * c, Ly->units, Ly->act, in, W, acts[i], grad, gW, gB, gin);
      }
      free(grad);
      grad = gin;
    }
    free(grad);
  }

  for (int i = 0; i < L; ++i) {
    free(acts[i]);
    free(pargs[i]);
  }
  free(acts);
  free(pargs);
  free(asz);
  free(lay);
  free(shapes);
  return st;
}

/* sgd_step (network.hpp:242-273): v = mom*v + g; w -= lr*v */
void orc_sgd_step(int64_t n, double* w, double* v, const double* g, double lr, double mom) {
  for (int64_t k = 0; k < n; ++k) {
    v[k] = mom * v[k] + g[k];
    w[k] -= lr * v[k];
  }
}

/* synth_bench_data (bench.cpp:29-45): one Rng(seed) stream: inputs U[0,1)
 * NCHW, then labels uniform_int(units) or MSE targets U[0,1). */
int orc_synth_bench_data(const orc_net* net, int B, uint64_t seed, float* x, int* cls,
                         float* values) {
  int* shapes = (int*)malloc(sizeof(int) * 3 * (size_t)(net->nlayers > 0 ? net->nlayers : 1));
  int st = orc_net_chain(net, shapes);
  if (st) {
    free(shapes);
    return st;
  }
  orc_rng rng;
  orc_rng_seed(&rng, seed);
  const int64_t n = (int64_t)net->in_h * net->in_w * net->in_c * B;
  for (int64_t i = 0; i < n; ++i) x[i] = (float)orc_rng_uniform(&rng);
  const int L = net->nlayers;
  const int units = L ? shapes[3 * (L - 1)] * shapes[3 * (L - 1) + 1] * shapes[3 * (L - 1) + 2]
                      : net->in_h * net->in_w * net->in_c;
  if (net->loss == ORC_LOSS_SOFTMAX_CE) {
    for (int b = 0; b < B; ++b) cls[b] = orc_rng_uniform_int(&rng, units);
  } else {
    for (int64_t i = 0; i < (int64_t)units * B; ++i) values[i] = (float)orc_rng_uniform(&rng);
  }
  free(shapes);
  return ORC_OK;
}

/* predict_classes (network.hpp:179-192): ties -> lowest index */
void orc_predict_classes(int B, int units, const double* out, int* cls) {
  for (int b = 0; b < B; ++b) {
    const double* p = out + (int64_t)b * units;
    int best = 0;
    for (int u = 1; u < units; ++u)
      if (p[u] > p[best]) best = u;
    cls[b] = best;
  }
}
