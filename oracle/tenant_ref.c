/* ORACLE / TEST INFRASTRUCTURE ONLY — the CPU restatement of the tenant-kernel math.
 *
 * The reference ships no GPU kernels (SURVEY.md §2 "Native / GPU inventory": none);
 * the tenant workloads are defined by SURVEY.md §8(d): bf16 GEMM with fp32
 * accumulation (LP batch GEMM, HP small-GEMM chain), bias+GELU epilogue, and a bf16
 * axpy HBM streamer.  This file states that math in plain C so tests can check the
 * sm_100a kernels (fp32 rel <= 1e-3, bf16 rel <= 1e-2, BASELINE.json north_star), and
 * defines the deterministic synthetic-tensor generator both sides share:
 *   value(seed, tensor, i) = bf16_rne( (2 * u24(splitmix64(hc(hc(seed, tensor), i))) - 1) * scale )
 * with u24(x) = (x >> 40) * 2^-24, hc = hash_combine of common.hpp:57-59.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

static uint64_t sm64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
static uint64_t hc(uint64_t a, uint64_t b) { return sm64(a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2))); }

static float bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static uint16_t f32_to_bf16(float f) { /* round to nearest even; NaN kept quiet */
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

float tr_synth_value(uint64_t seed, uint64_t tensor, uint64_t i, float scale) {
  const uint64_t x = sm64(hc(hc(seed, tensor), i));
  const float u = (float)(x >> 40) * 5.9604644775390625e-08f; /* 2^-24 */
  return (2.0f * u - 1.0f) * scale;
}

void tr_fill_bf16(uint16_t* out, size_t n, uint64_t seed, uint64_t tensor, float scale) {
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) out[i] = f32_to_bf16(tr_synth_value(seed, tensor, i, scale));
}

void tr_bf16_to_f32(const uint16_t* in, float* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = bf16_to_f32(in[i]);
}

/* C[r, :] = sum_k A[r, k] * W[n, k] for the listed rows (A: M x K, W: N x K, both
 * K-contiguous), fp32 accumulate in k order, double-checked in fp64 sum as well. */
void tr_gemm_rows(const uint16_t* A, const uint16_t* W, float* C, int M, int N, int K, const int* rows,
                  int nrows) {
  (void)M;
#pragma omp parallel for schedule(dynamic, 1)
  for (int ri = 0; ri < nrows; ++ri) {
    const int r = rows[ri];
    const uint16_t* a = A + (size_t)r * K;
    for (int n = 0; n < N; ++n) {
      const uint16_t* w = W + (size_t)n * K;
      double acc = 0.0;
      for (int k = 0; k < K; ++k) acc += (double)bf16_to_f32(a[k]) * (double)bf16_to_f32(w[k]);
      C[(size_t)ri * N + n] = (float)acc;
    }
  }
}

/* y <- bf16(fmaf(a, x, y)) over [begin, end) elements. */
void tr_axpy_bf16(uint16_t* y, const uint16_t* x, float a, size_t begin, size_t end) {
#pragma omp parallel for schedule(static)
  for (size_t i = begin; i < end; ++i) y[i] = f32_to_bf16(fmaf(a, bf16_to_f32(x[i]), bf16_to_f32(y[i])));
}

/* SwiGLU of a decode layer: out[m, n] = silu(x[m, n]) * x[m, N + n], x = [M x 2N] bf16,
   fp32 math (the device uses __expf; agreement is within the bf16 tolerance). */
void tr_silu_mul(const uint16_t* x, uint16_t* out, int M, int N) {
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      const float g = bf16_to_f32(x[(size_t)m * 2 * N + n]);
      const float u = bf16_to_f32(x[(size_t)m * 2 * N + N + n]);
      out[(size_t)m * N + n] = f32_to_bf16(g / (1.0f + expf(-g)) * u);
    }
}

/* tanh-approximated GELU of (x + bias[col]) over an M x N bf16 matrix, fp32 math. */
void tr_bias_gelu(const uint16_t* x, const uint16_t* bias, uint16_t* out, int M, int N) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      const float v = bf16_to_f32(x[(size_t)m * N + n]) + bf16_to_f32(bias[n]);
      const float g = 0.5f * v * (1.0f + tanhf(k0 * (v + k1 * v * v * v)));
      out[(size_t)m * N + n] = f32_to_bf16(g);
    }
}

/* ---- config-2 / config-3 tenant glue ops (hp_ops.cuh), NHWC batch 1, fp32 math, RNE out ---- */

/* conv patch matrix: out[m_pad x n_pad], row = output pixel oy*wo+ox, col = (ky*kw+kx)*cin+ch */
void tr_im2col(const uint16_t* in, uint16_t* out, int h, int w, int cin, int kh, int kw, int stride, int pad,
               int m_pad, int n_pad) {
  const int ho = (h + 2 * pad - kh) / stride + 1, wo = (w + 2 * pad - kw) / stride + 1;
  const int kvalid = kh * kw * cin;
  for (int r = 0; r < m_pad; ++r)
    for (int k = 0; k < n_pad; ++k) {
      uint16_t v = 0;
      if (r < ho * wo && k < kvalid) {
        const int oy = r / wo, ox = r % wo, tap = k / cin, ch = k % cin;
        const int iy = oy * stride - pad + tap / kw, ix = ox * stride - pad + tap % kw;
        if (iy >= 0 && iy < h && ix >= 0 && ix < w) v = in[((size_t)iy * w + ix) * cin + ch];
      }
      out[(size_t)r * n_pad + k] = v;
    }
}

/* out = act(x + bias[col] (+ resid)), relu when relu != 0; resid may be NULL */
void tr_bias_act(const uint16_t* x, const uint16_t* bias, const uint16_t* resid, uint16_t* out, int m, int n,
                 int relu) {
  for (int r = 0; r < m; ++r)
    for (int c = 0; c < n; ++c) {
      const size_t i = (size_t)r * n + c;
      float v = bf16_to_f32(x[i]) + bf16_to_f32(bias[c]);
      if (resid) v = v + bf16_to_f32(resid[i]);
      if (relu && v < 0.0f) v = 0.0f;
      out[i] = f32_to_bf16(v);
    }
}

void tr_maxpool(const uint16_t* in, uint16_t* out, int h, int w, int c, int k, int stride, int pad, int m_pad) {
  const int ho = (h + 2 * pad - k) / stride + 1, wo = (w + 2 * pad - k) / stride + 1;
  for (int r = 0; r < m_pad; ++r)
    for (int ch = 0; ch < c; ++ch) {
      float mx = -INFINITY;
      if (r < ho * wo) {
        const int oy = r / wo, ox = r % wo;
        for (int ky = 0; ky < k; ++ky)
          for (int kx = 0; kx < k; ++kx) {
            const int iy = oy * stride - pad + ky, ix = ox * stride - pad + kx;
            if (iy < 0 || iy >= h || ix < 0 || ix >= w) continue;
            const float v = bf16_to_f32(in[((size_t)iy * w + ix) * c + ch]);
            if (v > mx) mx = v;
          }
      } else {
        mx = 0.0f;
      }
      out[(size_t)r * c + ch] = f32_to_bf16(mx);
    }
}

/* out[0, :] = mean over rows of in [rows x n] (fp32 sum in row order); rows 1..m_pad-1 = 0 */
void tr_avgpool(const uint16_t* in, uint16_t* out, int rows, int n, int m_pad) {
  for (int c = 0; c < n; ++c) {
    float s = 0.0f;
    for (int q = 0; q < rows; ++q) s += bf16_to_f32(in[(size_t)q * n + c]);
    out[c] = f32_to_bf16(s * (1.0f / (float)rows));
  }
  for (size_t i = (size_t)n; i < (size_t)m_pad * n; ++i) out[i] = 0;
}

/* ctx[s x d] = per head softmax(Q K^T / 8) V; qkv = [s x 3d] = [Q | K | V], head dim 64;
   fp64 math (the device uses fp32 + __expf: agreement within the bf16 tolerance) */
void tr_attention(const uint16_t* qkv, uint16_t* ctx, int s, int d) {
  const int heads = d / 64;
  const size_t ld = (size_t)3 * d;
#pragma omp parallel for schedule(static)
  for (int hq = 0; hq < heads * s; ++hq) {
    const int hd = hq / s, q = hq % s;
    double p[1024];
    double mx = -1e300, sum = 0.0;
    for (int j = 0; j < s; ++j) {
      double acc = 0.0;
      for (int e = 0; e < 64; ++e)
        acc += (double)bf16_to_f32(qkv[q * ld + hd * 64 + e]) * (double)bf16_to_f32(qkv[j * ld + d + hd * 64 + e]);
      p[j] = acc * 0.125;
      if (p[j] > mx) mx = p[j];
    }
    for (int j = 0; j < s; ++j) {
      p[j] = exp(p[j] - mx);
      sum += p[j];
    }
    for (int e = 0; e < 64; ++e) {
      double acc = 0.0;
      for (int j = 0; j < s; ++j) acc += p[j] * (double)bf16_to_f32(qkv[j * ld + 2 * d + hd * 64 + e]);
      ctx[(size_t)q * d + hd * 64 + e] = f32_to_bf16((float)(acc / sum));
    }
  }
}

/* out = LayerNorm(x + resid) * gamma + beta over rows of n, eps 1e-12 (gb = [gamma | beta]) */
void tr_add_ln(const uint16_t* x, const uint16_t* resid, const uint16_t* gb, uint16_t* out, int m, int n) {
  for (int r = 0; r < m; ++r) {
    double mean = 0.0, var = 0.0;
    for (int c = 0; c < n; ++c)
      mean += (double)(bf16_to_f32(x[(size_t)r * n + c]) + bf16_to_f32(resid[(size_t)r * n + c]));
    mean /= n;
    for (int c = 0; c < n; ++c) {
      const double v = (double)(bf16_to_f32(x[(size_t)r * n + c]) + bf16_to_f32(resid[(size_t)r * n + c])) - mean;
      var += v * v;
    }
    const double rstd = 1.0 / sqrt(var / n + 1e-12);
    for (int c = 0; c < n; ++c) {
      const double v = (double)(bf16_to_f32(x[(size_t)r * n + c]) + bf16_to_f32(resid[(size_t)r * n + c]));
      out[(size_t)r * n + c] =
          f32_to_bf16((float)((v - mean) * rstd * bf16_to_f32(gb[c]) + bf16_to_f32(gb[n + c])));
    }
  }
}

/* Optimizer streamers (LP, config 2/3 training steps), element-wise over [begin, end):
   mode 0 = AdamW (fp32 p, m, v; bf16 g): m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
            p -= lr * (m * c1 / (sqrt(v * c2) + eps) + wd * p)   (c1, c2 = bias corrections)
   mode 1 = SGD momentum: m = mu m + g; p -= lr * (m + wd * p)   (v unused)
   Float math in this exact order (the device kernel uses the same operations, no FMA
   contraction: bit-exact). */
void tr_optim(float* p, float* m, float* v, const uint16_t* g, size_t begin, size_t end, int mode, float lr,
              float b1, float b2, float eps, float wd, float c1, float c2) {
#pragma omp parallel for schedule(static)
  for (size_t i = begin; i < end; ++i) {
    const float gi = bf16_to_f32(g[i]);
    if (mode == 0) {
      const float mi = b1 * m[i] + (1.0f - b1) * gi;
      const float vi = b2 * v[i] + (1.0f - b2) * (gi * gi);
      const float upd = (mi * c1) / (sqrtf(vi * c2) + eps) + wd * p[i];
      m[i] = mi;
      v[i] = vi;
      p[i] = p[i] - lr * upd;
    } else {
      const float mi = b1 * m[i] + gi;
      m[i] = mi;
      p[i] = p[i] - lr * (mi + wd * p[i]);
    }
  }
}
