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
