// HP chain elementwise / gather / small-reduction ops of the config-2 (ResNet-50 bs=1)
// and config-3 (BERT-base bs=1, seq 128) inference tenants.
//
// The contractions of those networks run on the tcgen05 GEMM (tc_gemm.cuh, per-op chain
// path); these kernels are the HBM/L2-bound glue between them:
//   im2col_kernel   — NHWC activation [H*W, C] -> conv patch matrix [M_pad, K_pad]
//                     (row = output pixel, column = (ky, kx, c), zero padding / zero pad
//                     rows and columns), the A operand of a conv-as-GEMM;
//   bias_act_kernel — c = act(a + bias[col] (+ residual)) : folded-BN shift + ReLU and
//                     the bottleneck's residual add;
//   maxpool_kernel  — k x k / stride max pooling over NHWC;
//   avgpool_kernel  — global average pooling of [H*W, C] into row 0 (FC input);
//   attn_kernel     — softmax(Q K^T / 8) V per head over a packed [S, 3D] QKV matrix
//                     (head dim 64, S <= 256, no mask: bs = 1 encoder);
//   add_ln_kernel   — c = LayerNorm(a + b) * gamma + beta (BERT post-LN residual).
// All are non-preemptible HP chain kernels: PDL-released by their predecessor, exit
// accounting through cta_exit (the chain's completion record is written by the last one).
// Math is fp32 on bf16 inputs with one RNE rounding at the output, restated in
// oracle/tenant_ref.c (tr_im2col, tr_bias_act, tr_maxpool, tr_avgpool, tr_attention,
// tr_add_ln).
#pragma once

#include "tile_run.cuh"

namespace msdev {

struct HpOpParams {
  TileRun run;
  const __nv_bfloat16* a;
  const __nv_bfloat16* b;     // residual (bias_act, add_ln) or null
  const __nv_bfloat16* bias;  // per-column bias / [gamma | beta]
  __nv_bfloat16* c;
  int m, n;                   // output rows (padded) x columns
  int h, w, cin, kh, kw, stride, pad, ho, wo;  // conv / pool geometry (NHWC, batch 1)
  int flags;                  // bias_act: bit 0 = ReLU
};

constexpr int kHpOpThreads = 256;
constexpr int kAttnMaxS = 256;
constexpr int kAttnRowStride = 66;  // bf16 per smem row of K / V (33 words: conflict-free)
constexpr int kAttnSmemBytes = 2 * kAttnMaxS * kAttnRowStride * 2 + 4 * kAttnMaxS * 4 + 4 * 64 * 4;

__device__ __forceinline__ void hp_op_begin(const HpOpParams& p) {
  if (threadIdx.x == 0) cta_started(p.run);
  if (p.run.hp_ctl) {
    pdl_launch_dependents();
    if (p.run.pdl_wait) pdl_wait();
  }
}

__device__ __forceinline__ void hp_op_end(const HpOpParams& p) {
  __syncthreads();
  if (threadIdx.x == 0) cta_exit(p.run, 0);
}

__device__ __forceinline__ float bf(const __nv_bfloat16 v) { return __bfloat162float(v); }

// ------------------------------------------------------------------ im2col
__global__ void __launch_bounds__(kHpOpThreads) im2col_kernel(const __grid_constant__ HpOpParams p) {
  hp_op_begin(p);
  const long long vec_per_row = p.n / 8;
  const long long total = static_cast<long long>(p.m) * vec_per_row;
  const int kvalid = p.kh * p.kw * p.cin;
  const bool vec_ok = (p.cin % 8) == 0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / vec_per_row);
    const int k0 = static_cast<int>(i - static_cast<long long>(r) * vec_per_row) * 8;
    uint4 out = make_uint4(0, 0, 0, 0);
    if (r < p.ho * p.wo && k0 < kvalid) {
      const int oy = r / p.wo, ox = r - (r / p.wo) * p.wo;
      if (vec_ok) {  // 8 consecutive channels of one tap
        const int tap = k0 / p.cin, ch = k0 - tap * p.cin;
        const int iy = oy * p.stride - p.pad + tap / p.kw, ix = ox * p.stride - p.pad + tap % p.kw;
        if (iy >= 0 && iy < p.h && ix >= 0 && ix < p.w)
          out = *reinterpret_cast<const uint4*>(p.a + (static_cast<long long>(iy) * p.w + ix) * p.cin + ch);
      } else {
        __nv_bfloat16 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int kk = k0 + j;
          v[j] = __float2bfloat16_rn(0.0f);
          if (kk < kvalid) {
            const int tap = kk / p.cin, ch = kk - tap * p.cin;
            const int iy = oy * p.stride - p.pad + tap / p.kw, ix = ox * p.stride - p.pad + tap % p.kw;
            if (iy >= 0 && iy < p.h && ix >= 0 && ix < p.w) v[j] = p.a[(static_cast<long long>(iy) * p.w + ix) * p.cin + ch];
          }
        }
        out = *reinterpret_cast<const uint4*>(v);
      }
    }
    *reinterpret_cast<uint4*>(p.c + static_cast<long long>(r) * p.n + k0) = out;
  }
  hp_op_end(p);
}

// ------------------------------------------------------------------ bias + residual + ReLU
__global__ void __launch_bounds__(kHpOpThreads) bias_act_kernel(const __grid_constant__ HpOpParams p) {
  hp_op_begin(p);
  const long long vec_per_row = p.n / 8;
  const long long total = static_cast<long long>(p.m) * vec_per_row;
  const bool relu = p.flags & 1;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int col = static_cast<int>(i % vec_per_row) * 8;
    const uint4 xv = *reinterpret_cast<const uint4*>(p.a + i * 8);
    const uint4 bv = *reinterpret_cast<const uint4*>(p.bias + col);
    uint4 rv = make_uint4(0, 0, 0, 0);
    if (p.b) rv = *reinterpret_cast<const uint4*>(p.b + i * 8);
    const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&xv);
    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&bv);
    const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&rv);
    uint4 o;
    uint32_t* os = &o.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float v0 = __fadd_rn(__low2float(x2[j]), __low2float(b2[j]));
      float v1 = __fadd_rn(__high2float(x2[j]), __high2float(b2[j]));
      if (p.b) {
        v0 = __fadd_rn(v0, __low2float(r2[j]));
        v1 = __fadd_rn(v1, __high2float(r2[j]));
      }
      if (relu) {
        v0 = fmaxf(v0, 0.0f);
        v1 = fmaxf(v1, 0.0f);
      }
      os[j] = pack_bf16x2(v0, v1);
    }
    *reinterpret_cast<uint4*>(p.c + i * 8) = o;
  }
  hp_op_end(p);
}

// ------------------------------------------------------------------ pooling
__global__ void __launch_bounds__(kHpOpThreads) maxpool_kernel(const __grid_constant__ HpOpParams p) {
  hp_op_begin(p);
  const int vec_per_row = p.cin / 8;
  const long long total = static_cast<long long>(p.m) * vec_per_row;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / vec_per_row);
    const int ch = static_cast<int>(i - static_cast<long long>(r) * vec_per_row) * 8;
    uint4 o = make_uint4(0, 0, 0, 0);
    if (r < p.ho * p.wo) {
      const int oy = r / p.wo, ox = r - (r / p.wo) * p.wo;
      float mx[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) mx[j] = -INFINITY;
      for (int ky = 0; ky < p.kh; ++ky)
        for (int kx = 0; kx < p.kw; ++kx) {
          const int iy = oy * p.stride - p.pad + ky, ix = ox * p.stride - p.pad + kx;
          if (iy < 0 || iy >= p.h || ix < 0 || ix >= p.w) continue;
          const uint4 v = *reinterpret_cast<const uint4*>(p.a + (static_cast<long long>(iy) * p.w + ix) * p.cin + ch);
          const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
          for (int j = 0; j < 8; ++j) mx[j] = fmaxf(mx[j], bf(e[j]));
        }
      uint32_t* os = &o.x;
#pragma unroll
      for (int j = 0; j < 4; ++j) os[j] = pack_bf16x2(mx[2 * j], mx[2 * j + 1]);
    }
    *reinterpret_cast<uint4*>(p.c + static_cast<long long>(r) * p.cin + ch) = o;
  }
  hp_op_end(p);
}

// out[0, c] = mean over the h * w valid input rows; rows 1 .. m-1 = 0 (the FC GEMM's pad rows)
__global__ void __launch_bounds__(kHpOpThreads) avgpool_kernel(const __grid_constant__ HpOpParams p) {
  hp_op_begin(p);
  const int vec_per_row = p.n / 8;
  const long long total = static_cast<long long>(p.m) * vec_per_row;
  const int rows = p.h * p.w;
  const float inv = 1.0f / static_cast<float>(rows);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / vec_per_row);
    const int ch = static_cast<int>(i - static_cast<long long>(r) * vec_per_row) * 8;
    uint4 o = make_uint4(0, 0, 0, 0);
    if (r == 0) {
      float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int q = 0; q < rows; ++q) {
        const uint4 v = *reinterpret_cast<const uint4*>(p.a + static_cast<long long>(q) * p.n + ch);
        const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
        for (int j = 0; j < 8; ++j) s[j] = __fadd_rn(s[j], bf(e[j]));
      }
      uint32_t* os = &o.x;
#pragma unroll
      for (int j = 0; j < 4; ++j) os[j] = pack_bf16x2(__fmul_rn(s[2 * j], inv), __fmul_rn(s[2 * j + 1], inv));
    }
    *reinterpret_cast<uint4*>(p.c + static_cast<long long>(r) * p.n + ch) = o;
  }
  hp_op_end(p);
}

// ------------------------------------------------------------------ attention (bs = 1 encoder)
// Unit = (head, block of 16 query rows); 4 warps x 4 rows.  K_h and V_h of the head are
// staged in shared memory (33-word rows: lane j reads row j conflict-free).
__global__ void __launch_bounds__(128) attn_kernel(const __grid_constant__ HpOpParams p) {
  extern __shared__ __align__(16) unsigned char attn_smem[];
  __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(attn_smem);
  __nv_bfloat16* Vs = Ks + kAttnMaxS * kAttnRowStride;
  float* Ps = reinterpret_cast<float*>(Vs + kAttnMaxS * kAttnRowStride);  // [4 warps][S]
  float* Qs = Ps + 4 * kAttnMaxS;                                          // [4 warps][64]
  hp_op_begin(p);
  const int S = p.m, D = p.n, heads = D / 64, qblocks = S / 16;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const long long ld = 3ll * D;
  const float scale = 0.125f;  // 1 / sqrt(64)
  for (int u = blockIdx.x; u < heads * qblocks; u += gridDim.x) {
    const int hd = u / qblocks, qb = u - hd * qblocks;
    __syncthreads();
    for (int idx = threadIdx.x; idx < S * 32; idx += blockDim.x) {  // bf16 pairs
      const int j = idx / 32, e = (idx & 31) * 2;
      const __nv_bfloat162 kv = *reinterpret_cast<const __nv_bfloat162*>(p.a + j * ld + D + hd * 64 + e);
      const __nv_bfloat162 vv = *reinterpret_cast<const __nv_bfloat162*>(p.a + j * ld + 2 * D + hd * 64 + e);
      *reinterpret_cast<__nv_bfloat162*>(Ks + j * kAttnRowStride + e) = kv;
      *reinterpret_cast<__nv_bfloat162*>(Vs + j * kAttnRowStride + e) = vv;
    }
    __syncthreads();
    float* P = Ps + warp * kAttnMaxS;
    float* Q = Qs + warp * 64;
    for (int rr = 0; rr < 4; ++rr) {
      const int q = qb * 16 + warp * 4 + rr;
      const __nv_bfloat162 qv = *reinterpret_cast<const __nv_bfloat162*>(p.a + q * ld + hd * 64 + lane * 2);
      Q[lane * 2] = __low2float(qv);
      Q[lane * 2 + 1] = __high2float(qv);
      __syncwarp();
      float mx = -INFINITY;
      for (int j = lane; j < S; j += 32) {
        float s = 0.0f;
        const __nv_bfloat16* kr = Ks + j * kAttnRowStride;
#pragma unroll 8
        for (int e = 0; e < 64; e += 2) {
          const __nv_bfloat162 k2 = *reinterpret_cast<const __nv_bfloat162*>(kr + e);
          s = __fmaf_rn(Q[e], __low2float(k2), s);
          s = __fmaf_rn(Q[e + 1], __high2float(k2), s);
        }
        s *= scale;
        P[j] = s;
        mx = fmaxf(mx, s);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      float sum = 0.0f;
      for (int j = lane; j < S; j += 32) {
        const float e = __expf(P[j] - mx);
        P[j] = e;
        sum += e;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      __syncwarp();
      float acc0 = 0.0f, acc1 = 0.0f;
      for (int j = 0; j < S; ++j) {
        const __nv_bfloat162 v2 = *reinterpret_cast<const __nv_bfloat162*>(Vs + j * kAttnRowStride + lane * 2);
        acc0 = __fmaf_rn(P[j], __low2float(v2), acc0);
        acc1 = __fmaf_rn(P[j], __high2float(v2), acc1);
      }
      const float inv = 1.0f / sum;
      *reinterpret_cast<uint32_t*>(p.c + static_cast<long long>(q) * D + hd * 64 + lane * 2) =
          pack_bf16x2(acc0 * inv, acc1 * inv);
      __syncwarp();
    }
  }
  hp_op_end(p);
}

// ------------------------------------------------------------------ residual + LayerNorm
// One row per CTA iteration; n <= 8 * 256 (each thread holds <= 8 values in registers).
__global__ void __launch_bounds__(kHpOpThreads) add_ln_kernel(const __grid_constant__ HpOpParams p) {
  __shared__ float red[2][kHpOpThreads / 32];
  hp_op_begin(p);
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int vecs = p.n / 8;
  const bool act = threadIdx.x < vecs;
  const int col = threadIdx.x * 8;
  for (int r = blockIdx.x; r < p.m; r += gridDim.x) {
    float v[8];
    float s = 0.0f;
    if (act) {
      const uint4 xv = *reinterpret_cast<const uint4*>(p.a + static_cast<long long>(r) * p.n + col);
      const uint4 rv = *reinterpret_cast<const uint4*>(p.b + static_cast<long long>(r) * p.n + col);
      const __nv_bfloat16* xe = reinterpret_cast<const __nv_bfloat16*>(&xv);
      const __nv_bfloat16* re = reinterpret_cast<const __nv_bfloat16*>(&rv);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        v[j] = __fadd_rn(bf(xe[j]), bf(re[j]));
        s += v[j];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[0][warp] = s;
    __syncthreads();
    float tot = 0.0f;
#pragma unroll
    for (int w = 0; w < kHpOpThreads / 32; ++w) tot += red[0][w];
    const float mean = tot / static_cast<float>(p.n);
    float q = 0.0f;
    if (act) {
#pragma unroll
      for (int j = 0; j < 8; ++j) q += (v[j] - mean) * (v[j] - mean);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    if (lane == 0) red[1][warp] = q;
    __syncthreads();
    float var = 0.0f;
#pragma unroll
    for (int w = 0; w < kHpOpThreads / 32; ++w) var += red[1][w];
    const float rstd = rsqrtf(var / static_cast<float>(p.n) + 1e-12f);
    if (act) {
      const uint4 gv = *reinterpret_cast<const uint4*>(p.bias + col);
      const uint4 bv = *reinterpret_cast<const uint4*>(p.bias + p.n + col);
      const __nv_bfloat16* ge = reinterpret_cast<const __nv_bfloat16*>(&gv);
      const __nv_bfloat16* be = reinterpret_cast<const __nv_bfloat16*>(&bv);
      uint4 o;
      uint32_t* os = &o.x;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        os[j] = pack_bf16x2((v[2 * j] - mean) * rstd * bf(ge[2 * j]) + bf(be[2 * j]),
                            (v[2 * j + 1] - mean) * rstd * bf(ge[2 * j + 1]) + bf(be[2 * j + 1]));
      *reinterpret_cast<uint4*>(p.c + static_cast<long long>(r) * p.n + col) = o;
    }
    __syncthreads();  // red[] reused by the next row
  }
  hp_op_end(p);
}

}  // namespace msdev
