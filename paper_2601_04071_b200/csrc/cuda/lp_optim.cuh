// LP persistent preemptible optimizer streamer (config-2 / config-3 training steps,
// "+ AdamW EW over 110 M params", "+ SGD ... (25.6 M params)").
//
// Same tile machinery as the axpy streamer (stream_kernels.cuh): ONE CTA per SM with three
// 256-thread streaming groups that claim linear tiles (claim_tile: redo entries first,
// harvest budget), a mirror poller warp, and CTA 0's host poller.  A claimed tile always
// completes (the update is not idempotent), so preempt / resume is exact.  Per element:
//   AdamW (mode 0): fp32 p, m, v and bf16 g -> 14 B read + 12 B written = 26 B
//   SGD momentum (mode 1): fp32 p, m and bf16 g -> 10 B read + 8 B written = 18 B
// Math uses explicitly rounded intrinsics in the order of oracle/tenant_ref.c tr_optim,
// so the result is bit-exact with the C restatement.
#pragma once

#include "stream_kernels.cuh"

namespace msdev {

struct OptimParams {
  TileRun run;
  float* p;
  float* m;
  float* v;
  const __nv_bfloat16* g;
  unsigned long long n;
  int tile_elems;  // multiple of 1024 (256 threads x 4 elements)
  int mode;        // 0 AdamW, 1 SGD momentum
  float lr, b1, b2, eps, wd, c1, c2;
};

__device__ __forceinline__ float4 ld_f4(const float* p) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_f4(float* p, const float4& v) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

__device__ __forceinline__ void optim_elem(const OptimParams& q, float& p, float& m, float& v, float g) {
  if (q.mode == 0) {
    const float mi = __fadd_rn(__fmul_rn(q.b1, m), __fmul_rn(__fsub_rn(1.0f, q.b1), g));
    const float vi = __fadd_rn(__fmul_rn(q.b2, v), __fmul_rn(__fsub_rn(1.0f, q.b2), __fmul_rn(g, g)));
    const float den = __fadd_rn(__fsqrt_rn(__fmul_rn(vi, q.c2)), q.eps);
    const float upd = __fadd_rn(__fdiv_rn(__fmul_rn(mi, q.c1), den), __fmul_rn(q.wd, p));
    m = mi;
    v = vi;
    p = __fsub_rn(p, __fmul_rn(q.lr, upd));
  } else {
    const float mi = __fadd_rn(__fmul_rn(q.b1, m), g);
    m = mi;
    p = __fsub_rn(p, __fmul_rn(q.lr, __fadd_rn(mi, __fmul_rn(q.wd, p))));
  }
}

template <int VPT>  // 4-element vectors per thread per tile
__global__ void __launch_bounds__(kAxpyGroups * kStreamThreads + 64, 1) optim_kernel(const __grid_constant__ OptimParams q) {
  constexpr int GROUPS = kAxpyGroups;
  __shared__ uint32_t preempt, producer_done, tiles_done, groups_left;
  __shared__ long long tile_sh[GROUPS][2];
  constexpr int kStreamWarps = GROUPS * kStreamThreads / 32;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    preempt = 0;
    producer_done = 0;
    tiles_done = 0;
    groups_left = GROUPS;
    cta_started(q.run);
  }
  __syncthreads();
  if (warp == kStreamWarps) {
    if ((threadIdx.x & 31) == 0 && q.run.preemptible) poll_mirror(q.run, &preempt, &producer_done);
  } else if (warp == kStreamWarps + 1) {
    if ((threadIdx.x & 31) == 0 && q.run.preemptible && blockIdx.x == 0) poll_host(q.run, &preempt, &producer_done);
    if ((threadIdx.x & 31) == 0 && q.run.preemptible && blockIdx.x >= 1 && blockIdx.x <= kAuxPollers)
      poll_host_aux(q.run, &preempt, &producer_done, 300u * blockIdx.x);
  } else {
    const int g = warp / (kStreamThreads / 32);
    const int tid = threadIdx.x % kStreamThreads;
    for (int j = 0;; ++j) {
      if (tid == 0) {
        long long t = -1;
        if (!(q.run.preemptible && ld_volatile_smem(&preempt))) t = claim_tile(q.run);
        tile_sh[g][j & 1] = t;
      }
      group_bar<GROUPS>(g);
      const long long t = tile_sh[g][j & 1];
      if (t < 0) break;
      const unsigned long long base = static_cast<unsigned long long>(t) * q.tile_elems;
      float4 pv[VPT], mv[VPT], vv[VPT];
      uint2 gv[VPT];
      bool ok[VPT];
#pragma unroll
      for (int u = 0; u < VPT; ++u) {
        const unsigned long long e = base + (static_cast<unsigned long long>(u) * kStreamThreads + tid) * 4;
        ok[u] = e + 4 <= q.n;
        if (ok[u]) {
          pv[u] = ld_f4(q.p + e);
          mv[u] = ld_f4(q.m + e);
          if (q.mode == 0) vv[u] = ld_f4(q.v + e);
          gv[u] = *reinterpret_cast<const uint2*>(q.g + e);
        }
      }
#pragma unroll
      for (int u = 0; u < VPT; ++u) {
        if (!ok[u]) continue;
        const unsigned long long e = base + (static_cast<unsigned long long>(u) * kStreamThreads + tid) * 4;
        const __nv_bfloat162 g01 = *reinterpret_cast<const __nv_bfloat162*>(&gv[u].x);
        const __nv_bfloat162 g23 = *reinterpret_cast<const __nv_bfloat162*>(&gv[u].y);
        optim_elem(q, pv[u].x, mv[u].x, vv[u].x, __low2float(g01));
        optim_elem(q, pv[u].y, mv[u].y, vv[u].y, __high2float(g01));
        optim_elem(q, pv[u].z, mv[u].z, vv[u].z, __low2float(g23));
        optim_elem(q, pv[u].w, mv[u].w, vv[u].w, __high2float(g23));
        st_f4(q.p + e, pv[u]);
        st_f4(q.m + e, mv[u]);
        if (q.mode == 0) st_f4(q.v + e, vv[u]);
      }
      if (tid == 0) atomicAdd(&tiles_done, 1u);
    }
    if (tid == 0 && atomicSub(&groups_left, 1u) == 1u) st_volatile_smem(&producer_done, 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) cta_exit(q.run, tiles_done);
}

// Deterministic fp32 fill (optimizer state / master weights): the bf16 synthetic value,
// widened (oracle: tr_synth_value rounded through bf16).
__global__ void synth_fill_f32_kernel(float* out, unsigned long long n, unsigned long long seed,
                                      unsigned long long tensor, float scale) {
  const uint64_t base = d_hash_combine(seed, tensor);
  for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const uint64_t x = d_splitmix64(d_hash_combine(base, i));
    const float u = static_cast<float>(x >> 40) * 5.9604644775390625e-08f;
    out[i] = __bfloat162float(__float2bfloat16_rn(__fmul_rn(__fsub_rn(__fmul_rn(2.0f, u), 1.0f), scale)));
  }
}

}  // namespace msdev
