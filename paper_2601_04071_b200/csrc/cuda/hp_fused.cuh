// Fused HP chain: one persistent launch runs a whole HP segment (the
// config-1 decode step: 4 x skinny GEMM [128 x 4096] * [4096 x 4096]^T + bias/GELU).
//
// Why: as separate kernels each 32 MB weight stream paid ~5 us of launch/drain and a
// cold start (HBM latency with an empty pipeline), so the chain ran at ~1 TB/s and
// co-location (an L2 the LP just flushed) cost it another ~40 us.  Here the weights of
// op i+1 stream while op i finishes: the producer issues B (weights do not depend on the
// previous op) into free smem stages and L2-prefetches the rest of its next unit before
// it waits for op i's output, and ops are separated by grid-wide phase counters instead
// of kernel boundaries.  All CTAs are co-resident (grid <= SMs, 1 CTA/SM), so the phase
// waits cannot deadlock; the HP stream is never preempted.
//
// Work decomposition of a GEMM op (BN = 128): unit u = (tile u / split, k-slice u % split),
// unit u runs on CTA u % grid.  split > 1: every unit writes an fp32 partial (coalesced
// [BN/4][128] float4 layout), then after a phase barrier all CTAs reduce the slices in
// slice order (deterministic) into bf16 C.  BIAS_GELU: a grid-stride elementwise phase.
//
// Warp roles as in tc_gemm.cuh (0 producer, 1 MMA, 2 TMEM alloc, 4-7 epilogue + phases).
#pragma once

#include "tc_gemm.cuh"

namespace msdev {

#ifndef MS_FUSED_MAX_STAGES
#define MS_FUSED_MAX_STAGES 8  // ring depth cap (A/B builds: make NVEXTRA=-DMS_FUSED_MAX_STAGES=n)
#endif

constexpr int kFusedMaxOps = 96;
constexpr int kFusedBN = 128;
constexpr int kFusedGemm = 1;
constexpr int kFusedBiasGelu = 2;
constexpr int kFusedSiluMul = 5;
constexpr int kFusedAbsorbed = 6;  // BIAS_GELU computed by the previous GEMM's epilogue (gelu_c)

// Scalar description of one op; copied into shared memory at kernel start (the grid-phase
// acquires invalidate L1, so re-reading these from global on every use costs L2 trips).
struct FusedOpDesc {
  int kind;
  int m, n, k;
  int tiles_m, tiles_n, split, kb_per_unit, units;
  int b_kmajor;
  int swiglu;       // GEMM whose 128-column tiles hold [64 gate | 64 up] features (n = output cols)
  int in_phase;     // phase whose completion makes this op's input readable (-1: chain input)
  int mma_phase;    // GEMM: every unit's epilogue done (C or partials written)
  int ready_phase;  // output complete
  __nv_bfloat16* c;
  float* ws;
  const __nv_bfloat16* x;  // BIAS_GELU input
  const __nv_bfloat16* bias;
  __nv_bfloat16* gelu_c;            // GEMM (cluster epilogue): also store gelu(C + gelu_bias) here
  const __nv_bfloat16* gelu_bias;
};

struct alignas(64) FusedOp {
  CUtensorMap tma_a;
  CUtensorMap tma_b;
  FusedOpDesc d;
};

// Shared-memory plan.  CS > 1: the k-slices of a tile run on the CS CTAs of one thread-
// block cluster and are reduced through distributed shared memory (no fp32 partials in
// HBM/L2, no extra grid phase): CTA rank r owns output columns [r*W, r*W + W), W = BN/CS,
// and receives the other CS-1 slices of that strip into `recv` with st.async.
template <int CS, int BN = kFusedBN>
struct FusedCfg {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStripCols = BN / CS;
  static constexpr int kRecvSliceBytes = CS > 1 ? kBM * kStripCols * 4 : 0;
  static constexpr int kRecvBytes = CS > 1 ? (CS - 1) * kRecvSliceBytes : 0;
  static constexpr int kStagesRaw = (220 * 1024 - kRecvBytes) / kStageBytes;
  static constexpr int kStages = kStagesRaw > MS_FUSED_MAX_STAGES ? MS_FUSED_MAX_STAGES : kStagesRaw;
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + kRecvBytes + 1024;
  static constexpr uint32_t kIdesc = umma_idesc_bf16(kBM, BN);
  static_assert(CS == 1 || CS == 2 || CS == 4, "cluster split must be 1, 2 or 4");
};

struct FusedProgram {
  FusedOp ops[kFusedMaxOps];
  int n_ops;
  int n_phases;
  int l2_prefetch;  // warm the L2 with the next op's weights (1) or not (0)
};

// Kernel parameters (constant bank): the op descriptors live here rather than in global or
// shared memory — reads go through the constant cache, which the grid-phase acquires do not
// invalidate, and the compiler may re-load them freely instead of pinning registers.
struct FusedParams {
  TileRun run;  // HP bookkeeping (first-CTA stamp, completion record, phase-counter reset)
  const FusedProgram* prog;  // tensor maps (global memory, 64 B aligned)
  uint32_t* phase_cnt;
  int n_ops;
  int l2_prefetch;
  int full_fence;  // 1: __threadfence before each phase release (MS_FUSED_FULL_FENCE=1; default 0)
  FusedOpDesc ops[kFusedMaxOps];
};

__device__ __forceinline__ void fused_unit_coords(const FusedOpDesc& o, int u, int& mb, int& nb, int& kb0) {
  const int tile = u / o.split;
  mb = tile % o.tiles_m;
  nb = tile / o.tiles_m;
  kb0 = (u % o.split) * o.kb_per_unit;
}

__device__ __forceinline__ void phase_wait(const uint32_t* cnt, uint32_t target) {
  while (ld_acquire_gpu(cnt) < target) __nanosleep(32);
}

// Epilogue-warp group (128 threads, named barrier 1): publish this CTA's part of a phase.
// The release reduction alone orders the group's writes (bar.sync makes them precede the
// leader's release, which is cumulative); `full_fence` adds the older __threadfence
// (MEMBAR.SC.GPU) in front of it.
__device__ __forceinline__ void group_arrive(uint32_t* cnt, bool leader, const TileRun* run = nullptr, int slot = 0,
                                             bool full_fence = true) {
  fence_proxy_async_global();  // results may be read by other CTAs' TMA loads
  if (leader && run) dbg_stamp_ext(*run, slot);
  asm volatile("bar.sync 1, 128;" ::: "memory");
  if (leader) {
    if (run) dbg_stamp_ext(*run, slot + 1);
    if (full_fence) __threadfence();
    if (run) dbg_stamp_ext(*run, slot + 2);
    red_release_gpu_add(cnt, 1u);
  }
}
__device__ __forceinline__ void group_wait(const uint32_t* cnt, uint32_t target, bool leader) {
  if (leader) phase_wait(cnt, target);
  asm volatile("bar.sync 1, 128;" ::: "memory");
}

// ---- grid phases (epilogue warps, 128 threads per CTA).  Each thread owns items
// blockIdx.x * 128 + t + b * G * 128; all loads of a batch are issued before the first
// add so one L2 latency covers the batch (the phases are latency-, not bandwidth-bound).
template <int BN>
__device__ __forceinline__ void reduce_store(const FusedOpDesc& o, int i, const float4& x) {
  constexpr int quads = BN / 4;
  const int row = i % kBM;
  const int tq = i / kBM;
  const int cq = tq % quads;
  const int tile = tq / quads;
  const int mb = tile % o.tiles_m, nb = tile / o.tiles_m;
  uint2 out;
  out.x = pack_bf16x2(x.x, x.y);
  out.y = pack_bf16x2(x.z, x.w);
  *reinterpret_cast<uint2*>(o.c + static_cast<size_t>(mb * kBM + row) * o.n + static_cast<size_t>(nb) * BN + cq * 4) = out;
}
template <int BN>
__device__ __forceinline__ const float4* reduce_src(const FusedOpDesc& o, int i) {
  constexpr int quads = BN / 4;
  const int row = i % kBM;
  const int tq = i / kBM;
  const int cq = tq % quads;
  const int tile = tq / quads;
  return reinterpret_cast<const float4*>(o.ws) + static_cast<size_t>(tile) * o.split * (kBM * quads) +
         static_cast<size_t>(cq) * kBM + row;
}

template <int SPLIT, int B, int BN>
__device__ __forceinline__ void reduce_slices(const FusedOpDesc& o, int t, int G) {
  constexpr size_t slice_stride = kBM * BN / 4;
  const int total = o.tiles_m * o.tiles_n * (BN / 4) * kBM;
  const int step = G * 128;
  for (int i0 = blockIdx.x * 128 + t; i0 < total; i0 += step * B) {
    float4 v[B][SPLIT];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int i = i0 + b * step;
      if (i < total) {
        const float4* src = reduce_src<BN>(o, i);
#pragma unroll
        for (int sl = 0; sl < SPLIT; ++sl) v[b][sl] = src[sl * slice_stride];
      }
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int i = i0 + b * step;
      if (i < total) {
        float4 x = v[b][0];
#pragma unroll
        for (int sl = 1; sl < SPLIT; ++sl) {  // slice order: deterministic
          x.x += v[b][sl].x; x.y += v[b][sl].y; x.z += v[b][sl].z; x.w += v[b][sl].w;
        }
        reduce_store<BN>(o, i, x);
      }
    }
  }
}

template <int BN>
__device__ __forceinline__ void reduce_slices_any(const FusedOpDesc& o, int t, int G) {
  constexpr size_t slice_stride = kBM * BN / 4;
  const int total = o.tiles_m * o.tiles_n * (BN / 4) * kBM;
  for (int i = blockIdx.x * 128 + t; i < total; i += G * 128) {
    const float4* src = reduce_src<BN>(o, i);
    float4 x = src[0];
    for (int sl = 1; sl < o.split; ++sl) {
      const float4 u = src[sl * slice_stride];
      x.x += u.x; x.y += u.y; x.z += u.z; x.w += u.w;
    }
    reduce_store<BN>(o, i, x);
  }
}

// BIAS_GELU (tanh form; same arithmetic as bias_gelu_kernel and oracle tr_bias_gelu).
__device__ __forceinline__ void bias_gelu_phase(const FusedOpDesc& o, int t, int G) {
  constexpr int B = 4;
  const long long chunks = static_cast<long long>(o.m) * o.n / 8;
  const long long step = static_cast<long long>(G) * 128;
  for (long long i0 = static_cast<long long>(blockIdx.x) * 128 + t; i0 < chunks; i0 += step * B) {
    uint4 xv[B], bv[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const long long i = i0 + b * step;
      if (i < chunks) {
        xv[b] = *reinterpret_cast<const uint4*>(o.x + i * 8);
        bv[b] = *reinterpret_cast<const uint4*>(o.bias + (i * 8) % o.n);
      }
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const long long i = i0 + b * step;
      if (i >= chunks) continue;
      const uint32_t* xs = &xv[b].x;
      const uint32_t* bs = &bv[b].x;
      uint4 out;
      uint32_t* os = &out.x;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const __nv_bfloat162 x2 = *reinterpret_cast<const __nv_bfloat162*>(&xs[e]);
        const __nv_bfloat162 b2 = *reinterpret_cast<const __nv_bfloat162*>(&bs[e]);
        os[e] = pack_bf16x2(bias_gelu_tanh(__low2float(x2), __low2float(b2)),
                            bias_gelu_tanh(__high2float(x2), __high2float(b2)));
      }
      *reinterpret_cast<uint4*>(o.c + i * 8) = out;
    }
  }
}

// k-slice exchange of one unit through distributed shared memory.  (Through L2 instead —
// global stores, a release reduction per destination, acquire + loads — measured 64 vs 57 us
// per config-1 chain: the 48 KB of stores + release per CTA took 5.9 us against 3.0 us over
// DSMEM, competing with the next op's weight stream for L2; profiles/r02c_fused_xchg_*.txt.)
template <int CS>
__device__ __forceinline__ void exchange_dsmem(uint32_t tmem_row, uint8_t* recv, uint64_t* recv_full,
                                               uint32_t recv_parity, uint32_t r, int row, bool leader,
                                               const TileRun& run, int oi, float (&out)[FusedCfg<CS>::kStripCols]) {
  using Cfg = FusedCfg<CS>;
  constexpr int W = Cfg::kStripCols;
  constexpr int kChunks = W / 4;
  if (leader) mbar_arrive_expect_tx(recv_full, static_cast<uint32_t>(Cfg::kRecvBytes));
  const uint32_t recv_local = smem_u32(recv);
  const uint32_t bar_local = smem_u32(recv_full);
#pragma unroll 1
  for (uint32_t dq = 1; dq < CS; ++dq) {
    const uint32_t dst = (r + dq) % CS;               // destination rank
    const uint32_t slot = r < dst ? r : r - 1;        // my slot in its receive buffer
    const uint32_t rbase = mapa_shared(recv_local, dst) + slot * Cfg::kRecvSliceBytes + row * (W * 4);
    const uint32_t rbar = mapa_shared(bar_local, dst);
#pragma unroll
    for (int cc = 0; cc < W / 32; ++cc) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tmem_row + dst * W + cc * 32, v);
      tmem_ld_wait();
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int chunk = cc * 8 + k;
        const int swz = (chunk & ~7) | ((chunk ^ row) & 7);
        st_async_v4(rbase + swz * 16, v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3], rbar);
      }
    }
  }
  // own strip stays in registers
  float acc[W];
  {
#pragma unroll
    for (int cc = 0; cc < W / 32; ++cc) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tmem_row + r * W + cc * 32, v);
      tmem_ld_wait();
#pragma unroll
      for (int k = 0; k < 32; ++k) acc[cc * 32 + k] = __uint_as_float(v[k]);
    }
  }
  if (leader) dbg_stamp_ext(run, 40 + oi * 6 + 0);
  mbar_wait(recv_full, recv_parity);
  if (leader) dbg_stamp_ext(run, 40 + oi * 6 + 1);
  // slice order 0..CS-1 (bit-identical to the global-partial reduction)
#pragma unroll
  for (int i = 0; i < W; ++i) out[i] = 0.f;
#pragma unroll
  for (uint32_t sl = 0; sl < CS; ++sl) {
    if (sl == r) {
#pragma unroll
      for (int i = 0; i < W; ++i) out[i] = sl == 0 ? acc[i] : out[i] + acc[i];
    } else {
      const uint32_t slot = sl < r ? sl : sl - 1;
      const uint8_t* src = recv + slot * Cfg::kRecvSliceBytes + row * (W * 4);
#pragma unroll
      for (int chunk = 0; chunk < kChunks; ++chunk) {
        const int swz = (chunk & ~7) | ((chunk ^ row) & 7);
        const float4 x = *reinterpret_cast<const float4*>(src + swz * 16);
        if (sl == 0) {
          out[4 * chunk] = x.x; out[4 * chunk + 1] = x.y; out[4 * chunk + 2] = x.z; out[4 * chunk + 3] = x.w;
        } else {
          out[4 * chunk] += x.x; out[4 * chunk + 1] += x.y; out[4 * chunk + 2] += x.z; out[4 * chunk + 3] += x.w;
        }
      }
    }
  }
}

// Cluster-mode epilogue of one unit (CS > 1): send the other ranks' strips of this CTA's
// fp32 partial, sum the received slices with its own strip in slice order, store bf16.
template <int CS>
__device__ __forceinline__ void cluster_epilogue(const FusedOpDesc& o, int u, uint32_t tmem_row, uint8_t* recv,
                                                 uint64_t* recv_full, uint32_t recv_parity, int q, int lane,
                                                 bool leader, const TileRun& run, int oi) {
  using Cfg = FusedCfg<CS>;
  constexpr int W = Cfg::kStripCols;
  const uint32_t r = cluster_ctarank();
  const int row = q * 32 + lane;
  int mb, nb, kb0;
  fused_unit_coords(o, u, mb, nb, kb0);
  uint4 gbias[W / 8];  // bias strip of the absorbed gelu op: its L2 trips overlap the exchange
  if (o.gelu_c) {
#pragma unroll
    for (int v = 0; v < W / 8; ++v)
      gbias[v] = *reinterpret_cast<const uint4*>(o.gelu_bias + static_cast<size_t>(nb) * kFusedBN + r * W + 8 * v);
  }
  float out[W];
  exchange_dsmem<CS>(tmem_row, recv, recv_full, recv_parity, r, row, leader, run, oi, out);
  uint4* dst = reinterpret_cast<uint4*>(o.c + static_cast<size_t>(mb * kBM + row) * o.n +
                                        static_cast<size_t>(nb) * kFusedBN + r * W);
#pragma unroll
  for (int v = 0; v < W / 8; ++v) {
    uint4 w;
    w.x = pack_bf16x2(out[8 * v + 0], out[8 * v + 1]);
    w.y = pack_bf16x2(out[8 * v + 2], out[8 * v + 3]);
    w.z = pack_bf16x2(out[8 * v + 4], out[8 * v + 5]);
    w.w = pack_bf16x2(out[8 * v + 6], out[8 * v + 7]);
    dst[v] = w;
    if (o.gelu_c) {  // the chain's next op, gelu(C + bias), on the bf16-rounded C as the phase does
      const size_t col = static_cast<size_t>(nb) * kFusedBN + r * W + 8 * v;
      const uint32_t* ws = &w.x;
      const uint32_t* bs = &gbias[v].x;
      uint4 g;
      uint32_t* gs = &g.x;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const __nv_bfloat162 x2 = *reinterpret_cast<const __nv_bfloat162*>(&ws[e]);
        const __nv_bfloat162 b2 = *reinterpret_cast<const __nv_bfloat162*>(&bs[e]);
        gs[e] = pack_bf16x2(bias_gelu_tanh(__low2float(x2), __low2float(b2)),
                            bias_gelu_tanh(__high2float(x2), __high2float(b2)));
      }
      reinterpret_cast<uint4*>(o.gelu_c + static_cast<size_t>(mb * kBM + row) * o.n + col)[0] = g;
    }
  }
}

// SILU_MUL: out[r, j] = silu(x[r, j]) * x[r, n + j] (x = [m x 2n]); same arithmetic as
// silu_mul_kernel and oracle tr_silu_mul.
__device__ __forceinline__ void silu_mul_phase(const FusedOpDesc& o, int t, int G) {
  constexpr int B = 4;  // chunks in flight per thread
  const int chunks = o.m * o.n / 8;
  const int cpr = o.n / 8;  // chunks per output row
  const int step = G * 128;
  for (int i0 = blockIdx.x * 128 + t; i0 < chunks; i0 += step * B) {
    uint4 gv[B], uv[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int i = i0 + b * step;
      if (i < chunks) {
        const int row = i / cpr, c = (i - row * cpr) * 8;
        gv[b] = *reinterpret_cast<const uint4*>(o.x + static_cast<size_t>(row) * 2 * o.n + c);
        uv[b] = *reinterpret_cast<const uint4*>(o.x + static_cast<size_t>(row) * 2 * o.n + o.n + c);
      }
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int i = i0 + b * step;
      if (i >= chunks) continue;
      const int row = i / cpr, c = (i - row * cpr) * 8;
      const uint32_t* gs = &gv[b].x;
      const uint32_t* us = &uv[b].x;
      uint4 out;
      uint32_t* os = &out.x;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const __nv_bfloat162 g2 = *reinterpret_cast<const __nv_bfloat162*>(&gs[e]);
        const __nv_bfloat162 u2 = *reinterpret_cast<const __nv_bfloat162*>(&us[e]);
        os[e] = pack_bf16x2(silu_mul(__low2float(g2), __low2float(u2)), silu_mul(__high2float(g2), __high2float(u2)));
      }
      *reinterpret_cast<uint4*>(o.c + static_cast<size_t>(row) * o.n + c) = out;
    }
  }
}

template <int CS, int BN = kFusedBN>
__global__ void __launch_bounds__(256, 1) hp_fused_kernel(const __grid_constant__ FusedParams p) {
  using Cfg = FusedCfg<CS, BN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + S * Cfg::kABytes;
  uint8_t* recv = smem + S * Cfg::kStageBytes;
  GemmSmemCtl* s = reinterpret_cast<GemmSmemCtl*>(recv + Cfg::kRecvBytes);
  uint64_t* recv_full = &s->mma_drain;  // (no drain in the HP chain) cluster receive barrier
  const FusedProgram& prog = *p.prog;
  const int n_ops = p.n_ops;
  const int G = static_cast<int>(gridDim.x);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    dbg_stamp(p.run, 7);
    for (int i = 0; i < S; ++i) {
      mbar_init(&s->full[i], 1);
      mbar_init(&s->empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s->tmem_full[i], 1);
      mbar_init(&s->tmem_empty[i], 1);
    }
    mbar_init(recv_full, 1);
    fence_mbar_init();
    cta_started(p.run);
  }
  for (int i = threadIdx.x; i < n_ops; i += blockDim.x)
    if (p.ops[i].kind == kFusedGemm) {
      prefetch_tmap(&prog.ops[i].tma_a);
      prefetch_tmap(&prog.ops[i].tma_b);
    }
  if (warp == 2) tmem_alloc(&s->tmem_base, Cfg::kTmemCols);
  tc_fence_before();
  if constexpr (CS > 1) cluster_sync_all();  // peers' barriers initialised before any st.async
  else __syncthreads();
  tc_fence_after();
  if (p.run.pdl_wait) pdl_wait();
  const uint32_t tmem_base = s->tmem_base;

  if (warp == 0) {
    // ===================== TMA producer (runs ahead across ops) =====================
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (int oi = 0; oi < n_ops; ++oi) {
        const FusedOpDesc& o = p.ops[oi];
        if (o.kind != kFusedGemm) continue;
        const CUtensorMap* tma_a = &prog.ops[oi].tma_a;
        const CUtensorMap* tma_b = &prog.ops[oi].tma_b;
        bool a_ready = o.in_phase < 0;
        const int dslot = oi * 8;
        dbg_stamp_ext(p.run, dslot + 0);
        for (int u = blockIdx.x; u < o.units; u += G) {
          int mb, nb, kb0;
          fused_unit_coords(o, u, mb, nb, kb0);
          // Stages whose weights were issued before the op's input was ready.
          uint32_t d_stage = stage;
          int d_kb = 0, deferred = 0;
          for (int kb = 0; kb < o.kb_per_unit; ++kb) {
            if (!a_ready && deferred == S) {
              phase_wait(p.phase_cnt + o.in_phase, static_cast<uint32_t>(G));
              dbg_stamp_ext(p.run, dslot + 1);
              fence_proxy_async_global();
              for (int i = 0; i < deferred; ++i) {
                tma_load_2d(smem_a + d_stage * Cfg::kABytes, tma_a, &s->full[d_stage], (kb0 + d_kb + i) * kBK,
                            mb * kBM);
                if (++d_stage == S) d_stage = 0;
              }
              a_ready = true;
            }
            mbar_wait(&s->empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&s->full[stage], Cfg::kStageBytes);
            if (o.b_kmajor)
              tma_load_3d(smem_b + stage * Cfg::kBBytes, tma_b, &s->full[stage], 0, nb * BN, kb0 + kb);
            else
              tma_load_2d(smem_b + stage * Cfg::kBBytes, tma_b, &s->full[stage], (kb0 + kb) * kBK, nb * BN);
            if (a_ready)
              tma_load_2d(smem_a + stage * Cfg::kABytes, tma_a, &s->full[stage], (kb0 + kb) * kBK, mb * kBM);
            else
              ++deferred;
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
          }
          if (!a_ready) {  // unit shorter than the ring
            phase_wait(p.phase_cnt + o.in_phase, static_cast<uint32_t>(G));
            fence_proxy_async_global();
            for (int i = 0; i < deferred; ++i) {
              tma_load_2d(smem_a + d_stage * Cfg::kABytes, tma_a, &s->full[d_stage], (kb0 + d_kb + i) * kBK,
                          mb * kBM);
              if (++d_stage == S) d_stage = 0;
            }
            a_ready = true;
          }
        }
        dbg_stamp_ext(p.run, dslot + 2);
        // This CTA's loads of op oi are all issued: warm the L2 with the weights of its
        // units in the next GEMM op (their HBM latency overlaps op oi's tail + phases).
        for (int oj = oi + 1; oj < n_ops && p.l2_prefetch; ++oj) {
          const FusedOpDesc& q = p.ops[oj];
          if (q.kind != kFusedGemm) continue;
          const CUtensorMap* qtma_b = &prog.ops[oj].tma_b;
          for (int u = blockIdx.x; u < q.units; u += G) {
            int mb, nb, kb0;
            fused_unit_coords(q, u, mb, nb, kb0);
            for (int kb = S; kb < q.kb_per_unit; ++kb) {  // the first S go straight to smem
              if (q.b_kmajor)
                tma_prefetch_l2_3d(qtma_b, 0, nb * BN, kb0 + kb);
              else
                tma_prefetch_l2_2d(qtma_b, (kb0 + kb) * kBK, nb * BN);
            }
          }
          break;
        }
      }
    }
  } else if (warp == 1) {
    // ===================== UMMA issuer =====================
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      int j = 0;
      for (int oi = 0; oi < n_ops; ++oi) {
        const FusedOpDesc& o = p.ops[oi];
        if (o.kind != kFusedGemm) continue;
        for (int u = blockIdx.x; u < o.units; u += G, ++j) {
          const int slot = j & 1;
          if (j >= 2) mbar_wait(&s->tmem_empty[slot], ((j >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(slot * BN);
          for (int kb = 0; kb < o.kb_per_unit; ++kb) {
            mbar_wait(&s->full[stage], phase);
            tc_fence_after();
            if (kb == 0) dbg_stamp_ext(p.run, oi * 8 + 3);
            const uint64_t a0 = umma_desc_k_sw128(smem_u32(smem_a + stage * Cfg::kABytes));
            const uint64_t b0 = umma_desc_k_sw128(smem_u32(smem_b + stage * Cfg::kBBytes));
#pragma unroll
            for (int k = 0; k < kBK / kUmmaK; ++k)
              umma_bf16(d_tmem, a0 + 2ull * k, b0 + 2ull * k, Cfg::kIdesc, (kb | k) != 0 ? 1u : 0u);
            umma_commit(&s->empty[stage]);
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit(&s->tmem_full[slot]);
          dbg_stamp_ext(p.run, oi * 8 + 4);
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue + grid phases =====================
    const int q = warp - 4;
    const int t = threadIdx.x - 128;  // 0..127
    const bool leader = t == 0;
    int j = 0;
    uint32_t recv_parity = 0;
    for (int oi = 0; oi < n_ops; ++oi) {
      const FusedOpDesc& o = p.ops[oi];
      if constexpr (CS > 1) {
        if (o.kind == kFusedGemm && o.split > 1) {
          // one unit per CTA per op (host plan), slices of a tile = the CTAs of a cluster
          const int u = blockIdx.x;
          if (u < o.units) {
            const int slot = j & 1;
            mbar_wait(&s->tmem_full[slot], (j >> 1) & 1);
            tc_fence_after();
            if (leader) dbg_stamp_ext(p.run, oi * 8 + 5);
            const uint32_t tmem_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(slot * BN);
            cluster_epilogue<CS>(o, u, tmem_row, recv, recv_full, recv_parity, q, lane, leader, p.run, oi);
            recv_parity ^= 1;
            tc_fence_before();
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (leader) mbar_arrive(&s->tmem_empty[slot]);
            ++j;
          }
          if (leader) dbg_stamp_ext(p.run, oi * 8 + 6);
          group_arrive(p.phase_cnt + o.ready_phase, leader, &p.run, 40 + oi * 6 + 2, p.full_fence);
          if (leader) dbg_stamp_ext(p.run, oi * 8 + 7);
          continue;
        }
      }
      if (o.kind == kFusedGemm) {
        for (int u = blockIdx.x; u < o.units; u += G, ++j) {
          const int slot = j & 1;
          mbar_wait(&s->tmem_full[slot], (j >> 1) & 1);
          tc_fence_after();
          if (leader) dbg_stamp_ext(p.run, oi * 8 + 5);
          int mb, nb, kb0;
          fused_unit_coords(o, u, mb, nb, kb0);
          const int row_in_tile = q * 32 + lane;
          const uint32_t trow = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(slot * BN);
          if (BN == kFusedBN && o.swiglu) {  // (narrow plans never carry SwiGLU ops)
            // columns [0, 64) = gate, [64, 128) = up of output features [64 nb, 64 nb + 64)
            __nv_bfloat16* crow = o.c + static_cast<size_t>(mb * kBM + row_in_tile) * o.n + static_cast<size_t>(nb) * 64;
#pragma unroll 1
            for (int c0 = 0; c0 < 64; c0 += 32) {
              uint32_t g[32], u[32];
              tmem_ld_32x32b_x32(trow + c0, g);
              tmem_ld_32x32b_x32(trow + 64 + c0, u);
              tmem_ld_wait();
              uint4* dst = reinterpret_cast<uint4*>(crow + c0);
#pragma unroll
              for (int v = 0; v < 4; ++v) {
                uint32_t w[4];
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  w[e] = pack_bf16x2(silu_mul(__uint_as_float(g[8 * v + 2 * e]), __uint_as_float(u[8 * v + 2 * e])),
                                     silu_mul(__uint_as_float(g[8 * v + 2 * e + 1]), __uint_as_float(u[8 * v + 2 * e + 1])));
                dst[v] = make_uint4(w[0], w[1], w[2], w[3]);
              }
            }
          } else {
          __nv_bfloat16* crow = o.c + static_cast<size_t>(mb * kBM + row_in_tile) * o.n + static_cast<size_t>(nb) * BN;
          float4* wunit = o.split > 1 ? reinterpret_cast<float4*>(o.ws) + static_cast<size_t>(u) * (kBM * BN / 4) : nullptr;
#pragma unroll 1
          for (int c0 = 0; c0 < BN; c0 += 32) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(trow + c0, r);
            tmem_ld_wait();
            if (CS == 1 && o.split > 1) {  // (cluster launches reduce k-slices in DSMEM)
#pragma unroll
              for (int v = 0; v < 8; ++v)
                wunit[static_cast<size_t>(c0 / 4 + v) * kBM + row_in_tile] =
                    make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
            } else {
              uint4* dst = reinterpret_cast<uint4*>(crow + c0);
#pragma unroll
              for (int v = 0; v < 4; ++v) {
                uint4 w;
                w.x = pack_bf16x2(__uint_as_float(r[8 * v + 0]), __uint_as_float(r[8 * v + 1]));
                w.y = pack_bf16x2(__uint_as_float(r[8 * v + 2]), __uint_as_float(r[8 * v + 3]));
                w.z = pack_bf16x2(__uint_as_float(r[8 * v + 4]), __uint_as_float(r[8 * v + 5]));
                w.w = pack_bf16x2(__uint_as_float(r[8 * v + 6]), __uint_as_float(r[8 * v + 7]));
                dst[v] = w;
              }
            }
          }
          }
          tc_fence_before();
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (leader) mbar_arrive(&s->tmem_empty[slot]);
        }
        if (leader) dbg_stamp_ext(p.run, oi * 8 + 6);
        group_arrive(p.phase_cnt + o.mma_phase, leader, nullptr, 0, p.full_fence);
        if (leader) dbg_stamp_ext(p.run, oi * 8 + 7);
        if (CS == 1 && o.split > 1) {
          // Reduce the k-slices (slice order) into bf16 C across the whole grid.
          group_wait(p.phase_cnt + o.mma_phase, static_cast<uint32_t>(G), leader);
          if (leader) dbg_stamp_ext(p.run, 40 + oi * 2);
          switch (o.split) {
            case 2: reduce_slices<2, 6, BN>(o, t, G); break;
            case 4: reduce_slices<4, 3, BN>(o, t, G); break;
            case 8: reduce_slices<8, 1, BN>(o, t, G); break;
            default: reduce_slices_any<BN>(o, t, G); break;
          }
          if (leader) dbg_stamp_ext(p.run, 41 + oi * 2);
          group_arrive(p.phase_cnt + o.ready_phase, leader, nullptr, 0, p.full_fence);
        }
      } else if (o.kind == kFusedAbsorbed) {
        continue;  // written by the previous GEMM's epilogue, published with its phase
      } else {
        // BIAS_GELU (tanh form, same arithmetic as bias_gelu_kernel / oracle tr_bias_gelu)
        if (leader) dbg_stamp_ext(p.run, oi * 8 + 4);
        if (o.in_phase >= 0) group_wait(p.phase_cnt + o.in_phase, static_cast<uint32_t>(G), leader);
        if (leader) dbg_stamp_ext(p.run, oi * 8 + 5);
        if (o.kind == kFusedSiluMul)
          silu_mul_phase(o, t, G);
        else
          bias_gelu_phase(o, t, G);
        if (leader) dbg_stamp_ext(p.run, oi * 8 + 6);
        group_arrive(p.phase_cnt + o.ready_phase, leader, nullptr, 0, p.full_fence);
        if (leader) dbg_stamp_ext(p.run, oi * 8 + 7);
      }
    }
    if (leader) dbg_stamp(p.run, 6);
  }

  tc_fence_before();
  if constexpr (CS > 1) cluster_sync_all();  // no CTA leaves while a peer may still write to it
  else __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, Cfg::kTmemCols);
  if (threadIdx.x == 0) cta_exit(p.run, 0);
}

}  // namespace msdev
