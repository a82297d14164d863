// HP decode chain for batch-1 requests (Llama-style decode, bs=1).
//
// A bs=1 decode step is a chain of matrix-VECTOR products: every weight byte is read once
// and used for one multiply-add, so the step is bound by HBM (2.47 GB of bf16 weights per
// token for the 1B geometry), not by the tensor cores.  One persistent launch runs the
// whole chain:
//
//   * warp 0 (one elected thread) streams weight units — a few whole rows of W, <= 16 KB —
//     with cp.async.bulk into a 12-stage shared-memory ring (192 KB per SM, evict-first L2
//     policy).  Weights do not depend on the previous op's output, so the producer runs
//     straight through op boundaries: while the consumers wait for op i's output vector,
//     the ring keeps filling with op i+1's rows, and an L2 lookahead of 16 units past the
//     issue point (cp.async.bulk.prefetch.L2) keeps HBM busy once the ring is full.
//   * warps 1-12 consume: they copy the op's input vector (<= 16 KB) into shared memory, then
//     a unit belongs to one warp (unit j of the CTA's stream -> warp j % 12 = its stage): up to 4 rows
//     at a time against each unpacked x chunk (16-byte smem reads, fp32 accumulation,
//     shuffle reduction); lanes 0-3 store the bf16 outputs.  GEMV_SWIGLU units carry gate
//     and up rows; silu(g) * u is applied to the fp32 dot products.
//   * op -> op handoff without fences: an output consumed later in the chain is also
//     written to a "wire" of 32-bit words {16-bit launch tag, bf16 value} (the LL-protocol
//     idea: data and flag in one store).  The next op's CTAs poll the wire words of their
//     input until every tag matches this launch.  A grid phase counter (MEMBAR + atomic,
//     measured ~2 us per op under full HBM load) is used only for inputs that are not
//     produced in the chain.
//   * units are dealt to CTAs round-robin on a counter that continues across ops, so each
//     CTA's total byte count over the chain is balanced to within one unit (DYN = false), or
//     (DYN = true) each CTA's producer CLAIMS batches of B units of the op from a per-op
//     counter, so a CTA that starts late (its SM still draining a preempted LP CTA when the
//     doorbell fires) takes fewer units instead of holding back every later op by its start
//     delay.  The producer writes each stage's (op, unit) before arming its barrier and,
//     once an op's claims run out, the ring position where the op ends in this CTA; a
//     consumer warp leaves the op at that position (or, racing the producer, at a landed
//     stage that holds a later op's unit).  The L2 lookahead keeps the static unit plan
//     (whichever CTA claims a prefetched unit finds it in L2).  The two variants are
//     separate instantiations: the static one is the round-1 code path unchanged.
//
// Per-unit algorithmic bytes = the unit's weight bytes (the vectors are L2-resident and
// small).  Roofline: HBM (MEASURED_PEAKS.json hbm_gbs).
#pragma once

#include "stream_kernels.cuh"

namespace msdev {

constexpr int kGemvMaxOps = 96;
constexpr int kGemvStageBytes = 16384;
constexpr int kGemvStages = 12;
constexpr int kGemvMaxK = kGemvStageBytes / 2;  // input vector (bf16) held in smem
constexpr int kGemvConsumers = kGemvStages;     // consumer warp w owns ring stage w (no parity ABA)
constexpr int kGemvThreads = 32 * (1 + kGemvConsumers);
constexpr int kGemvSmemBytes = kGemvStages * kGemvStageBytes + kGemvMaxK * 2 + 256;

constexpr int kGemvMatvec = 1;   // y[n] = W[n,k] . x[k]
constexpr int kGemvSwiglu = 6;   // y[j] = silu(Wg[j] . x) * (Wu[j] . x), W = [gate rows; up rows]
constexpr int kGemvBiasGelu = 2; // y = gelu(x + bias) over n
constexpr int kGemvSiluMul = 5;  // y[j] = silu(x[j]) * x[n + j]

struct GemvOpDesc {
  int kind;
  int n, k;
  int rows;       // rows of W (gate/up pairs for SWIGLU) per unit
  int units;      // ceil(n / rows)
  int unit_base;  // chain-wide unit counter at this op's first unit (CTA = counter % grid)
  int wait_phase; // 1: input not produced in the chain -> wait for op i-1's phase counter
  int arrive;     // 1: publish completion on this op's phase counter (next op waits on it)
  const __nv_bfloat16* x;
  const uint32_t* x_wire;  // input from an earlier op's wire (null: plain x)
  const __nv_bfloat16* w;
  const __nv_bfloat16* bias;
  __nv_bfloat16* y;
  uint32_t* y_wire;  // tagged copy of y for later ops (null: none)
};

static_assert(sizeof(GemvOpDesc) % 16 == 0, "descriptors are bulk-copied (16-byte granules)");

struct GemvParams {
  TileRun run;  // HP bookkeeping (first-CTA stamp, completion record, phase-counter reset)
  uint32_t* phase_cnt;  // [n_ops]: CTAs that finished op i
  uint32_t* claim;      // [n_ops]: DYN unit-claim counters (reset by the last CTA)
  int claim_batch;      // DYN: units per claim
  const GemvOpDesc* ops;  // [n_ops] in global memory (16-byte aligned), bulk-copied to smem
  int n_ops;
  uint32_t tag;  // this launch's wire tag (16 bits)
  int inflight;  // max units issued but not yet landed (the rest of the ring buffers landed data)
  int prefetch;  // L2 lookahead in units past the issue point
  // Head prefetch: the first kGemvHeadCtas CTAs to start prefetch the first head_kb KB of the
  // chain's weights (op order, every CTA's units) into L2.  When the doorbell fires while a
  // preempted LP grid still drains, the CTAs that start on free SMs keep HBM busy for the
  // CTAs that start late; those then find their first units in L2 and catch up, instead of
  // holding back every op of the static unit plan by their start delay.
  int head_kb;
  uint32_t* start_cnt;  // CTAs started (reset by the last CTA)
};

constexpr int kGemvHeadCtas = 8;
constexpr uint32_t kGemvHeadChunk = 64 * 1024;

__device__ __forceinline__ uint4 ld_relaxed_v4(const uint32_t* p) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ bool wire_ok(const uint4& v, uint32_t tag) {
  return (v.x >> 16) == tag && (v.y >> 16) == tag && (v.z >> 16) == tag && (v.w >> 16) == tag;
}
__device__ __forceinline__ void store_out(const GemvOpDesc& o, int idx, float v, uint32_t tag) {
  const __nv_bfloat16 b = __float2bfloat16_rn(v);
  o.y[idx] = b;
  if (o.y_wire) st_relaxed_u32(o.y_wire + idx, (tag << 16) | __bfloat16_as_ushort(b));
}

__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void bulk_load(void* smem_dst, const void* src, uint32_t bytes, uint64_t* bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(smem_dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint4 ld_cg_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// Diagnostics: SM-cycle stamps (clock64) in the extended debug block.  %globaltimer
// readings of warps released by the same barrier were measured up to 5 us apart on this
// part, so intra-CTA timelines use the SM clock; slot 63 holds the CTA's start cycle.
// Stamps taken right after bar.sync go through a shared load first: BAR.SYNC is
// DEFER_BLOCKING (the warp keeps issuing independent instructions, e.g. a clock read,
// until one needs the barrier), so an unguarded stamp records the ARRIVAL at the barrier.
__device__ __forceinline__ void gemv_stamp(const TileRun& r, int slot, uint32_t guard_smem = 0) {
  if (!r.dbg || slot >= 64) return;
  uint32_t g = 0;
  if (guard_smem) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(g) : "r"(guard_smem) : "memory");
  if (g != 0x7FEDCBA9u) r.dbg[2048 + blockIdx.x * 64 + slot] = clock64();
}

__device__ __forceinline__ void gemv_phase_wait(const uint32_t* cnt, uint32_t target) {
  while (ld_acquire_gpu(cnt) < target) __nanosleep(32);
}

__device__ __forceinline__ int gemv_first_unit(const GemvOpDesc& o, int G) {
  // first unit u of this op with (unit_base + u) % G == blockIdx.x
  return ((static_cast<int>(blockIdx.x) - o.unit_base % G) % G + G) % G;
}

__device__ __forceinline__ int gemv_unit_rows(const GemvOpDesc& o, int u) {
  const int r0 = u * o.rows;
  return min(o.rows, o.n - r0);
}

// acc.x += even products, acc.y += odd products (two independent FMA chains)
__device__ __forceinline__ void dot8(const uint4& w, const float (&x)[8], float2& acc) {
  const uint32_t* ws = &w.x;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    acc.x = fmaf(__uint_as_float(ws[e] << 16), x[2 * e], acc.x);
    acc.y = fmaf(__uint_as_float(ws[e] & 0xFFFF0000u), x[2 * e + 1], acc.y);
  }
}

__device__ __forceinline__ void unpack8(const uint4& v, float (&x)[8]) {
  const uint32_t* vs = &v.x;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    x[2 * e] = __uint_as_float(vs[e] << 16);
    x[2 * e + 1] = __uint_as_float(vs[e] & 0xFFFF0000u);
  }
}

__device__ __forceinline__ float warp_sum(float s) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  return s;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// One warp, 4 rows of one unit (shared-space addresses) against the smem input vector:
// each x chunk is unpacked once and used for every row; 8 independent FMA chains.
__device__ __forceinline__ void rows4_dot(const uint32_t (&row)[4], uint32_t xs, int chunks, int lane, float (&out)[4]) {
  float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll 2
  for (int c = lane; c < chunks; c += 32) {
    float x[8];
    unpack8(lds128(xs + c * 16), x);
#pragma unroll
    for (int r = 0; r < 4; ++r) dot8(lds128(row[r] + c * 16), x, acc[r]);
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) out[r] = warp_sum(acc[r].x + acc[r].y);
}

// One row (long K): four chunks in flight per lane, 8 independent FMA chains.
__device__ __forceinline__ float row1_dot(uint32_t row, uint32_t xs, int chunks, int lane) {
  float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  int c = lane;
  for (; c + 96 < chunks; c += 128) {
    uint4 w[4], xv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      w[q] = lds128(row + (c + 32 * q) * 16);
      xv[q] = lds128(xs + (c + 32 * q) * 16);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float x[8];
      unpack8(xv[q], x);
      dot8(w[q], x, acc[q]);
    }
  }
  for (; c < chunks; c += 32) {
    float x[8];
    unpack8(lds128(xs + c * 16), x);
    dot8(lds128(row + c * 16), x, acc[0]);
  }
  return warp_sum((acc[0].x + acc[0].y) + (acc[1].x + acc[1].y) + ((acc[2].x + acc[2].y) + (acc[3].x + acc[3].y)));
}

// Consume one unit (whole rows of W in one stage, <= 32 outputs): returns output r of the
// unit in lane r.  Stores happen after the stage is released (see the consumer loop).
__device__ __forceinline__ float gemv_unit(const GemvOpDesc& o, int u, uint32_t st, uint32_t xs, int lane) {
  const int nr = gemv_unit_rows(o, u);
  const uint32_t rb = static_cast<uint32_t>(o.k) * 2;
  const int chunks = o.k / 8;
  float mine = 0.f;
  if (o.kind == kGemvSwiglu) {
    for (int r0 = 0; r0 < nr; r0 += 2) {  // gate r0, gate r0+1, up r0, up r0+1
      const int r1 = r0 + 1 < nr ? r0 + 1 : r0;
      const uint32_t up = st + static_cast<uint32_t>(o.rows) * rb;
      const uint32_t row[4] = {st + r0 * rb, st + r1 * rb, up + r0 * rb, up + r1 * rb};
      float d[4];
      rows4_dot(row, xs, chunks, lane, d);
      if (lane == r0) mine = silu_mul(d[0], d[2]);
      if (lane == r0 + 1) mine = silu_mul(d[1], d[3]);
    }
  } else if (nr == 1) {
    mine = row1_dot(st, xs, chunks, lane);
  } else {
    for (int r0 = 0; r0 < nr; r0 += 4) {
      uint32_t row[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) row[q] = st + static_cast<uint32_t>(min(r0 + q, nr - 1)) * rb;
      float d[4];
      rows4_dot(row, xs, chunks, lane, d);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (lane == r0 + q) mine = d[q];
    }
  }
  return mine;
}

__device__ __forceinline__ float gemv_in(const GemvOpDesc& o, int j, uint32_t tag) {
  if (!o.x_wire) return __bfloat162float(o.x[j]);
  uint32_t w;
  while (((w = ld_relaxed_u32(o.x_wire + j)) >> 16) != tag) __nanosleep(20);
  return __uint_as_float(w << 16);
}

__device__ __forceinline__ void gemv_elementwise(const GemvOpDesc& o, int t, int G, uint32_t tag) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  for (int j = blockIdx.x * (32 * kGemvConsumers) + t; j < o.n; j += G * 32 * kGemvConsumers) {
    float v;
    if (o.kind == kGemvSiluMul) {
      v = silu_mul(gemv_in(o, j, tag), gemv_in(o, o.n + j, tag));
    } else {
      v = gemv_in(o, j, tag) + __bfloat162float(o.bias[j]);
      v = 0.5f * v * (1.0f + tanhf(k0 * (v + k1 * v * v * v)));
    }
    store_out(o, j, v, tag);
  }
}

// Input vector -> shared memory (bf16).  Wire input: poll until every word carries this
// launch's tag; all of a thread's loads are in flight at once (one L2 round trip).
__device__ __forceinline__ void gemv_load_x(const GemvOpDesc& o, uint8_t* xs, int t, uint32_t tag) {
  constexpr int kT = 32 * kGemvConsumers;
  if (!o.x_wire) {
    constexpr int kPer = (kGemvMaxK / 8 + kT - 1) / kT;
    uint4 v[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i)
      if (t + i * kT < o.k / 8) v[i] = ld_cg_v4(o.x + (t + i * kT) * 8);
#pragma unroll
    for (int i = 0; i < kPer; ++i)
      if (t + i * kT < o.k / 8) *reinterpret_cast<uint4*>(xs + (t + i * kT) * 16) = v[i];
    return;
  }
  constexpr int kPer = (kGemvMaxK / 4 + kT - 1) / kT;  // 16-byte vectors of 4 wire words
  const int nv = o.k / 4;
  uint4 v[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i)
    if (t + i * kT < nv) v[i] = ld_relaxed_v4(o.x_wire + (t + i * kT) * 4);
  for (;;) {
    bool all = true;
#pragma unroll
    for (int i = 0; i < kPer; ++i)
      if (t + i * kT < nv && !wire_ok(v[i], tag)) all = false;
    if (all) break;
    __nanosleep(20);
#pragma unroll
    for (int i = 0; i < kPer; ++i)
      if (t + i * kT < nv && !wire_ok(v[i], tag)) v[i] = ld_relaxed_v4(o.x_wire + (t + i * kT) * 4);
  }
#pragma unroll
  for (int i = 0; i < kPer; ++i)
    if (t + i * kT < nv)
      *reinterpret_cast<uint2*>(xs + (t + i * kT) * 8) =
          make_uint2((v[i].x & 0xFFFFu) | (v[i].y << 16), (v[i].z & 0xFFFFu) | (v[i].w << 16));
}

template <bool DYN>
__global__ void __launch_bounds__(kGemvThreads, 1) hp_gemv_kernel(const __grid_constant__ GemvParams p) {
  extern __shared__ __align__(128) uint8_t gsm_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(gsm_raw) + 127) & ~uintptr_t(127));
  uint8_t* xs = ring + kGemvStages * kGemvStageBytes;
  const uint32_t ring_s = smem_u32(ring), xs_s = smem_u32(xs);
  __shared__ uint64_t full[kGemvStages], empty[kGemvStages], desc_bar;
  // DYN: (op, unit) in each stage, and where each op ends in this CTA's ring stream
  __shared__ int2 stage_meta[DYN ? kGemvStages : 1];
  __shared__ uint32_t op_end[DYN ? kGemvMaxOps : 1];
  // Op descriptors live in shared memory (one bulk copy from global at entry): dynamically
  // indexed kernel-parameter reads go through the constant cache, whose misses wait behind
  // the saturated memory system, and small parameters keep the launch itself short.
  __shared__ __align__(16) GemvOpDesc sops[kGemvMaxOps];
  const int G = static_cast<int>(gridDim.x);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    cta_started(p.run);  // first HP CTA dispatched (the preemption-latency end point)
    gemv_stamp(p.run, 63);
    for (int i = 0; i < kGemvStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&desc_bar, 1);
    fence_mbar_init();
    const uint32_t bytes = static_cast<uint32_t>(p.n_ops * sizeof(GemvOpDesc));
    mbar_arrive_expect_tx(&desc_bar, bytes);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sops)),
                 "l"(p.ops), "r"(bytes), "r"(smem_u32(&desc_bar))
                 : "memory");
  }
  if constexpr (DYN)
    for (int i = threadIdx.x; i < kGemvMaxOps; i += blockDim.x) op_end[i] = 0xFFFFFFFFu;
  __syncthreads();
  mbar_wait(&desc_bar, 0);
  if (p.run.pdl_wait) pdl_wait();

  if (warp == 0) {
    // ===================== weight producer (runs ahead across ops) =====================
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      uint32_t stage = 0, phase = 0, issued = 0;
      const uint32_t D = static_cast<uint32_t>(p.inflight);
      // L2 lookahead: the next P units past the issue point are prefetched into L2, so
      // while the ring is full (consumers waiting for an op's input vector) HBM keeps
      // streaming.  (Waits stay blocking try_waits: a test_wait spin interleaved with the
      // prefetches measured 20% slower on a single long op.)
      const uint32_t P = static_cast<uint32_t>(p.prefetch);
      uint32_t pf_count = 0;
      int pf_oi = 0, pf_u = 0;
      auto pf_seek = [&](int oi, int u) {  // first gemv unit at or after (oi, u)
        for (; oi < p.n_ops; ++oi) {
          const GemvOpDesc& q = sops[oi];
          if ((q.kind == kGemvMatvec || q.kind == kGemvSwiglu) && u < q.units) break;
          if (oi + 1 < p.n_ops) u = gemv_first_unit(sops[oi + 1], G);
        }
        pf_oi = oi;
        pf_u = u;
      };
      pf_seek(0, gemv_first_unit(sops[0], G));
      if (p.head_kb > 0) {
        const uint32_t r = atomicAdd(p.start_cnt, 1u);
        if (r < static_cast<uint32_t>(kGemvHeadCtas)) {
          // chunk c of the head (64 KB, op order, contiguous weight ranges) -> CTA c % 8
          const size_t head = static_cast<size_t>(p.head_kb) * 1024;
          size_t pos = 0;
          uint32_t c = 0;
          for (int oi = 0; oi < p.n_ops && pos < head; ++oi) {
            const GemvOpDesc& q = sops[oi];
            if (q.kind != kGemvMatvec && q.kind != kGemvSwiglu) continue;
            const size_t bytes = static_cast<size_t>(q.kind == kGemvSwiglu ? 2 * q.n : q.n) * q.k * 2;
            const uint8_t* base = reinterpret_cast<const uint8_t*>(q.w);
            for (size_t off = 0; off < bytes && pos < head; off += kGemvHeadChunk, pos += kGemvHeadChunk, ++c)
              if (c % kGemvHeadCtas == r)
                bulk_prefetch_l2(base + off, static_cast<uint32_t>(min(static_cast<size_t>(kGemvHeadChunk), bytes - off)));
          }
        }
      }
      auto pf_step = [&]() -> bool {
        if (pf_oi >= p.n_ops || pf_count >= issued + P) return false;
        const GemvOpDesc& q = sops[pf_oi];
        const size_t rb = static_cast<size_t>(q.k) * 2;
        const uint32_t bytes = static_cast<uint32_t>(gemv_unit_rows(q, pf_u) * rb);
        const uint8_t* src = reinterpret_cast<const uint8_t*>(q.w) + static_cast<size_t>(pf_u) * q.rows * rb;
        bulk_prefetch_l2(src, bytes);
        if (q.kind == kGemvSwiglu) bulk_prefetch_l2(src + static_cast<size_t>(q.n) * rb, bytes);
        ++pf_count;
        pf_seek(pf_oi, pf_u + G);
        return true;
      };
      for (int oi = 0; oi < p.n_ops && DYN; ++oi) {
        const GemvOpDesc& o = sops[oi];
        if (o.kind != kGemvMatvec && o.kind != kGemvSwiglu) continue;
        const size_t row_bytes = static_cast<size_t>(o.k) * 2;
        const int B = p.claim_batch;
        int next = static_cast<int>(atomicAdd(p.claim + oi, static_cast<unsigned>(B)));
        for (;;) {
          const int b0 = next;
          if (b0 >= o.units) break;
          // the next batch's claim is in flight while this batch's stages are waited for
          next = static_cast<int>(atomicAdd(p.claim + oi, static_cast<unsigned>(B)));
          for (int u = b0; u < min(b0 + B, o.units); ++u, ++issued) {
            const int r0 = u * o.rows, nr = gemv_unit_rows(o, u);
            const uint32_t bytes = static_cast<uint32_t>(nr * row_bytes);
            if (issued >= D) {
              const uint32_t back = issued - D;
              mbar_wait(&full[back % kGemvStages], (back / kGemvStages) & 1);
            }
            mbar_wait(&empty[stage], phase ^ 1);
            stage_meta[stage] = make_int2(oi, u);  // published by the barrier's arrive (release)
            uint8_t* dst = ring + stage * kGemvStageBytes;
            const uint8_t* src = reinterpret_cast<const uint8_t*>(o.w) + r0 * row_bytes;
            if (o.kind == kGemvSwiglu) {
              mbar_arrive_expect_tx(&full[stage], 2 * bytes);
              bulk_load(dst, src, bytes, &full[stage], pol);
              bulk_load(dst + o.rows * row_bytes, src + static_cast<size_t>(o.n) * row_bytes, bytes, &full[stage], pol);
            } else {
              mbar_arrive_expect_tx(&full[stage], bytes);
              bulk_load(dst, src, bytes, &full[stage], pol);
            }
            if (++stage == kGemvStages) {
              stage = 0;
              phase ^= 1;
            }
            while (pf_step()) {
            }
          }
        }
        st_volatile_smem(&op_end[oi], issued);  // op oi ends at ring position `issued` here
        if (oi < 16) gemv_stamp(p.run, 48 + oi);
      }
      if constexpr (DYN) {  // end of the chain: one terminal entry per consumer warp (no data)
        for (int w = 0; w < kGemvConsumers; ++w, ++issued) {
          mbar_wait(&empty[stage], phase ^ 1);
          stage_meta[stage] = make_int2(p.n_ops, 0);
          mbar_arrive(&full[stage]);
          if (++stage == kGemvStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      for (int oi = 0; oi < p.n_ops && !DYN; ++oi) {
        const GemvOpDesc& o = sops[oi];
        if (o.kind != kGemvMatvec && o.kind != kGemvSwiglu) continue;
        const size_t row_bytes = static_cast<size_t>(o.k) * 2;
        for (int u = gemv_first_unit(o, G); u < o.units; u += G, ++issued) {
          const int r0 = u * o.rows, nr = gemv_unit_rows(o, u);
          const uint32_t bytes = static_cast<uint32_t>(nr * row_bytes);
          // Bound the loads in flight: a full 12-stage queue on every SM inflates HBM latency
          // (and the op->op handoff traffic behind it); landed units may still fill the
          // whole ring while the consumers wait for an op's input.
          if (issued >= D) {
            const uint32_t back = issued - D;
            mbar_wait(&full[back % kGemvStages], (back / kGemvStages) & 1);
          }
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* dst = ring + stage * kGemvStageBytes;
          const uint8_t* src = reinterpret_cast<const uint8_t*>(o.w) + r0 * row_bytes;
          if (o.kind == kGemvSwiglu) {
            mbar_arrive_expect_tx(&full[stage], 2 * bytes);
            bulk_load(dst, src, bytes, &full[stage], pol);  // gate rows
            bulk_load(dst + o.rows * row_bytes, src + static_cast<size_t>(o.n) * row_bytes, bytes, &full[stage], pol);
          } else {
            mbar_arrive_expect_tx(&full[stage], bytes);
            bulk_load(dst, src, bytes, &full[stage], pol);
          }
          if (++stage == kGemvStages) {
            stage = 0;
            phase ^= 1;
          }
          while (pf_step()) {
          }  // keep the L2 lookahead P units past the issue point
        }
        if (oi < 16) gemv_stamp(p.run, 48 + oi);  // last unit of op oi issued
      }
    }
  } else {
    // ===================== consumers: dot products + grid phases =====================
    // Unit j of this CTA's stream (counted across ops) lives in stage j % S and belongs to
    // consumer warp j % S: each warp is the only consumer of its stage, so it always waits
    // for the stage's current phase (a warp owning several stages could run a whole
    // phase ahead of a stage another warp has not released: mbarrier parity ABA).
    const int cw = warp - 1;
    const int t = threadIdx.x - 32;  // 0..255
    uint32_t j = DYN ? static_cast<uint32_t>(cw) : 0u;  // DYN: this warp's next ring position
    const uint32_t tag = p.tag;
    for (int oi = 0; oi < p.n_ops; ++oi) {
      const GemvOpDesc& o = sops[oi];
      if (o.wait_phase) {  // input not produced in the chain: order behind op oi-1
        if (t == 0) gemv_phase_wait(p.phase_cnt + oi - 1, static_cast<uint32_t>(G));
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kGemvConsumers) : "memory");
      }
      if (o.kind == kGemvMatvec || o.kind == kGemvSwiglu) {
        if (t == 0 && oi < 12) gemv_stamp(p.run, 4 * oi);
        gemv_load_x(o, xs, t, tag);
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kGemvConsumers) : "memory");
        if (t == 0 && oi < 12) gemv_stamp(p.run, 4 * oi + 1, xs_s);
        if (t == 0 && p.run.dbg && oi >= 1 && oi <= 8) {  // global time: x of ops 1..8 ready
          uint32_t g;
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(g) : "r"(xs_s) : "memory");
          if (g != 0x7FEDCBA9u) p.run.dbg[2048 + 148 * 64 + blockIdx.x * 16 + oi] = globaltimer();
        }
        if constexpr (DYN) {
          for (;;) {
            if (j >= ld_volatile_smem(&op_end[oi])) break;  // the producer knows where op oi ends
            const uint32_t stage = j % kGemvStages;
            mbar_wait(&full[stage], (j / kGemvStages) & 1);
            const int2 meta = stage_meta[stage];
            if (meta.x != oi) break;  // (raced the producer: a later op's unit, kept for that op)
            const int u = meta.y;
            const float v = gemv_unit(o, u, ring_s + stage * kGemvStageBytes, xs_s, lane);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (lane < gemv_unit_rows(o, u)) store_out(o, u * o.rows + lane, v, tag);
            j += kGemvConsumers;
          }
        }
        for (int u = gemv_first_unit(o, G); u < o.units && !DYN; u += G, ++j) {
          if (static_cast<int>(j % kGemvConsumers) != cw) continue;
          const uint32_t stage = j % kGemvStages;
          mbar_wait(&full[stage], (j / kGemvStages) & 1);
          const float v = gemv_unit(o, u, ring_s + stage * kGemvStageBytes, xs_s, lane);
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[stage]);  // release the stage before any global store
          if (lane < gemv_unit_rows(o, u)) store_out(o, u * o.rows + lane, v, tag);
        }
      } else {
        gemv_elementwise(o, t, G, tag);
      }
      // every consumer warp is done with op oi (x is rewritten next)
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kGemvConsumers) : "memory");
      if (t == 0) {
        if (oi < 12) gemv_stamp(p.run, 4 * oi + 2, xs_s);
        if (p.run.dbg && oi <= 8) {  // global time: op done in this CTA
          uint32_t g;
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(g) : "r"(xs_s) : "memory");
          if (g != 0x7FEDCBA9u) p.run.dbg[2048 + 148 * 64 + blockIdx.x * 16 + 8 + oi] = globaltimer();
        }
        if (o.arrive) {  // same pattern as hp_fused.cuh group_arrive
          __threadfence();
          red_release_gpu_add(p.phase_cnt + oi, 1u);
        }
        if (oi < 12) gemv_stamp(p.run, 4 * oi + 3);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cta_exit(p.run, 0);
}

}  // namespace msdev
