// HBM-streaming tenant kernels and the HP doorbell gate.
//
//  * axpy_kernel     — LP persistent preemptible streamer:
//                      y <- bf16(fma(a, x, y)) over linear tiles of `tile_elems` bf16,
//                      16 B vector loads, 8 loads in flight per thread, 4 CTAs/SM;
//                      one tile (8192 elems = 48 KB of traffic) is the preemption grain.
//  * bias_gelu_kernel— HP epilogue kernel of the config-1 chain (tanh-GELU(x + bias)).
//  * gate_kernel     — HP doorbell (north_star (b)): a 1-warp kernel
//                      pre-enqueued at the head of each armed HP chain on the
//                      highest-priority stream; it spins on the host-mapped doorbell
//                      (ld.acquire.sys) and exits when the host rings, releasing the
//                      already-enqueued chain kernels with no host launch on the path.
//  * synth_fill_kernel — deterministic synthetic tensors (same generator as
//                      oracle/tenant_ref.c: splitmix64-keyed uniform, bf16 RNE).
#pragma once

#include "tile_run.cuh"

namespace msdev {

struct StreamParams {
  TileRun run;
  const __nv_bfloat16* x;
  __nv_bfloat16* y;
  float alpha;
  unsigned long long n;
  int tile_elems;  // multiple of 256 * 8
  // Off-device admission (memory tier, ms_lp_set_slow_tiles): tiles of group
  // t / slow_group with slow[group] != 0 touch host-DRAM / peer chunks; at most slow_max of
  // them are in flight device-wide (slow_sem), so a preemption drains at most
  // slow_max tiles over the slow link instead of one per CTA.
  const uint8_t* slow;
  unsigned int* slow_sem;
  int slow_group, slow_max;
};

constexpr int kStreamThreads = 256;  // one streaming group = 8 warps; then mirror poller + host poller (CTA 0) warps
constexpr int kAxpyGroups = 3;       // streaming groups of the one-CTA-per-SM streamer (ctas_per_sm == 1)

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ld_plain(const void* p) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_stream(void* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint32_t axpy2(float a, uint32_t xv, uint32_t yv) {
  const __nv_bfloat162 x2 = *reinterpret_cast<const __nv_bfloat162*>(&xv);
  const __nv_bfloat162 y2 = *reinterpret_cast<const __nv_bfloat162*>(&yv);
  const float lo = __fmaf_rn(a, __low2float(x2), __low2float(y2));
  const float hi = __fmaf_rn(a, __high2float(x2), __high2float(y2));
  return pack_bf16x2(lo, hi);
}

// GROUPS independent 256-thread streaming groups per CTA (each claims its own tiles, own
// named barrier), then the two poller warps.  GROUPS = 1: 4 CTAs per SM (register-capped).
// GROUPS = 3: ONE CTA per SM (832 threads) — a capped grid (governor, SM reserve) then
// really leaves whole SMs empty for the HP chain, which several small CTAs per SM never
// do (the block scheduler spreads them over every SM).
// Named barrier of streaming group g (ids 1..GROUPS; id 0 = __syncthreads).  Immediate ids
// so ptxas reserves only the barriers used (a register id reserves all 16).
template <int GROUPS>
__device__ __forceinline__ void group_bar(int g) {
  if constexpr (GROUPS == 1) {
    asm volatile("bar.sync 1, %0;" ::"n"(kStreamThreads) : "memory");
  } else {
    static_assert(GROUPS == 3, "group_bar: add the ids");
    if (g == 0) asm volatile("bar.sync 1, %0;" ::"n"(kStreamThreads) : "memory");
    else if (g == 1) asm volatile("bar.sync 2, %0;" ::"n"(kStreamThreads) : "memory");
    else asm volatile("bar.sync 3, %0;" ::"n"(kStreamThreads) : "memory");
  }
}

template <int VPT, int GROUPS>  // 16-byte vectors per thread per tile
__global__ void __launch_bounds__(GROUPS * kStreamThreads + 64, GROUPS == 1 ? 4 : 1)
    axpy_kernel(const __grid_constant__ StreamParams p) {
  __shared__ uint32_t preempt, producer_done, tiles_done, groups_left;
  __shared__ long long tile_sh[GROUPS][2];
  constexpr int kStreamWarps = GROUPS * kStreamThreads / 32;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    preempt = 0;
    producer_done = 0;
    tiles_done = 0;
    groups_left = GROUPS;
    cta_started(p.run);
  }
  __syncthreads();
  if (warp == kStreamWarps) {
    if ((threadIdx.x & 31) == 0 && p.run.preemptible) poll_mirror(p.run, &preempt, &producer_done);
  } else if (warp == kStreamWarps + 1) {
    if ((threadIdx.x & 31) == 0 && p.run.preemptible && blockIdx.x == 0) poll_host(p.run, &preempt, &producer_done);
    if ((threadIdx.x & 31) == 0 && p.run.preemptible && blockIdx.x >= 1 && blockIdx.x <= kAuxPollers)
      poll_host_aux(p.run, &preempt, &producer_done, 300u * blockIdx.x);
  } else {
    const int g = warp / (kStreamThreads / 32);
    const int tid = threadIdx.x % kStreamThreads;
    for (int j = 0;; ++j) {
      bool slow_held = false;
      if (tid == 0) {
        long long t = -1;
        if (!(p.run.preemptible && ld_volatile_smem(&preempt))) t = claim_tile(p.run);
        if (t >= 0 && p.slow && p.slow[t / p.slow_group]) {
          // admission: wait for one of slow_max slots; a preemption meanwhile parks the tile
          // (read, then CAS: waiters never inflate the count the way add-then-undo would)
          for (;;) {
            const unsigned c = *reinterpret_cast<volatile unsigned int*>(p.slow_sem);
            if (c < static_cast<unsigned>(p.slow_max) && atomicCAS(p.slow_sem, c, c + 1) == c) {
              slow_held = true;
              break;
            }
            if (p.run.preemptible && ld_volatile_smem(&preempt)) {
              push_redo(p.run, static_cast<unsigned long long>(t));
              t = -1;
              break;
            }
            __nanosleep(256);
          }
        }
        tile_sh[g][j & 1] = t;
      }
      group_bar<GROUPS>(g);
      const long long t = tile_sh[g][j & 1];
      if (t < 0) break;
      const unsigned long long base = static_cast<unsigned long long>(t) * p.tile_elems;
      uint4 xv[VPT], yv[VPT];
      bool ok[VPT];
#pragma unroll
      for (int v = 0; v < VPT; ++v) {
        const unsigned long long e = base + (static_cast<unsigned long long>(v) * kStreamThreads + tid) * 8;
        ok[v] = e + 8 <= p.n;
        if (ok[v]) {
          xv[v] = ld_stream(p.x + e);
          yv[v] = ld_plain(p.y + e);
        }
      }
#pragma unroll
      for (int v = 0; v < VPT; ++v) {
        if (!ok[v]) continue;
        const unsigned long long e = base + (static_cast<unsigned long long>(v) * kStreamThreads + tid) * 8;
        uint4 o;
        o.x = axpy2(p.alpha, xv[v].x, yv[v].x);
        o.y = axpy2(p.alpha, xv[v].y, yv[v].y);
        o.z = axpy2(p.alpha, xv[v].z, yv[v].z);
        o.w = axpy2(p.alpha, xv[v].w, yv[v].w);
        st_stream(p.y + e, o);
      }
      if (p.slow) {
        // every thread's slow-tile loads have returned once all reach this barrier
        group_bar<GROUPS>(g);
        if (slow_held) atomicSub(p.slow_sem, 1u);
      }
      if (tid == 0) atomicAdd(&tiles_done, 1u);
    }
    if (tid == 0 && atomicSub(&groups_left, 1u) == 1u) st_volatile_smem(&producer_done, 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) cta_exit(p.run, tiles_done);
}

// ---------------------------------------------------------------- HP elementwise
struct BiasGeluParams {
  TileRun run;  // non-preemptible; tiles = rows
  const __nv_bfloat16* x;
  const __nv_bfloat16* bias;
  __nv_bfloat16* out;
  int rows, cols;
};

__global__ void __launch_bounds__(256) bias_gelu_kernel(const __grid_constant__ BiasGeluParams p) {
  __shared__ long long tile_sh;
  __shared__ uint32_t tiles_done;
  if (threadIdx.x == 0) {
    tiles_done = 0;
    cta_started(p.run);
  }
  if (p.run.hp_ctl) {  // PDL-launched chain kernel
    pdl_launch_dependents();
    if (p.run.pdl_wait) pdl_wait();
  }
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) tile_sh = claim_tile(p.run);
    __syncthreads();
    const long long r = tile_sh;
    if (r < 0) break;
    for (int c = threadIdx.x * 8; c < p.cols; c += blockDim.x * 8) {
      const uint4 xv = *reinterpret_cast<const uint4*>(p.x + static_cast<size_t>(r) * p.cols + c);
      const uint4 bv = *reinterpret_cast<const uint4*>(p.bias + c);
      const uint32_t* xs = &xv.x;
      const uint32_t* bs = &bv.x;
      uint4 o;
      uint32_t* os = &o.x;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const __nv_bfloat162 x2 = *reinterpret_cast<const __nv_bfloat162*>(&xs[i]);
        const __nv_bfloat162 b2 = *reinterpret_cast<const __nv_bfloat162*>(&bs[i]);
        os[i] = pack_bf16x2(bias_gelu_tanh(__low2float(x2), __low2float(b2)),
                            bias_gelu_tanh(__high2float(x2), __high2float(b2)));
      }
      *reinterpret_cast<uint4*>(p.out + static_cast<size_t>(r) * p.cols + c) = o;
    }
    if (threadIdx.x == 0) ++tiles_done;
  }
  if (threadIdx.x == 0) cta_exit(p.run, tiles_done);
}

// SwiGLU activation of a decode layer: out[r, j] = silu(x[r, j]) * x[r, cols + j], x = [rows x 2 cols].
__device__ __forceinline__ float silu_mul(float g, float u) { return __fdividef(g, 1.0f + __expf(-g)) * u; }

__global__ void __launch_bounds__(256) silu_mul_kernel(const __grid_constant__ BiasGeluParams p) {
  __shared__ long long tile_sh;
  __shared__ uint32_t tiles_done;
  if (threadIdx.x == 0) {
    tiles_done = 0;
    cta_started(p.run);
  }
  if (p.run.hp_ctl) {
    pdl_launch_dependents();
    if (p.run.pdl_wait) pdl_wait();
  }
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) tile_sh = claim_tile(p.run);
    __syncthreads();
    const long long r = tile_sh;
    if (r < 0) break;
    for (int c = threadIdx.x * 8; c < p.cols; c += blockDim.x * 8) {
      const uint4 gv = *reinterpret_cast<const uint4*>(p.x + static_cast<size_t>(r) * 2 * p.cols + c);
      const uint4 uv = *reinterpret_cast<const uint4*>(p.x + static_cast<size_t>(r) * 2 * p.cols + p.cols + c);
      const uint32_t* gs = &gv.x;
      const uint32_t* us = &uv.x;
      uint4 o;
      uint32_t* os = &o.x;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const __nv_bfloat162 g2 = *reinterpret_cast<const __nv_bfloat162*>(&gs[i]);
        const __nv_bfloat162 u2 = *reinterpret_cast<const __nv_bfloat162*>(&us[i]);
        os[i] = pack_bf16x2(silu_mul(__low2float(g2), __low2float(u2)), silu_mul(__high2float(g2), __high2float(u2)));
      }
      *reinterpret_cast<uint4*>(p.out + static_cast<size_t>(r) * p.cols + c) = o;
    }
    if (threadIdx.x == 0) ++tiles_done;
  }
  if (threadIdx.x == 0) cta_exit(p.run, tiles_done);
}

// ---------------------------------------------------------------- HP doorbell gate
// The doorbell word carries (epoch << 32 | seq).  On release the gate (already resident,
// no launch needed) first pushes the preempt epoch into the device mirror — every LP CTA
// sees it on its next L2 poll, without waiting for the LP leader's own PCIe round trip —
// then lets the PDL-launched chain kernel be scheduled.
// Eight pollers (lane 0 of warps 0-7), started ~75 ns apart, so a PCIe read reaches the
// host page every ~RTT/8 instead of every RTT: the doorbell is seen sooner after it lands.
// Live config-1 A/B (tools/gate_pollers_ab.py, profiles/r02s3_gate_pollers_ab.json, 4 x 2.5 s
// windows each): ring -> first HP CTA p50 / p99 3.90 / 7.81 us with 4 pollers, 3.75 / 7.42
// with 8, 3.65 / 7.34 with 16 (LP in flight p99 8.05 / 7.82 / 7.59).  But the LP drain of
// configs 2/3 (single-CTA k-split GEMMs + optimizer streamer) degrades with the poll rate:
// flag -> last LP exit p99 config 2 / 3 = 11-12 / 15 us with 4 pollers, 13 / 14-15 with 8,
// 17-19 / 20-21 with 16 (tools/drain23_probe.py, profiles/r02s3_drain23_gate_warps/), so 8.
// MS_GATE_WARPS overrides.
constexpr int kGateWarps = 8;

__global__ void gate_kernel(const uint64_t* doorbell, unsigned int seq, MsHpRecord* rec, MsDevMirror* mirror,
                            const MsTrace* trace) {
  __shared__ uint32_t rung;
  __shared__ uint64_t word;
  if (threadIdx.x == 0) rung = 0;
  __syncthreads();
  const int warp = threadIdx.x / 32;
  if ((threadIdx.x & 31) == 0) {
    __nanosleep(600u / (blockDim.x / 32) * warp);  // pollers spread over ~600 ns
    // Relaxed polling: the doorbell value itself is the only datum consumed.
    for (;;) {
      if (ld_volatile_smem(&rung)) break;
      uint64_t v;
      asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(doorbell) : "memory");
      if (static_cast<int>(static_cast<uint32_t>(v) - seq) >= 0) {
        if (atomicExch(&rung, 1u) == 0) {
          word = v;
          const uint32_t epoch = static_cast<uint32_t>(v >> 32);
          if (mirror) {
#pragma unroll
            for (int c = 0; c < MS_MIRROR_COPIES; ++c) atomicMax(&mirror->epoch[c * MS_MIRROR_STRIDE], epoch);
          }
          pdl_launch_dependents();
          if (rec) {  // (the e2e input-copy gate carries no record)
            const unsigned long long t = globaltimer();
            st_relaxed_sys_u64(&rec->t_gate, t);
            st_release_sys_u32(&rec->seq_gate, seq);
            trace_emit(trace, 6u, seq, v, 0, t);
          }
        }
        break;
      }
      __nanosleep(64);
    }
  }
}

// e2e request input, pulled by SMs from pinned host memory (PCIe reads, many 16-byte loads
// in flight) into HBM as the first HP kernel of an armed chain: PDL-released by the gate at
// the ring (no copy-engine start, no event -> launch hop), and the chain's first kernel is
// PDL-released by it in turn.  Its last CTA stamps the chain's t_first_cta when the input is
// resident: the e2e preemption latency = ring -> HP input in HBM (its compute then starts
// at the dependent's griddepcontrol.wait).
struct PullParams {
  const uint4* src;      // device view of the pinned host buffer
  uint4* dst;
  unsigned long long n16;  // 16-byte words
  MsHpCtl* hp_ctl;
  unsigned int* done;    // CTAs finished (self-resetting)
};
// Grid: 56 CTAs (16 KB of reads in flight each).  The pull is bound by reads in flight, and
// with LP resident the PCIe read latency grows: 7 CTAs took ring -> input resident p50 43 us
// with LP in flight vs 25 us on an idle GPU; 28 / 56 CTAs 29 / 27 us (split-kernel p99 30.4 /
// 29.2 vs 46.6 us, exclusive ~25-26 either way; tools/e2e_tail_probe.py,
// profiles/r02s3_e2e_tail_probe_*.json).  The CTAs need no shared memory, so they fit beside
// the LP CTAs on any SM.  MS_PULL_CTAS overrides.
constexpr int kPullThreads = 256, kPullCtas = 56, kPullCtasPerSm = 7, kPullUnroll = 4;

__global__ void __launch_bounds__(kPullThreads, kPullCtasPerSm) hp_pull_kernel(const __grid_constant__ PullParams p) {
  pdl_launch_dependents();  // the chain kernel may become resident now; it waits for our completion
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * kPullThreads;
  for (unsigned long long i0 = blockIdx.x * static_cast<unsigned long long>(kPullThreads) + threadIdx.x; i0 < p.n16;
       i0 += stride * kPullUnroll) {
    uint4 v[kPullUnroll];
#pragma unroll
    for (int u = 0; u < kPullUnroll; ++u) {
      const unsigned long long i = i0 + u * stride;
      if (i < p.n16) v[u] = p.src[i];
    }
#pragma unroll
    for (int u = 0; u < kPullUnroll; ++u) {
      const unsigned long long i = i0 + u * stride;
      if (i < p.n16) p.dst[i] = v[u];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(p.done, 1u) + 1 == gridDim.x) {
      atomicMin(&p.hp_ctl->t_first_cta, static_cast<unsigned long long>(globaltimer()));
      *p.done = 0;
    }
  }
}

// Completion record of a chain whose last op is a copy (e2e mode): written after the D2H.
__global__ void hp_notify_kernel(MsHpCtl* ctl, MsHpRecord* rec, unsigned int seq, const MsTrace* trace, int chain) {
  const unsigned long long t = globaltimer();
  const unsigned long long first = ctl->t_first_cta;
  trace_emit(trace, 4u, static_cast<uint32_t>(chain), seq, 0, first);
  trace_emit(trace, 5u, static_cast<uint32_t>(chain), seq, 0, t);
  st_relaxed_sys_v2(&rec->done_first, first, (static_cast<uint64_t>(seq) << 32) | ((t - first) & 0xFFFFFFFFull));
  ctl->t_first_cta = ~0ull;
}

// ---------------------------------------------------------------- clock calibration echo
__global__ void echo_kernel(const uint32_t* ping, uint32_t* pong, unsigned long long* stamps, int rounds) {
  for (int k = 1; k <= rounds; ++k) {
    while (ld_acquire_sys(ping) < static_cast<uint32_t>(k)) {
    }
    stamps[k - 1] = globaltimer();
    st_release_sys_u32(pong, static_cast<uint32_t>(k));
  }
}

// ---------------------------------------------------------------- synthetic tensors
__device__ __forceinline__ uint64_t d_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t d_hash_combine(uint64_t a, uint64_t b) {
  return d_splitmix64(a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2)));
}

__global__ void synth_fill_kernel(__nv_bfloat16* out, unsigned long long n, unsigned long long seed,
                                  unsigned long long tensor, float scale) {
  const uint64_t base = d_hash_combine(seed, tensor);
  for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const uint64_t x = d_splitmix64(d_hash_combine(base, i));
    const float u = static_cast<float>(x >> 40) * 5.9604644775390625e-08f;
    const float v = __fmul_rn(__fsub_rn(__fmul_rn(2.0f, u), 1.0f), scale);
    out[i] = __float2bfloat16_rn(v);
  }
}

// [N, K] row-major -> [K/64][N][64] (k-block-major), 16 B per thread-iteration.
__global__ void kblock_major_kernel(const __nv_bfloat16* src, __nv_bfloat16* dst, unsigned long long n,
                                    unsigned long long k) {
  const unsigned long long vecs = n * k / 8;
  for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < vecs;
       i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const unsigned long long row = i / (k / 8);
    const unsigned long long k8 = i - row * (k / 8);
    const unsigned long long kb = k8 / 8;
    const unsigned long long kin = (k8 & 7) * 8;
    *reinterpret_cast<uint4*>(dst + (kb * n + row) * 64 + kin) = *reinterpret_cast<const uint4*>(src + row * k + k8 * 8);
  }
}

// SwiGLU weights [2F][K] (gate rows, then up rows) -> k-block-major [K/64][2F][64] with the
// rows interleaved in 64-row blocks: block t = gate rows [64t, 64t + 64) then up rows
// [64t, 64t + 64), so one 128-column GEMM tile holds the gate and up halves of 64 features.
__global__ void kblock_major_swiglu_kernel(const __nv_bfloat16* src, __nv_bfloat16* dst, unsigned long long f,
                                           unsigned long long k) {
  const unsigned long long n = 2 * f;
  const unsigned long long vecs = n * k / 8;
  for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < vecs;
       i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const unsigned long long row = i / (k / 8);  // interleaved row
    const unsigned long long k8 = i - row * (k / 8);
    const unsigned long long t = row / 128, w = row % 128;
    const unsigned long long srow = w < 64 ? 64 * t + w : f + 64 * t + (w - 64);
    const unsigned long long kb = k8 / 8;
    const unsigned long long kin = (k8 & 7) * 8;
    *reinterpret_cast<uint4*>(dst + (kb * n + row) * 64 + kin) = *reinterpret_cast<const uint4*>(src + srow * k + k8 * 8);
  }
}

__global__ void init_ctl_kernel(MsLpCtl* ctl, int n, MsHpCtl* hp, int n_hp) {  // n = MS_N_CTL
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    ctl[i].claim = 0;
    ctl[i].t_free = 0;
    ctl[i].t_start = ~0ull;
    ctl[i].t_seen = ~0ull;
    ctl[i].exited = 0;
    ctl[i].redo_out_n = 0;
    ctl[i].preempted = 0;
    ctl[i].top = 0;
  }
  if (i < n_hp) hp[i].t_first_cta = ~0ull;
}

}  // namespace msdev
