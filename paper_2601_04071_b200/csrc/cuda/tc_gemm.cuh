// Persistent, preemptible tcgen05/TMA GEMM tile loop.
//
//   C[M, N] (bf16) = A[M, K] (bf16, K-contiguous) * B[N, K]^T (bf16, K-contiguous), fp32 accumulate in TMEM.
//
// One CTA per SM (256 threads, warp-specialised):
//   warp 0  lane 0 : tile scheduler + TMA producer (STAGES-deep smem ring, 128B swizzle)
//   warp 1  lane 0 : UMMA issuer (tcgen05.mma.cta_group::1.kind::f16, M=128, N=BN, K=16)
//   warp 2         : TMEM allocator; lane 0 then polls the preempt epoch
//   warps 4-7      : epilogue (tcgen05.ld 32x32b -> bf16 -> st.global), TMEM double-buffered
// so the epilogue of tile j overlaps the MMAs of tile j+1.
//
// Preemption (north_star (a)): tiles are claimed from a device counter over linear tile
// ids [begin, end) — the same contiguous index space as the reference's row-major slice
// boxes (splitter.hpp:41-113).  CTA 0's poller reads the host-mapped epoch with
// ld.acquire.sys and mirrors it into device memory; every other CTA's poller reads the
// mirror (gpu scope).  The producer checks the CTA's smem preempt bit before claiming a
// tile and before every k-block: on preempt it stops issuing TMA, the MMA warp drains the
// in-flight stages, the partially accumulated tile is abandoned (pushed to the redo list,
// recomputed on resume — C is only written for completed tiles), and the CTA exits.  The
// last CTA to exit publishes the run's cursor / redo count / timestamps to the host page.
// Preemption latency floor = flag propagation + <= STAGES k-blocks of MMA + exit.
#pragma once

#include "tile_run.cuh"

namespace msdev {

constexpr int kBM = 128;  // UMMA M (one TMEM lane per row)
constexpr int kBK = 64;   // k-block = one 128 B swizzle row of bf16
constexpr int kUmmaK = 16;

struct GemmParams {
  TileRun run;
  int m, n, k;
  int tiles_m, tiles_n, group_m;
  __nv_bfloat16* c;
  // split-K (skinny HP GEMMs): a work unit is (tile, k-slice); unit u -> tile u / split_k,
  // slice u % split_k.  Partials go to ws in fp32; the last unit of a tile to finish
  // reduces the slices in slice order (deterministic) and writes C.
  int split_k;
  float* ws;
  unsigned int* tile_cnt;
  // B stored k-block-major ([K/64][N][64], a 3-D tensor map): every B box is one
  // contiguous BN x 128 B chunk of HBM (DRAM-page friendly streaming of HP weights).
  int b_kblock_major;
  // Preemptible runs keep at most mma_lag k-blocks of MMAs queued on the tensor core
  // (1..4; 0 = unbounded): an abort then drains <= mma_lag k-blocks.
  int mma_lag;
  // Preemptible runs keep at most tma_inflight stages issued but not yet landed (0 =
  // unbounded): an abort waits for the in-flight loads to land before the CTA can leave, and
  // for an HBM-bound shape (skinny training GEMMs with K up to 802,816) a full ring of loads
  // queued at the SM's share of HBM bandwidth is ~5 us of drain.
  int tma_inflight;
  // Off-device admission (memory tier, ms_lp_set_slow_tiles): units u with slow[u / slow_group]
  // read operand chunks that live in host DRAM / a peer's HBM; at most slow_max of them run
  // at once device-wide (slow_sem), so a preemption drains at most slow_max units' loads
  // over the slow link instead of one per CTA.
  const uint8_t* slow;
  unsigned int* slow_sem;
  int slow_group, slow_max;
  // CTA-pair kernel, 256 x 512 tiles (tc_gemm2.cuh): the last wave's tiles run as
  // tail_parts column parts on as many pairs — units u >= half_base (half_units of them, 0 =
  // none) are (tile half_base + (u - half_base) / tail_parts, part (u - half_base) % tail_parts).
  long long half_base;
  int half_units;
  int tail_parts;  // 2: the last wave's units are 256-column halves, 4: 128-column quarters
  // HP epilogue (split_k == 1 here; the split-K reduce kernel applies it otherwise):
  // C = act(acc + bias[col] (+ resid[row, col])), act 0 none / 1 ReLU / 2 tanh-GELU.
  const __nv_bfloat16* bias;
  const __nv_bfloat16* resid;
  int act;
};

// fp32 epilogue of 8 consecutive columns: + bias, + residual, activation (tanh-GELU as in
// bias_gelu_kernel / oracle tr_bias_gelu).
__device__ __forceinline__ void epilogue8(float (&v)[8], const __nv_bfloat16* bias8, const __nv_bfloat16* resid8,
                                          int act) {
  if (bias8) {
    const uint4 b = *reinterpret_cast<const uint4*>(bias8);
    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[2 * e] += __low2float(b2[e]);
      v[2 * e + 1] += __high2float(b2[e]);
    }
  }
  if (resid8) {
    const uint4 r = *reinterpret_cast<const uint4*>(resid8);
    const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[2 * e] += __low2float(r2[e]);
      v[2 * e + 1] += __high2float(r2[e]);
    }
  }
  if (act == 1) {
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = fmaxf(v[e], 0.0f);
  } else if (act == 2) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = 0.5f * v[e] * (1.0f + tanhf(k0 * (v[e] + k1 * v[e] * v[e] * v[e])));
  }
}

template <int BN>
struct GemmCfg {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (200 * 1024 / kStageBytes) > 8 ? 8 : (200 * 1024 / kStageBytes);
  static constexpr int kTmemCols = 2 * BN < 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  // C staging for the TMA-store epilogue: per epilogue warp 2 x [32 rows x 32 cols] bf16
  // (64 B rows, 64B-swizzled), double-buffered.
  static constexpr int kCStageBytes = 4 * 2 * 32 * 64;
  static constexpr int kSmemBytes = 1024 /*align slack*/ + kStages * kStageBytes + kCStageBytes + 1024 /*barriers etc.*/;
  static constexpr uint32_t kIdesc = umma_idesc_bf16(kBM, BN);
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN must be a multiple of 32 in [32, 256]");
};

struct GemmSmemCtl {
  uint64_t full[8], empty[8];
  uint64_t tmem_full[2], tmem_empty[2];
  uint64_t tile_full[2], tile_empty[2];
  uint64_t mma_drain;
  long long tile_id[2];
  uint32_t tile_abort[2];
  uint32_t tile_slow[2];  // the unit holds an off-device admission slot (released by the MMA warp)
  uint32_t stage_flag[8];  // 0: data, 1: data + last k-block, 2: aborted (no data)
  uint32_t tmem_base;
  uint32_t preempt;
  uint32_t producer_done;
  uint32_t tiles_done;
  uint32_t fix_last;
  uint32_t red_stop;
  uint32_t epi_done;  // epilogue warps finished (the CTA's mirror poller may stop)
};

__device__ __forceinline__ void tile_coords(long long t, const GemmParams& p, int& mb, int& nb) {
  const long long group_span = static_cast<long long>(p.group_m) * p.tiles_n;
  const int group = static_cast<int>(t / group_span);
  const int first_m = group * p.group_m;
  const int gm = min(p.tiles_m - first_m, p.group_m);
  const int in_group = static_cast<int>(t - group * group_span);
  mb = first_m + in_group % gm;
  nb = in_group / gm;
}

// ---------------------------------------------------------------- split-K reduction tree
// An LP unit is (tile, k-slice).  Its fp32 partial goes to ws slot `slice`.  Slices are
// reduced by a fixed tree of fan-in kRedFan: level 0 holds the S partials, the group
// (level l, g) sums partials [g*F, g*F + F) of level l (in index order) into partial g of
// level l + 1, which lives in ws slot g * F^(l+1) (the group's first slot, in place).  The
// last unit to arrive at a group's counter reduces it; the top group (<= F partials) writes
// bf16 C.  The summation order is fixed by the tree, never by timing, so a preempted and
// resumed GEMM is bit-identical to an uninterrupted one.  A reducer reads at most F partials
// (<= 512 KB) instead of all S (25 MB for the 128 x 192 x 802,816 wgrad at S = 256, which
// made one CTA spend ~0.5 ms in a non-preemptible reduction), and it stops at 32-column
// chunk boundaries when preempted, parking the rest as a continuation entry on the redo
// list (kRedEntry | tile << 32 | level << 24 | group << 8 | chunk).
constexpr int kRedFan = 4;
constexpr unsigned long long kRedEntry = 1ull << 62;

// Off-device admission of one unit (memory tier): when the unit's operands touch off-device
// chunks (slow map entry map_idx: the unit itself, or a CTA-pair unit's tile), wait for one of slow_max device-wide slots (read, then CAS: waiters never inflate
// the count).  A preemption meanwhile parks the unit on the redo list and sets tile = -1.
// Returns 1 when a slot was taken (the MMA warp returns it after the unit's last k-block).
__device__ __forceinline__ uint32_t slow_admit(const GemmParams& p, const uint32_t* preempt, long long& tile,
                                               long long map_idx) {
  if (tile < 0 || (tile & kRedEntry) || !p.slow || !p.slow[map_idx / p.slow_group]) return 0;
  for (;;) {
    const unsigned c = *reinterpret_cast<volatile unsigned int*>(p.slow_sem);
    if (c < static_cast<unsigned>(p.slow_max) && atomicCAS(p.slow_sem, c, c + 1) == c) return 1;
    if (p.run.preemptible && ld_volatile_smem(preempt)) {
      push_redo(p.run, static_cast<unsigned long long>(tile));
      tile = -1;
      return 0;
    }
    __nanosleep(256);
  }
}

__device__ __forceinline__ int red_level_count(int S, int level) {
  int n = S;
  for (int i = 0; i < level; ++i) n = (n + kRedFan - 1) / kRedFan;
  return n;
}
// counter index of group (level, g) inside the tile's block of S counters
__device__ __forceinline__ int red_counter(int S, int level, int g) {
  int base = 0, n = S;
  for (int i = 0; i < level; ++i) {
    base += (n + kRedFan - 1) / kRedFan;
    n = (n + kRedFan - 1) / kRedFan;
  }
  return base + g;
}

__device__ __forceinline__ float4 f4add(float4 a, const float4 b) {
  a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
  return a;
}

// Run by the 128 epilogue threads (named barrier 1).  `arrive`: this unit just wrote its
// level-0 partial into slot `g * F + j` and arrives at group (0, g); otherwise resume the
// already-won group (level, g) at `chunk`.  Returns when the tree above this unit needs no
// more work from it (another unit will arrive later), when C is written, or after parking a
// continuation because of a preemption.
template <int BN>
__device__ void split_tree_reduce(const GemmParams& p, GemmSmemCtl* s, long long tile, int level, int g, int chunk,
                                  bool arrive, int mb, int nb, int row) {
  const int S = p.split_k;
  float4* const ws = reinterpret_cast<float4*>(p.ws) + static_cast<size_t>(tile) * S * (kBM * BN / 4);
  unsigned int* const cnt = p.tile_cnt + static_cast<size_t>(tile) * S;
  const int tid = threadIdx.x - 128;
  for (;;) {
    const int n = red_level_count(S, level);
    const int gsize = min(kRedFan, n - g * kRedFan);
    const bool top = n <= kRedFan;
    if (arrive) {
      __threadfence();  // release this thread's partial stores (gpu scope) ...
      asm volatile("bar.sync 1, 128;" ::: "memory");  // ... before the group counter moves
      if (tid == 0) {
        unsigned int* c = cnt + red_counter(S, level, g);
        const bool last = atomicAdd(c, 1u) + 1 == static_cast<unsigned>(gsize);
        if (last) *c = 0;  // self-resetting: nobody else arrives at this group in this pass
        s->fix_last = last ? 1u : 0u;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (tid == 0) dbg_stamp_ext(p.run, 12);  // arrival done
      if (!s->fix_last) return;
      __threadfence();
    }
    size_t stride = 1;  // ws slots between consecutive partials of this level: F^level
    for (int i = 0; i < level; ++i) stride *= kRedFan;
    const size_t slot0 = static_cast<size_t>(g) * kRedFan * stride;
    for (int c = chunk; c < BN / 32; ++c) {
      if (c > chunk || arrive) {
        // preemption point before every 32-column chunk (one decision for all 128 threads); a
        // resumed continuation always makes at least one chunk of progress
        if (tid == 0) s->red_stop = (p.run.preemptible && ld_volatile_smem(&s->preempt)) ? 1u : 0u;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const bool stop = s->red_stop != 0;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (stop) {
          if (tid == 0) dbg_stamp_ext(p.run, 14);  // parked at a chunk boundary
          if (tid == 0)
            push_redo(p.run, kRedEntry | (static_cast<unsigned long long>(tile) << 32) |
                                 (static_cast<unsigned long long>(level) << 24) |
                                 (static_cast<unsigned long long>(g) << 8) | static_cast<unsigned long long>(c));
          return;
        }
      }
      // partial j of the group, column quad cq: ws[(slot0 + j*stride) * (128*BN/4) + cq*128 + row]
      // every partial of the group in flight at once for half a chunk (16 x 16 B per thread,
      // 32 KB per CTA), then summed in index order
      float4 acc[8];
      const float4* b0 = ws + slot0 * (kBM * BN / 4) + static_cast<size_t>(c * 8) * kBM + row;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float4 x[kRedFan][4];
#pragma unroll
        for (int j = 0; j < kRedFan; ++j)
          if (j < gsize) {
#pragma unroll
            for (int v = 0; v < 4; ++v) x[j][v] = __ldcg(b0 + j * stride * (kBM * BN / 4) + (h * 4 + v) * kBM);
          }
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[h * 4 + v] = x[0][v];
#pragma unroll
        for (int j = 1; j < kRedFan; ++j)
          if (j < gsize) {
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[h * 4 + v] = f4add(acc[h * 4 + v], x[j][v]);
          }
      }
      if (top) {
        __nv_bfloat16* crow = p.c + static_cast<size_t>(mb * kBM + row) * p.n + static_cast<size_t>(nb) * BN + c * 32;
#pragma unroll
        for (int v = 0; v < 8; v += 2) {
          uint4 o;
          o.x = pack_bf16x2(acc[v].x, acc[v].y);
          o.y = pack_bf16x2(acc[v].z, acc[v].w);
          o.z = pack_bf16x2(acc[v + 1].x, acc[v + 1].y);
          o.w = pack_bf16x2(acc[v + 1].z, acc[v + 1].w);
          *reinterpret_cast<uint4*>(crow + v * 4) = o;
        }
      } else {
        float4* d0 = ws + slot0 * (kBM * BN / 4) + static_cast<size_t>(c * 8) * kBM + row;
#pragma unroll
        for (int v = 0; v < 8; ++v) __stcg(d0 + v * kBM, acc[v]);
      }
    }
    if (tid == 0) dbg_stamp_ext(p.run, 13);  // a group reduced
    if (top) return;
    // this group's sum is partial g of the next level, in group g / F there
    level += 1;
    g /= kRedFan;
    chunk = 0;
    arrive = true;
  }
}

template <int BN>
__global__ void __launch_bounds__(256, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                   const __grid_constant__ CUtensorMap tma_c, const __grid_constant__ GemmParams p) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + S * Cfg::kABytes;
  uint8_t* smem_c = smem + S * Cfg::kStageBytes;
  GemmSmemCtl* s = reinterpret_cast<GemmSmemCtl*>(smem_c + Cfg::kCStageBytes);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (threadIdx.x == 0) dbg_stamp(p.run, 7);

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&s->full[i], 1);
      mbar_init(&s->empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s->tmem_full[i], 1);
      mbar_init(&s->tmem_empty[i], 1);
      mbar_init(&s->tile_full[i], 1);
      mbar_init(&s->tile_empty[i], 1);
    }
    mbar_init(&s->mma_drain, 1);
    s->preempt = 0;
    s->producer_done = 0;
    s->epi_done = 0;
    s->tiles_done = 0;
    fence_mbar_init();
    cta_started(p.run);
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tma_a);
    prefetch_tmap(&tma_b);
    if (p.split_k <= 1) prefetch_tmap(&tma_c);
  }
  if (warp == 2) tmem_alloc(&s->tmem_base, Cfg::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // HP chains are PDL-launched: let the next chain kernel get scheduled now, and wait for
  // the previous one's results before touching them (no-ops for ordinary launches).
  if (p.run.hp_ctl) {
    pdl_launch_dependents();
    if (p.run.pdl_wait) pdl_wait();
  }
  if (threadIdx.x == 0) dbg_stamp(p.run, 0);  // prologue done (HP) / overwritten by "seen" (LP)
  const uint32_t tmem_base = s->tmem_base;
  const int split = p.split_k > 1 ? p.split_k : 1;
  const int num_kb = p.k / kBK / split;  // k-blocks per work unit

  if (warp == 0) {
    // ===================== tile scheduler + TMA producer =====================
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      uint32_t issued = 0;  // ring positions issued (for the in-flight bound)
      const uint32_t D = p.run.preemptible ? static_cast<uint32_t>(p.tma_inflight) : 0u;
      for (int j = 0;; ++j) {
        const int slot = j & 1;
        if (j >= 2) mbar_wait(&s->tile_empty[slot], ((j >> 1) & 1) ^ 1);
        long long tile = -1;
        if (!(p.run.preemptible && ld_volatile_smem(&s->preempt))) tile = claim_tile(p.run);
        const uint32_t slow_held = slow_admit(p, &s->preempt, tile, tile);
        s->tile_id[slot] = tile;
        s->tile_abort[slot] = 0;
        s->tile_slow[slot] = slow_held;
        mbar_arrive(&s->tile_full[slot]);
        if (tile < 0) break;
        if (tile & kRedEntry) continue;  // reduction continuation: no MMA work
        int mb, nb;
        tile_coords(tile / split, p, mb, nb);
        const int kb0 = static_cast<int>(tile % split) * num_kb;
        for (int kb = 0; kb < num_kb; ++kb) {
          if (D > 0 && issued >= D) {  // position issued - D has landed (its full phase completed)
            const uint32_t back = issued - D;
            mbar_wait(&s->full[back % S], (back / S) & 1);
          }
          const bool abort = p.run.preemptible && kb > 0 && ld_volatile_smem(&s->preempt);
          mbar_wait(&s->empty[stage], phase ^ 1);
          if (abort) {
            s->stage_flag[stage] = 2;  // the MMA warp owns the redo push for this tile
            mbar_arrive(&s->full[stage]);
          } else {
            s->stage_flag[stage] = (kb == num_kb - 1) ? 1u : 0u;
            mbar_arrive_expect_tx(&s->full[stage], Cfg::kStageBytes);
            tma_load_2d(smem_a + stage * Cfg::kABytes, &tma_a, &s->full[stage], (kb0 + kb) * kBK, mb * kBM);
            if (p.b_kblock_major)
              tma_load_3d(smem_b + stage * Cfg::kBBytes, &tma_b, &s->full[stage], 0, nb * BN, kb0 + kb);
            else
              tma_load_2d(smem_b + stage * Cfg::kBBytes, &tma_b, &s->full[stage], (kb0 + kb) * kBK, nb * BN);
          }
          ++issued;
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
          if (abort) break;
        }
      }
      st_volatile_smem(&s->producer_done, 1u);
      dbg_stamp(p.run, 1);
    }
  } else if (warp == 1) {
    // ===================== UMMA issuer =====================
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, drain_phase = 0;
      // Preemptible runs keep at most mma_lag k-blocks of MMAs queued on the tensor core: an
      // abort then drains <= mma_lag k-blocks instead of the whole smem ring (lower
      // preemption latency; the queue still never runs dry).
      // (Stages are consumed in ring order, so the k-block `lag` steps back sits at stage
      // - lag with the phase flipped on wrap-around: no history arrays, which would live in
      // local memory and slow this issue loop by ~9%.)
      const int lag = p.run.preemptible ? p.mma_lag : 0;
      int consumed = 0;
      for (int j = 0;; ++j) {
        const int slot = j & 1;
        mbar_wait(&s->tile_full[slot], (j >> 1) & 1);
        if (s->tile_id[slot] < 0) break;
        if (s->tile_id[slot] & kRedEntry) {  // reduction continuation: hand the slot on
          if (j >= 2) mbar_wait(&s->tmem_empty[slot], ((j >> 1) & 1) ^ 1);
          mbar_arrive(&s->tmem_full[slot]);
          continue;
        }
        // A preemption seen while the epilogue still holds this accumulator slot (a previous
        // unit's epilogue, e.g. a k-split reduction): consume this unit's ring positions right
        // away without MMAs, so the producer's stop is not held behind the epilogue, and take
        // the slot (in order) afterwards.
        bool aborted = false, have_slot = j < 2;
        if (!have_slot) {
          if (mbar_wait_unless(&s->tmem_empty[slot], ((j >> 1) & 1) ^ 1, p.run.preemptible ? &s->preempt : nullptr, 1u))
            have_slot = true;
          else
            aborted = true;
        }
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(slot * BN);
        for (int kb = 0;; ++kb) {
          mbar_wait(&s->full[stage], phase);
          tc_fence_after();
          const uint32_t flag = s->stage_flag[stage];
          // Once preempted, stop feeding the tensor core: the tile is abandoned anyway.
          if (!aborted && p.run.preemptible && ld_volatile_smem(&s->preempt)) aborted = true;
          if (flag == 2) aborted = true;
          if (aborted) {
            mbar_arrive(&s->empty[stage]);
          } else {
            if (lag > 0 && consumed >= lag) {
              int ps = static_cast<int>(stage) - lag;
              uint32_t pp = phase;
              if (ps < 0) {
                ps += S;
                pp ^= 1;
              }
              mbar_wait(&s->empty[ps], pp);
            }
            const uint64_t a0 = umma_desc_k_sw128(smem_u32(smem_a + stage * Cfg::kABytes));
            const uint64_t b0 = umma_desc_k_sw128(smem_u32(smem_b + stage * Cfg::kBBytes));
#pragma unroll
            for (int k = 0; k < kBK / kUmmaK; ++k) {
              // advance 16 elements (32 B) along K inside the 128 B swizzle atom: +2 in addr>>4 units
              umma_bf16(d_tmem, a0 + 2ull * k, b0 + 2ull * k, Cfg::kIdesc, (kb | k) != 0 ? 1u : 0u);
            }
            umma_commit(&s->empty[stage]);
          }
          ++consumed;
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
          if (flag != 0) break;
        }
        if (s->tile_slow[slot]) atomicSub(p.slow_sem, 1u);  // every load of the unit has landed
        if (aborted) {
          if (!have_slot) mbar_wait(&s->tmem_empty[slot], ((j >> 1) & 1) ^ 1);  // keep the slot order
          // Tell the epilogue to skip the tile (it reads nothing of it) with a plain arrive,
          // then drain this tile's issued MMAs (TMEM must be quiescent before dealloc) and park
          // the tile on the redo list: both before this thread reaches the teardown barrier.
          s->tile_abort[slot] = 1;
          mbar_arrive(&s->tmem_full[slot]);
          umma_commit(&s->mma_drain);
          mbar_wait(&s->mma_drain, drain_phase);
          drain_phase ^= 1;
          push_redo(p.run, static_cast<unsigned long long>(s->tile_id[slot]));
        } else {
          umma_commit(&s->tmem_full[slot]);
        }
      }
      dbg_stamp(p.run, 2);
    }
  } else if (warp == 2) {
    // The mirror poller stays up until the epilogue is done, not just the producer: an epilogue
    // still reducing split-K partials must see a preemption (it stops at a chunk boundary).
    if (lane == 0 && p.run.preemptible) poll_mirror(p.run, &s->preempt, &s->epi_done);
  } else if (warp == 3) {
    if (lane == 0 && p.run.preemptible && blockIdx.x == 0) poll_host(p.run, &s->preempt, &s->producer_done);
    if (lane == 0 && p.run.preemptible && blockIdx.x >= 1 && blockIdx.x <= kAuxPollers)
      poll_host_aux(p.run, &s->preempt, &s->producer_done, 300u * blockIdx.x);
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int q = warp - 4;  // TMEM lane quarter
    int cbuf_idx = 0;
    for (int j = 0;; ++j) {
      const int slot = j & 1;
      mbar_wait(&s->tile_full[slot], (j >> 1) & 1);
      const long long tile = s->tile_id[slot];
      if (tile < 0) break;
      mbar_wait(&s->tmem_full[slot], (j >> 1) & 1);
      if (q == 0 && lane == 0) dbg_stamp_ext(p.run, 10);  // diagnostics: epilogue unit start
      tc_fence_after();
      const bool cont = (tile & kRedEntry) != 0;  // reduction continuation (split-K tree)
      const bool keep = !cont && !s->tile_abort[slot];
      const long long unit_tile = cont ? static_cast<long long>((tile >> 32) & 0x3FFFFFFF) : tile / split;
      const int unit_slice = cont ? 0 : static_cast<int>(tile % split);
      int mb = 0, nb = 0;
      if (keep || cont) tile_coords(unit_tile, p, mb, nb);
      bool abandoned = false;  // preempted while storing: the unit goes to the redo list
      if (keep) {
        const int row_in_tile = q * 32 + lane;
        const int row = mb * kBM + row_in_tile;
        // split-K partial layout (per unit, 128 x BN fp32): [BN / 4][128 rows] of float4, so for a
        // fixed column quad the 32 lanes of a warp touch 512 contiguous bytes (coalesced).
        float4* wunit = split > 1 ? reinterpret_cast<float4*>(p.ws) +
                                        (static_cast<size_t>(unit_tile) * split + unit_slice) * (kBM * BN / 4)
                                  : nullptr;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          if (p.run.preemptible) {  // one decision per 32-column chunk for the 4 epilogue warps
            if (q == 0 && lane == 0) s->red_stop = ld_volatile_smem(&s->preempt) != 0 ? 1u : 0u;
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const bool stop = s->red_stop != 0;
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (stop) {
              if (q == 0 && lane == 0) push_redo(p.run, static_cast<unsigned long long>(tile));
              abandoned = true;
              break;
            }
          }
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(slot * BN + c0), r);
          tmem_ld_wait();
          if (split > 1) {
#pragma unroll
            for (int v = 0; v < 8; ++v)
              wunit[static_cast<size_t>(c0 / 4 + v) * kBM + row_in_tile] =
                  make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                              __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
          } else {
            // bf16 -> this warp's staging buffer (64B swizzle: chunk ^= (row >> 1) & 3, conflict
            // free) -> one TMA store of the 32 x 32 box.  The buffer is reused two stores later.
            uint8_t* cbuf = smem_c + (q * 2 + cbuf_idx) * (32 * 64);
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
            const bool epi = p.bias || p.resid || p.act;
            const size_t col0 = static_cast<size_t>(nb) * BN + c0;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              float f[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(r[8 * v + e]);
              if (epi)
                epilogue8(f, p.bias ? p.bias + col0 + 8 * v : nullptr,
                          p.resid ? p.resid + static_cast<size_t>(row) * p.n + col0 + 8 * v : nullptr, p.act);
              uint4 w;
              w.x = pack_bf16x2(f[0], f[1]);
              w.y = pack_bf16x2(f[2], f[3]);
              w.z = pack_bf16x2(f[4], f[5]);
              w.w = pack_bf16x2(f[6], f[7]);
              *reinterpret_cast<uint4*>(cbuf + lane * 64 + ((v ^ ((lane >> 1) & 3)) * 16)) = w;
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tma_c, cbuf, nb * BN + c0, mb * kBM + q * 32);
              bulk_commit();
            }
            cbuf_idx ^= 1;
          }
        }
        if (q == 0 && lane == 0 && !abandoned) ++s->tiles_done;
      }
      tc_fence_before();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (q == 0 && lane == 0) {
        mbar_arrive(&s->tmem_empty[slot]);
        mbar_arrive(&s->tile_empty[slot]);
      }
      if (q == 0 && lane == 0) dbg_stamp_ext(p.run, 11);  // unit's TMEM drained / partial stored
      if (split > 1 && p.tile_cnt && ((keep && !abandoned) || cont)) {
        // split-K: arrive at this slice's level-0 group (or resume a parked group) and
        // reduce up the tree as far as this unit is the last arrival
        const int row_in_tile = q * 32 + lane;
        if (cont)
          split_tree_reduce<BN>(p, s, unit_tile, static_cast<int>((tile >> 24) & 0xFF),
                                static_cast<int>((tile >> 8) & 0xFFFF), static_cast<int>(tile & 0xFF), false, mb, nb,
                                row_in_tile);
        else
          split_tree_reduce<BN>(p, s, unit_tile, 0, unit_slice / kRedFan, 0, true, mb, nb, row_in_tile);
      }
    }
    if (lane == 0) bulk_wait_read<0>();  // staging must stay valid until the TMA read it
    if (q == 0 && lane == 0) {
      st_volatile_smem(&s->epi_done, 1u);
      dbg_stamp(p.run, 3);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, Cfg::kTmemCols);
  if (threadIdx.x == 0) dbg_stamp(p.run, 4);

  if (threadIdx.x == 0) cta_exit(p.run, s->tiles_done);
}

// Split-K reduction (runs as the next PDL-chained kernel): C tile = sum over slices (in
// slice order: deterministic) of the fp32 partials, written as bf16.  One thread per
// (tile, column quad, row): coalesced float4 reads, all SMs.
struct SplitReduceParams {
  TileRun run;  // HP bookkeeping only (non-preemptible)
  const float4* ws;
  __nv_bfloat16* c;
  int n, tiles_m, tiles_n, group_m, bn, split;
  long long total;  // tiles * (bn / 4) * 128
  const __nv_bfloat16* bias;  // GEMM epilogue (GemmParams::bias / resid / act)
  const __nv_bfloat16* resid;
  int act;
};

__global__ void __launch_bounds__(256) splitk_reduce_kernel(const __grid_constant__ SplitReduceParams p) {
  if (threadIdx.x == 0) cta_started(p.run);
  if (p.run.hp_ctl) {
    pdl_launch_dependents();
    if (p.run.pdl_wait) pdl_wait();
  }
  const int quads = p.bn / 4;
  GemmParams gp{};
  gp.tiles_m = p.tiles_m;
  gp.tiles_n = p.tiles_n;
  gp.group_m = p.group_m;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < p.total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(i % kBM);
    const long long tq = i / kBM;
    const int cq = static_cast<int>(tq % quads);
    const long long tile = tq / quads;
    const float4* base = p.ws + static_cast<size_t>(tile) * p.split * (kBM * quads) + static_cast<size_t>(cq) * kBM + row;
    float4 x = base[0];
    for (int sl = 1; sl < p.split; ++sl) {
      const float4 u = base[static_cast<size_t>(sl) * (kBM * quads)];
      x.x += u.x; x.y += u.y; x.z += u.z; x.w += u.w;
    }
    int mb, nb;
    tile_coords(tile, gp, mb, nb);
    if (p.bias || p.resid || p.act) {
      const size_t col = static_cast<size_t>(nb) * p.bn + cq * 4;
      const size_t rr = static_cast<size_t>(mb * kBM + row);
      float f[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (p.bias) f[e] += __bfloat162float(p.bias[col + e]);
        if (p.resid) f[e] += __bfloat162float(p.resid[rr * p.n + col + e]);
        if (p.act == 1) f[e] = fmaxf(f[e], 0.0f);
        if (p.act == 2) {
          const float k0 = 0.7978845608028654f, k1 = 0.044715f;
          f[e] = 0.5f * f[e] * (1.0f + tanhf(k0 * (f[e] + k1 * f[e] * f[e] * f[e])));
        }
      }
      x = make_float4(f[0], f[1], f[2], f[3]);
    }
    uint2 o;
    o.x = pack_bf16x2(x.x, x.y);
    o.y = pack_bf16x2(x.z, x.w);
    *reinterpret_cast<uint2*>(p.c + static_cast<size_t>(mb * kBM + row) * p.n + static_cast<size_t>(nb) * p.bn + cq * 4) = o;
  }
  __syncthreads();
  if (threadIdx.x == 0) cta_exit(p.run, 0);
}

}  // namespace msdev
