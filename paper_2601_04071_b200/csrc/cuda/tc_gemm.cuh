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
};

template <int BN>
struct GemmCfg {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (200 * 1024 / kStageBytes) > 8 ? 8 : (200 * 1024 / kStageBytes);
  static constexpr int kTmemCols = 2 * BN < 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  static constexpr int kSmemBytes = 1024 /*align slack*/ + kStages * kStageBytes + 1024 /*barriers etc.*/;
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
  uint32_t stage_flag[8];  // 0: data, 1: data + last k-block, 2: aborted (no data)
  uint32_t tmem_base;
  uint32_t preempt;
  uint32_t producer_done;
  uint32_t tiles_done;
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

template <int BN>
__global__ void __launch_bounds__(256, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                   const __grid_constant__ GemmParams p) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + S * Cfg::kABytes;
  GemmSmemCtl* s = reinterpret_cast<GemmSmemCtl*>(smem + S * Cfg::kStageBytes);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

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
    s->tiles_done = 0;
    fence_mbar_init();
    cta_started(p.run);
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tma_a);
    prefetch_tmap(&tma_b);
  }
  if (warp == 2) tmem_alloc(&s->tmem_base, Cfg::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = s->tmem_base;
  const int num_kb = p.k / kBK;

  if (warp == 0) {
    // ===================== tile scheduler + TMA producer =====================
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (int j = 0;; ++j) {
        const int slot = j & 1;
        if (j >= 2) mbar_wait(&s->tile_empty[slot], ((j >> 1) & 1) ^ 1);
        long long tile = -1;
        if (!(p.run.preemptible && ld_volatile_smem(&s->preempt))) tile = claim_tile(p.run);
        s->tile_id[slot] = tile;
        s->tile_abort[slot] = 0;
        mbar_arrive(&s->tile_full[slot]);
        if (tile < 0) break;
        int mb, nb;
        tile_coords(tile, p, mb, nb);
        for (int kb = 0; kb < num_kb; ++kb) {
          const bool abort = p.run.preemptible && kb > 0 && ld_volatile_smem(&s->preempt);
          mbar_wait(&s->empty[stage], phase ^ 1);
          if (abort) {
            s->stage_flag[stage] = 2;
            mbar_arrive(&s->full[stage]);
            push_redo(p.run, static_cast<unsigned long long>(tile));
          } else {
            s->stage_flag[stage] = (kb == num_kb - 1) ? 1u : 0u;
            mbar_arrive_expect_tx(&s->full[stage], Cfg::kStageBytes);
            tma_load_2d(smem_a + stage * Cfg::kABytes, &tma_a, &s->full[stage], kb * kBK, mb * kBM);
            tma_load_2d(smem_b + stage * Cfg::kBBytes, &tma_b, &s->full[stage], kb * kBK, nb * BN);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
          if (abort) break;
        }
      }
      st_volatile_smem(&s->producer_done, 1u);
    }
  } else if (warp == 1) {
    // ===================== UMMA issuer =====================
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (int j = 0;; ++j) {
        const int slot = j & 1;
        mbar_wait(&s->tile_full[slot], (j >> 1) & 1);
        if (s->tile_id[slot] < 0) break;
        if (j >= 2) mbar_wait(&s->tmem_empty[slot], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(slot * BN);
        bool aborted = false;
        for (int kb = 0;; ++kb) {
          mbar_wait(&s->full[stage], phase);
          tc_fence_after();
          const uint32_t flag = s->stage_flag[stage];
          if (flag == 2) {
            mbar_arrive(&s->empty[stage]);
            aborted = true;
          } else {
            const uint64_t a0 = umma_desc_k_sw128(smem_u32(smem_a + stage * Cfg::kABytes));
            const uint64_t b0 = umma_desc_k_sw128(smem_u32(smem_b + stage * Cfg::kBBytes));
#pragma unroll
            for (int k = 0; k < kBK / kUmmaK; ++k) {
              // advance 16 elements (32 B) along K inside the 128 B swizzle atom: +2 in addr>>4 units
              umma_bf16(d_tmem, a0 + 2ull * k, b0 + 2ull * k, Cfg::kIdesc, (kb | k) != 0 ? 1u : 0u);
            }
            umma_commit(&s->empty[stage]);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
          if (flag != 0) break;
        }
        if (aborted) {
          // Drain the abandoned tile's MMAs (TMEM must be quiescent before dealloc), then
          // tell the epilogue to skip it with a plain (release) arrive.  At most once per CTA.
          umma_commit(&s->mma_drain);
          mbar_wait(&s->mma_drain, 0);
          s->tile_abort[slot] = 1;
          mbar_arrive(&s->tmem_full[slot]);
        } else {
          umma_commit(&s->tmem_full[slot]);
        }
      }
    }
  } else if (warp == 2) {
    if (lane == 0 && p.run.preemptible) run_poller(p.run, &s->preempt, &s->producer_done);
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int q = warp - 4;  // TMEM lane quarter
    for (int j = 0;; ++j) {
      const int slot = j & 1;
      mbar_wait(&s->tile_full[slot], (j >> 1) & 1);
      const long long tile = s->tile_id[slot];
      if (tile < 0) break;
      mbar_wait(&s->tmem_full[slot], (j >> 1) & 1);
      tc_fence_after();
      if (!s->tile_abort[slot]) {
        int mb, nb;
        tile_coords(tile, p, mb, nb);
        const int row = mb * kBM + q * 32 + lane;
        __nv_bfloat16* crow = p.c + static_cast<size_t>(row) * p.n + static_cast<size_t>(nb) * BN;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(slot * BN + c0), r);
          tmem_ld_wait();
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
        if (q == 0 && lane == 0) ++s->tiles_done;
      }
      tc_fence_before();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (q == 0 && lane == 0) {
        mbar_arrive(&s->tmem_empty[slot]);
        mbar_arrive(&s->tile_empty[slot]);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, Cfg::kTmemCols);

  if (threadIdx.x == 0) cta_exit(p.run, s->tiles_done);
}

}  // namespace msdev
