// Persistent, preemptible tcgen05 GEMM on CTA PAIRS (cta_group::2) — the LP GEMM tenant
// for 256-aligned shapes.
//
//   C[M, N] (bf16) = A[M, K] * B[N, K]^T, bf16 in, fp32 accumulate in TMEM; 256 x 256 tiles.
//
// Why pairs: a single-CTA 128 x 256 x 64 k-block moves 48 KB into one SM's shared memory
// per 512 MMA cycles; the pair's M=256 x N=256 UMMA needs only each CTA's 128 rows of A and
// 128 columns of B (32 KB per SM per k-block), which is what cuBLAS's own B200 kernel for
// this shape does (nvjet ..._256x256_64x4_2x1_2cta: 96% tensor-pipe activity vs 72-78% for
// the single-CTA kernel, profiles/r02_ncu_gemm_vs_cublas.txt).
//
// Steady state has no per-stage cross-CTA messages (the round-1 pair kernel sent every
// stage's command from the leader to the peer and ran at parity with the single kernel):
//   leader warp 0 : claims a tile, announces {tile, first ring position} to the peer (one
//                   DSMEM store + remote arrive per TILE), then streams its halves of A/B
//                   into its ring; it arms each stage's full barrier for BOTH CTAs' bytes
//   peer   warp 0 : on each announcement streams its halves into its own ring, completing
//                   the bytes on the leader's full barrier (cp.async.bulk.tensor .cta_group::2);
//                   it waits only on its own empty barriers
//   leader warp 1 : single-thread UMMA issuer (tcgen05.mma.cta_group::2, M=256, N=256, K=16);
//                   every commit is multicast to both CTAs' empty barriers, accumulator-ready
//                   commits to both CTAs' tmem_full barriers
//   warp 2        : TMEM allocator (cta_group::2, 512 columns = 2 x 256 fp32 accumulators);
//                   leader lane 0 then polls the preempt epoch
//   warp 3 (CTA 0): host poller
//   warps 4-7     : epilogue of this CTA's 128 rows (tcgen05.ld -> bf16 -> TMA store)
//
// Preemption (same semantics as tc_gemm.cuh: claim counter, abort at a k-block, abandoned
// tiles on the redo list, C written only for complete tiles).  The two producers run ahead
// independently, so they must agree where the aborted tile's stream ends before either
// moves on: the leader stops at k-block L, asks the peer to stop, the peer answers with the
// k-block P it stopped at (or num_kb if it had issued everything).  Ring positions [P, L)
// were armed for both halves but get only the leader's: the leader completes the missing
// bytes itself (mbarrier.complete_tx); positions [L, P) get only the peer's bytes: the
// leader arms them for those bytes and flags them "discard"; then one terminal position ends
// the tile.  The MMA warp consumes every position (no MMAs once aborted) and releases it in
// both CTAs, so both rings stay phase-aligned; the next announcement carries the ring
// position both producers resume from.
#pragma once

#include "tc_gemm.cuh"

namespace msdev {

// TN = pair tile width: 256 (one M=256 x N=256 UMMA per k-step, two accumulators in TMEM)
// or 512 (two UMMAs per k-step over the tile's column halves; the accumulator fills all 512
// TMEM columns, so the epilogue of tile j and the MMAs of tile j+1 do not overlap, but each
// SM stages 48 KB per 1024 MMA cycles instead of 32 KB per 512 — the shape of cuBLAS's own
// kernel for 8192^3 on this part).
template <int TN>
struct Gemm2Cfg {
  static constexpr int kHalfBytes = 128 * kBK * 2;      // 16 KB: 128 rows (A) or columns (B) x 64 k
  static constexpr int kBHalves = TN / 256;             // UMMAs (N = 256) per k-step
  static constexpr int kStageBytes = (1 + kBHalves) * kHalfBytes;  // one CTA's bytes of a k-block
  static constexpr int kStages = TN == 256 ? 6 : 4;
  static constexpr int kSlots = 512 / TN;               // accumulators in TMEM
  static constexpr int kTmemCols = 512;
  static constexpr int kCStageBytes = 4 * 2 * 32 * 64;
  static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + kCStageBytes + 1024;
  static constexpr uint32_t kIdesc = umma_idesc_bf16(256, 256);
  static constexpr uint32_t kIdescQ = umma_idesc_bf16(256, 128);  // quarter units (TN = 512)
};
constexpr int kGemm2MaxStages = 6;

// Work unit -> (tile, its columns [c_lo, c_lo + cw) of the TN-wide tile): see
// GemmParams::half_base.  Whole tiles have cw = TN; the last wave's units are the tile's
// 256-column halves or 128-column quarters (p.tail_parts).
template <int TN>
__device__ __forceinline__ long long pair_unit(long long u, const GemmParams& p, int& c_lo, int& cw) {
  if (p.half_units > 0 && u >= p.half_base) {
    const long long v = u - p.half_base;
    cw = TN / p.tail_parts;
    c_lo = static_cast<int>(v % p.tail_parts) * cw;
    return p.half_base + v / p.tail_parts;
  }
  c_lo = 0;
  cw = TN;
  return u;
}

// Stage flags (leader): 0 data, 1 data + last k-block, 2 terminal (no data), 3 peer-only
// bytes of an aborted tile (discard).
struct Gemm2Ctl {
  uint64_t full[kGemm2MaxStages];   // leader: producer's arrive.expect_tx + both CTAs' TMA bytes
  uint64_t empty[kGemm2MaxStages];  // both: MMA commit multicast (or the abort path's arrives)
  uint64_t tile_full[2];              // both: tile announcement
  uint64_t tile_empty[2];             // leader: both epilogues
  uint64_t tmem_full[2];              // both: accumulator ready / aborted
  uint64_t tmem_empty[2];             // leader: both epilogues
  uint64_t stop_bar;                  // leader: the peer's stop report
  uint64_t mma_drain;
  long long tile_id[2];
  uint32_t tile_start[2];  // ring position of the tile's first k-block
  uint32_t tile_abort[2];
  uint32_t stage_flag[kGemm2MaxStages];
  alignas(16) uint32_t peer_stop[4];  // leader: k-block at which the peer stopped (st.async)
  uint32_t stop_req;   // peer: ordinal (j + 1) of the tile the leader asks it to stop
  uint32_t tmem_base;
  uint32_t preempt;
  uint32_t producer_done;
  uint32_t tiles_done;
  uint32_t epi_abort;  // peer: ordinal (j + 1) of the tile whose epilogue the leader abandoned
  uint32_t epi_stop;   // epilogue warps' shared stop decision
  uint32_t epi_done;   // epilogue finished (the leader's mirror poller may stop)
  uint32_t tile_slow[2];  // leader: the tile holds an off-device admission slot (tc_gemm.cuh slow_admit)
};

// ---- cluster helpers ----------------------------------------------------------------
__device__ __forceinline__ void st_cluster_u64(uint32_t addr, unsigned long long v) {
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "MS_WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra MS_WAITC_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(uint32_t smem_dst, const CUtensorMap* map, uint32_t bar_cluster,
                                                 int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_dst),
      "l"(map), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void umma_commit_pair_mc(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* smem_dst, uint32_t ncols) {  // whole warp, both CTAs
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_complete_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
template <int TN>
__global__ void __launch_bounds__(256, 1)
    tc_gemm2_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                    const __grid_constant__ CUtensorMap tma_bq,  // B, 64-row boxes (quarter units)
                    const __grid_constant__ CUtensorMap tma_c, const __grid_constant__ GemmParams p) {
  using Cfg = Gemm2Cfg<TN>;
  constexpr int S = Cfg::kStages;
  constexpr int NS = Cfg::kSlots;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;                              // [S][128 x 64] bf16, SW128
  uint8_t* smem_b = smem + S * Cfg::kHalfBytes;        // [S][kBHalves][128 x 64] bf16, SW128
  uint8_t* smem_c = smem + S * Cfg::kStageBytes;
  Gemm2Ctl* s = reinterpret_cast<Gemm2Ctl*>(smem_c + Cfg::kCStageBytes);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0 && p.run.dbg) {  // diagnostics: SM of each CTA (pair placement)
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.run.dbg[2048 + blockIdx.x * 64 + 60] = smid;
  }

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&s->full[i], 1);
      mbar_init(&s->empty[i], 1);
      s->stage_flag[i] = 0;
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s->tile_full[i], 1);
      mbar_init(&s->tile_empty[i], 2);  // both CTAs' epilogues
      mbar_init(&s->tmem_full[i], 1);
      mbar_init(&s->tmem_empty[i], 2);  // both CTAs' epilogues
    }
    mbar_init(&s->stop_bar, 1);
    mbar_init(&s->mma_drain, 1);
    s->stop_req = 0;
    s->epi_abort = 0;
    s->epi_done = 0;
    s->preempt = 0;
    s->producer_done = 0;
    s->tiles_done = 0;
    fence_mbar_init();
    cta_started(p.run);
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tma_a);
    prefetch_tmap(&tma_b);
    prefetch_tmap(&tma_bq);
    prefetch_tmap(&tma_c);
  }
  if (warp == 2) tmem_alloc_pair(&s->tmem_base, Cfg::kTmemCols);
  tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs initialised, TMEM allocated in both
  tc_fence_after();
  const uint32_t tmem_base = s->tmem_base;
  const int num_kb = p.k / kBK;

  if (warp == 0) {
    if (lane == 0 && leader) {
      // ===================== leader: tile scheduler + producer =====================
      const uint32_t peer_tile_id = mapa_shared(smem_u32(&s->tile_id[0]), 1);
      const uint32_t peer_tile_start = mapa_shared(smem_u32(&s->tile_start[0]), 1);
      const uint32_t peer_tile_abort = mapa_shared(smem_u32(&s->tile_abort[0]), 1);
      const uint32_t peer_tile_full = mapa_shared(smem_u32(&s->tile_full[0]), 1);
      const uint32_t peer_stop_req = mapa_shared(smem_u32(&s->stop_req), 1);
      uint32_t pos = 0, stop_phase = 0;
      for (int j = 0;; ++j) {
        const int slot = j & 1;
        if (j >= 2) mbar_wait_cluster(&s->tile_empty[slot], ((j >> 1) & 1) ^ 1);
        long long tile = -1;
        if (!(p.run.preemptible && ld_volatile_smem(&s->preempt))) tile = claim_tile(p.run);
        int c_lo = 0, cw = TN;
        const long long tl = tile >= 0 ? pair_unit<TN>(tile, p, c_lo, cw) : -1;
        s->tile_slow[slot] = slow_admit(p, &s->preempt, tile, tl);
        s->tile_id[slot] = tile;
        s->tile_start[slot] = pos;
        s->tile_abort[slot] = 0;
        st_cluster_u64(peer_tile_id + slot * 8, static_cast<unsigned long long>(tile));
        st_cluster_u32(peer_tile_start + slot * 4, pos);
        st_cluster_u32(peer_tile_abort + slot * 4, 0u);
        mbar_arrive(&s->tile_full[slot]);
        mbar_arrive_cluster(peer_tile_full + slot * 8);  // release.cluster: the stores above first
        if (tile < 0) break;
        int mb, nb;
        tile_coords(tl, p, mb, nb);
        // one CTA's bytes per k-block: 128 rows of A + cw / 2 columns of B
        const uint32_t stage_bytes = Cfg::kHalfBytes + static_cast<uint32_t>(cw) * kBK;
        const uint32_t pos0 = pos;
        int lead_stop = num_kb;
        for (int kb = 0; kb < num_kb; ++kb) {
          const bool may_stop = p.run.preemptible && kb > 0;
          if (may_stop && ld_volatile_smem(&s->preempt)) {
            lead_stop = kb;
            break;
          }
          const uint32_t st = pos % S;
          if (!mbar_wait_unless(&s->empty[st], ((pos / S) & 1) ^ 1, may_stop ? &s->preempt : nullptr, 1u)) {
            lead_stop = kb;
            break;
          }
          s->stage_flag[st] = (kb == num_kb - 1) ? 1u : 0u;
          mbar_arrive_expect_tx(&s->full[st], 2 * stage_bytes);  // both CTAs' halves
          const uint32_t fb = smem_u32(&s->full[st]);
          tma_load_2d_pair(smem_u32(smem_a + st * Cfg::kHalfBytes), &tma_a, fb, kb * kBK, mb * 256);
          if (cw == TN) {
#pragma unroll
            for (int h = 0; h < Cfg::kBHalves; ++h)
              tma_load_2d_pair(smem_u32(smem_b + (st * Cfg::kBHalves + h) * Cfg::kHalfBytes), &tma_b, fb, kb * kBK,
                               nb * TN + h * 256);
          } else {  // a part unit: its columns into the stage's first B slot
            tma_load_2d_pair(smem_u32(smem_b + st * Cfg::kBHalves * Cfg::kHalfBytes), cw == 128 ? &tma_bq : &tma_b, fb,
                             kb * kBK, nb * TN + c_lo);
          }
          ++pos;
        }
        if (lead_stop < num_kb) {
          dbg_stamp_ext(p.run, 20);  // diagnostics (drain probe): leader producer stopped
          // agree on the end of this tile's stream with the peer (see the header); the answer
          // is one st.async completing the armed stop barrier (no release fence on the path)
          mbar_arrive_expect_tx(&s->stop_bar, 16);
          st_cluster_u32(peer_stop_req, static_cast<uint32_t>(j + 1));
          mbar_wait(&s->stop_bar, stop_phase);
          stop_phase ^= 1;
          dbg_stamp_ext(p.run, 21);  // peer's stop report received
          const int ps = static_cast<int>(ld_volatile_smem(&s->peer_stop[0]));
          for (int kb = ps; kb < lead_stop; ++kb)  // armed for both halves, the peer's never comes
            mbar_complete_tx(&s->full[(pos0 + kb) % S], stage_bytes);
          for (int kb = lead_stop; kb < ps; ++kb) {  // only the peer's half comes
            const uint32_t st = pos % S;
            mbar_wait(&s->empty[st], ((pos / S) & 1) ^ 1);
            s->stage_flag[st] = 3u;
            mbar_arrive_expect_tx(&s->full[st], stage_bytes);
            ++pos;
          }
          const uint32_t st = pos % S;  // terminal position: ends the tile for the MMA warp
          mbar_wait(&s->empty[st], ((pos / S) & 1) ^ 1);
          s->stage_flag[st] = 2u;
          mbar_arrive(&s->full[st]);
          ++pos;
          dbg_stamp_ext(p.run, 22);  // terminal position issued
        }
      }
      st_volatile_smem(&s->producer_done, 1u);
      dbg_stamp(p.run, 1);
    } else if (lane == 0) {
      // ===================== peer: producer of its halves =====================
      const uint32_t lead_peer_stop = mapa_shared(smem_u32(&s->peer_stop[0]), 0);
      const uint32_t lead_stop_bar = mapa_shared(smem_u32(&s->stop_bar), 0);
      auto report = [&](int kb) {  // data and completion in one async store
        st_async_v4(lead_peer_stop, static_cast<uint32_t>(kb), 0u, 0u, 0u, lead_stop_bar);
      };
      mbar_wait_cluster(&s->tile_full[0], 0);
      for (int j = 0;; ++j) {
        const int slot = j & 1;
        const long long tile = *reinterpret_cast<volatile long long*>(&s->tile_id[slot]);
        if (tile < 0) break;
        uint32_t pos = *reinterpret_cast<volatile uint32_t*>(&s->tile_start[slot]);
        int c_lo, cw, mb, nb;
        tile_coords(pair_unit<TN>(tile, p, c_lo, cw), p, mb, nb);
        const uint32_t ord = static_cast<uint32_t>(j + 1);
        bool reported = false;
        for (int kb = 0; kb < num_kb; ++kb) {
          const uint32_t st = pos % S;
          if (!mbar_wait_unless(&s->empty[st], ((pos / S) & 1) ^ 1, &s->stop_req, ord) ||
              ld_volatile_smem(&s->stop_req) == ord) {
            report(kb);
            reported = true;
            dbg_stamp_ext(p.run, 23);  // peer producer stopped
            break;
          }
          const uint32_t fb = mapa_shared(smem_u32(&s->full[st]), 0);
          tma_load_2d_pair(smem_u32(smem_a + st * Cfg::kHalfBytes), &tma_a, fb, kb * kBK, mb * 256 + 128);
          if (cw == TN) {
#pragma unroll
            for (int h = 0; h < Cfg::kBHalves; ++h)
              tma_load_2d_pair(smem_u32(smem_b + (st * Cfg::kBHalves + h) * Cfg::kHalfBytes), &tma_b, fb, kb * kBK,
                               nb * TN + h * 256 + 128);
          } else {  // the second half of the part unit's columns (cta_group::2 splits N)
            tma_load_2d_pair(smem_u32(smem_b + st * Cfg::kBHalves * Cfg::kHalfBytes), cw == 128 ? &tma_bq : &tma_b, fb,
                             kb * kBK, nb * TN + c_lo + cw / 2);
          }
          ++pos;
        }
        // Next announcement; a stop request for this tile that comes after every k-block was
        // issued is answered with num_kb.
        const int ns = (j + 1) & 1;
        const uint32_t np = static_cast<uint32_t>(((j + 1) >> 1) & 1);
        for (;;) {
          if (mbar_try_wait_cluster(&s->tile_full[ns], np)) break;
          if (!reported && ld_volatile_smem(&s->stop_req) == ord) {
            report(num_kb);
            reported = true;
          }
        }
      }
      st_volatile_smem(&s->producer_done, 1u);
    }
  } else if (warp == 1) {
    // ===================== leader: UMMA issuer (cta_group::2) =====================
    if (lane == 0 && leader) {
      uint32_t pos = 0, drain_phase = 0;
      const int lag = p.run.preemptible ? p.mma_lag : 0;  // see tc_gemm.cuh
      uint32_t consumed = 0;
      const uint32_t peer_tile_abort = mapa_shared(smem_u32(&s->tile_abort[0]), 1);
      const uint32_t peer_tmem_full = mapa_shared(smem_u32(&s->tmem_full[0]), 1);
      const uint32_t peer_empty = mapa_shared(smem_u32(&s->empty[0]), 1);
      for (int j = 0;; ++j) {
        const int slot = j & 1;
        mbar_wait(&s->tile_full[slot], (j >> 1) & 1);
        if (s->tile_id[slot] < 0) break;
        int c_lo, cw;
        pair_unit<TN>(s->tile_id[slot], p, c_lo, cw);
        const int ts = j % NS;  // accumulator slot
        // (see tc_gemm.cuh: a preemption seen while the epilogue holds the accumulator lets the
        // MMA warp consume this tile's positions first, so the stop agreement is not held
        // behind the previous tile's epilogue)
        bool aborted = false, have_slot = j < NS;
        if (!have_slot) {
          if (mbar_wait_cluster_unless(&s->tmem_empty[ts], ((j / NS) & 1) ^ 1,
                                       p.run.preemptible ? &s->preempt : nullptr, 1u))
            have_slot = true;
          else
            aborted = true;
        }
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(ts * TN);
        for (int kb = 0;; ++kb) {
          const uint32_t st = pos % S;
          mbar_wait(&s->full[st], (pos / S) & 1);
          tc_fence_after();
          const uint32_t flag = s->stage_flag[st];
          if (!aborted && p.run.preemptible && ld_volatile_smem(&s->preempt)) {
            aborted = true;
            dbg_stamp_ext(p.run, 24);  // MMA warp saw the preemption
          }
          if (flag >= 2) aborted = true;
          if (aborted) {
            // no MMA reads this position: release it in both CTAs
            mbar_arrive(&s->empty[st]);
            mbar_arrive_remote_relaxed(peer_empty + st * 8);
          } else {
            if (lag > 0 && consumed >= static_cast<uint32_t>(lag)) {
              const uint32_t bp = pos - lag;
              mbar_wait(&s->empty[bp % S], (bp / S) & 1);
            }
            const uint64_t a0 = umma_desc_k_sw128(smem_u32(smem_a + st * Cfg::kHalfBytes));
            if (cw == TN) {
#pragma unroll
              for (int k = 0; k < kBK / kUmmaK; ++k)
#pragma unroll
                for (int h = 0; h < Cfg::kBHalves; ++h) {
                  const uint64_t b0 = umma_desc_k_sw128(smem_u32(smem_b + (st * Cfg::kBHalves + h) * Cfg::kHalfBytes));
                  umma_bf16_pair(d_tmem + h * 256, a0 + 2ull * k, b0 + 2ull * k, Cfg::kIdesc, (kb | k) != 0 ? 1u : 0u);
                }
            } else {  // part unit: one UMMA (N = cw) into its columns of the accumulator
              const uint64_t b0 = umma_desc_k_sw128(smem_u32(smem_b + st * Cfg::kBHalves * Cfg::kHalfBytes));
              const uint32_t idesc = cw == 128 ? Cfg::kIdescQ : Cfg::kIdesc;
#pragma unroll
              for (int k = 0; k < kBK / kUmmaK; ++k)
                umma_bf16_pair(d_tmem + static_cast<uint32_t>(c_lo), a0 + 2ull * k, b0 + 2ull * k, idesc,
                               (kb | k) != 0 ? 1u : 0u);
            }
            umma_commit_pair_mc(&s->empty[st], 0x3);
          }
          ++consumed;
          ++pos;
          if (flag == 1 || flag == 2) break;
        }
        if (s->tile_slow[slot]) atomicSub(p.slow_sem, 1u);  // every load of the tile has landed
        if (aborted) {
          dbg_stamp_ext(p.run, 25);  // aborted tile's ring positions consumed
          if (!have_slot) mbar_wait_cluster(&s->tmem_empty[ts], ((j / NS) & 1) ^ 1);  // keep the slot order
          // The epilogues read nothing of an aborted tile: tell them first, so their teardown
          // does not wait behind the MMA drain and the redo push (an L2 round trip); both
          // complete before this thread reaches the teardown barrier (TMEM dealloc, cta_exit).
          s->tile_abort[slot] = 1;
          st_cluster_u32(peer_tile_abort + slot * 4, 1u);
          mbar_arrive(&s->tmem_full[ts]);
          mbar_arrive_cluster(peer_tmem_full + ts * 8);  // release.cluster: the abort flag first
          dbg_stamp_ext(p.run, 27);  // epilogues told
          umma_commit_pair(&s->mma_drain);
          mbar_wait(&s->mma_drain, drain_phase);
          drain_phase ^= 1;
          dbg_stamp_ext(p.run, 26);  // queued MMAs drained
          push_redo(p.run, static_cast<unsigned long long>(s->tile_id[slot]));
        } else {
          umma_commit_pair_mc(&s->tmem_full[ts], 0x3);
        }
      }
      dbg_stamp(p.run, 2);
    }
  } else if (warp == 2) {
    // up until the epilogue is done: an epilogue in progress abandons its tile on a preemption
    if (lane == 0 && leader && p.run.preemptible) {
      poll_mirror(p.run, &s->preempt, &s->epi_done);
      dbg_stamp_ext(p.run, 31);  // mirror poller left
    }
  } else if (warp == 3) {
    // (CTA 0's peer cannot exit before CTA 0 reaches the teardown cluster barrier)
    if (lane == 0 && p.run.preemptible && blockIdx.x == 0) {
      poll_host(p.run, &s->preempt, &s->producer_done, 2);
      dbg_stamp_ext(p.run, 30);  // host poller left
    }
    // auxiliary host pollers on the next leaders (see tile_run.cuh poll_host_aux)
    if (lane == 0 && p.run.preemptible && leader && blockIdx.x >= 2 && blockIdx.x <= 2 * kAuxPollers)
      poll_host_aux(p.run, &s->preempt, &s->producer_done, 150u * blockIdx.x);
  } else if (warp >= 4) {
    // ===================== epilogue (this CTA's 128 rows of the pair tile) =====================
    const int q = warp - 4;
    int cbuf_idx = 0;
    const uint32_t lead_tmem_empty = mapa_shared(smem_u32(&s->tmem_empty[0]), 0);
    const uint32_t lead_tile_empty = mapa_shared(smem_u32(&s->tile_empty[0]), 0);
    const uint32_t peer_epi_abort = mapa_shared(smem_u32(&s->epi_abort), 1);
    const int tid = threadIdx.x - 128;
    for (int j = 0;; ++j) {
      const int slot = j & 1;
      mbar_wait_cluster(&s->tile_full[slot], (j >> 1) & 1);
      const long long tile = *reinterpret_cast<volatile long long*>(&s->tile_id[slot]);
      if (tile < 0) break;
      const int ts = j % NS;
      mbar_wait_cluster(&s->tmem_full[ts], (j / NS) & 1);
      tc_fence_after();
      const bool keep = !*reinterpret_cast<volatile uint32_t*>(&s->tile_abort[slot]);
      if (!keep && q == 0 && lane == 0) dbg_stamp_ext(p.run, 28);  // epilogue: aborted tile seen
      bool abandoned = false;
      if (keep) {
        int c_lo, cw, mb, nb;
        tile_coords(pair_unit<TN>(tile, p, c_lo, cw), p, mb, nb);
        const int c_hi = c_lo + cw;  // the unit's columns
        const int row0 = mb * 256 + static_cast<int>(rank) * 128 + q * 32;
        // A preemption during the store of a completed tile abandons it (the leader decides, at
        // 32-column chunk boundaries, tells the peer, and parks the tile on the redo list): the
        // 512-column epilogue is ~2.5 us of TMEM reads that a preempted grid need not wait for.
#pragma unroll 1
        for (int c0 = c_lo; c0 < c_hi; c0 += 32) {
          if (p.run.preemptible) {
            if (tid == 0)
              s->epi_stop = leader ? (ld_volatile_smem(&s->preempt) != 0 ? 1u : 0u)
                                   : (ld_volatile_smem(&s->epi_abort) == static_cast<uint32_t>(j + 1) ? 1u : 0u);
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const bool stop = s->epi_stop != 0;
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (stop) {
              if (tid == 0 && leader) st_cluster_u32(peer_epi_abort, static_cast<uint32_t>(j + 1));
              abandoned = true;  // (parked on the redo list after the slot is released)
              break;
            }
          }
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(ts * TN + c0), r);
          tmem_ld_wait();
          uint8_t* cbuf = smem_c + (q * 2 + cbuf_idx) * (32 * 64);
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            uint4 w;
            w.x = pack_bf16x2(__uint_as_float(r[8 * v + 0]), __uint_as_float(r[8 * v + 1]));
            w.y = pack_bf16x2(__uint_as_float(r[8 * v + 2]), __uint_as_float(r[8 * v + 3]));
            w.z = pack_bf16x2(__uint_as_float(r[8 * v + 4]), __uint_as_float(r[8 * v + 5]));
            w.w = pack_bf16x2(__uint_as_float(r[8 * v + 6]), __uint_as_float(r[8 * v + 7]));
            *reinterpret_cast<uint4*>(cbuf + lane * 64 + ((v ^ ((lane >> 1) & 3)) * 16)) = w;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tma_c, cbuf, nb * TN + c0, row0);
            bulk_commit();
          }
          cbuf_idx ^= 1;
        }
        if (q == 0 && lane == 0 && leader && !abandoned) ++s->tiles_done;
      }
      tc_fence_before();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (q == 0 && lane == 0) {
        mbar_arrive_cluster(lead_tmem_empty + ts * 8);
        mbar_arrive_cluster(lead_tile_empty + slot * 8);
      }
      if (abandoned && tid == 0 && leader) push_redo(p.run, static_cast<unsigned long long>(tile));
    }
    if (q == 0 && lane == 0) dbg_stamp_ext(p.run, 29);  // epilogue: end announcement seen
    if (lane == 0) bulk_wait_read<0>();
    if (q == 0 && lane == 0) {
      st_volatile_smem(&s->epi_done, 1u);
      dbg_stamp(p.run, 3);
    }
  }

  tc_fence_before();
  cluster_sync_all();  // no CTA frees TMEM or leaves while its peer may still signal it
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair(tmem_base, Cfg::kTmemCols);
  if (threadIdx.x == 0) dbg_stamp(p.run, 4);
  if (threadIdx.x == 0 && leader) cta_exit(p.run, s->tiles_done, 2);  // accounts for the pair
}

}  // namespace msdev
