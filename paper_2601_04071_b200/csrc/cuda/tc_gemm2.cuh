// Persistent, preemptible tcgen05 GEMM on CTA PAIRS (cta_group::2) — the LP GEMM tenant
// for 256-aligned shapes.
//
//   C[M, N] (bf16) = A[M, K] * B[N, K]^T, bf16 in, fp32 accumulate in TMEM; 256 x 256 tiles.
//
// Why pairs: a single-CTA 128 x 256 x 64 k-block moves 48 KB into shared memory and reads
// 48 KB back into the tensor core every 512 MMA cycles — ~192 B/clk of smem traffic against
// ~128 B/clk available, which held the single-CTA kernel at ~72% tensor-pipe activity
// (profiles/r01_ncu_gemm_details.csv).  With cta_group::2 the two SMs of a TPC run one
// M=256 x N=256 UMMA: each CTA stages only its 128 rows of A and its 128 columns of B
// (32 KB per k-block), so the smem traffic halves and a 6-stage ring fits in 192 KB.
//
// Roles (256 threads per CTA, cluster of 2; rank 0 = leader):
//   leader warp 0  : tile scheduler + TMA producer; decides every stage (load / abort /
//                    end) and forwards the decision to the peer through DSMEM (command word +
//                    remote mbarrier arrive), so both CTAs always agree on a preemption point
//   peer   warp 0  : command follower: issues its half of each stage's TMA loads, completing
//                    their bytes on the LEADER's full barrier (cp.async.bulk.tensor .cta_group::2)
//   leader warp 1  : single-thread UMMA issuer (tcgen05.mma.cta_group::2, M=256, N=256, K=16);
//                    accumulator-ready commits multicast to both CTAs
//   warp 2         : TMEM allocator (cta_group::2, 512 columns = 2 x 256 fp32 accumulators);
//                    leader lane 0 then polls the preempt epoch
//   warp 3 (CTA 0) : host poller
//   warps 4-7      : epilogue of this CTA's 128 rows (tcgen05.ld -> bf16 -> TMA store)
// Preemption semantics are those of tc_gemm.cuh (tile claim counter, abort at a k-block,
// abandoned tiles on the redo list, C written only for complete tiles); tile ids count
// 256 x 256 pair tiles.
#pragma once

#include "tc_gemm.cuh"

namespace msdev {

struct Gemm2Cfg {
  static constexpr int kHalfBytes = 128 * kBK * 2;  // 16 KB: 128 rows (A) or columns (B) x 64 k
  static constexpr int kStageBytes = 2 * kHalfBytes;
  static constexpr int kStages = 6;
  static constexpr int kTmemCols = 512;
  static constexpr int kCStageBytes = 4 * 2 * 32 * 64;
  static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + kCStageBytes + 1024;
  static constexpr uint32_t kIdesc = umma_idesc_bf16(256, 256);
};

struct Gemm2Ctl {
  uint64_t full[Gemm2Cfg::kStages];   // leader: one arrive_expect_tx + both CTAs' TMA bytes
  uint64_t empty[Gemm2Cfg::kStages];  // leader: MMA commit (both CTAs' stage reads done)
  uint64_t go[Gemm2Cfg::kStages];     // peer: leader's command for this stage
  uint64_t tmem_full[2], tmem_empty[2], tile_full[2], tile_empty[2];
  uint64_t mma_drain;
  long long tile_id[2];
  alignas(16) int4 cmd[Gemm2Cfg::kStages];  // peer: {tile lo, tile hi, kb, 0}; tile -1 skip, -2 end
  uint32_t tile_abort[2];
  uint32_t stage_flag[Gemm2Cfg::kStages];  // leader: 0 data, 1 data + last k-block, 2 aborted
  uint32_t tmem_base;
  uint32_t preempt;
  uint32_t producer_done;
  uint32_t tiles_done;
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

__global__ void __launch_bounds__(256, 1)
    tc_gemm2_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                    const __grid_constant__ CUtensorMap tma_c, const __grid_constant__ GemmParams p) {
  using Cfg = Gemm2Cfg;
  constexpr int S = Cfg::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;                              // [S][128 x 64] bf16, SW128
  uint8_t* smem_b = smem + S * Cfg::kHalfBytes;        // [S][128 x 64] bf16, SW128
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
      mbar_init(&s->go[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s->tmem_full[i], 1);
      mbar_init(&s->tmem_empty[i], 2);  // both CTAs' epilogues
      mbar_init(&s->tile_full[i], 1);
      mbar_init(&s->tile_empty[i], 2);  // both CTAs' epilogues
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
    prefetch_tmap(&tma_c);
  }
  if (warp == 2) tmem_alloc_pair(&s->tmem_base, Cfg::kTmemCols);
  tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs initialised, TMEM allocated in both
  tc_fence_after();
  const uint32_t tmem_base = s->tmem_base;
  const int num_kb = p.k / kBK;
  if (!leader && threadIdx.x == 0)
    for (int i = 0; i < S; ++i) mbar_arrive_expect_tx(&s->go[i], 16);  // first command of each slot

  if (warp == 0) {
    if (lane == 0) {
      if (leader) {
        // ===================== leader: scheduler + producer + peer commands =====================
        uint32_t stage = 0, phase = 0;
        const uint32_t peer_cmd = mapa_shared(smem_u32(&s->cmd[0]), 1);
        const uint32_t peer_go = mapa_shared(smem_u32(&s->go[0]), 1);
        const uint32_t peer_tile_id = mapa_shared(smem_u32(&s->tile_id[0]), 1);
        const uint32_t peer_tile_abort = mapa_shared(smem_u32(&s->tile_abort[0]), 1);
        const uint32_t peer_tile_full = mapa_shared(smem_u32(&s->tile_full[0]), 1);
        // Command to the peer: load (tile, kb) / skip (-1) / end (-2).  One 16-byte st.async
        // carries the data and completes the peer's go barrier (no release fence: a
        // release.cluster arrive costs a MEMBAR.GPU per stage, which capped this loop at one
        // stage per ~0.9 us).
        auto command = [&](long long tile, int kb) {
          const unsigned long long t = static_cast<unsigned long long>(tile);
          st_async_v4(peer_cmd + stage * 16, static_cast<uint32_t>(t), static_cast<uint32_t>(t >> 32),
                      static_cast<uint32_t>(kb), 0u, peer_go + stage * 8);
        };
        for (int j = 0;; ++j) {
          const int slot = j & 1;
          if (j >= 2) mbar_wait_cluster(&s->tile_empty[slot], ((j >> 1) & 1) ^ 1);
          long long tile = -1;
          if (!(p.run.preemptible && ld_volatile_smem(&s->preempt))) tile = claim_tile(p.run);
          s->tile_id[slot] = tile;
          s->tile_abort[slot] = 0;
          st_cluster_u64(peer_tile_id + slot * 8, static_cast<unsigned long long>(tile));
          st_cluster_u32(peer_tile_abort + slot * 4, 0u);
          mbar_arrive(&s->tile_full[slot]);
          mbar_arrive_cluster(peer_tile_full + slot * 8);
          if (tile < 0) {
            command(-2, 0);  // the peer's producer leaves (its stage counter is not reused)
            break;
          }
          int mb, nb;
          tile_coords(tile, p, mb, nb);
          for (int kb = 0; kb < num_kb; ++kb) {
            const bool abort = p.run.preemptible && kb > 0 && ld_volatile_smem(&s->preempt);
            mbar_wait(&s->empty[stage], phase ^ 1);
            if (abort) {
              s->stage_flag[stage] = 2;  // the MMA warp owns the redo push for this tile
              command(-1, kb);
              mbar_arrive(&s->full[stage]);
            } else {
              s->stage_flag[stage] = (kb == num_kb - 1) ? 1u : 0u;
              mbar_arrive_expect_tx(&s->full[stage], 2 * Cfg::kStageBytes);  // before any peer byte lands
              command(tile, kb);
              const uint32_t fb = smem_u32(&s->full[stage]);
              tma_load_2d_pair(smem_u32(smem_a + stage * Cfg::kHalfBytes), &tma_a, fb, kb * kBK, mb * 256);
              tma_load_2d_pair(smem_u32(smem_b + stage * Cfg::kHalfBytes), &tma_b, fb, kb * kBK, nb * 256);
            }
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
            if (abort) break;
          }
        }
      } else {
        // ===================== peer: follow the leader's stage commands =====================
        uint32_t stage = 0, phase = 0;
        for (;;) {
          mbar_wait(&s->go[stage], phase);
          uint32_t c0, c1, c2, c3;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(c0), "=r"(c1), "=r"(c2), "=r"(c3)
                       : "r"(smem_u32(&s->cmd[stage]))
                       : "memory");
          const long long tile = static_cast<long long>((static_cast<unsigned long long>(c1) << 32) | c0);
          const int kb = static_cast<int>(c2);
          (void)c3;
          if (tile == -2) break;
          mbar_arrive_expect_tx(&s->go[stage], 16);  // arm the slot's next command
          if (tile >= 0) {
            int mb, nb;
            tile_coords(tile, p, mb, nb);
            const uint32_t fb = mapa_shared(smem_u32(&s->full[stage]), 0);
            tma_load_2d_pair(smem_u32(smem_a + stage * Cfg::kHalfBytes), &tma_a, fb, kb * kBK, mb * 256 + 128);
            tma_load_2d_pair(smem_u32(smem_b + stage * Cfg::kHalfBytes), &tma_b, fb, kb * kBK, nb * 256 + 128);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      st_volatile_smem(&s->producer_done, 1u);
    }
  } else if (warp == 1) {
    // ===================== leader: UMMA issuer (cta_group::2) =====================
    if (lane == 0 && leader) {
      uint32_t stage = 0, phase = 0, drain_phase = 0;
      const int lag = p.run.preemptible ? p.mma_lag : 0;  // see tc_gemm.cuh
      int consumed = 0;
      const uint32_t peer_tile_abort = mapa_shared(smem_u32(&s->tile_abort[0]), 1);
      const uint32_t peer_tmem_full = mapa_shared(smem_u32(&s->tmem_full[0]), 1);
      for (int j = 0;; ++j) {
        const int slot = j & 1;
        mbar_wait(&s->tile_full[slot], (j >> 1) & 1);
        if (s->tile_id[slot] < 0) break;
        if (j >= 2) mbar_wait_cluster(&s->tmem_empty[slot], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(slot * 256);
        bool aborted = false;
        for (int kb = 0;; ++kb) {
          mbar_wait(&s->full[stage], phase);
          tc_fence_after();
          const uint32_t flag = s->stage_flag[stage];
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
            const uint64_t a0 = umma_desc_k_sw128(smem_u32(smem_a + stage * Cfg::kHalfBytes));
            const uint64_t b0 = umma_desc_k_sw128(smem_u32(smem_b + stage * Cfg::kHalfBytes));
#pragma unroll
            for (int k = 0; k < kBK / kUmmaK; ++k)
              umma_bf16_pair(d_tmem, a0 + 2ull * k, b0 + 2ull * k, Cfg::kIdesc, (kb | k) != 0 ? 1u : 0u);
            umma_commit_pair(&s->empty[stage]);
          }
          ++consumed;
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
          if (flag != 0) break;
        }
        if (aborted) {
          umma_commit_pair(&s->mma_drain);
          mbar_wait(&s->mma_drain, drain_phase);
          drain_phase ^= 1;
          push_redo(p.run, static_cast<unsigned long long>(s->tile_id[slot]));
          s->tile_abort[slot] = 1;
          st_cluster_u32(peer_tile_abort + slot * 4, 1u);
          mbar_arrive(&s->tmem_full[slot]);
          mbar_arrive_cluster(peer_tmem_full + slot * 8);
        } else {
          umma_commit_pair_mc(&s->tmem_full[slot], 0x3);
        }
      }
    }
  } else if (warp == 2) {
    if (lane == 0 && leader && p.run.preemptible) poll_mirror(p.run, &s->preempt, &s->producer_done);
  } else if (warp == 3) {
    // (CTA 0's peer cannot exit before CTA 0 reaches the teardown cluster barrier)
    if (lane == 0 && p.run.preemptible && blockIdx.x == 0) poll_host(p.run, &s->preempt, &s->producer_done, 2);
  } else if (warp >= 4) {
    // ===================== epilogue (this CTA's 128 rows of the pair tile) =====================
    const int q = warp - 4;
    int cbuf_idx = 0;
    const uint32_t lead_tmem_empty = mapa_shared(smem_u32(&s->tmem_empty[0]), 0);
    const uint32_t lead_tile_empty = mapa_shared(smem_u32(&s->tile_empty[0]), 0);
    for (int j = 0;; ++j) {
      const int slot = j & 1;
      mbar_wait_cluster(&s->tile_full[slot], (j >> 1) & 1);
      const long long tile = *reinterpret_cast<volatile long long*>(&s->tile_id[slot]);
      if (tile < 0) break;
      mbar_wait_cluster(&s->tmem_full[slot], (j >> 1) & 1);
      tc_fence_after();
      const bool keep = !*reinterpret_cast<volatile uint32_t*>(&s->tile_abort[slot]);
      if (keep) {
        int mb, nb;
        tile_coords(tile, p, mb, nb);
        const int row0 = mb * 256 + static_cast<int>(rank) * 128 + q * 32;
#pragma unroll 1
        for (int c0 = 0; c0 < 256; c0 += 32) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(slot * 256 + c0), r);
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
            tma_store_2d(&tma_c, cbuf, nb * 256 + c0, row0);
            bulk_commit();
          }
          cbuf_idx ^= 1;
        }
        if (q == 0 && lane == 0 && leader) ++s->tiles_done;
      }
      tc_fence_before();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (q == 0 && lane == 0) {
        mbar_arrive_cluster(lead_tmem_empty + slot * 8);
        mbar_arrive_cluster(lead_tile_empty + slot * 8);
      }
    }
    if (lane == 0) bulk_wait_read<0>();
  }

  tc_fence_before();
  cluster_sync_all();  // no CTA frees TMEM or leaves while its peer may still signal it
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair(tmem_base, Cfg::kTmemCols);
  if (threadIdx.x == 0) cta_exit(p.run, s->tiles_done);
}

}  // namespace msdev
