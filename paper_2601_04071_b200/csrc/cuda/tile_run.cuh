// Preemptible persistent tile-loop machinery shared by every LP kernel (GEMM and HBM
// streamer) and reused, non-preemptibly, by the HP chain kernels.
//
//  * claim_tile   : one atomic on the run's claim counter hands out redo entries first,
//                   then fresh linear tile ids of [begin, end); a fresh tile past the
//                   host's soft budget is parked on the redo list (cursor stays exact).
//  * run_poller   : the preempt-epoch poller.  CTA 0 reads the host-
//                   mapped epoch + budget with ld.acquire.sys and mirrors them into device
//                   memory (8 copies on separate L2 lines); all other CTAs read a mirror.
//                   Measured on B200 (profiles/r01_latency_probe.txt): 148 CTAs polling
//                   host memory directly take ~130 us to all observe a store; one elected
//                   poller + device mirror: p99 1.5 us.
//  * cta_exit     : exit accounting; the last CTA publishes {cursor, redo count, tiles
//                   done, t_start, t_seen, t_exit} to the host page with a release and
//                   self-resets the control block for the next (stream-ordered) run.
#pragma once

#include "ms_ctl.h"
#include "ms_ptx.cuh"

namespace msdev {

struct TileRun {
  unsigned long long begin, end, budget0;
  unsigned int nr_in;
  const unsigned long long* redo_in;
  unsigned long long* redo_out;
  MsLpCtl* ctl;
  int preemptible;
  unsigned int run_epoch;
  const uint32_t* host_epoch;
  const uint64_t* host_budget;
  MsDevMirror* mirror;
  int slot;
  MsLpExit* exit_rec;
  unsigned long long* host_progress;  // CTA 0's poller publishes the claim counter here
  unsigned long long run_id;
  // HP chain notification (null for LP runs)
  MsHpCtl* hp_ctl;
  MsHpRecord* hp_rec;
  int hp_first, hp_last;
  unsigned int hp_seq;
};

__device__ __forceinline__ unsigned long long current_budget(const TileRun& r) {
  if (!r.preemptible) return r.end;
  const uint64_t w = ld_relaxed_gpu_u64(&r.mirror->budget[r.slot][0]);
  const bool ours = (w >> 40) == (r.run_id & 0xFFFFFFull);
  const unsigned long long b = ours ? (w & ((1ull << 40) - 1)) : r.budget0;
  return b < r.end ? b : r.end;
}

__device__ __forceinline__ void push_redo(const TileRun& r, unsigned long long t) {
  r.redo_out[atomicAdd(&r.ctl->redo_out_n, 1u)] = t;
}

__device__ __forceinline__ long long claim_tile(const TileRun& r) {
  const unsigned long long idx = atomicAdd(&r.ctl->claim, 1ull);
  if (idx < r.nr_in) return static_cast<long long>(r.redo_in[idx]);
  const unsigned long long t = r.begin + (idx - r.nr_in);
  if (t >= r.end) return -1;
  if (t >= current_budget(r)) {
    push_redo(r, t);
    return -1;
  }
  return static_cast<long long>(t);
}

__device__ __forceinline__ void cta_started(const TileRun& r) {
  const unsigned long long now = globaltimer();
  atomicMin(&r.ctl->t_start, now);
  if (r.hp_ctl && r.hp_first) atomicMin(&r.hp_ctl->t_first_cta, now);
}

// Runs on one thread per CTA.  `preempt` / `producer_done` are the CTA's smem words.
__device__ __forceinline__ void run_poller(const TileRun& r, uint32_t* preempt, const uint32_t* producer_done) {
  const bool leader = blockIdx.x == 0;
  const uint32_t* mine = &r.mirror->epoch[(blockIdx.x % MS_MIRROR_COPIES) * MS_MIRROR_STRIDE];
  uint32_t mirrored = 0;
  for (;;) {
    if (ld_volatile_smem(producer_done)) {
      if (!leader) break;
      if (*reinterpret_cast<volatile unsigned int*>(&r.ctl->exited) + 1 >= gridDim.x) break;
    }
    uint32_t e;
    if (leader) {
      if (r.host_progress)
        st_relaxed_sys_u64(reinterpret_cast<uint64_t*>(r.host_progress), ld_relaxed_gpu_u64(reinterpret_cast<const uint64_t*>(&r.ctl->claim)));
      e = ld_acquire_sys(r.host_epoch);
      st_relaxed_gpu_u64(&r.mirror->budget[r.slot][0], ld_acquire_sys_u64(r.host_budget));
      if (e > mirrored) {
#pragma unroll
        for (int c = 0; c < MS_MIRROR_COPIES; ++c) st_relaxed_gpu(&r.mirror->epoch[c * MS_MIRROR_STRIDE], e);
        mirrored = e;
      }
    } else {
      e = ld_relaxed_gpu(mine);
    }
    if (e > r.run_epoch) {
      st_volatile_smem(preempt, 1u);
      atomicMin(&r.ctl->t_seen, static_cast<unsigned long long>(globaltimer()));
      r.ctl->preempted = 1u;
      break;
    }
    __nanosleep(leader ? 32 : 128);
  }
}

// Called by thread 0 of each CTA after all of the CTA's work (and TMEM traffic) is done.
__device__ __forceinline__ void cta_exit(const TileRun& r, unsigned int tiles_done_cta) {
  MsLpCtl* ctl = r.ctl;
  atomicAdd(&ctl->tiles_done, static_cast<unsigned long long>(tiles_done_cta));
  __threadfence();
  const unsigned int prev = atomicAdd(&ctl->exited, 1u);
  if (prev + 1 != gridDim.x) return;
  __threadfence();
  const unsigned long long claimed = *reinterpret_cast<volatile unsigned long long*>(&ctl->claim);
  // Redo entries nobody claimed carry over to the next run.
  for (unsigned long long idx = claimed; idx < r.nr_in; ++idx) r.redo_out[ctl->redo_out_n++] = r.redo_in[idx];
  unsigned long long cursor = r.begin;
  if (claimed > r.nr_in) cursor = min(r.end, r.begin + (claimed - r.nr_in));
  const unsigned long long t_exit = globaltimer();
  if (r.exit_rec) {
    MsLpExit* e = r.exit_rec;
    st_relaxed_sys_u64(&e->cursor, cursor);
    st_relaxed_sys_u64(&e->redo_count, ctl->redo_out_n);
    st_relaxed_sys_u64(&e->tiles_done, ctl->tiles_done);
    st_relaxed_sys_u64(&e->t_start, ctl->t_start);
    st_relaxed_sys_u64(&e->t_seen, ctl->t_seen == ~0ull ? 0ull : ctl->t_seen);
    st_relaxed_sys_u64(&e->t_exit, t_exit);
    st_relaxed_sys_u64(&e->preempted, ctl->preempted);
    fence_sys();
    st_relaxed_sys_u64(&e->run_id, r.run_id);
  }
  if (r.hp_ctl && r.hp_last && r.hp_rec) {
    st_relaxed_sys_u64(&r.hp_rec->t_first_cta, r.hp_ctl->t_first_cta);
    st_relaxed_sys_u64(&r.hp_rec->t_done, t_exit);
    fence_sys();
    st_release_sys_u32(&r.hp_rec->seq_done, r.hp_seq);
    r.hp_ctl->t_first_cta = ~0ull;
  }
  ctl->claim = 0;
  ctl->tiles_done = 0;
  ctl->t_start = ~0ull;
  ctl->t_seen = ~0ull;
  ctl->redo_out_n = 0;
  ctl->preempted = 0;
  __threadfence();
  ctl->exited = 0;
}

}  // namespace msdev
