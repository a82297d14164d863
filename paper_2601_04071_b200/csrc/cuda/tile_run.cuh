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
  const uint64_t* host_line;  // MsLpLine of this slot: {epoch, budget}
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
  int pdl_wait;  // HP chain kernel whose inputs come from the previous chain kernel
  unsigned long long* dbg;  // optional per-CTA phase timestamps [gridDim][8] (diagnostics)
  uint32_t* reset_words;    // zeroed by the last CTA to exit (grid-phase counters of a fused chain)
  int n_reset;
  const MsTrace* trace;     // device-side event trace (null: off)
};

// One event into the trace ring (any thread; posted system-scope stores, seq last).
__device__ __forceinline__ void trace_emit(const MsTrace* tr, uint32_t kind, uint32_t id, uint64_t a, uint64_t b,
                                           uint64_t t) {
  if (!tr) return;
  const unsigned long long idx = atomicAdd(tr->head, 1ull);
  MsTraceEvent* e = tr->ev + (idx & tr->cap_mask);
  st_relaxed_sys_u64(&e->t_ns, t);
  st_relaxed_sys_u64(reinterpret_cast<uint64_t*>(&e->kind), (static_cast<uint64_t>(id) << 32) | kind);
  st_relaxed_sys_u64(&e->a, a);  // (40-byte events: 8-byte aligned fields only)
  st_relaxed_sys_u64(&e->b, b);
  st_release_sys_u64(&e->seq, idx + 1);
}

__device__ __forceinline__ void dbg_stamp(const TileRun& r, int phase) {
  if (r.dbg) r.dbg[blockIdx.x * 8 + phase] = globaltimer();
}

// Extended per-CTA stamps (64 slots per CTA after the [gridDim][8] block).
__device__ __forceinline__ void dbg_stamp_ext(const TileRun& r, int slot) {
  if (r.dbg && slot < 64) r.dbg[2048 + blockIdx.x * 64 + slot] = globaltimer();
}

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

// Mirror poller: one thread per CTA, L2 reads of the device mirror only (never PCIe).
__device__ __forceinline__ void poll_mirror(const TileRun& r, uint32_t* preempt, const uint32_t* producer_done) {
  const uint32_t* mine = &r.mirror->epoch[(blockIdx.x % MS_MIRROR_COPIES) * MS_MIRROR_STRIDE];
  for (;;) {
    if (ld_volatile_smem(producer_done)) break;
    if (ld_relaxed_gpu(mine) > r.run_epoch) {
      st_volatile_smem(preempt, 1u);
      dbg_stamp(r, 0);
      atomicMin(&r.ctl->t_seen, static_cast<unsigned long long>(globaltimer()));
      r.ctl->preempted = 1u;
      break;
    }
    __nanosleep(64);
  }
}

// Host poller: one thread of CTA 0 (an otherwise idle warp).  Fetches {epoch, budget}
// from the host-mapped line with one 16-byte ld.acquire.sys per iteration, forwards them
// to the device mirror, and publishes the claim counter to the host.  Stays alive until
// every other CTA has exited so scheduler-initiated preemptions keep propagating.
// `group`: CTAs (this one included) that cannot exit before this CTA does — 1, or 2 for a
// CTA pair whose teardown cluster barrier waits for this CTA.
__device__ __forceinline__ void poll_host(const TileRun& r, const uint32_t* preempt, const uint32_t* producer_done,
                                          unsigned int group = 1) {
  uint32_t mirrored = 0;
  for (;;) {
    if (ld_volatile_smem(preempt)) break;  // CTA 0 is leaving anyway
    // every other CTA has left (LP grids count exits in the low half of `top`, cta_exit)
    if (ld_volatile_smem(producer_done) &&
        static_cast<unsigned int>(*reinterpret_cast<volatile unsigned long long*>(&r.ctl->top)) + group >= gridDim.x)
      break;
    if (r.host_progress)
      st_relaxed_sys_u64(reinterpret_cast<uint64_t*>(r.host_progress),
                         ld_relaxed_gpu_u64(reinterpret_cast<const uint64_t*>(&r.ctl->claim)));
    uint64_t ep, bud;
    ld_acquire_sys_v2(r.host_line, ep, bud);
    st_relaxed_gpu_u64(&r.mirror->budget[r.slot][0], bud);
    const uint32_t e = static_cast<uint32_t>(ep);
    if (e > mirrored) {
#pragma unroll
      for (int c = 0; c < MS_MIRROR_COPIES; ++c) atomicMax(&r.mirror->epoch[c * MS_MIRROR_STRIDE], e);
      mirrored = e;
    }
  }
}

// Auxiliary host pollers (CTAs 1 .. kAuxPollers of an LP grid, one otherwise idle lane
// each): the same 16-byte ld.acquire.sys of {epoch, budget} as CTA 0's poller, started
// `stagger` ns apart, forwarding only the epoch to the device mirror.  With P pollers a host
// store is seen ~RTT/(2P) + RTT/2 after it lands instead of ~RTT (one PCIe round trip is
// ~1.2 us here).  Each leaves with its own CTA (no cross-CTA wait).
constexpr int kAuxPollers = 3;

__device__ __forceinline__ void poll_host_aux(const TileRun& r, const uint32_t* preempt, const uint32_t* producer_done,
                                              unsigned stagger_ns) {
  __nanosleep(stagger_ns);
  for (;;) {
    if (ld_volatile_smem(preempt) || ld_volatile_smem(producer_done)) break;
    uint64_t ep, bud;
    ld_acquire_sys_v2(r.host_line, ep, bud);
    const uint32_t e = static_cast<uint32_t>(ep);
    if (e > r.run_epoch) {
#pragma unroll
      for (int c = 0; c < MS_MIRROR_COPIES; ++c) atomicMax(&r.mirror->epoch[c * MS_MIRROR_STRIDE], e);
      break;
    }
  }
}

// Called by thread 0 of each CTA after all of the CTA's work (and TMEM traffic) is done.
// One acq_rel atomic per CTA on MsLpCtl::top ((tiles << 32) | 1) publishes this CTA's
// tile / redo accounting (ordered by the CTA barrier before cta_exit) and lets the last
// CTA acquire everyone else's.  (A two-level tree measured slower: the last CTA then pays
// two L2 round trips while the preempted CTAs' in-flight loads drain.)
// `ctas`: CTAs this call accounts for (2: the leader of a CTA pair exits for both, after the
// pair's teardown cluster barrier — half the atomics on `top` while a preempted grid drains).
//
// LP grids (persistent, at most one wave, no HP bookkeeping) publish differently: every CTA
// but CTA 0 adds its count with a fire-and-forget release reduction and leaves at once — no
// L2 round trip on its way out, so a preempted grid frees its SMs sooner — and CTA 0, which
// stays until the others are gone anyway (its host poller), waits for the count and
// publishes.  (HP kernels keep the last-arrival scheme: a spinning CTA 0 could hold a slot a
// not-yet-resident CTA of a larger or PDL-overlapped grid needs.)
__device__ __forceinline__ void cta_exit(const TileRun& r, unsigned int tiles_done_cta, unsigned int ctas = 1) {
  MsLpCtl* ctl = r.ctl;
  dbg_stamp(r, 5);
  const unsigned long long mine = (static_cast<unsigned long long>(tiles_done_cta) << 32) | ctas;
  unsigned long long w, t_free = 0;
  if (r.hp_ctl == nullptr) {
    if (blockIdx.x != 0) {
      // this CTA's SMs are free from here: the max over CTAs is the grid's SM-release time
      // (CTA 0 then spends an L2 round trip or two aggregating the exit record on one SM)
      red_relaxed_gpu_max_u64(&ctl->t_free, globaltimer());
      red_release_gpu_add_u64(&ctl->top, mine);  // after this CTA's redo pushes (release)
      return;
    }
    const unsigned long long t_own = globaltimer();
    const unsigned int others = gridDim.x - ctas;
    // relaxed polling (no L1 invalidation per iteration), one acquire fence once complete
    while (static_cast<unsigned int>((w = ld_relaxed_gpu_u64(reinterpret_cast<const uint64_t*>(&ctl->top)))) < others)
      __nanosleep(32);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    dbg_stamp_ext(r, 1);
    const unsigned long long tf = ld_relaxed_gpu_u64(reinterpret_cast<const uint64_t*>(&ctl->t_free));
    t_free = tf > t_own ? tf : t_own;
  } else {
    atomicAdd(&ctl->exited, ctas);  // relaxed: only CTA 0's host poller reads it
    w = atom_add_acqrel_gpu_u64(&ctl->top, mine);
    dbg_stamp_ext(r, 1);
    if (static_cast<unsigned int>(w) + ctas != gridDim.x) return;
  }
  const unsigned long long tiles_total = (w >> 32) + tiles_done_cta;
  // Issue every control-block read at once (each is an L2 round trip, slow while the
  // preempted CTAs' in-flight loads still drain).
  const unsigned long long claimed = ld_relaxed_gpu_u64(reinterpret_cast<const uint64_t*>(&ctl->claim));
  unsigned int redo_n = ld_relaxed_gpu(&ctl->redo_out_n);
  const unsigned long long t_start = ld_relaxed_gpu_u64(reinterpret_cast<const uint64_t*>(&ctl->t_start));
  const unsigned long long t_seen = ld_relaxed_gpu_u64(reinterpret_cast<const uint64_t*>(&ctl->t_seen));
  const unsigned int preempted = ld_relaxed_gpu(&ctl->preempted);
  // Redo entries nobody claimed carry over to the next run.
  for (unsigned long long idx = claimed; idx < r.nr_in; ++idx) r.redo_out[redo_n++] = r.redo_in[idx];
  unsigned long long cursor = r.begin;
  if (claimed > r.nr_in) cursor = min(r.end, r.begin + (claimed - r.nr_in));
  const unsigned long long t_exit = globaltimer();
  dbg_stamp(r, 6);
  if (r.exit_rec) {
    MsLpExit* e = r.exit_rec;
    st_relaxed_sys_u64(&e->cursor, cursor);
    st_relaxed_sys_u64(&e->redo_count, redo_n);
    st_relaxed_sys_u64(&e->tiles_done, tiles_total);
    st_relaxed_sys_u64(&e->t_start, t_start);
    st_relaxed_sys_u64(&e->t_seen, t_seen == ~0ull ? 0ull : t_seen);
    st_relaxed_sys_u64(&e->t_exit, t_exit);
    st_relaxed_sys_u64(&e->preempted, preempted);
    st_relaxed_sys_u64(&e->t_free, t_free ? t_free : t_exit);
    st_release_sys_u64(&e->run_id, r.run_id);  // host acquires run_id, then reads the rest
  }
  if (r.trace && r.exit_rec) {
    trace_emit(r.trace, 1u, static_cast<uint32_t>(r.slot), r.run_id, 0, t_start);
    if (preempted && t_seen != ~0ull) trace_emit(r.trace, 2u, static_cast<uint32_t>(r.slot), r.run_id, 0, t_seen);
    trace_emit(r.trace, 3u, static_cast<uint32_t>(r.slot), r.run_id, (tiles_total << 32) | redo_n, t_exit);
  }
  if (r.hp_ctl && r.hp_last && r.hp_rec) {
    const unsigned long long first = r.hp_ctl->t_first_cta;
    trace_emit(r.trace, 4u, static_cast<uint32_t>(r.slot), r.hp_seq, 0, first);
    trace_emit(r.trace, 5u, static_cast<uint32_t>(r.slot), r.hp_seq, 0, t_exit);
    st_relaxed_sys_v2(&r.hp_rec->done_first, first,
                      (static_cast<uint64_t>(r.hp_seq) << 32) | ((t_exit - first) & 0xFFFFFFFFull));
    r.hp_ctl->t_first_cta = ~0ull;
  }
  for (int i = 0; i < r.n_reset; ++i) r.reset_words[i] = 0;
  ctl->top = 0;
  ctl->claim = 0;
  ctl->t_start = ~0ull;
  ctl->t_seen = ~0ull;
  ctl->redo_out_n = 0;
  ctl->preempted = 0;
  ctl->t_free = 0;
  __threadfence();
  ctl->exited = 0;
}

}  // namespace msdev
