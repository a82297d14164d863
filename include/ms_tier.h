/* ms_tier.h — C-ABI of the live memory tier.
 *
 * LP tenants whose footprint overflows HBM keep running: their buffers are ONE virtual
 * range (CUDA VMM) whose 2 MB chunks are backed by local HBM, an NVLink peer's HBM, or
 * pinned host DRAM, so the unmodified LP kernels (ms_lp_register) read them in place.
 * Placement decisions are the replay engine's MemoryManager (microslice/memory.hpp —
 * reference memory.hpp:138-323) fed with LIVE link measurements:
 *   priority isolation : HP chunks are pinned local; when the tier's HBM budget is full an
 *                        HP allocation displaces the oldest unpinned LP chunk (its data is
 *                        copied to the eviction target and the VA is remapped in place)
 *   interference-aware : contention-first eviction ping-probes every peer link (a timed
 *                        probe_mb copy on a low-priority stream) and spills to the least
 *                        congested peer whose score t_now / t_base is under the threshold,
 *                        else to DRAM; round_robin ignores congestion (HUVM's policy)
 * Reference call sites: Engine setup allocation (engine.hpp:396-411), ProbeTick
 * (engine.hpp:1263-1276).
 *
 * options_json: {"hbm_gb": tier budget in local HBM (default: free HBM at open - 8 GB),
 *                "peers": [{"device": ordinal, "free_gb": g}, ...]  (P2P-capable GPUs),
 *                "eviction": "contention_first" | "round_robin", "score_threshold": 1.5,
 *                "probe_mb": 4, "probe_cache_us": 1000, "numa": host NUMA node (default:
 *                the GPU's)}
 * Relocation (an HP allocation displacing LP chunks) remaps LP memory: it waits for the
 * LP stream (preempt first — ms_preempt_raise — to keep that short); ms_tier_free waits
 * for the LP stream too.  A buffer an ARMED HP chain uses must not be freed.
 * Threading: one owner thread per tier.  Errors as in ms_b200.h (ms_last_error).
 */
#ifndef MS_TIER_H_
#define MS_TIER_H_

#include "ms_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ms_tier ms_tier;

#define MS_TIER_LOCAL 0
#define MS_TIER_PEER 1
#define MS_TIER_DRAM 2

typedef struct ms_tier_chunk {
  int32_t tier;   /* MS_TIER_* */
  int32_t peer;   /* link index when tier == MS_TIER_PEER, else -1 */
  int32_t owner;  /* task id */
  int32_t pinned; /* 1 for HP chunks */
} ms_tier_chunk;

typedef struct ms_tier_stats {
  int64_t local_capacity_chunks, local_used_chunks;
  int64_t chunks_local, chunks_peer, chunks_dram;
  int64_t relocations;      /* LP chunks moved out of HBM by HP allocations */
  int64_t relocated_bytes;  /* bytes copied by those moves */
  int64_t relocate_copy_ns;  /* host time in relocation: granules + staging + copies */
  int64_t relocate_remap_ns; /* host time in relocation: VA unmap / map / access */
  int64_t probes;           /* live link probes issued */
  int32_t n_links;
  int32_t pad;
} ms_tier_stats;

int ms_tier_open(ms_dev* dev, const char* options_json, ms_tier** tier);
/* Allocate `bytes` (rounded up to 2 MB chunks) for `task`; *dptr is a device pointer
 * usable by any kernel on the device.  high_priority != 0 pins the chunks in HBM. */
int ms_tier_alloc(ms_tier* t, int task, int high_priority, uint64_t bytes, uint64_t* dptr,
                  uint64_t* n_chunks);
/* Placement of the chunks of the allocation starting at dptr (n = its chunk count). */
int ms_tier_chunks(ms_tier* t, uint64_t dptr, ms_tier_chunk* out, uint64_t n);
/* Live ping-probe of peer link `link`: score = t_now / t_base, t_now in ns. */
int ms_tier_probe(ms_tier* t, int link, double* score, int64_t* t_ns);
int ms_tier_get_stats(ms_tier* t, ms_tier_stats* st);
int ms_tier_free(ms_tier* t, uint64_t dptr);
int ms_tier_close(ms_tier* t);

#ifdef __cplusplus
}
#endif
#endif /* MS_TIER_H_ */
