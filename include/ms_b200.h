/* ms_b200.h — C-ABI of the B200 device layer (sm_100a preemptible tenant kernels,
 * preempt flag, HP doorbell, device-side timing).
 *
 * The reference has no device layer: its "device" is the simulated wave model
 * (engine.hpp:682-945) and its host<->device crossings are modelled events.  Each entry
 * point below is the live counterpart of one of those modelled crossings (SURVEY.md
 * §8b), and is what the C++ scheduler core's B200 backend (csrc/live) binds:
 *   issue_instance (LP slice)        engine.hpp:702-720   -> ms_lp_run
 *   p_flag_ = true on HP activation  engine.hpp:949-968   -> ms_preempt_raise
 *   scheduler SyncBegin/SyncEnd      engine.hpp:621-627   -> ms_lp_wait / ms_lp_poll
 *   tick launcher / consolidation    engine.hpp:1047-1115 -> ms_lp_set_budget / ms_lp_run ranges
 *   issue_instance (HP kernel) +     engine.hpp:548-560,  -> ms_hp_arm (ahead of time) + ms_hp_ring
 *   its modelled launch_overhead       705, 718              (no launch on the critical path)
 *   KernelDone of an HP segment      engine.hpp:871-889   -> ms_hp_poll / ms_hp_wait
 *
 * Conventions: return 0 on success, negative on error (MS_E_CUDA = CUDA failure, text via
 * ms_last_error); no exceptions cross the ABI; device pointers are uint64_t; device
 * timestamps are %globaltimer ns; host timestamps are CLOCK_MONOTONIC ns.
 * Threading: one owner thread per ms_dev drives launches; ms_preempt_raise and
 * ms_hp_ring are plain release stores to the host-mapped page and may be called from any
 * thread.
 */
#ifndef MS_B200_H_
#define MS_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#ifndef MS_OK
#define MS_OK 0
#define MS_E_ARG (-1)
#endif
#define MS_E_CUDA (-5)
#define MS_E_TIMEOUT (-6)
#define MS_E_NODEV (-7)

typedef struct ms_dev ms_dev;

typedef struct ms_dev_info {
  int32_t ordinal, sm_count, cc_major, cc_minor;
  int32_t stream_memops; /* 1 if cuStreamWaitValue32 is usable on this driver */
  int32_t prio_low, prio_high;
  int64_t hbm_bytes;
  char name[64];
} ms_dev_info;

int ms_dev_open(int ordinal, ms_dev** dev);
int ms_dev_close(ms_dev* dev);
int ms_dev_get_info(ms_dev* dev, ms_dev_info* info);
int ms_dev_sync(ms_dev* dev);
const char* ms_last_error(void);
int64_t ms_host_now_ns(void);

/* pinned host memory (e2e request buffers) */
int ms_host_alloc(ms_dev* dev, size_t bytes, uint64_t* hptr);
int ms_host_free(ms_dev* dev, uint64_t hptr);

/* device memory helpers (tests / bench data setup) */
int ms_mem_alloc(ms_dev* dev, size_t bytes, uint64_t* dptr);
int ms_mem_free(ms_dev* dev, uint64_t dptr);
int ms_memcpy_h2d(ms_dev* dev, uint64_t dst, const void* src, size_t bytes);
int ms_memcpy_d2h(ms_dev* dev, void* dst, uint64_t src, size_t bytes);
int ms_memset(ms_dev* dev, uint64_t dst, int value, size_t bytes);
/* deterministic synthetic bf16 tensor (generator of oracle/tenant_ref.c) */
int ms_fill_synth_bf16(ms_dev* dev, uint64_t dst, uint64_t n, uint64_t seed, uint64_t tensor, float scale);
/* fp32 tensor holding the same synthetic values (widened from bf16): optimizer state */
int ms_fill_synth_f32(ms_dev* dev, uint64_t dst, uint64_t n, uint64_t seed, uint64_t tensor, float scale);

/* ---- LP (preemptible) kernels ------------------------------------------------------ */
#define MS_LP_GEMM 1 /* C[m,n] = A[m,k] * B[n,k]^T, bf16 in/out, fp32 accumulate (tcgen05) */
#define MS_LP_AXPY 2 /* y = alpha * x + y over n_elems bf16 (HBM streamer) */
#define MS_LP_OPTIM 3 /* optimizer step over n_elems parameters (HBM streamer): a = fp32 params, b = fp32
                         first moment, c = fp32 second moment (AdamW only), x = bf16 gradients;
                         opt_mode 0 = AdamW, 1 = SGD momentum (opt[1] = momentum); tile_elems multiple
                         of 1024 (default 4096) */

typedef struct ms_lp_desc {
  int32_t kind;
  int32_t block_n;    /* GEMM tile N: 64, 128 or 256 (tile M is 128, k-block 64) */
  int32_t group_m;    /* GEMM raster group (L2 reuse), 0 = default 16 */
  int32_t tile_elems; /* AXPY tile (elements, multiple of 2048), 0 = default 8192 */
  int32_t ctas_per_sm;/* AXPY layout: 1 (default, 0) = ONE CTA per SM with 3 x 256 streaming
                         threads, so a capped grid leaves whole SMs free for HP; 2..4 = that
                         many 256-thread CTAs per SM (the block scheduler spreads them) */
  int32_t split_k;    /* GEMM: k-slices per output tile (0/1: none).  Work unit = (tile, slice):
                         fp32 partials, the tile's last unit reduces them in slice order
                         (deterministic).  Bounds a unit's duration (the preemption grain) and
                         fills the GPU when a GEMM has few tiles and a long K (wgrad) */
  uint64_t a, b, c;
  int64_t m, n, k;
  uint64_t x, y;
  float alpha;
  float pad2;
  int64_t n_elems;
  int32_t opt_mode;   /* MS_LP_OPTIM: 0 = AdamW, 1 = SGD momentum */
  float opt[7];       /* MS_LP_OPTIM: lr, beta1 (momentum), beta2, eps, weight decay, bias corrections c1, c2 */
} ms_lp_desc;

typedef struct ms_lp_status {
  uint64_t run_id;
  uint64_t begin, end;        /* range of the last launch (fresh tiles) */
  uint64_t redo_in;           /* redo tiles the last launch started with */
  uint64_t cursor;            /* next never-claimed fresh tile */
  uint64_t redo_count;        /* claimed-but-unfinished tiles carried to the next run */
  uint64_t tiles_done;        /* tiles completed by the last run */
  int32_t preempted;          /* the run ended because the epoch advanced */
  int32_t done;               /* the run has exited */
  int64_t t_launch_host;      /* host ns at ms_lp_run */
  uint64_t t_start, t_seen, t_exit; /* device ns: first CTA start, first epoch observation, last exit */
  uint64_t t_free;            /* device ns: LP grids' SMs released (every CTA but the one that
                                 aggregates the exit record gone, and that one's work done) */
} ms_lp_status;

/* Register a preemptible LP kernel; *total_tiles = size of its linear tile space. */
int ms_lp_register(ms_dev* dev, const ms_lp_desc* desc, int* id, uint64_t* total_tiles);
/* Release a slot (waits for the LP stream). */
int ms_lp_unregister(ms_dev* dev, int id);
/* Launch (async, low-priority stream) over fresh tiles [begin, end) plus the redo tiles
 * carried from the previous run; tiles >= budget are not started (budget <= end). */
int ms_lp_run(ms_dev* dev, int id, uint64_t begin, uint64_t end, uint64_t budget);
/* Same with flags: MS_RUN_NONPREEMPTIBLE runs the range to completion without polling the
 * epoch (kernel-boundary temporal-sharing baseline). */
#define MS_RUN_NONPREEMPTIBLE 1
int ms_lp_run_ex(ms_dev* dev, int id, uint64_t begin, uint64_t end, uint64_t budget, int flags);
/* Claim counter of the running launch as last published by its poller (redo entries
 * first, then fresh tiles), for harvest-budget pacing. */
uint64_t ms_lp_progress(ms_dev* dev, int id);
uint64_t ms_lp_total_tiles(ms_dev* dev, int id);
/* SMs (CTAs) one tile of the kernel occupies: 2 for GEMMs on CTA pairs (256 x 512 tiles),
 * else 1.  A wave of an LP run over n SMs covers n / ms_lp_tile_ctas tiles. */
int ms_lp_tile_ctas(ms_dev* dev, int id);
/* Number of SMs a preemptible LP GEMM grid leaves free (default 0). */
int ms_set_lp_sm_reserve(ms_dev* dev, int n);
/* Diagnostics: enable=1 arms per-CTA phase timestamps for subsequent LP runs; enable=0
 * copies [cta][8] globaltimer stamps (seen, producer done, mma done, epilogue done,
 * teardown, exit begin, last-exit) into `out` and disarms. */
int ms_debug_stamps(ms_dev* dev, int enable, unsigned long long* out, size_t n);
/* Move the running launch's soft end (harvest budget word). */
int ms_lp_set_budget(ms_dev* dev, int id, uint64_t budget);
/* Memory tier (ms_tier.h): tiles [g * tiles_per_group, (g + 1) * tiles_per_group) of the
 * LP kernel `id` touch off-device chunks when slow_groups[g] != 0; at most max_inflight
 * such tiles run at once device-wide, which bounds the preemption drain over PCIe /
 * NVLink to max_inflight tiles.  slow_groups == NULL disables.  Streamers (MS_LP_AXPY) and
 * GEMMs, single-CTA or on CTA pairs (tiles = the kernel's linear work units, k-split units
 * included; the host maps each unit's A / B panels onto the tier's chunks, tier.py
 * gemm_slow_units). */
int ms_lp_set_slow_tiles(ms_dev* dev, int id, const uint8_t* slow_groups, uint64_t n_groups, int tiles_per_group,
                         int max_inflight);
/* Non-blocking: fills *st; returns 1 if the last launch has exited, 0 if running. */
int ms_lp_poll(ms_dev* dev, int id, ms_lp_status* st);
int ms_lp_wait(ms_dev* dev, int id, int64_t timeout_ns, ms_lp_status* st);
/* Drop the redo carry-over (start a fresh pass). */
int ms_lp_reset(ms_dev* dev, int id);

/* ---- preemption flag ---------------------------------------------------------------- */
/* epoch += 1 (release store to the host-mapped word); every LP run launched with an older
 * epoch drains its current tile / k-blocks and exits. */
int ms_preempt_raise(ms_dev* dev, uint32_t* epoch, int64_t* t_host_ns);
uint32_t ms_preempt_epoch(ms_dev* dev);

/* ---- HP chains --------------------------------------------------------------------- */
#define MS_HP_GEMM 1      /* C = A * B^T (non-preemptible tcgen05 GEMM); m == 1: batch-1 matrix-vector
                             product — a chain whose GEMM ops all have m == 1 runs as one HBM-streaming
                             GEMV launch (weights row-major [n,k] read in place, k <= 8192) */
#define MS_HP_BIAS_GELU 2 /* c = gelu(a + bias) over m x n */
#define MS_HP_SILU_MUL 5  /* c[m, n] = silu(a[m, j]) * a[m, n + j]: a is [m x 2n] = [gate | up] */
#define MS_HP_GEMM_SWIGLU 6 /* c[m, n] = silu(a b_gate^T) * (a b_up^T); b = [2n x k] = [gate rows; up
                               rows] (row-major); the SwiGLU is applied to the fp32 accumulators
                               (m == 1: GEMV chain, k <= 4096) */
#define MS_HP_H2D 3       /* copy m bytes: pinned host a -> device c (e2e request input) */
#define MS_HP_D2H 4       /* copy m bytes: device a -> pinned host c (e2e request output) */
/* Config-2 / config-3 tenants (ResNet-50 bs=1, BERT-base bs=1): per-op chain kernels,
 * hp_ops.cuh.  Geometry in ms_hp_op.geo (NHWC, batch 1). */
#define MS_HP_IM2COL 7    /* c[m x n] = conv patches of the NHWC input a [h*w x cin]: row = output pixel
                             (oy * wo + ox, rows >= ho*wo zero), column = (ky, kx, ch) (cols >= kh*kw*cin
                             zero); m, n padded to the GEMM tile (128, 64) */
#define MS_HP_BIAS_ACT 8  /* c = act(a + bias[col] (+ b when b != 0)) over m x n; geo.flags bit 0 = ReLU */
#define MS_HP_MAXPOOL 9   /* c[m x cin] = geo.kh x geo.kw / stride / pad max pooling of NHWC a [h*w x cin] */
#define MS_HP_AVGPOOL 10  /* c[0, :] = mean of the h*w rows of a [h*w x n]; rows 1 .. m-1 of c = 0 */
#define MS_HP_ATTN 11     /* c[m x n] = per head softmax(Q K^T / 8) V, a = [m x 3n] = [Q | K | V], head dim 64,
                             m <= 256 and a multiple of 16 (no mask) */
#define MS_HP_ADD_LN 12   /* c = LayerNorm(a + b) * gamma + beta over rows of n (eps 1e-12), bias = [gamma | beta] */

typedef struct ms_hp_geo {
  int32_t h, w, cin;      /* input spatial size and channels */
  int32_t kh, kw;         /* window */
  int32_t stride, pad;
  int32_t flags;          /* MS_HP_BIAS_ACT: bit 0 = ReLU */
} ms_hp_geo;

typedef struct ms_hp_op {
  int32_t kind;
  int32_t block_n;   /* GEMM tile N (0: 128) */
  uint64_t a, b, c, bias;
  int64_t m, n, k;
  int32_t split_k;   /* GEMM k-slices per tile (0: auto — enough units to cover the SMs) */
  int32_t b_layout;  /* GEMM weights: 0 = row-major [N,K], captured k-block-major at registration
                        (DRAM-page friendly); 1 = read row-major in place; 2 = b already k-block-major
                        [K/64][N][64] */
  int64_t lda;       /* GEMM: row stride of a in elements (0: k) — e.g. a column slice of a wider
                        activation */
  ms_hp_geo geo;     /* IM2COL / MAXPOOL / AVGPOOL geometry, BIAS_ACT flags (zero otherwise) */
  uint64_t resid;    /* MS_HP_GEMM epilogue (per-op chains, m >= 128): C = act(A B^T + bias[col] + resid),
                        bias != 0 adds a per-column bf16 bias, resid != 0 an [m x n] bf16 residual,
                        geo.flags bit 0 = ReLU, bit 1 = tanh-GELU; applied to the fp32 accumulators
                        (one rounding) — the folded-BN / residual / activation of a conv, FFN1 + GELU */
} ms_hp_op;

typedef struct ms_hp_times {
  uint32_t seq;
  uint32_t done;
  uint64_t t_gate;      /* device ns the gate saw the doorbell (0 for direct launches) */
  uint64_t t_first_cta; /* first CTA of the first chain kernel */
  uint64_t t_done;      /* last CTA of the last chain kernel */
} ms_hp_times;

int ms_hp_register_chain(ms_dev* dev, const ms_hp_op* ops, int n_ops, int* chain_id);
/* Next value of the device's monotonic doorbell sequence (never reused on this ms_dev). */
uint32_t ms_hp_next_seq(ms_dev* dev);
/* Release a chain's device buffers (its slot becomes reusable).  The chain must be idle. */
int ms_hp_unregister_chain(ms_dev* dev, int chain_id);
/* Pre-enqueue gate(seq) + the chain's kernels on the highest-priority stream. */
int ms_hp_arm(ms_dev* dev, int chain_id, uint32_t seq);
/* Chain execution mode, applied by later ms_hp_register_chain / arm / launch calls:
   1 (default): a chain whose kernel ops are contiguous and tile-aligned runs as ONE
   persistent launch (weights of op i+1 stream during op i; grid phase counters between
   ops; k-slices of a tile reduced through cluster DSMEM when the split is 2 or 4).
   2: fused, k-slices reduced through global memory (no clusters).  0: one kernel per op
   (PDL-linked).  The cluster/no-cluster choice is fixed when the chain is registered. */
int ms_hp_set_fused(ms_dev* dev, int mode);
/* Fused plan of a registered chain: grid size and cluster size (0, 0: not fusable). */
int ms_hp_chain_info(ms_dev* dev, int chain_id, int* fused_grid, int* cluster);
/* Ring the doorbell: release store doorbell = seq (host ns of the store in *t_host_ns). */
int ms_hp_ring(ms_dev* dev, uint32_t seq, int64_t* t_host_ns);
/* Baseline path: launch the chain now with no gate (host launch on the critical path). */
int ms_hp_launch_direct(ms_dev* dev, int chain_id, uint32_t seq);
int ms_hp_poll(ms_dev* dev, int chain_id, uint32_t seq, ms_hp_times* t);
int ms_hp_wait(ms_dev* dev, int chain_id, uint32_t seq, int64_t timeout_ns, ms_hp_times* t);

/* ---- clocks ------------------------------------------------------------------------- */
/* Ping-pong through the host page; device_ns ~= host_ns + *offset_ns (min-RTT sample). */
int ms_clock_calibrate(ms_dev* dev, int rounds, int64_t* offset_ns, int64_t* rtt_min_ns);

/* ---- device-side event trace -------------------------------------------------------- */
/* A ring of %globaltimer events written by the kernels themselves (posted stores into
 * pinned host memory, no copy): the exit record of every LP run (start, first CTA that saw
 * a preemption, exit), every HP chain (first CTA, done) and every doorbell gate release.
 * A long live run can be logged incrementally by draining it (SURVEY.md §8b
 * ms_trace_drain); the live scheduler's own Timeline is unaffected. */
typedef struct ms_event {
  uint64_t seq;   /* 1-based position in the trace */
  uint64_t t_ns;  /* %globaltimer */
  uint32_t kind;  /* MS_EV_* */
  uint32_t id;    /* LP slot, HP chain control block, or doorbell seq (gate) */
  uint64_t a, b;  /* per kind, see below */
} ms_event;
#define MS_EV_LP_START 1 /* a = run id */
#define MS_EV_LP_SEEN 2  /* a = run id (first CTA that observed the preempt epoch) */
#define MS_EV_LP_EXIT 3  /* a = run id, b = (tiles done << 32) | redo entries left; t = last exit */
#define MS_EV_HP_FIRST 4 /* a = doorbell seq of the chain run */
#define MS_EV_HP_DONE 5  /* a = doorbell seq */
#define MS_EV_GATE 6     /* a = doorbell word (epoch << 32 | seq) as the gate saw it */
/* capacity (events, a power of two) > 0 allocates and enables the ring; 0 disables it. */
int ms_trace_enable(ms_dev* dev, size_t capacity);
/* Copy up to `max` events in order, oldest first; returns the count (>= 0).  `lost` (may be
 * null) receives the number of events overwritten before they were drained. */
int ms_trace_drain(ms_dev* dev, ms_event* out, size_t max, uint64_t* lost);

/* ---- kernel timing (CUDA events on the launching stream) ---------------------------- */
/* Time `reps` back-to-back full runs of LP kernel `id` over [0, total); returns mean ms. */
int ms_lp_time_full(ms_dev* dev, int id, int reps, float* ms_per_run);
/* Same over the tile range [begin, end) (the on-B200 profiler behind KernelSpec.measured_time,
 * which the reference consumes at engine.hpp:461-481 / splitter.hpp:141-207). */
int ms_lp_time_range(ms_dev* dev, int id, uint64_t begin, uint64_t end, int reps, float* ms_per_run);
/* Time `reps` direct launches of an HP chain; returns mean ms per chain. */
int ms_hp_time_chain(ms_dev* dev, int chain_id, int reps, float* ms_per_chain);

#ifdef __cplusplus
}
#endif
#endif /* MS_B200_H_ */
