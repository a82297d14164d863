/* ms_replay.h — C-ABI of the microslice-b200 scheduler core (replay / planning side).
 *
 * The reference exposes its scheduler only as a header-only C++20 API
 * (/root/reference/proj/include/microslice, namespace microslice) and ships no FFI.
 * This header is the binding surface a non-C++ host (Python ctypes, cgo, JNI) would
 * use for the same entry points; each function cites the reference call it replaces.
 * The C++ drop-in (the headers under include/microslice) is the primary boundary; this C-ABI is a
 * thin wrapper over it (paper_2601_04071_b200/csrc/host/capi_replay.cpp).
 *
 * Conventions
 *   - plain pointers + sizes; complex inputs (GpuConfig / KernelSpec / ScenarioSpec)
 *     are passed as JSON text in the reference's scenario schema (scenario_io.hpp)
 *   - return 0 on success; MS_E_VALIDATION (-2) for ValidationError (SPEC exit code 2),
 *     MS_E_ENGINE (-3) for EngineError (exit code 3), MS_E_ARG (-1) for bad arguments,
 *     MS_E_CAPACITY (-4) when an output buffer is too small (required size reported)
 *   - `err`/`err_len` (optional) receive the exception text
 *   - strings returned through char** are malloc'd; release with ms_free
 *   - thread safety: every function is reentrant; independent replays may run concurrently
 */
#ifndef MS_REPLAY_H_
#define MS_REPLAY_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MS_OK 0
#define MS_E_ARG (-1)
#define MS_E_VALIDATION (-2)
#define MS_E_ENGINE (-3)
#define MS_E_CAPACITY (-4)

typedef struct ms_box {
  int32_t ox, oy, oz, sx, sy, sz;
} ms_box;

typedef struct ms_split_plan {
  int64_t blocks_per_slice;
  int64_t predicted_slice_time_ns;
  int64_t cap_ns;
  int32_t memory_bound;
  int32_t uncappable;
  int64_t n_slices;
} ms_split_plan;

/* ---- keyed randomness (common.hpp:50-97) ---- */
uint64_t ms_splitmix64(uint64_t x);
uint64_t ms_hash_combine(uint64_t a, uint64_t b);
uint64_t ms_hash_str(const char* s, size_t n);
double ms_u01_from_key(uint64_t key);

/* DurationDist::sample / sample_keyed / mean (distribution.hpp:54-93).
 * dist_json: {"dist":"point|uniform|empirical|default_cdf", ...} (scenario_io.hpp:44-67). */
int ms_dist_sample(const char* dist_json, const double* u, size_t n, int64_t* out, char* err, size_t err_len);
int ms_dist_sample_keyed(const char* dist_json, const uint64_t* keys, size_t n, int64_t* out, char* err,
                         size_t err_len);
int ms_dist_mean(const char* dist_json, int64_t* out, char* err, size_t err_len);

/* Eq. 1 and the wave model (exec_model.hpp:17-57).  gpu_json / kernel_json use the
 * scenario schema's "gpu" object and one "kernels[]" entry. rounding: 0 per-SM, 1 global. */
int ms_concurrent_capacity(const char* gpu_json, const char* kernel_json, int rounding, int64_t* out,
                           char* err, size_t err_len);
int ms_exec_time_model(const char* gpu_json, const char* kernel_json, int64_t n_blocks, double load,
                       int rounding, int64_t* out, char* err, size_t err_len);

/* find_optimal_split with the wave-model oracle, or the kernel's measured_time table
 * when present (splitter.hpp:141-220; engine.hpp:461-504).  slices may be NULL. */
int ms_find_optimal_split(const char* gpu_json, const char* kernel_json, double epsilon, int64_t cap_ns,
                          int square_tiling, int rounding, ms_split_plan* plan, ms_box* slices,
                          size_t slices_cap, char* err, size_t err_len);

/* slice_boxes / consolidate (splitter.hpp:89-113, 245-286). *n_out = boxes written/required. */
int ms_slice_boxes(int32_t gx, int32_t gy, int32_t gz, int64_t blocks_per_slice, int square_tiling,
                   ms_box* out, size_t cap, size_t* n_out);
int ms_consolidate(int32_t gx, int32_t gy, int32_t gz, const ms_box* pending, size_t n_pending, ms_box* out,
                   size_t cap, size_t* n_out);

/* Idle-slice predictor and harvest sizing (scheduler.hpp:18-85). */
int64_t ms_predict_interval(const int64_t* gaps, size_t n, double alpha, int32_t k, int64_t fallback);
int64_t ms_tick_interval(int64_t predicted_slice_time, int64_t launch_overhead);
/* consolidation_prefix with merged_time(k) = exec_time_model(sum of first k box sizes). */
int ms_consolidation_prefix(const char* gpu_json, const char* kernel_json, const int64_t* box_blocks,
                            size_t n, int64_t predicted_interval, double safety_factor, int64_t* out,
                            char* err, size_t err_len);

/* Metrics (metrics.hpp:21-105). */
int64_t ms_percentile(const int64_t* samples, size_t n, double q);

/* Bursty MMPP arrivals (tracegen.hpp:14-61). */
int ms_generate_bursty_arrivals(double rate, double burstiness, int64_t horizon_ns, uint64_t seed,
                                int64_t dwell_ns, int64_t* out, size_t cap, size_t* n_out, char* err,
                                size_t err_len);

/* Engine(ScenarioSpec, Policy).run() (engine.hpp:92-99, 1233-1333) on the replay device.
 * policy: "exclusive" | "spatial" | "reef" | "splitkernel" | "exclusive_lp".
 * flags: MS_RUN_NDJSON includes the rendered decision log in the result,
 *        MS_RUN_REPORT also runs exclusive + exclusive_lp and adds build_report().
 * *out_json receives the artifacts digest (counters + FNV-1a hashes of every
 * RunArtifacts vector, the decision-log hash, DES events, wall time). */
#define MS_RUN_NDJSON 1
#define MS_RUN_REPORT 2
#define MS_RUN_DELAYS 4
#define MS_RUN_ROWS 8   /* per-request rows [arrival, ttft, tpot, iterations, completed] (the live
                           runtime's ms_live_run row format), for decision-level comparisons */
int ms_replay_run(const char* scenario_json, const char* policy, int flags, char** out_json, char* err,
                  size_t err_len);

/* Same with EngineOptions (engine.hpp:84-90) as JSON:
 * {"hint_filter": ["tagA+tagB", ...], "global_floor": bool, "util_sample_period_ns": n}. */
int ms_replay_run_opts(const char* scenario_json, const char* policy, const char* options_json, int flags,
                       char** out_json, char* err, size_t err_len);

/* Scenario JSON round trip through ScenarioSpec (scenario_io.hpp:128-465). */
int ms_scenario_normalize(const char* scenario_json, char** out_json, char* err, size_t err_len);

void ms_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* MS_REPLAY_H_ */
