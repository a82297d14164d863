/* ms_live.h — C-ABI of the live B200 scheduler (Algorithm 1 on a host thread driving
 * the device layer of ms_b200.h in real time).
 *
 * It is the live counterpart of Engine(ScenarioSpec, Policy).run()
 * (/root/reference/proj/include/microslice/engine.hpp:92-99, 1233-1327): same scenario
 * schema, same policies, same keyed iteration counts / hint durations, same decision
 * events in the Timeline — but kernels execute on the GPU and every timestamp is real.
 *
 * scenario_json : reference scenario schema (scenario_io.hpp)
 * policy        : "splitkernel" | "exclusive" | "exclusive_lp" | "reef" | "reef_req"
 *                 reef = kernel-boundary temporal sharing as the reference's Reef policy
 *                 models it (engine.hpp:949-997, 1129-1143): unsplit, non-preemptible LP
 *                 kernels relaunched whenever HP drains (after the scheduler sync); an HP
 *                 segment arriving meanwhile waits for the running LP kernel.
 *                 reef_req = the same with LP only between HP requests.
 * binding_json  : {"lp": {"<kernel name>": <ms_lp id>, ...},
 *                  "hp": {"<task name>": [<chain id of segment 0>, ...], ...}}
 * options_json  : {"eager": bool, "slo": {"ttft_ns": .., "tpot_ns": ..},
 *                  "tile_ns": {"<lp kernel name>": ns}, "timeline": bool,
 *                  "start_delay_ns": ns, "ndjson_path": str,
 *                  LP SM footprint (B200 power cap):
 *                  "lp_sm_reserve": n (SMs every LP launch leaves free, default 1),
 *                  "lp_max_sms": n (fixed LP SM budget), "small_bubble_sms": n (budget
 *                  while harvesting a bubble inside an HP request),
 *                  "power_governor": bool (NVML SM-clock feedback sizes the LP budget),
 *                  "governor_min_sms", "governor_start_sms", "governor_slack_mhz",
 *                  hint bubbles: "bound_hint_harvest": bool (default true: LP stops at the
 *                  predicted end / safety), "hint_quantile": q (size from the q-quantile of
 *                  the hint's duration profile instead of its mean)}
 * *result_json  : requests, preemption delays (ring -> first HP CTA, and flag -> last LP
 *                 CTA exit), LP tiles / parents completed, SLO report, timeline summary,
 *                 power-governor summary (mean LP SMs, SM clock).
 */
#ifndef MS_LIVE_H_
#define MS_LIVE_H_

#include "ms_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

int ms_live_run(ms_dev* dev, const char* scenario_json, const char* policy, const char* binding_json,
                const char* options_json, char** result_json);
void ms_live_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* MS_LIVE_H_ */
