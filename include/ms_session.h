/* ms_session.h — C-ABI of the live scheduler for an EXTERNAL HP tenant (SURVEY.md §8f
 * next #3: bubble hints from real tenants).
 *
 * ms_live_run (ms_live.h) replays a synthetic scenario; a session instead serves a real
 * HP process: the tenant submits its pre-registered HP chains and announces its
 * CPU-side bubbles (sampling / detokenize, memcpy + sync, collective waits) as they
 * happen, and a scheduler thread harvests those bubbles with the registered preemptible
 * LP kernels — the live counterpart of the reference's hint-driven small-bubble path
 * (fire_hints / on_bubble_over, engine.hpp:576-661; BubbleHint, model.hpp:85-114) and of
 * the large-bubble check (engine.hpp:970-997).
 *
 *   submit : one epoch raise (LP drains) + one doorbell store releasing the chain the
 *            session pre-armed behind its gate — both plain stores to the host-mapped
 *            page, issued on the caller's thread (no launch, no lock on the path)
 *   hint   : a bubble of predicted length starts now — LP batches are sized to it
 *            (IntervalPredictor-free: the tenant knows its own bubble profile)
 *   idle   : no HP activity for large_bubble_ns (default 2 ms) — LP runs unbounded
 *            (budget extended while the tenant stays idle)
 *
 * Arming: the chain a submit releases is enqueued behind its doorbell gate at start and
 * then at each hint (the start of the tenant's bubble), so no launch sits on the submit
 * path; a submit with no hint before it arms on demand (one launch latency).  A chain
 * armed by a trailing hint that no submit follows runs once when the session stops.
 * Threading: submit / hint / wait may be called from one tenant thread; the session's
 * scheduler thread owns every CUDA call on the ms_dev.  Errors as in ms_b200.h.
 * options_json : {"large_bubble_ns": ns, "safety_factor": f, "power_governor": bool,
 *                 "tile_ns": [ns per LP kernel] (measured at start when absent)}
 */
#ifndef MS_SESSION_H_
#define MS_SESSION_H_

#include "ms_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ms_session ms_session;

/* lp_ids: registered LP kernels to harvest with (round-robin over parents);
 * hp_chain: the chain the first submit runs (pre-armed at start). */
int ms_session_start(ms_dev* dev, const int* lp_ids, int n_lp, int hp_chain, const char* options_json,
                     ms_session** session);
/* Chain that the NEXT submit runs (armed at the next hint; default: the same chain). */
int ms_session_hp_prepare(ms_session* s, int hp_chain);
/* Release the armed chain now; *seq identifies it for ms_session_hp_wait.  Fails with
 * MS_E_ARG when `hp_chain` is not the armed chain or a chain is still running. */
int ms_session_hp_submit(ms_session* s, int hp_chain, uint32_t* seq);
int ms_session_hp_wait(ms_session* s, uint32_t seq, int64_t timeout_ns, ms_hp_times* t);
/* A CPU-side bubble of predicted length starts now (call after the HP work completed). */
int ms_session_hint(ms_session* s, int64_t predicted_ns);
/* Stop LP, drain, and return a JSON report (free with ms_live_free). */
int ms_session_stop(ms_session* s, char** result_json);

#ifdef __cplusplus
}
#endif
#endif /* MS_SESSION_H_ */
