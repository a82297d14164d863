// Live scheduler session for an external HP tenant (include/ms_session.h).
//
// The tenant's thread calls submit / hint / wait; a scheduler thread owns every CUDA call
// on the ms_dev (LP launches, budgets, HP arming) and reacts like the reference's
// hint-driven small-bubble path and large-bubble check (engine.hpp:576-661, 970-997):
//   hint(p)   -> LP batch sized to p / safety_factor, stopped at that deadline
//   idle      -> after large_bubble_ns without HP activity, LP runs with its budget
//                extended while the tenant stays idle
//   submit    -> (tenant thread) hp_pending = 1, epoch raise, doorbell ring; the running
//                LP run drains and exits, the pre-armed chain starts behind its gate
// Race rule: the tenant sets hp_pending BEFORE raising; the scheduler never launches LP
// while it is set and re-checks it right after every launch (raising again if a submit
// slipped in between, since the launch may have captured the tenant's epoch).
#include <time.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "microslice/json.hpp"
#include "microslice/metrics.hpp"
#include "ms_session.h"
#include "power_governor.hpp"

namespace microslice {
namespace {

int64_t now_mono() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return static_cast<int64_t>(ts.tv_sec) * 1000000000ll + ts.tv_nsec;
}

struct LpState {
  int id = -1;
  uint64_t total = 0, cursor = 0, redo = 0;
  bool has_parent = false;
  int64_t tile_ns = 50000;
  uint64_t tiles_done = 0, parents = 0;
};

struct Sample {
  int64_t ring;  // host ns
  uint64_t gate, first, done;
};

}  // namespace
}  // namespace microslice

using namespace microslice;

struct ms_session {
  ms_dev* dev = nullptr;
  int n_sm = 148;
  double safety = 1.2;
  int64_t large_bubble = 2'000'000;
  std::vector<LpState> lp;
  std::unique_ptr<PowerGovernor> governor;
  std::thread th;
  std::atomic<bool> stop{false};
  // tenant <-> scheduler
  std::atomic<uint64_t> armed{0};      // (chain << 32) | seq of the pre-armed chain, 0 = none
  std::atomic<uint64_t> running{0};    // (chain << 32) | seq released by the last submit, 0 = idle
  std::atomic<int> hp_pending{0};      // set by submit before its raise, cleared on completion
  std::atomic<int> next_chain{-1};
  std::atomic<int> last_chain{-1};     // chain of the last submit (for wait)
  std::atomic<int> want_arm{0};        // a submit found nothing armed
  int last_armed_chain = -1;
  std::mutex mu;
  std::deque<int64_t> hints;           // predicted bubble lengths
  std::vector<int64_t> ring_times;     // per submit (tenant thread), consumed by the scheduler
  // scheduler-owned state
  int lp_cur = -1, lp_rr = 0;
  bool lp_running = false, bounded = false;
  int64_t deadline = 0, harvest_gap = 0, last_hp = 0;
  uint64_t run_begin = 0, run_redo_in = 0, budget = 0;
  uint64_t launches = 0, preemptions = 0, extensions = 0, submits = 0, hints_n = 0;
  std::vector<Sample> samples;
  int64_t off0 = 0, off1 = 0, c0 = 0, c1 = 0;
  std::string error;

  int lp_sms() const {
    int n = n_sm - 1;
    if (governor && governor->ok()) n = std::min(n, governor->target());
    return std::max(1, n);
  }
  uint64_t batch(const LpState& l, int64_t gap) const {
    const double waves = std::floor(static_cast<double>(gap) / safety / static_cast<double>(l.tile_ns));
    return static_cast<uint64_t>(std::max(1.0, waves) * lp_sms());
  }
  void raise() { ms_preempt_raise(dev, nullptr, nullptr); }

  void arm_next(int chain) {
    const uint32_t seq = ms_hp_next_seq(dev);
    if (ms_hp_arm(dev, chain, seq) != 0) error = std::string("ms_hp_arm: ") + ms_last_error();
    armed.store((static_cast<uint64_t>(chain) << 32) | seq, std::memory_order_release);
  }

  bool launch_lp(int64_t now) {
    if (lp.empty() || hp_pending.load(std::memory_order_seq_cst)) return false;
    if (lp_cur < 0 || !lp[lp_cur].has_parent) {
      lp_cur = lp_rr;
      lp_rr = (lp_rr + 1) % static_cast<int>(lp.size());
    }
    LpState& l = lp[lp_cur];
    if (!l.has_parent) {
      ms_lp_reset(dev, l.id);
      l.cursor = 0;
      l.redo = 0;
      l.has_parent = true;
    }
    int64_t gap = harvest_gap;
    if (bounded) {
      gap = static_cast<int64_t>(static_cast<double>(deadline - now) * safety);
      if (deadline - now < l.tile_ns) return false;  // not even one wave left
    }
    const uint64_t want = batch(l, gap);
    const uint64_t fresh = want > l.redo ? want - l.redo : 0;
    budget = std::min<uint64_t>(l.total, l.cursor + fresh);
    const int reserve = std::max(1, n_sm - lp_sms());
    ms_set_lp_sm_reserve(dev, reserve);
    if (ms_lp_run(dev, l.id, l.cursor, l.total, budget) != 0) {
      error = std::string("ms_lp_run: ") + ms_last_error();
      return false;
    }
    lp_running = true;
    run_begin = l.cursor;
    run_redo_in = l.redo;
    ++launches;
    if (hp_pending.load(std::memory_order_seq_cst)) raise();  // a submit slipped in: drain now
    return true;
  }

  void lp_exited(const ms_lp_status& st) {
    LpState& l = lp[lp_cur];
    lp_running = false;
    l.cursor = st.cursor;
    l.redo = st.redo_count;
    l.tiles_done += st.tiles_done;
    if (st.preempted) ++preemptions;
    if (l.cursor >= l.total && l.redo == 0) {
      l.has_parent = false;
      ++l.parents;
      lp_cur = -1;
    }
  }

  void maybe_extend(int64_t now) {
    (void)now;
    if (!lp_running || bounded || hp_pending.load()) return;
    LpState& l = lp[lp_cur];
    if (budget >= l.total) return;
    const uint64_t claimed = ms_lp_progress(dev, l.id);
    const uint64_t pos = run_begin + (claimed > run_redo_in ? claimed - run_redo_in : 0);
    if (pos + 2ull * n_sm < budget) return;
    budget = std::min<uint64_t>(l.total, budget + batch(l, harvest_gap));
    ms_lp_set_budget(dev, l.id, budget);
    ++extensions;
  }

  void loop() {
    last_hp = now_mono();
    bool harvesting = false;
    while (!stop.load(std::memory_order_acquire)) {
      const int64_t now = now_mono();
      // HP completion
      const uint64_t run = running.load(std::memory_order_acquire);
      if (run) {
        ms_hp_times t{};
        const int chain = static_cast<int>(run >> 32);
        if (ms_hp_poll(dev, chain, static_cast<uint32_t>(run), &t) == 1) {
          int64_t ring = 0;
          {
            std::lock_guard<std::mutex> g(mu);
            if (!ring_times.empty()) {
              ring = ring_times.front();
              ring_times.erase(ring_times.begin());
            }
          }
          samples.push_back({ring, t.t_gate, t.t_first_cta, t.t_done});
          last_armed_chain = chain;
          // hp_pending first: once running reads 0 a submit may proceed and set
          // hp_pending = 1 for the next chain, which a later clear would wipe.
          hp_pending.store(0, std::memory_order_seq_cst);
          running.store(0, std::memory_order_release);
          last_hp = now_mono();
          harvesting = false;
        }
      }
      // bubble hints: taken once the HP work they follow has completed
      const bool hp_busy = hp_pending.load(std::memory_order_seq_cst) != 0;
      int64_t hint = -1;
      if (!hp_busy) {
        std::lock_guard<std::mutex> g(mu);
        if (!hints.empty()) {
          hint = hints.front();
          hints.pop_front();
        }
      }
      // Arm the next chain at the start of the tenant's bubble (it is on the GPU long before
      // the next submit), or right away when a submit is waiting for it.
      if ((hint > 0 || want_arm.load(std::memory_order_acquire)) && !armed.load() && !running.load() &&
          !hp_pending.load(std::memory_order_seq_cst)) {
        const int nc = next_chain.load();
        arm_next(nc >= 0 ? nc : last_armed_chain);
        want_arm.store(0, std::memory_order_release);
      }
      if (hint > 0) {
        bounded = true;
        harvest_gap = hint;
        deadline = now + static_cast<int64_t>(static_cast<double>(hint) / safety);
        harvesting = lp_running || launch_lp(now);
      } else if (!hp_busy && !harvesting && !lp_running && now - last_hp >= large_bubble) {
        bounded = false;  // large bubble: unbounded, extended while idle
        harvest_gap = large_bubble;
        harvesting = launch_lp(now);
      }
      if (hp_busy) harvesting = false;
      // LP progress / exit
      if (lp_running && lp_cur >= 0) {
        ms_lp_status st{};
        if (ms_lp_poll(dev, lp[lp_cur].id, &st) == 1) {
          lp_exited(st);
          if (harvesting && !hp_pending.load()) harvesting = launch_lp(now_mono());
        } else {
          maybe_extend(now);
        }
      }
    }
  }
};

extern "C" {

int ms_session_start(ms_dev* dev, const int* lp_ids, int n_lp, int hp_chain, const char* options_json,
                     ms_session** out) {
  try {
    const json opts = json::parse(options_json ? options_json : "{}");
    auto* s = new ms_session();
    s->dev = dev;
    ms_dev_info info{};
    ms_dev_get_info(dev, &info);
    s->n_sm = info.sm_count;
    s->safety = opts.value("safety_factor", 1.2);
    s->large_bubble = opts.value("large_bubble_ns", static_cast<long long>(2'000'000));
    const json tile_ns = opts.contains("tile_ns") ? opts.at("tile_ns") : json::array();
    for (int i = 0; i < n_lp; ++i) {
      LpState l;
      l.id = lp_ids[i];
      l.total = ms_lp_total_tiles(dev, l.id);
      if (l.total == 0) {
        delete s;
        return MS_E_ARG;
      }
      if (tile_ns.is_array() && static_cast<int>(tile_ns.size()) > i) {
        l.tile_ns = tile_ns.at(static_cast<std::size_t>(i)).get<long long>();
      } else {  // measure: one full run, per-wave time
        float ms = 0;
        if (ms_lp_time_full(dev, l.id, 1, &ms) != 0) {
          delete s;
          return MS_E_CUDA;
        }
        const double waves = std::ceil(static_cast<double>(l.total) / (s->n_sm - 1));
        l.tile_ns = std::max<int64_t>(1000, static_cast<int64_t>(ms * 1e6 / waves));
      }
      ms_lp_reset(dev, l.id);
      s->lp.push_back(l);
    }
    if (opts.value("power_governor", false))
      s->governor = std::make_unique<PowerGovernor>(info.ordinal, info.sm_count, 37, info.sm_count / 2, 40u);
    int64_t rtt = 0;
    const int64_t a = now_mono();
    if (ms_clock_calibrate(dev, 100, &s->off0, &rtt) != 0) {
      delete s;
      return MS_E_CUDA;
    }
    s->c0 = (a + now_mono()) / 2;
    s->last_armed_chain = hp_chain;
    s->arm_next(hp_chain);
    s->th = std::thread([s] { s->loop(); });
    *out = s;
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ms_session_start: %s\n", e.what());
    return MS_E_ARG;
  }
}

int ms_session_hp_prepare(ms_session* s, int hp_chain) {
  s->next_chain.store(hp_chain);
  return 0;
}

int ms_session_hp_submit(ms_session* s, int hp_chain, uint32_t* seq) {
  // The scheduler re-arms right after the previous chain completes; a submit that follows
  // a very short bubble may have to wait those few microseconds.
  uint64_t a = 0;
  const int64_t t0 = now_mono();
  for (;;) {
    a = s->armed.load(std::memory_order_acquire);
    if (a && !s->running.load(std::memory_order_acquire)) break;
    if (!a) {
      s->next_chain.store(hp_chain);
      s->want_arm.store(1, std::memory_order_release);  // no bubble hint preceded: arm now
    }
    if (now_mono() - t0 > 5'000'000) return MS_E_TIMEOUT;
  }
  if (static_cast<int>(a >> 32) != hp_chain) return MS_E_ARG;
  s->armed.store(0, std::memory_order_relaxed);
  const uint32_t sq = static_cast<uint32_t>(a);
  s->hp_pending.store(1, std::memory_order_seq_cst);  // before the raise (see the race rule)
  ms_preempt_raise(s->dev, nullptr, nullptr);
  int64_t t_ring = 0;
  ms_hp_ring(s->dev, sq, &t_ring);
  {
    std::lock_guard<std::mutex> g(s->mu);
    s->ring_times.push_back(t_ring);
    s->hints.clear();  // a bubble ends when HP work arrives
  }
  s->last_chain.store(hp_chain, std::memory_order_relaxed);
  s->running.store(a, std::memory_order_release);
  ++s->submits;
  if (seq) *seq = sq;
  return 0;
}

int ms_session_hp_wait(ms_session* s, uint32_t seq, int64_t timeout_ns, ms_hp_times* t) {
  const int64_t t0 = now_mono();
  const int chain = s->last_chain.load(std::memory_order_relaxed);
  if (chain < 0) return MS_E_ARG;
  for (;;) {  // the completion record of a chain stays until its next completion
    if (ms_hp_poll(s->dev, chain, seq, t) == 1) return 0;
    if (timeout_ns >= 0 && now_mono() - t0 > timeout_ns) return MS_E_TIMEOUT;
  }
}

int ms_session_hint(ms_session* s, int64_t predicted_ns) {
  if (predicted_ns <= 0) return MS_E_ARG;
  std::lock_guard<std::mutex> g(s->mu);
  s->hints.push_back(predicted_ns);
  ++s->hints_n;
  return 0;
}

int ms_session_stop(ms_session* s, char** result_json) {
  // wait for in-flight HP work, stop the scheduler, drain LP
  for (int i = 0; i < 100000 && s->running.load(); ++i) std::this_thread::sleep_for(std::chrono::microseconds(10));
  s->stop.store(true, std::memory_order_release);
  if (s->th.joinable()) s->th.join();
  ms_preempt_raise(s->dev, nullptr, nullptr);
  if (s->lp_running && s->lp_cur >= 0) {
    ms_lp_status st{};
    ms_lp_wait(s->dev, s->lp[s->lp_cur].id, 30'000'000'000ll, &st);
    s->lp_exited(st);
  }
  // release the still-armed gate so the HP stream drains
  const uint64_t a = s->armed.load();
  if (a) ms_hp_ring(s->dev, static_cast<uint32_t>(a), nullptr);
  ms_dev_sync(s->dev);
  int64_t rtt = 0;
  const int64_t a1 = now_mono();
  ms_clock_calibrate(s->dev, 100, &s->off1, &rtt);
  s->c1 = (a1 + now_mono()) / 2;
  auto to_host = [s](uint64_t dev_ns) -> int64_t {
    double off = static_cast<double>(s->off0);
    if (s->c1 > s->c0) {
      const double h = static_cast<double>(dev_ns) - off;
      off += static_cast<double>(s->off1 - s->off0) * (h - static_cast<double>(s->c0)) / static_cast<double>(s->c1 - s->c0);
    }
    return static_cast<int64_t>(static_cast<double>(dev_ns) - off);
  };
  std::vector<Ns> r2f, g2f, dur;
  for (const Sample& x : s->samples) {
    if (x.ring && x.first) r2f.push_back(to_host(x.first) - x.ring);
    if (x.gate && x.first >= x.gate) g2f.push_back(static_cast<Ns>(x.first - x.gate));
    if (x.done >= x.first) dur.push_back(static_cast<Ns>(x.done - x.first));
  }
  auto summ = [](std::vector<Ns> v) {
    json j = json::object();
    j["n"] = json(static_cast<unsigned long long>(v.size()));
    if (!v.empty()) {
      std::sort(v.begin(), v.end());
      j["p50_ns"] = json(static_cast<long long>(percentile(v, 0.5)));
      j["p99_ns"] = json(static_cast<long long>(percentile(v, 0.99)));
      j["max_ns"] = json(static_cast<long long>(v.back()));
    }
    return j;
  };
  json out = json::object();
  out["submits"] = json(static_cast<unsigned long long>(s->submits));
  out["hints"] = json(static_cast<unsigned long long>(s->hints_n));
  out["lp_launches"] = json(static_cast<unsigned long long>(s->launches));
  out["lp_preemptions"] = json(static_cast<unsigned long long>(s->preemptions));
  out["lp_budget_extensions"] = json(static_cast<unsigned long long>(s->extensions));
  json lps = json::array();
  for (const LpState& l : s->lp) {
    json e = json::object();
    e["id"] = json(l.id);
    e["tiles_done"] = json(static_cast<unsigned long long>(l.tiles_done));
    e["parents_completed"] = json(static_cast<unsigned long long>(l.parents));
    e["tile_ns"] = json(static_cast<long long>(l.tile_ns));
    lps.push_back(std::move(e));
  }
  out["lp"] = std::move(lps);
  out["ring_to_first_hp_cta"] = summ(r2f);
  out["gate_to_first_hp_cta"] = summ(g2f);
  out["hp_chain_duration"] = summ(dur);
  if (s->governor) out["power_governor"] = s->governor->summary();
  if (!s->error.empty()) out["error"] = json(s->error);
  const std::string str = out.dump();
  *result_json = static_cast<char*>(std::malloc(str.size() + 1));
  std::memcpy(*result_json, str.c_str(), str.size() + 1);
  delete s;
  return 0;
}

}  // extern "C"
