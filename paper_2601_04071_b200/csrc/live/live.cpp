// Live B200 scheduler: Algorithm 1 (reference engine.hpp:508-1115) on
// a dedicated host thread, driving the sm_100a device layer (include/ms_b200.h).
//
// Mapping of the reference's modelled mechanisms to the live path:
//   HP kernel issue + 7 us launch overhead   -> ring the pre-armed chain's doorbell
//   p_flag_ = true (engine.hpp:951)          -> ms_preempt_raise: LP CTAs drain and exit
//   PreemptEnd at first HP wave              -> first HP CTA %globaltimer (device clock)
//   tick launcher + 2-outstanding pacing     -> one persistent LP run whose soft budget
//                                               (harvest word) is sized from the predicted
//                                               gap and extended while HP stays idle
//   Parent::pending resume cursor            -> device claim cursor + redo list
//   SyncBegin/End "scheduler"                -> LP stream quiescence check (ms_lp_poll)
// The HP tenant's host-side bubble (hint) is reproduced from the keyed duration draw of
// the reference (engine.hpp:583-588), so a live run and a replay of the same scenario
// see the same arrivals, iteration counts and bubble lengths.
#include <cuda_runtime_api.h>
#include <dlfcn.h>
#include <pthread.h>
#include <sched.h>
#include <nvml.h>
#include <time.h>

#include <algorithm>
#include <atomic>
#include <memory>
#include <thread>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <fstream>
#include <map>
#include <queue>
#include <string>
#include <vector>

#include "microslice/engine.hpp"
#include "microslice/json.hpp"
#include "microslice/metrics.hpp"
#include "microslice/scenario_io.hpp"
#include "ms_live.h"
#include "power_governor.hpp"

namespace microslice {
namespace {

struct Timer {
  Ns t;
  long seq;
  int kind;
  int a;
  long b;
  bool operator>(const Timer& o) const { return t != o.t ? t > o.t : seq > o.seq; }
};
enum TimerKind { kArrival, kBubbleOver, kLargeBubble, kReefRefill };

struct HpTask {
  const TaskSpec* spec = nullptr;
  const RequestTrace* trace = nullptr;
  int index = 0;
  std::vector<std::vector<int>> seg_hints;  // per segment: hint indices (empty = none)
  std::vector<int> seg_kernels;             // per segment: kernel count
  std::vector<int> chain;                   // per segment: device chain id
  std::deque<std::size_t> backlog;
  bool busy = false;
  std::size_t request = 0;
  int iteration = 0, n_iterations = 0;
  std::size_t seg = 0;
  // device chain state
  bool inflight = false;
  uint32_t seq = 0;
  std::vector<uint32_t> armed;  // per segment: armed seq (0 = not armed)
  Ns ring_t = 0;
  std::uint64_t name_hash = 0, hint_hash = 0;
};

struct LpTask {
  const TaskSpec* spec = nullptr;
  std::vector<std::string> expanded;  // kernel names of the cyclic sequence
  std::size_t seq_cursor = 0;
  // current parent
  bool has_parent = false;
  int dev_id = -1;
  std::string kernel;
  uint64_t total = 0, cursor = 0;
  uint64_t redo = 0;
  Ns tile_ns = 50000;
  int tile_ctas = 1;  // SMs one tile occupies (ms_lp_tile_ctas)
};

// Host clock of the device layer (CLOCK_MONOTONIC; the ring / raise timestamps use the same
// clock).  Taken through the C-ABI so a virtual-time model of the device layer can drive
// this scheduler unchanged (tests/livemock, tests/test_live_decisions.py).
int64_t mono_ns() { return ms_host_now_ns(); }

class LiveRun {
 public:
  LiveRun(ms_dev* dev, ScenarioSpec sc, std::string policy, const json& binding, const json& opts)
      : dev_(dev), sc_(std::move(sc)), policy_(std::move(policy)), opts_(opts),
        predictor_(sc_.sched.ema_alpha, sc_.sched.ema_k, sc_.sched.large_bubble_threshold) {
    harvest_ = policy_ == "splitkernel";
    // Kernel-boundary temporal sharing (the reference's Reef policy, engine.hpp:949-997,
    // 1129-1143): non-preemptible LP kernels are (re)launched whenever HP drains; an HP
    // segment that arrives meanwhile waits for the running LP kernel to finish.
    // "reef_req": the same, but LP only between HP requests (request-level boundary).
    reef_ = policy_ == "reef" || policy_ == "reef_req";
    reef_req_ = policy_ == "reef_req";
    want_hp_ = policy_ != "exclusive_lp";
    want_lp_ = policy_ != "exclusive";
    eager_ = opts.value("eager", false);
    direct_hp_ = opts.value("direct_hp", false);  // profiler-safe: no gate kernels
    debug_runs_ = opts.value("debug_stamps", 0);   // diagnostics: per-CTA exit phases
    calibrate_ = opts.value("calibrate", true);
    // LP SM footprint: `lp_sm_reserve` SMs stay free in every LP launch (the HP gate's home);
    // `small_bubble_sms` > 0 caps LP at that many SMs while harvesting a bubble INSIDE an HP
    // request (hint bubbles), so the co-running GEMM draws less power between HP iterations
    // and the HP chain keeps its clocks (B200 runs into its 1 kW cap under a full-GPU GEMM).
    base_reserve_ = opts.value("lp_sm_reserve", getenv("MS_LP_SM_RESERVE") ? std::max(0, atoi(getenv("MS_LP_SM_RESERVE"))) : 1);
    small_sms_ = opts.value("small_bubble_sms", 0);
    max_sms_ = opts.value("lp_max_sms", 0);  // > 0: LP never uses more SMs (power budget)
    // Hint bubbles are harvested up to their predicted end / safety and not extended past
    // it (config 4, 3 x 15 s A/B: HP SLO attainment 0.92-0.93 vs 0.84-0.86 unbounded, LP
    // 0.37-0.39 vs 0.43-0.47 of exclusive).  false: extend while the bubble is open.
    bound_hints_ = opts.value("bound_hint_harvest", true);
    hint_quantile_ = opts.value("hint_quantile", -1.0);
    record_ = opts.value("timeline", true);
    ms_dev_info info{};
    ms_dev_get_info(dev_, &info);
    n_sm_ = info.sm_count;
    if (opts.value("power_governor", false))
      governor_ = std::make_unique<PowerGovernor>(info.ordinal, info.sm_count, opts.value("governor_min_sms", 37),
                                                  opts.value("governor_start_sms", info.sm_count / 2),
                                                  opts.value("governor_slack_mhz", 40u));
    for (const TaskSpec& t : sc_.tasks) {
      if (t.priority == Priority::High && want_hp_) {
        HpTask h;
        h.spec = &t;
        h.trace = sc_.find_trace(t.trace);
        h.index = static_cast<int>(hp_.size());
        build_segments(h);
        const json& chains = binding.at("hp").at(t.name);
        for (std::size_t s = 0; s < h.seg_kernels.size(); ++s)
          h.chain.push_back(h.seg_kernels[s] ? chains.at(s).get<int>() : -1);
        h.armed.assign(h.seg_kernels.size(), 0);
        h.name_hash = hash_str(t.name);
        h.hint_hash = hash_str(t.name + "#hint");
        hp_.push_back(std::move(h));
      } else if (t.priority == Priority::Low && want_lp_) {
        LpTask l;
        l.spec = &t;
        for (const KernelRef& kr : t.kernel_sequence)
          for (int r = 0; r < kr.repeat; ++r) l.expanded.push_back(kr.kernel);
        lp_.push_back(std::move(l));
      }
    }
    // One HP doorbell lane per device: every armed gate sits on the one HP stream and opens
    // for doorbell >= its seq, so a second HP task's ring would release the first task's
    // pre-armed chain.  The replay core models any number of HP streams; live runs refuse.
    if (hp_.size() > 1)
      throw ValidationError("tasks", "live B200 runtime supports one high-priority task per device (got " +
                                         std::to_string(hp_.size()) + ")");
    lp_bind_ = binding.contains("lp") ? binding.at("lp") : json::object();
    if (opts.contains("tile_ns")) tile_ns_ = opts.at("tile_ns");
    art_.policy = policy_ == "splitkernel" ? Policy::SplitKernel
                  : policy_ == "exclusive" ? Policy::Exclusive
                  : policy_ == "exclusive_lp" ? Policy::ExclusiveLp
                                              : Policy::Reef;
    art_.scenario = sc_.name;
    art_.seed = sc_.seed;
    art_.horizon = sc_.horizon;
  }

  json run();

 private:
  // ---------------------------------------------------------------- helpers
  void build_segments(HpTask& h) {
    // Same segmentation as the replay core (engine.hpp:434-459).
    std::size_t n = 0;
    for (const KernelRef& kr : h.spec->kernel_sequence) n += static_cast<std::size_t>(kr.repeat);
    std::vector<std::vector<int>> after(n + 1);
    for (std::size_t i = 0; i < h.spec->bubble_hints.size(); ++i) {
      const int pos = h.spec->bubble_hints[i].position;
      after[pos < 0 ? n : std::min<std::size_t>(static_cast<std::size_t>(pos) + 1, n)].push_back(static_cast<int>(i));
    }
    int cur = 0;
    for (std::size_t i = 0; i <= n; ++i) {
      if (i > 0) ++cur;
      if (after[i].empty()) continue;
      h.seg_kernels.push_back(cur);
      h.seg_hints.push_back(after[i]);
      cur = 0;
    }
    if (cur) {
      h.seg_kernels.push_back(cur);
      h.seg_hints.emplace_back();
    }
  }

  Ns now() const { return mono_ns() - t0_; }
  // device %globaltimer -> run-relative host ns, linear in time between the start and
  // end calibrations (the two clocks drift by ~10 ppm on this host).
  Ns dev_to_host(uint64_t dev_ns) const {
    const double d = static_cast<double>(dev_ns);
    double off = static_cast<double>(off0_);
    if (c1_ > c0_) {
      const double h = d - off;  // first approximation of the host time
      off += static_cast<double>(off1_ - off0_) * (h - static_cast<double>(c0_)) / static_cast<double>(c1_ - c0_);
    }
    return static_cast<Ns>(d - off) - t0_;
  }
  void push_timer(Ns t, int kind, int a = 0, long b = 0) { timers_.push(Timer{t, ++timer_seq_, kind, a, b}); }
  void emit(Ns ts, EventKind k, int stream, const std::string& kernel, const std::string& detail = {}) {
    if (record_) art_.timeline.emit(ts, k, stream, kernel, detail);
  }
  int check(int rc, const char* what) {
    if (rc < 0) throw EngineError(std::string(what) + ": " + ms_last_error());
    return rc;
  }

  // ---------------------------------------------------------------- HP driver
  void arm(HpTask& h, std::size_t seg) {
    if (direct_hp_ || h.chain[seg] < 0 || h.armed[seg]) return;
    const uint32_t s = ms_hp_next_seq(dev_);
    last_seq_ = s;
    check(ms_hp_arm(dev_, h.chain[seg], s), "ms_hp_arm");
    h.armed[seg] = s;
  }

  void request_arrival(int task, std::size_t idx) {
    HpTask& h = hp_[task];
    RequestStat rs;
    rs.task = task;
    rs.index = idx;
    rs.arrival = now_;
    rs.iterations = h.trace->iterations_for(sc_.seed, idx);
    art_.requests.push_back(rs);
    h.backlog.push_back(art_.requests.size() - 1);
    if (last_arrival_ >= 0) predictor_.observe_gap(now_ - last_arrival_);
    last_arrival_ = now_;
    if (h.busy) return;
    h.busy = true;
    begin_request(h);
  }

  void begin_request(HpTask& h) {
    h.request = h.backlog.front();
    h.backlog.pop_front();
    h.iteration = 0;
    h.n_iterations = art_.requests[h.request].iterations;
    h.seg = 0;
    issue_segment(h);
  }

  void issue_segment(HpTask& h) {
    if (h.seg_kernels[h.seg] == 0) {
      fire_hints(h);
      return;
    }
    arm(h, h.seg);  // normally armed long before; this is the cold path
    if (hp_active_ == 0) hp_turned_active();
    ++hp_active_;
    int64_t t_ring = 0;
    if (direct_hp_) {
      // Baseline / profiler-safe path: a host launch sits on the critical path.
      h.seq = ms_hp_next_seq(dev_);
      t_ring = mono_ns();
      check(ms_hp_launch_direct(dev_, h.chain[h.seg], h.seq), "ms_hp_launch_direct");
    } else {
      // Kernel-boundary sharing (reef) also rings immediately: the released chain cannot
      // get SMs before the running non-preemptible LP kernel drains.
      h.seq = h.armed[h.seg];
      h.armed[h.seg] = 0;
      check(ms_hp_ring(dev_, h.seq, &t_ring), "ms_hp_ring");
    }
    h.ring_t = t_ring - t0_;
    h.inflight = true;
    emit(h.ring_t, EventKind::Launch, h.index, h.spec->name, "seq=" + std::to_string(h.seq));
    // Log order of the reference (engine.hpp:707-713): Launch, then PreemptBegin at the same
    // instant — physically the flag was raised just before the ring.
    if (preempt_emit_pending_) {
      emit(h.ring_t, EventKind::PreemptBegin, -1, "");
      preempt_emit_pending_ = false;
    }
  }

  void hp_turned_active() {
    if (policy_ == "exclusive") return;
    p_flag_ = true;
    harvest_open_ = false;
    ++generation_;
    PreemptionRecord rec;
    rec.begin = now_;
    rec.lp_in_flight = lp_running_;
    pending_preempt_ = rec;
    preempt_emit_pending_ = true;  // logged right after the segment's Launch (issue_segment)
    if (harvest_ && lp_running_ && !preempt_raised_) {
      int64_t t_raise = 0;
      check(ms_preempt_raise(dev_, nullptr, &t_raise), "ms_preempt_raise");
      preempt_raised_ = true;
      t_raise_ = t_raise - t0_;
    }
  }

  void hp_chain_done(HpTask& h, const ms_hp_times& tm) {
    h.inflight = false;
    // Device timestamps are converted after the run with a drift-corrected clock fit.
    HpSample smp{h.ring_t, tm.t_first_cta, tm.t_done, tm.t_gate, pending_preempt_.has_value(),
                 pending_preempt_.has_value() && pending_preempt_->lp_in_flight, h.index, tm.seq, now_};
    hp_samples_.push_back(smp);
    if (pending_preempt_) {
      art_.preemptions.push_back(*pending_preempt_);  // delay filled in at the end
      pending_preempt_.reset();
    }
    --hp_active_;
    last_hp_activity_ = now_;
    // pre-arm the next segment this task will issue
    arm(h, (h.seg + 1) % h.seg_kernels.size());
    if (hp_active_ == 0) hp_drained();
    segment_done(h);
  }

  void hp_drained() {
    if (policy_ == "exclusive") return;
    p_flag_ = false;
    if (reef_ && !reef_req_) {  // refill after the scheduler's sync (engine.hpp:986-990)
      art_.sync_cost_total += sc_.gpu.sync_overhead;
      push_timer(now_ + sc_.gpu.sync_overhead, kReefRefill, 0);
      return;
    }
    if (!harvest_ || open_hint_ >= 0) return;
    if (eager_) {
      start_harvest(predictor_.predict());
      return;
    }
    push_timer(now_ + sc_.sched.large_bubble_threshold, kLargeBubble, 0, ++generation_);
  }

  void segment_done(HpTask& h) {
    if (!h.seg_hints[h.seg].empty()) {
      fire_hints(h);
      return;
    }
    if (++h.seg < h.seg_kernels.size()) issue_segment(h); else finish_iteration(h);
  }

  void fire_hints(HpTask& h) {
    // Keyed bubble length, identical to the replay core (engine.hpp:583-593).
    const std::uint64_t req_index = art_.requests[h.request].index;
    const std::uint64_t base = hash_combine(hash_combine(sc_.seed, h.hint_hash), req_index * 17);
    Ns dur = 0, predicted = 0;
    std::string key;
    for (const int hi : h.seg_hints[h.seg]) {
      const BubbleHint& hint = h.spec->bubble_hints[hi];
      // the scheduler sizes LP from the hint's profile, not the draw: its mean, or a low
      // quantile (option hint_quantile) so that most bubbles outlast the LP batch
      predicted += hint_quantile_ >= 0 ? hint.duration.sample(hint_quantile_) : hint.duration.mean();
      dur += hint.duration.sample_keyed(hash_combine(
          base, hash_combine(static_cast<std::uint64_t>(h.iteration), static_cast<std::uint64_t>(hi))));
      if (!key.empty()) key += '+';
      key += hint.pattern_key();
    }
    if (dur <= 0) dur = 1;
    emit(now_, EventKind::BubbleBegin, h.index, h.spec->name, "hint=" + key);
    art_.small_bubble_time += dur;
    if (harvest_ && !lp_.empty()) {
      open_hint_ = h.index;
      emit(now_, EventKind::SyncBegin, h.index, h.spec->name, "scheduler");
      emit(now_, EventKind::SyncEnd, h.index, h.spec->name, "scheduler");
      start_harvest(std::max<Ns>(1, predicted), bound_hints_);
    }
    push_timer(now_ + dur, kBubbleOver, h.index);
  }

  void bubble_over(int task) {
    HpTask& h = hp_[task];
    emit(now_, EventKind::BubbleEnd, h.index, h.spec->name);
    if (open_hint_ == task) {
      open_hint_ = -1;
      ++generation_;
      harvest_open_ = false;
      harvest_deadline_ = 0;
      const bool more = h.seg + 1 < h.seg_kernels.size() || h.iteration + 1 < h.n_iterations || !h.backlog.empty();
      if (!more && !eager_) stop_lp_soft();
      if (harvest_ && hp_active_ == 0 && !eager_)
        push_timer(now_ + sc_.sched.large_bubble_threshold, kLargeBubble, 0, generation_);
      if (eager_) harvest_open_ = true;
      if (eager_ && !lp_running_ && hp_active_ == 0) relaunch_if_allowed();
    }
    if (++h.seg < h.seg_kernels.size()) issue_segment(h); else finish_iteration(h);
  }

  void finish_iteration(HpTask& h) {
    RequestStat& rs = art_.requests[h.request];
    if (++h.iteration == 1) rs.first_token = now_;
    if (h.iteration < h.n_iterations) {
      h.seg = 0;
      issue_segment(h);
      return;
    }
    rs.done = now_;
    rs.completed = true;
    if (!h.backlog.empty()) return begin_request(h);
    h.busy = false;
    if (reef_req_) relaunch_if_allowed();  // request-level boundary: LP only between HP requests
  }

  void large_bubble_check(long gen) {
    if (!harvest_ || gen != generation_ || hp_active_ > 0) return;
    if (now_ - last_hp_activity_ < sc_.sched.large_bubble_threshold || lp_.empty()) return;
    emit(now_, EventKind::SyncBegin, -1, "", "scheduler");
    emit(now_, EventKind::SyncEnd, -1, "", "scheduler");
    start_harvest(predictor_.predict());
  }

  // ---------------------------------------------------------------- LP control
  LpTask& pick_lp() {
    LpTask& l = lp_[lp_rr_ % lp_.size()];
    lp_rr_ = (lp_rr_ + 1) % static_cast<int>(lp_.size());
    return l;
  }

  void ensure_parent(LpTask& l) {
    if (l.has_parent) return;
    l.kernel = l.expanded[l.seq_cursor % l.expanded.size()];
    ++l.seq_cursor;
    l.dev_id = lp_bind_.at(l.kernel).get<int>();
    l.tile_ns = tile_ns_.contains(l.kernel) ? tile_ns_.at(l.kernel).get<Ns>() : 50000;
    check(ms_lp_reset(dev_, l.dev_id), "ms_lp_reset");
    l.total = ms_lp_total_tiles(dev_, l.dev_id);
    l.tile_ctas = std::max(1, ms_lp_tile_ctas(dev_, l.dev_id));
    l.cursor = 0;
    l.redo = 0;
    l.has_parent = true;
    emit(now_, EventKind::Launch, -1, l.kernel, "parent");
  }

  // Tiles that fit `gap` at the kernel's measured per-tile time with every SM busy,
  // divided by the safety factor (consolidation_prefix sizing, scheduler.hpp:66-85).
  uint64_t batch_tiles(const LpTask& l, Ns gap) const {
    const double waves = static_cast<double>(gap) / sc_.sched.safety_factor / static_cast<double>(l.tile_ns);
    // one wave covers lp_sms() / (SMs per tile) tiles (2 SMs per tile on CTA pairs)
    const int per = std::max(1, l.tile_ctas);
    const uint64_t t = static_cast<uint64_t>(std::max(1.0, std::floor(waves)) * std::max(1, lp_sms() / per));
    return t;
  }
  // SMs the next LP launch may use
  int lp_sms() const {
    int n = n_sm_ - base_reserve_;
    if (max_sms_ > 0) n = std::min(n, max_sms_);
    if (governor_ && governor_->ok()) n = std::min(n, governor_->target());
    if (small_sms_ > 0 && open_hint_ >= 0) n = std::min(n, small_sms_);
    return std::max(1, n);
  }

  void start_harvest(Ns predicted_gap, bool bounded = false) {
    harvest_open_ = true;
    harvest_gap_ = predicted_gap;
    // bounded: a hint bubble of known profile — LP stops at the predicted end / safety
    // instead of being extended or relaunched into the next HP iteration
    harvest_deadline_ = bounded ? now_ + static_cast<Ns>(predicted_gap / sc_.sched.safety_factor) : 0;
    if (!lp_running_) launch_lp();
  }

  void launch_lp() {
    if (lp_.empty() || p_flag_) return;
    if (lp_cur_ < 0 || !lp_[lp_cur_].has_parent) lp_cur_ = static_cast<int>(&pick_lp() - lp_.data());
    LpTask* lt = &lp_[lp_cur_];
    ensure_parent(*lt);
    const bool np = reef_ || policy_ == "exclusive_lp";
    uint64_t budget = lt->total;
    if (harvest_) {
      // Tiles that fit the gap, less the parked (redo) tiles every run finishes first.  A
      // bounded hint bubble only gets what fits before its predicted end.
      Ns gap = harvest_gap_;
      if (harvest_deadline_ > 0) {
        gap = harvest_deadline_ - now_;
        if (gap * 1.0 < static_cast<double>(lt->tile_ns)) return;  // not even one wave left
        gap = static_cast<Ns>(gap * sc_.sched.safety_factor);  // batch_tiles divides it back out
      }
      const uint64_t want = batch_tiles(*lt, gap);
      const uint64_t fresh = want > lt->redo ? want - lt->redo : 0;
      budget = std::min<uint64_t>(lt->total, lt->cursor + fresh);
    }
    if (debug_runs_ > 0) ms_debug_stamps(dev_, 1, nullptr, 0);
    check(ms_set_lp_sm_reserve(dev_, lp_sms() < n_sm_ ? n_sm_ - lp_sms() : base_reserve_), "ms_set_lp_sm_reserve");
    check(ms_lp_run_ex(dev_, lt->dev_id, lt->cursor, lt->total, budget, np ? MS_RUN_NONPREEMPTIBLE : 0), "ms_lp_run");
    lp_budget_ = budget;
    lp_running_ = true;
    preempt_raised_ = false;
    run_begin_ = lt->cursor;
    run_redo_in_ = lt->redo;
    ++lp_launches_;
    emit(now_, EventKind::Launch, static_cast<int>(hp_.size()) + lp_cur_, lt->kernel,
         "range=" + std::to_string(lt->cursor) + ".." + std::to_string(budget) + ";redo=" + std::to_string(lt->redo));
  }

  void stop_lp_soft() {
    if (!lp_running_) return;
    LpTask& l = lp_[lp_cur_];
    // Pull the harvest budget back to the current claim point: CTAs finish their tiles and exit.
    const uint64_t claimed = ms_lp_progress(dev_, l.dev_id);
    const uint64_t fresh = claimed > run_redo_in_ ? claimed - run_redo_in_ : 0;
    check(ms_lp_set_budget(dev_, l.dev_id, run_begin_ + fresh), "ms_lp_set_budget");
    lp_budget_ = run_begin_ + fresh;
  }

  void maybe_extend_budget() {
    if (!harvest_ || !lp_running_ || !harvest_open_ || p_flag_ || harvest_deadline_ > 0) return;
    LpTask& l = lp_[lp_cur_];
    if (lp_budget_ >= l.total) return;
    const uint64_t claimed = ms_lp_progress(dev_, l.dev_id);
    const uint64_t fresh_pos = run_begin_ + (claimed > run_redo_in_ ? claimed - run_redo_in_ : 0);
    if (fresh_pos + 2ull * n_sm_ < lp_budget_) return;
    // The HP gap outlived the prediction: extend by another predicted batch.
    const uint64_t nb = std::min<uint64_t>(l.total, lp_budget_ + batch_tiles(l, harvest_gap_));
    check(ms_lp_set_budget(dev_, l.dev_id, nb), "ms_lp_set_budget");
    lp_budget_ = nb;
    ++budget_extensions_;
  }

  void lp_exited(const ms_lp_status& st) {
    LpTask& l = lp_[lp_cur_];
    lp_running_ = false;
    l.cursor = st.cursor;
    l.redo = st.redo_count;
    lp_tiles_done_ += st.tiles_done;
    if (st.t_exit > st.t_start) lp_busy_ns_ += st.t_exit - st.t_start;
    if (st.preempted) lp_preemptions_++;
    if (debug_runs_ > 0) {
      std::vector<uint64_t> buf(148 * 8 + 1, 0);
      ms_debug_stamps(dev_, 0, reinterpret_cast<unsigned long long*>(buf.data()), 148 * 8);
      if (st.preempted && preempt_raised_) {
        buf[148 * 8] = static_cast<uint64_t>(t_raise_);
        debug_.push_back(std::move(buf));
        debug_kernels_.push_back(l.kernel);
        --debug_runs_;
      }
    }
    lp_samples_.push_back(LpSample{st.preempted && preempt_raised_ ? t_raise_ : -1, st.t_seen, st.t_exit,
                                   st.t_free ? st.t_free : st.t_exit, st.t_start,
                                   static_cast<int>(hp_.size()) + lp_cur_, l.kernel,
                                   "tiles=" + std::to_string(st.tiles_done) + ";cursor=" + std::to_string(st.cursor) +
                                       ";redo=" + std::to_string(st.redo_count) +
                                       (st.preempted ? ";preempted=1" : "")});
    if (l.cursor >= l.total && l.redo == 0) {
      art_.lp_work_units += static_cast<double>(l.total);
      ++art_.lp_parent_completions;
      l.has_parent = false;
      lp_cur_ = -1;  // next parent round-robins across LP tasks
    }
    relaunch_if_allowed();
  }

  bool any_hp_busy() const {
    for (const HpTask& h : hp_)
      if (h.busy) return true;
    return false;
  }

  void relaunch_if_allowed() {
    if (lp_.empty() || lp_running_ || p_flag_) return;
    if (policy_ == "exclusive_lp") return launch_lp();
    if (reef_) {
      if (!reef_req_ || !any_hp_busy()) launch_lp();
      return;
    }
    if (harvest_ && harvest_open_) launch_lp();
  }

  // ---------------------------------------------------------------- state
  ms_dev* dev_;
  ScenarioSpec sc_;
  std::string policy_;
  json opts_;
  json lp_bind_ = json::object();
  json tile_ns_ = json::object();
  bool harvest_ = false, reef_ = false, reef_req_ = false, want_hp_ = true, want_lp_ = true, eager_ = false, record_ = true;
  bool direct_hp_ = false, calibrate_ = true;
  int debug_runs_ = 0;
  int base_reserve_ = 1, small_sms_ = 0, max_sms_ = 0;
  bool bound_hints_ = false;
  double hint_quantile_ = -1.0;  // < 0: size hint harvests from the hint's mean
  std::unique_ptr<PowerGovernor> governor_;
  std::vector<std::vector<uint64_t>> debug_;  // per preempted run: raw stamps + raise
  std::vector<std::string> debug_kernels_;    // kernel of each debug_ run
  std::vector<ms_event> trace_;               // device-side events drained during the run
  uint64_t trace_lost_ = 0;
  int n_sm_ = 148;
  int64_t t0_ = 0, off0_ = 0, off1_ = 0, c0_ = 0, c1_ = 0;
  uint32_t last_seq_ = 0;
  struct HpSample {
    Ns ring;
    uint64_t first, done, gate;
    bool preempt;
    bool lp_in_flight;  // an LP run was resident when HP turned active (engine.hpp:954-960)
    int stream;
    uint32_t seq;
    Ns detect;  // host time the scheduler saw the completion
  };
  struct LpSample {
    Ns raise;  // -1: not a preemption we raised
    uint64_t seen, exit, free, start;  // free: the grid's SMs released (ms_lp_status::t_free)
    int stream;
    std::string kernel, detail;
  };
  std::vector<HpSample> hp_samples_;
  std::vector<LpSample> lp_samples_;
  Ns now_ = 0;
  std::priority_queue<Timer, std::vector<Timer>, std::greater<Timer>> timers_;
  std::vector<Ns> timer_late_, detect_lag_;
  long timer_seq_ = 0;
  std::vector<HpTask> hp_;
  std::vector<LpTask> lp_;
  int hp_active_ = 0;
  bool p_flag_ = false;
  bool preempt_emit_pending_ = false;
  long generation_ = 0;
  int open_hint_ = -1;
  Ns last_hp_activity_ = 0, last_arrival_ = -1;
  IntervalPredictor predictor_;
  std::optional<PreemptionRecord> pending_preempt_;
  // LP
  bool lp_running_ = false, harvest_open_ = false, preempt_raised_ = false;
  int lp_cur_ = -1, lp_rr_ = 0;
  Ns harvest_gap_ = 0, t_raise_ = 0, harvest_deadline_ = 0;
  uint64_t lp_budget_ = 0, run_begin_ = 0, run_redo_in_ = 0;
  uint64_t lp_tiles_done_ = 0, lp_launches_ = 0, lp_preemptions_ = 0, budget_extensions_ = 0, lp_busy_ns_ = 0;
  std::vector<Ns> lp_free_lat_;
  std::vector<Ns> ring_to_first_, preempt_delays_, lp_exit_lat_, lp_seen_lat_, gate_to_first_, chain_durations_;
  std::vector<Ns> lp_queued_exit_lat_;
  std::vector<Ns> preempt_inflight_, preempt_idle_;  // HP activations with / without LP resident  // preempted runs that had not started at the raise
  RunArtifacts art_;

};

json summarize(const std::vector<Ns>& v) {
  json j = json::object();
  j["n"] = json(static_cast<unsigned long long>(v.size()));
  if (v.empty()) return j;
  std::vector<Ns> s = v;
  std::sort(s.begin(), s.end());
  double sum = 0;
  for (const Ns x : s) sum += static_cast<double>(x);
  j["mean_ns"] = json(sum / static_cast<double>(s.size()));
  j["p50_ns"] = json(static_cast<long long>(percentile(s, 0.50)));
  j["p90_ns"] = json(static_cast<long long>(percentile(s, 0.90)));
  j["p99_ns"] = json(static_cast<long long>(percentile(s, 0.99)));
  j["max_ns"] = json(static_cast<long long>(s.back()));
  j["min_ns"] = json(static_cast<long long>(s.front()));
  return j;
}

json LiveRun::run() {
  // Optional: pin the scheduler thread (the caller's) to one host core for the run — the
  // multi-GPU replicas each get a core on their GPU's NUMA node.  Helper threads created
  // before this point (power governor) keep the process mask.
  cpu_set_t saved;
  bool pinned = false;
  if (opts_.contains("pin_core") && opts_.at("pin_core").get<int>() >= 0) {
    const int core = opts_.at("pin_core").get<int>();
    if (pthread_getaffinity_np(pthread_self(), sizeof saved, &saved) == 0) {
      cpu_set_t one;
      CPU_ZERO(&one);
      CPU_SET(core, &one);
      pinned = pthread_setaffinity_np(pthread_self(), sizeof one, &one) == 0;
    }
  }
  struct Unpin {
    bool on;
    cpu_set_t* mask;
    ~Unpin() {
      if (on) pthread_setaffinity_np(pthread_self(), sizeof(cpu_set_t), mask);
    }
  } unpin{pinned, &saved};
  // Clock calibration: device %globaltimer -> host monotonic.
  int64_t rtt = 0, rtt1 = 0;
  {
    const int64_t a = mono_ns();
    if (calibrate_) check(ms_clock_calibrate(dev_, 200, &off0_, &rtt), "ms_clock_calibrate");
    c0_ = (a + mono_ns()) / 2;
  }
  // Optional device-side event trace (include/ms_b200.h ms_trace_*): drained while the run
  // goes on, so a long run is logged incrementally rather than rebuilt at the end.
  const long long trace_cap = opts_.value("device_trace", 0ll);
  if (trace_cap > 0) {
    check(ms_trace_enable(dev_, static_cast<size_t>(trace_cap)), "ms_trace_enable");
    ms_event sink[256];
    while (ms_trace_drain(dev_, sink, 256, nullptr) > 0) {
    }  // start from an empty window
  }
  auto drain_trace = [&]() {
    if (trace_cap <= 0) return;
    ms_event buf[256];
    int n;
    while ((n = ms_trace_drain(dev_, buf, 256, &trace_lost_)) > 0)
      for (int i = 0; i < n; ++i) trace_.push_back(buf[i]);
  };
  // Pre-arm segment 0 of every HP task; schedule arrivals.
  for (HpTask& h : hp_)
    if (!h.seg_kernels.empty()) arm(h, 0);
  const Ns start_delay = opts_.value("start_delay_ns", static_cast<long long>(2'000'000));
  t0_ = mono_ns() + start_delay;
  for (HpTask& h : hp_)
    for (std::size_t r = 0; r < h.trace->arrivals.size() && h.trace->arrivals[r] < sc_.horizon; ++r)
      push_timer(h.trace->arrivals[r], kArrival, h.index, static_cast<long>(r));
  while (mono_ns() < t0_) {
  }
  if (policy_ == "exclusive_lp" || reef_) relaunch_if_allowed();

  uint64_t loops = 0;
  for (;;) {
    now_ = now();
    if (now_ > sc_.horizon) break;
    ++loops;
    while (!timers_.empty() && timers_.top().t <= now_) {
      const Timer t = timers_.top();
      timers_.pop();
      switch (t.kind) {
        case kArrival: request_arrival(t.a, static_cast<std::size_t>(t.b)); break;
        case kBubbleOver:
          timer_late_.push_back(now_ - t.t);
          bubble_over(t.a);
          break;
        case kLargeBubble: large_bubble_check(t.b); break;
        case kReefRefill: relaunch_if_allowed(); break;  // flag checked before the first wave
      }
    }
    for (HpTask& h : hp_) {
      if (!h.inflight) continue;
      ms_hp_times tm{};
      if (check(ms_hp_poll(dev_, h.chain[h.seg], h.seq, &tm), "ms_hp_poll")) {
        now_ = now();
        hp_chain_done(h, tm);
      }
    }
    if (lp_running_) {
      ms_lp_status st{};
      if (check(ms_lp_poll(dev_, lp_[lp_cur_].dev_id, &st), "ms_lp_poll")) {
        now_ = now();
        lp_exited(st);
      } else {
        maybe_extend_budget();
      }
    }
    if ((loops & 1023) == 0) drain_trace();
  }
  // Drain: stop LP, release the armed gates (a parked gate holds an SM slot a late LP CTA
  // may need to start, see its exit and leave), finish in-flight HP.
  int64_t tr = 0;
  ms_preempt_raise(dev_, nullptr, &tr);
  if (!direct_hp_ && last_seq_) ms_hp_ring(dev_, last_seq_, nullptr);
  if (lp_running_) {
    ms_lp_status st{};
    check(ms_lp_wait(dev_, lp_[lp_cur_].dev_id, 30'000'000'000ll, &st), "ms_lp_wait");
    lp_tiles_done_ += st.tiles_done;
    if (st.t_exit > st.t_start) lp_busy_ns_ += st.t_exit - st.t_start;
  }
  for (HpTask& h : hp_)
    if (h.inflight) {
      ms_hp_times tm{};
      check(ms_hp_wait(dev_, h.chain[h.seg], h.seq, 10'000'000'000ll, &tm), "ms_hp_wait");
    }
  // Release any still-armed gates so the HP stream drains.
  ms_hp_ring(dev_, last_seq_, nullptr);
  ms_dev_sync(dev_);
  drain_trace();
  if (trace_cap > 0) ms_trace_enable(dev_, 0);
  // The LP SM reserve was moved per launch (governor, SM caps): leave the device at the
  // run's base reserve, so a later timing (calibration, profiler) sees the full LP grid.
  ms_set_lp_sm_reserve(dev_, base_reserve_);
  {
    const int64_t a = mono_ns();
    if (calibrate_) check(ms_clock_calibrate(dev_, 200, &off1_, &rtt1), "ms_clock_calibrate");
    else off1_ = off0_;
    c1_ = (a + mono_ns()) / 2;
  }
  // Convert the device-side samples and emit the device-timed decision events.
  std::size_t pi = 0;
  for (const HpSample& smp : hp_samples_) {
    const Ns first = dev_to_host(smp.first), done = dev_to_host(smp.done);
    ring_to_first_.push_back(first - smp.ring);
    if (smp.gate) gate_to_first_.push_back(static_cast<Ns>(smp.first) - static_cast<Ns>(smp.gate));
    chain_durations_.push_back(done - first);
    detect_lag_.push_back(smp.detect - done);
    if (smp.preempt && pi < art_.preemptions.size()) {
      art_.preemptions[pi].delay = first - smp.ring;
      preempt_delays_.push_back(first - smp.ring);
      (smp.lp_in_flight ? preempt_inflight_ : preempt_idle_).push_back(first - smp.ring);
      emit(first, EventKind::PreemptEnd, smp.stream, hp_[smp.stream].spec->name,
           "delay_ns=" + std::to_string(first - smp.ring));
      ++pi;
    }
    emit(done, EventKind::KernelDone, smp.stream, hp_[smp.stream].spec->name, "seq=" + std::to_string(smp.seq));
  }
  json preempted_runs = json::array();  // [kernel, exit - raise, start - raise, seen - raise, detail]
  for (const LpSample& smp : lp_samples_) {
    if (smp.raise >= 0) {
      json e = json::array();
      e.push_back(json(smp.kernel));
      e.push_back(json(static_cast<long long>(dev_to_host(smp.exit) - smp.raise)));
      e.push_back(json(static_cast<long long>(smp.start ? dev_to_host(smp.start) - smp.raise : 0)));
      e.push_back(json(static_cast<long long>(smp.seen ? dev_to_host(smp.seen) - smp.raise : 0)));
      e.push_back(json(smp.detail));
      preempted_runs.push_back(std::move(e));
      // A run whose first CTA started after the raise was still queued behind the HP chain
      // (its CTAs get SMs only when HP leaves them): it never occupied an SM HP needed, so
      // its exit time is reported apart from the drain of running LP work.
      if (smp.start && dev_to_host(smp.start) > smp.raise) {
        lp_queued_exit_lat_.push_back(dev_to_host(smp.exit) - smp.raise);
      } else {
        lp_exit_lat_.push_back(dev_to_host(smp.exit) - smp.raise);
        lp_free_lat_.push_back(dev_to_host(smp.free) - smp.raise);
        if (smp.seen) lp_seen_lat_.push_back(dev_to_host(smp.seen) - smp.raise);
      }
    }
    emit(dev_to_host(smp.exit), EventKind::KernelDone, smp.stream, smp.kernel, smp.detail);
  }
  art_.timeline.finalize();

  json out = json::object();
  out["policy"] = json(policy_);
  out["scenario"] = json(sc_.name);
  out["horizon_ns"] = json(static_cast<long long>(sc_.horizon));
  out["loops"] = json(static_cast<unsigned long long>(loops));
  out["pinned_core"] = json(pinned ? opts_.at("pin_core").get<int>() : -1);
  out["clock"] = json::object();
  out["clock"]["offset_ns"] = json(static_cast<long long>(off0_));
  out["clock"]["drift_ppm"] = json(c1_ > c0_ ? 1e6 * static_cast<double>(off1_ - off0_) / static_cast<double>(c1_ - c0_) : 0.0);
  out["clock"]["rtt_min_ns"] = json(static_cast<long long>(std::max(rtt, rtt1)));
  std::size_t completed = 0;
  json reqs = json::array();
  for (const RequestStat& r : art_.requests) {
    completed += r.completed ? 1 : 0;
    json e = json::array();
    e.push_back(json(static_cast<long long>(r.arrival)));
    e.push_back(json(static_cast<long long>(r.ttft())));
    e.push_back(json(static_cast<long long>(r.tpot())));
    e.push_back(json(r.iterations));
    e.push_back(json(r.completed));
    reqs.push_back(std::move(e));
  }
  out["requests"] = json::object();
  out["requests"]["n"] = json(static_cast<unsigned long long>(art_.requests.size()));
  out["requests"]["completed"] = json(static_cast<unsigned long long>(completed));
  out["requests"]["rows"] = std::move(reqs);  // [arrival, ttft, tpot, iterations, completed]
  out["preempt_ring_to_first_hp_cta"] = summarize(preempt_delays_);
  out["ring_to_first_hp_cta_all"] = summarize(ring_to_first_);
  // true preemptions (LP resident when HP turned active) vs activations on an LP-idle GPU
  out["preempt_ring_to_first_hp_cta_lp_in_flight"] = summarize(preempt_inflight_);
  out["preempt_ring_to_first_hp_cta_lp_idle"] = summarize(preempt_idle_);
  // host-side HP path: chain done (device) -> scheduler saw it; bubble end due -> handled
  out["hp_done_detect_lag"] = summarize(detect_lag_);
  out["bubble_timer_late"] = summarize(timer_late_);
  out["preempt_flag_to_last_lp_exit"] = summarize(lp_exit_lat_);
  out["preempt_flag_to_lp_sms_free"] = summarize(lp_free_lat_);
  out["preempt_flag_to_first_lp_seen"] = summarize(lp_seen_lat_);
  out["preempt_flag_to_exit_of_queued_lp_runs"] = summarize(lp_queued_exit_lat_);
  std::vector<Ns> g2f;
  for (const Ns x : gate_to_first_)
    if (x >= 0) g2f.push_back(x);
  out["gate_to_first_hp_cta_device"] = summarize(g2f);
  out["hp_chain_duration"] = summarize(chain_durations_);
  json raw = json::object();
  json a = json::array(), b = json::array();
  for (const Ns x : preempt_delays_) a.push_back(json(static_cast<long long>(x)));
  for (const Ns x : lp_exit_lat_) b.push_back(json(static_cast<long long>(x)));
  raw["preempt_ring_to_first_hp_cta"] = std::move(a);
  raw["preempt_flag_to_last_lp_exit"] = std::move(b);
  json bf = json::array();
  for (const Ns x : lp_free_lat_) bf.push_back(json(static_cast<long long>(x)));
  raw["preempt_flag_to_lp_sms_free"] = std::move(bf);
  json fi = json::array();
  for (const Ns x : preempt_inflight_) fi.push_back(json(static_cast<long long>(x)));
  raw["preempt_ring_to_first_hp_cta_lp_in_flight"] = std::move(fi);
  json fid = json::array();
  for (const Ns x : preempt_idle_) fid.push_back(json(static_cast<long long>(x)));
  raw["preempt_ring_to_first_hp_cta_lp_idle"] = std::move(fid);
  json c = json::array();
  for (const Ns x : ring_to_first_) c.push_back(json(static_cast<long long>(x)));
  raw["ring_to_first_hp_cta_all"] = std::move(c);
  raw["preempted_lp_runs"] = std::move(preempted_runs);
  if (opts_.value("device_trace", 0ll) > 0) {
    // [t (run-relative host ns), kind, id, a, b] of every drained device event
    json dt = json::object(), rows = json::array();
    std::map<uint32_t, long long> by_kind;
    for (const ms_event& e : trace_) {
      ++by_kind[e.kind];
      json r = json::array();
      r.push_back(json(static_cast<long long>(dev_to_host(e.t_ns))));
      r.push_back(json(static_cast<long long>(e.kind)));
      r.push_back(json(static_cast<long long>(e.id)));
      r.push_back(json(static_cast<unsigned long long>(e.a)));
      r.push_back(json(static_cast<unsigned long long>(e.b)));
      rows.push_back(std::move(r));
    }
    json bk = json::object();
    for (const auto& [k, n] : by_kind) bk[std::to_string(k)] = json(n);
    dt["events"] = json(static_cast<unsigned long long>(trace_.size()));
    dt["lost"] = json(static_cast<unsigned long long>(trace_lost_));
    dt["by_kind"] = std::move(bk);
    dt["rows"] = std::move(rows);
    out["device_trace"] = std::move(dt);
  }
  out["samples"] = std::move(raw);
  if (!debug_.empty()) {
    // phase p of CTA c relative to the raise, converted with the drift-corrected clock
    json dbg = json::array();
    for (const auto& buf : debug_) {
      const Ns raise = static_cast<Ns>(buf[148 * 8]);
      json run = json::array();
      for (int ph = 0; ph < 7; ++ph) {
        std::vector<Ns> v;
        for (int c = 0; c < 148; ++c)
          if (buf[c * 8 + ph]) v.push_back(dev_to_host(buf[c * 8 + ph]) - raise);
        json e = json::array();
        if (!v.empty()) {
          std::sort(v.begin(), v.end());
          e.push_back(json(static_cast<long long>(v.front())));
          e.push_back(json(static_cast<long long>(v[v.size() / 2])));
          e.push_back(json(static_cast<long long>(v.back())));
        }
        run.push_back(std::move(e));
      }
      // the latest observers: [cta, seen, exit_begin]
      std::vector<std::pair<Ns, int>> seen;
      for (int c = 0; c < 148; ++c)
        if (buf[c * 8]) seen.push_back({dev_to_host(buf[c * 8]) - raise, c});
      std::sort(seen.begin(), seen.end());
      json late = json::array();
      for (std::size_t i = seen.size() > 4 ? seen.size() - 4 : 0; i < seen.size(); ++i) {
        json t = json::array();
        t.push_back(json(seen[i].second));
        t.push_back(json(static_cast<long long>(seen[i].first)));
        t.push_back(json(static_cast<long long>(buf[seen[i].second * 8 + 5] ? dev_to_host(buf[seen[i].second * 8 + 5]) - raise : -1)));
        late.push_back(std::move(t));
      }
      run.push_back(std::move(late));
      json cnt = json::array();
      for (int ph = 0; ph < 7; ++ph) {
        int k = 0;
        for (int c = 0; c < 148; ++c) k += buf[c * 8 + ph] ? 1 : 0;
        cnt.push_back(json(k));
      }
      run.push_back(std::move(cnt));
      dbg.push_back(std::move(run));
    }
    out["debug_phases"] = std::move(dbg);  // [run][phase] = [min, p50, max] ns
    json dk = json::array();
    for (const std::string& k : debug_kernels_) dk.push_back(json(k));
    out["debug_kernels"] = std::move(dk);
  }
  out["hp_chains"] = json(static_cast<unsigned long long>(hp_samples_.size()));
  json lp = json::object();
  lp["tiles_done"] = json(static_cast<unsigned long long>(lp_tiles_done_));
  lp["tiles_per_s"] = json(static_cast<double>(lp_tiles_done_) / to_sec(sc_.horizon));
  lp["parents_completed"] = json(static_cast<long long>(art_.lp_parent_completions));
  lp["work_units"] = json(art_.lp_work_units);
  lp["launches"] = json(static_cast<unsigned long long>(lp_launches_));
  // device time the LP grids were resident (first CTA start -> exit record, summed over runs)
  lp["busy_ns"] = json(static_cast<unsigned long long>(lp_busy_ns_));
  lp["preemptions"] = json(static_cast<unsigned long long>(lp_preemptions_));
  lp["budget_extensions"] = json(static_cast<unsigned long long>(budget_extensions_));
  out["lp"] = std::move(lp);
  out["small_bubble_ns"] = json(static_cast<long long>(art_.small_bubble_time));
  if (governor_) out["power_governor"] = governor_->summary();
  out["timeline_events"] = json(static_cast<unsigned long long>(art_.timeline.size()));
  if (opts_.contains("slo")) {
    SloThresholds slo{opts_.at("slo").at("ttft_ns").get<Ns>(), opts_.at("slo").at("tpot_ns").get<Ns>()};
    out["slo_attainment"] = json(slo_attainment(art_.requests, slo));
  }
  if (art_.requests.size() >= 1) {
    try {
      const SloThresholds own = compute_slo(art_, 1);
      out["own_p99"] = json::object();
      out["own_p99"]["ttft_ns"] = json(static_cast<long long>(own.ttft));
      out["own_p99"]["tpot_ns"] = json(static_cast<long long>(own.tpot));
    } catch (const ValidationError&) {
    }
  }
  if (opts_.contains("ndjson_path")) {
    std::ofstream f(opts_.at("ndjson_path").get<std::string>());
    art_.timeline.write_ndjson(f);
  }
  return out;
}

}  // namespace
}  // namespace microslice

extern "C" int ms_live_run(ms_dev* dev, const char* scenario_json, const char* policy, const char* binding_json,
                           const char* options_json, char** result_json) {
  using namespace microslice;
  try {
    const ScenarioSpec sc = scenario_from_json(json::parse(scenario_json));
    const json binding = json::parse(binding_json ? binding_json : "{}");
    const json opts = json::parse(options_json ? options_json : "{}");
    const std::string pol = policy ? policy : "splitkernel";
    if (pol != "splitkernel" && pol != "exclusive" && pol != "exclusive_lp" && pol != "reef" && pol != "reef_req")
      throw ValidationError("policy", "unknown live policy '" + pol + "'");
    LiveRun run(dev, sc, pol, binding, opts);
    const std::string s = run.run().dump();
    *result_json = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(*result_json, s.c_str(), s.size() + 1);
    return 0;
  } catch (const ValidationError& e) {
    std::fprintf(stderr, "ms_live_run: %s\n", e.what());
    return -2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ms_live_run: %s\n", e.what());
    return -3;
  }
}

extern "C" void ms_live_free(void* p) { std::free(p); }
