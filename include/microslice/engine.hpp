// Engine: the SLO-oriented preemptive scheduler (Algorithm 1) plus the sharing-policy
// comparators, run either against the replay device model or (live.hpp) a B200.
// Reference public API: /root/reference/proj/include/microslice/engine.hpp:24-99, 1329-1333.
//
// Internally the reference's monolithic class is split into
//   * SchedulerCore   — HP serving driver, preempt/resume reactions, small/large bubble
//                       harvesting, kernel-tick launcher, consolidation, SLO records;
//   * Device seam     — where instances are submitted and completions come back;
//   * SimDevice       — replay backend reproducing the wave-quantised device model
//                       bit-exactly (decision-log parity);
// (see paper_2601_04071_b200/csrc/host/engine.cpp).  The public surface below is
// source-compatible with the reference.
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <set>
#include <string>
#include <vector>

#include "microslice/common.hpp"
#include "microslice/events.hpp"
#include "microslice/exec_model.hpp"
#include "microslice/model.hpp"
#include "microslice/scheduler.hpp"
#include "microslice/splitter.hpp"

namespace microslice {

/// One HP request's service record (engine.hpp:24-39).
struct RequestStat {
  int task = -1;
  std::size_t index = 0;
  Ns arrival = 0;
  Ns first_token = -1;
  Ns done = -1;
  int iterations = 0;
  bool completed = false;

  Ns ttft() const { return first_token < 0 ? -1 : first_token - arrival; }
  /// (done - first) / (iters - 1) with integer division; done - arrival for 1 iteration.
  Ns tpot() const {
    if (!completed) return -1;
    return iterations > 1 ? (done - first_token) / (iterations - 1) : done - arrival;
  }
};

/// Opened when HP goes idle->active (at the HP launch-issue time), closed at the first
/// dispatched HP wave: delay = that time - begin (engine.hpp:41-46, 826-834).
struct PreemptionRecord {
  Ns begin = 0;
  Ns delay = 0;
  bool lp_in_flight = false;
  bool consolidated = false;
};

struct RunArtifacts {
  Policy policy = Policy::Exclusive;
  std::string scenario;
  std::uint64_t seed = 0;
  Ns horizon = 0;
  Timeline timeline;
  std::vector<ApiTraceRow> api_rows;
  std::vector<UtilSample> util_samples;
  std::vector<RequestStat> requests;
  std::vector<PreemptionRecord> preemptions;

  std::int64_t lp_blocks_launched = 0;
  std::int64_t lp_blocks_done = 0;
  std::int64_t lp_waste_blocks = 0;
  std::int64_t lp_blocks_in_flight_at_cutoff = 0;
  std::int64_t hp_blocks_launched = 0;
  std::int64_t hp_blocks_done = 0;
  std::int64_t hp_blocks_in_flight_at_cutoff = 0;
  double lp_work_units = 0.0;
  std::int64_t lp_parent_completions = 0;
  std::int64_t relaunch_count = 0;
  Ns sync_cost_total = 0;
  double sm_active_fraction = 0.0;
  Ns small_bubble_time = 0;
  double hp_stretch_sum = 0.0;
  std::int64_t hp_stretch_waves = 0;

  double lp_throughput_per_s() const {
    return horizon > 0 ? lp_work_units / to_sec(horizon) : 0.0;
  }
  double mean_hp_stretch() const {
    return hp_stretch_waves > 0 ? hp_stretch_sum / static_cast<double>(hp_stretch_waves) : 1.0;
  }
};

struct EngineOptions {
  /// Only hints whose pattern key is in the set are harvested (engine.hpp:85-87).
  std::optional<std::set<std::string>> hint_filter;
  CapacityRounding rounding = CapacityRounding::PerSmFloor;
  Ns util_sample_period = us(100);
};

class Engine {
 public:
  Engine(ScenarioSpec scenario, Policy policy, EngineOptions opts = {});
  Engine(Engine&&) noexcept;
  Engine& operator=(Engine&&) noexcept;
  ~Engine();

  /// Replay the scenario to its horizon on the deterministic device model.
  RunArtifacts run();

  /// Number of DES events processed by the last run() (bench / CPU-baseline metric).
  std::uint64_t events_processed() const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

RunArtifacts run_scenario(const ScenarioSpec& sc, Policy policy, EngineOptions opts = {});

}  // namespace microslice
