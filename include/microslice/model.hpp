// Task / scheduler API value types: the drop-in surface the scheduler is driven by.
// Reference: /root/reference/proj/include/microslice/model.hpp:13-310.
// Field names, defaults and validation messages are kept identical so code written
// against the reference compiles unchanged and fails with the same ValidationError.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "microslice/common.hpp"
#include "microslice/distribution.hpp"

namespace microslice {

struct NvlinkPeer {  // model.hpp:13-18 (memory tier links, microslice/memory.hpp)
  int peer_id = 0;
  Ns baseline_latency = us(2);
  double bandwidth = 600.0e9;
  double background_load = 0.0;
};

/// Device description.  Defaults are the reference's A100 numbers; the B200 replay
/// configs override n_sm / hbm_bandwidth / launch / sync with measured values.
struct GpuConfig {
  int n_sm = 108;
  int sm_max_threads = 2048;
  double hbm_bandwidth = 2.0e12;  // bytes/s
  Ns launch_overhead = us(7);
  Ns sync_overhead = us(5);
  std::vector<NvlinkPeer> nvlink_peers;
  double dram_latency_factor = 4.0;

  void validate() const;
};

struct Grid {
  int x = 1, y = 1, z = 1;
  std::int64_t blocks() const { return static_cast<std::int64_t>(x) * y * z; }
};

/// One kernel as the scheduler sees it: grid geometry, Eq. 1 occupancy inputs, the
/// per-block time distribution and HBM demand; `measured_time` (n_blocks, time)
/// rows replace the analytic wave model as the split oracle when present.
struct KernelSpec {
  std::string name;
  Grid grid;
  int threads_per_block = 256;
  double occupancy = 1.0;
  DurationDist block_time = DurationDist::point(us(77));
  double bw_demand_per_block = 0.0;  // bytes/s while a block is resident
  bool splittable = true;
  std::vector<std::pair<std::int64_t, Ns>> measured_time;

  void validate(const GpuConfig& gpu) const;
};

enum class Priority { High, Low };
enum class TaskKind { Serving, Batch };
enum class HintKind { MemSync, InterGpuComm, CpuBound };

/// Host-side API marker sequence delimiting an idle interval of the HP tenant
/// (small bubble).  `position` = fire after kernel index (-1: iteration end).
struct BubbleHint {
  HintKind kind = HintKind::MemSync;
  std::vector<std::string> pattern;
  DurationDist duration = DurationDist::uniform(us(500), us(1000));
  int position = -1;
  bool contended = false;

  void validate() const;
  std::string pattern_key() const;  // tags joined with '+'
};

struct RequestTrace {
  std::string name;
  std::vector<Ns> arrivals;
  DurationDist iterations = DurationDist::point(8);  // dimensionless count

  void validate() const;
  /// Keyed iteration count of request `request_idx` (model.hpp:131-136), >= 1.
  int iterations_for(std::uint64_t seed, std::size_t request_idx) const;
};

struct KernelRef {
  std::string kernel;
  int repeat = 1;
};

struct TaskSpec {
  std::string name;
  Priority priority = Priority::Low;
  TaskKind kind = TaskKind::Batch;
  std::vector<KernelRef> kernel_sequence;
  std::vector<BubbleHint> bubble_hints;
  std::int64_t memory_footprint = 0;
  std::string trace;

  void validate() const;
};

/// Split-kernel scheduler knobs (model.hpp:167-190).
struct SchedParams {
  Ns large_bubble_threshold = ms(2);
  double ema_alpha = 0.3;
  int ema_k = 8;
  double safety_factor = 1.2;
  int resync_every = 64;
  Ns slice_cap = us(400);
  bool square_tiling = false;
  bool consolidation = true;

  void validate() const;
};

/// Kernel-boundary temporal-sharing comparator knobs (model.hpp:192-201).
struct ReefConfig {
  int queue_cap = 4;
  Ns evict_cost_per_kernel = us(1);

  void validate() const;
};

enum class EvictionPolicy { ContentionFirst, RoundRobin };

/// Memory-tier knobs (model.hpp:205-225); the tier is microslice/memory.hpp.
struct MemParams {
  bool enabled = false;
  double hbm_gb = 80.0;
  std::vector<double> peer_free_gb;
  double dram_factor = 4.0;
  double probe_mb = 4.0;
  double score_threshold = 1.5;
  EvictionPolicy eviction = EvictionPolicy::ContentionFirst;
  int accesses_per_wave = 4;

  void validate() const;
};

enum class Policy { Exclusive, Spatial, Reef, SplitKernel, ExclusiveLp };

std::string policy_name(Policy p);
std::optional<Policy> parse_policy(const std::string& s);

struct ScenarioSpec {
  std::string name;
  GpuConfig gpu;
  std::vector<KernelSpec> kernels;
  std::vector<TaskSpec> tasks;
  std::vector<RequestTrace> traces;
  std::uint64_t seed = 1;
  Ns horizon = seconds(30);
  SchedParams sched;
  ReefConfig reef;
  MemParams mem;

  const KernelSpec* find_kernel(const std::string& n) const;
  const RequestTrace* find_trace(const std::string& n) const;
  void validate() const;
  std::vector<const TaskSpec*> tasks_with(Priority p) const;
};

}  // namespace microslice
