// Value types, distributions and their validation.
// Reference: distribution.hpp:18-200, model.hpp:29-310.
#include <algorithm>
#include <cmath>

#include "microslice/distribution.hpp"
#include "microslice/model.hpp"

namespace microslice {

namespace {
void require(bool ok, const char* where, const char* what) {
  if (!ok) throw ValidationError(where, what);
}
}  // namespace

// ---------------------------------------------------------------- DurationDist
DurationDist DurationDist::point(Ns v) {
  DurationDist d;
  d.kind_ = Kind::Point;
  d.lo_ = d.hi_ = v;
  d.check();
  return d;
}

DurationDist DurationDist::uniform(Ns lo, Ns hi) {
  DurationDist d;
  d.kind_ = Kind::Uniform;
  d.lo_ = lo;
  d.hi_ = hi;
  d.check();
  return d;
}

DurationDist DurationDist::empirical(std::vector<CdfPoint> pts) {
  DurationDist d;
  d.kind_ = Kind::Empirical;
  d.cdf_ = std::move(pts);
  d.check();
  return d;
}

void DurationDist::check() const {
  if (kind_ != Kind::Empirical) {
    require(lo_ > 0 && hi_ >= lo_, "distribution", "duration bounds must be positive and ordered");
    return;
  }
  require(cdf_.size() >= 2, "distribution", "empirical CDF needs >= 2 points");
  require(cdf_.front().cum == 0.0 && cdf_.back().cum == 1.0, "distribution",
          "empirical CDF must span cum 0..1");
  for (std::size_t i = 1; i < cdf_.size(); ++i)
    require(cdf_[i].value >= cdf_[i - 1].value && cdf_[i].cum >= cdf_[i - 1].cum,
            "distribution", "empirical CDF breakpoints must be sorted");
  require(cdf_.front().value > 0, "distribution", "durations must be positive");
}

Ns DurationDist::sample(double u) const {
  if (kind_ == Kind::Point) return lo_;
  if (kind_ == Kind::Empirical) return sample_cdf(u);
  const double v = static_cast<double>(lo_) + u * static_cast<double>(hi_ - lo_);
  return std::clamp<Ns>(static_cast<Ns>(std::llround(v)), lo_, hi_);
}

Ns DurationDist::sample_cdf(double u) const {
  // First breakpoint whose cumulative probability is >= u.
  std::size_t lo_i = 0, hi_i = cdf_.size();
  while (lo_i < hi_i) {
    const std::size_t mid = lo_i + (hi_i - lo_i) / 2;
    if (cdf_[mid].cum < u) lo_i = mid + 1; else hi_i = mid;
  }
  if (lo_i == 0) return cdf_.front().value;
  if (lo_i == cdf_.size()) return cdf_.back().value;
  const CdfPoint& upper = cdf_[lo_i];
  const CdfPoint& lower = cdf_[lo_i - 1];
  const double dp = upper.cum - lower.cum;
  const double frac = dp <= 0.0 ? 0.0 : (u - lower.cum) / dp;
  const double v = static_cast<double>(lower.value) +
                   frac * static_cast<double>(upper.value - lower.value);
  return std::clamp<Ns>(static_cast<Ns>(std::llround(v)), lower.value, upper.value);
}

Ns DurationDist::mean() const {
  switch (kind_) {
    case Kind::Point: return lo_;
    case Kind::Uniform: return (lo_ + hi_) / 2;
    case Kind::Empirical: break;
  }
  double acc = 0.0;  // trapezoid rule over the piecewise-linear CDF
  for (std::size_t i = 1; i < cdf_.size(); ++i) {
    const double mass = cdf_[i].cum - cdf_[i - 1].cum;
    const double mid = 0.5 * (static_cast<double>(cdf_[i].value) +
                              static_cast<double>(cdf_[i - 1].value));
    acc += mass * mid;
  }
  return static_cast<Ns>(std::llround(acc));
}

double DurationDist::cdf_at(Ns t) const {
  if (kind_ == Kind::Point) return t >= lo_ ? 1.0 : 0.0;
  if (kind_ == Kind::Uniform) {
    if (t < lo_) return 0.0;
    if (t >= hi_) return 1.0;
    return static_cast<double>(t - lo_) / static_cast<double>(hi_ - lo_);
  }
  if (t < cdf_.front().value) return 0.0;
  if (t >= cdf_.back().value) return 1.0;
  for (std::size_t i = 1; i < cdf_.size(); ++i) {
    if (t >= cdf_[i].value) continue;
    const double span = static_cast<double>(cdf_[i].value - cdf_[i - 1].value);
    const double frac =
        span == 0.0 ? 1.0 : static_cast<double>(t - cdf_[i - 1].value) / span;
    return cdf_[i - 1].cum + frac * (cdf_[i].cum - cdf_[i - 1].cum);
  }
  return 1.0;
}

DurationDist default_block_time_cdf() {
  return DurationDist::empirical({{us(5), 0.0},
                                  {us(100), 0.90},
                                  {us(300), 0.999},
                                  {us(400), 0.999995},
                                  {us(1000), 1.0}});
}

std::string kind_name(DurationDist::Kind k) {
  static const char* const kNames[] = {"point", "uniform", "empirical"};
  const int i = static_cast<int>(k);
  return (i >= 0 && i < 3) ? kNames[i] : "?";
}

// ---------------------------------------------------------------- model types
void GpuConfig::validate() const {
  require(n_sm >= 1, "gpu.n_sm", "must be >= 1");
  require(sm_max_threads >= 32, "gpu.sm_max_threads", "must be >= 32");
  require(launch_overhead > 0, "gpu.launch_overhead", "must be > 0");
  require(sync_overhead > 0, "gpu.sync_overhead", "must be > 0");
  require(hbm_bandwidth > 0, "gpu.hbm_bandwidth", "must be > 0");
  require(dram_latency_factor >= 1.0, "gpu.dram_latency_factor", "must be >= 1");
}

void KernelSpec::validate(const GpuConfig& gpu) const {
  require(!name.empty(), "kernel.name", "must be nonempty");
  require(grid.blocks() >= 1, "kernel.grid", "grid must contain >= 1 block");
  require(threads_per_block >= 1, "kernel.threads_per_block", "must be >= 1");
  require(occupancy > 0.0 && occupancy <= 1.0, "kernel.occupancy", "must be in (0, 1]");
  require(block_time.min_value() > 0, "kernel.block_time", "durations must be > 0");
  require(bw_demand_per_block >= 0.0, "kernel.bw_demand_per_block", "must be >= 0");
  if (occupancy * gpu.sm_max_threads < threads_per_block)
    throw ValidationError("kernel." + name,
                          "no block fits an SM: occupancy * sm_max_threads < threads_per_block");
}

void BubbleHint::validate() const {
  require(!pattern.empty(), "hint.pattern", "must be nonempty");
  require(duration.min_value() > 0, "hint.duration", "durations must be > 0");
}

std::string BubbleHint::pattern_key() const {
  std::string key;
  for (std::size_t i = 0; i < pattern.size(); ++i) {
    if (i) key.push_back('+');
    key += pattern[i];
  }
  return key;
}

void RequestTrace::validate() const {
  if (arrivals.empty()) throw ValidationError("trace." + name, "arrivals must be nonempty");
  if (std::adjacent_find(arrivals.begin(), arrivals.end(),
                         [](Ns a, Ns b) { return b <= a; }) != arrivals.end())
    throw ValidationError("trace." + name, "arrivals must be strictly increasing");
}

int RequestTrace::iterations_for(std::uint64_t seed, std::size_t request_idx) const {
  const std::uint64_t key =
      hash_combine(hash_combine(seed, hash_str(name)), 0x9000 + request_idx);
  return static_cast<int>(std::max<Ns>(1, iterations.sample_keyed(key)));
}

void TaskSpec::validate() const {
  require(!name.empty(), "task.name", "must be nonempty");
  const std::string where = "task." + name;
  if (kernel_sequence.empty()) throw ValidationError(where, "kernel_sequence must be nonempty");
  for (const BubbleHint& h : bubble_hints) h.validate();
  if (kind == TaskKind::Serving && trace.empty())
    throw ValidationError(where, "serving tasks must reference a trace");
  if (memory_footprint < 0) throw ValidationError(where, "memory_footprint must be >= 0");
}

void SchedParams::validate() const {
  require(large_bubble_threshold > 0, "scheduler.threshold_ms", "must be > 0");
  require(ema_alpha > 0.0 && ema_alpha <= 1.0, "scheduler.ema_alpha", "must be in (0, 1]");
  require(ema_k >= 1, "scheduler.ema_k", "must be >= 1");
  require(safety_factor >= 1.0, "scheduler.safety_factor", "must be >= 1");
  require(resync_every >= 1, "scheduler.resync_every", "must be >= 1");
  require(slice_cap > 0, "scheduler.slice_cap_us", "must be > 0");
}

void ReefConfig::validate() const {
  require(queue_cap >= 1, "reef.queue_cap", "must be >= 1");
  require(evict_cost_per_kernel >= 0, "reef.evict_cost_us", "must be >= 0");
}

void MemParams::validate() const {
  require(hbm_gb > 0, "memory.hbm_gb", "must be > 0");
  require(probe_mb > 0, "memory.probe_mb", "must be > 0");
  require(score_threshold > 0, "memory.score_threshold", "must be > 0");
  require(dram_factor >= 1.0, "memory.dram_factor", "must be >= 1");
  require(accesses_per_wave >= 0, "memory.accesses_per_wave", "must be >= 0");
}

namespace {
struct PolicyName {
  Policy p;
  const char* name;
};
constexpr PolicyName kPolicyNames[] = {{Policy::Exclusive, "exclusive"},
                                       {Policy::Spatial, "spatial"},
                                       {Policy::Reef, "reef"},
                                       {Policy::SplitKernel, "splitkernel"},
                                       {Policy::ExclusiveLp, "exclusive_lp"}};
}  // namespace

std::string policy_name(Policy p) {
  for (const auto& e : kPolicyNames)
    if (e.p == p) return e.name;
  return "?";
}

std::optional<Policy> parse_policy(const std::string& s) {
  for (const auto& e : kPolicyNames)
    if (s == e.name) return e.p;
  return std::nullopt;
}

const KernelSpec* ScenarioSpec::find_kernel(const std::string& n) const {
  auto it = std::find_if(kernels.begin(), kernels.end(),
                         [&](const KernelSpec& k) { return k.name == n; });
  return it == kernels.end() ? nullptr : &*it;
}

const RequestTrace* ScenarioSpec::find_trace(const std::string& n) const {
  auto it = std::find_if(traces.begin(), traces.end(),
                         [&](const RequestTrace& t) { return t.name == n; });
  return it == traces.end() ? nullptr : &*it;
}

void ScenarioSpec::validate() const {
  gpu.validate();
  sched.validate();
  reef.validate();
  mem.validate();
  require(horizon > 0, "horizon", "must be > 0");
  for (const KernelSpec& k : kernels) k.validate(gpu);
  for (const TaskSpec& t : tasks) {
    t.validate();
    const std::string where = "task." + t.name;
    for (const KernelRef& kr : t.kernel_sequence) {
      if (!find_kernel(kr.kernel))
        throw ValidationError(where, "references unknown kernel '" + kr.kernel + "'");
      if (kr.repeat < 1) throw ValidationError(where, "repeat must be >= 1");
    }
    if (t.kind != TaskKind::Serving) continue;
    const RequestTrace* tr = find_trace(t.trace);
    if (!tr) throw ValidationError(where, "references unknown trace '" + t.trace + "'");
    tr->validate();
  }
}

std::vector<const TaskSpec*> ScenarioSpec::tasks_with(Priority p) const {
  std::vector<const TaskSpec*> out;
  for (const TaskSpec& t : tasks)
    if (t.priority == p) out.push_back(&t);
  return out;
}

}  // namespace microslice
