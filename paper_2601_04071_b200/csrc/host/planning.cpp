// Eq. 1 / wave model, slice geometry, optimal-split search, consolidation, and the
// bursty arrival generator.
// Reference: exec_model.hpp:17-68, splitter.hpp:41-286, tracegen.hpp:14-61.
#include <algorithm>
#include <cmath>

#include "microslice/exec_model.hpp"
#include "microslice/splitter.hpp"
#include "microslice/tracegen.hpp"

namespace microslice {

// ------------------------------------------------------------------ Eq. 1 + waves
std::int64_t concurrent_capacity(const GpuConfig& gpu, const KernelSpec& kernel,
                                 CapacityRounding rounding) {
  const double threads_per_sm = kernel.occupancy * gpu.sm_max_threads;
  std::int64_t cap;
  if (rounding == CapacityRounding::GlobalFloor) {
    cap = static_cast<std::int64_t>(gpu.n_sm * threads_per_sm / kernel.threads_per_block);
  } else {
    const auto blocks_per_sm =
        static_cast<std::int64_t>(threads_per_sm / kernel.threads_per_block);
    cap = blocks_per_sm * static_cast<std::int64_t>(gpu.n_sm);
  }
  if (cap < 1)
    throw ValidationError("concurrent_capacity",
                          "block exceeds SM capacity for kernel '" + kernel.name + "'");
  return cap;
}

Ns exec_time_model(const GpuConfig& gpu, const KernelSpec& kernel, std::int64_t n_blocks,
                   double concurrent_bw_load, CapacityRounding rounding) {
  if (n_blocks < 1) throw ValidationError("exec_time_model", "n_blocks must be >= 1");
  const std::int64_t cap = concurrent_capacity(gpu, kernel, rounding);
  const std::int64_t waves = (n_blocks + cap - 1) / cap;
  const double resident = static_cast<double>(n_blocks < cap ? n_blocks : cap);
  const double stretch = std::max(
      1.0, (resident * kernel.bw_demand_per_block + concurrent_bw_load) / gpu.hbm_bandwidth);
  const double t =
      static_cast<double>(waves) * static_cast<double>(kernel.block_time.mean()) * stretch;
  return static_cast<Ns>(std::llround(t));
}

double bandwidth_stretch(const GpuConfig& gpu, const KernelSpec& kernel,
                         std::int64_t resident_blocks, double other_bw_load) {
  const double demand =
      static_cast<double>(resident_blocks) * kernel.bw_demand_per_block + other_bw_load;
  return std::max(1.0, demand / gpu.hbm_bandwidth);
}

// ------------------------------------------------------------------ geometry
namespace detail {

void linear_to_coord(std::int64_t p, const Grid& g, int& x, int& y, int& z) {
  const std::int64_t row = p / g.x;
  x = static_cast<int>(p - row * g.x);
  y = static_cast<int>(row % g.y);
  z = static_cast<int>(p / (static_cast<std::int64_t>(g.x) * g.y));
}

GridBox next_box(std::int64_t p, const Grid& g, std::int64_t budget) {
  GridBox b;
  linear_to_coord(p, g, b.ox, b.oy, b.oz);
  b.sy = b.sz = 1;
  // Mid-row start, or not even one full row of budget: a run along x.
  if (b.ox != 0 || budget < g.x) {
    b.sx = static_cast<int>(std::min<std::int64_t>(g.x - b.ox, budget));
    return b;
  }
  b.sx = g.x;
  const std::int64_t plane = static_cast<std::int64_t>(g.x) * g.y;
  // Mid-plane start, or less than a plane of budget: whole rows.
  if (b.oy != 0 || budget < plane) {
    b.sy = static_cast<int>(std::min<std::int64_t>(g.y - b.oy, budget / g.x));
    return b;
  }
  b.sy = g.y;
  b.sz = static_cast<int>(std::min<std::int64_t>(g.z - b.oz, budget / plane));
  return b;
}

void box_ranges(const GridBox& b, const Grid& g, std::vector<LinRange>& out) {
  const std::int64_t plane = static_cast<std::int64_t>(g.x) * g.y;
  for (int dz = 0; dz < b.sz; ++dz)
    for (int dy = 0; dy < b.sy; ++dy) {
      const std::int64_t lo =
          (b.oz + dz) * plane + static_cast<std::int64_t>(b.oy + dy) * g.x + b.ox;
      out.push_back({lo, lo + b.sx});
    }
}

}  // namespace detail

std::vector<GridBox> slice_boxes(const Grid& grid, std::int64_t blocks_per_slice,
                                 bool square_tiling) {
  if (blocks_per_slice < 1) throw ValidationError("splitter", "blocks_per_slice must be >= 1");
  const bool quadrants = square_tiling && grid.z == 1 && grid.x == grid.y &&
                         grid.x % 2 == 0 &&
                         blocks_per_slice == static_cast<std::int64_t>(grid.x / 2) * (grid.y / 2);
  std::vector<GridBox> out;
  if (quadrants) {
    const int h = grid.x / 2;
    for (int qy = 0; qy < 2; ++qy)
      for (int qx = 0; qx < 2; ++qx) out.push_back({qx * h, qy * h, 0, h, h, 1});
    return out;
  }
  const std::int64_t total = grid.blocks();
  for (std::int64_t p = 0; p < total;) {
    out.push_back(detail::next_box(p, grid, std::min(blocks_per_slice, total - p)));
    p += out.back().blocks();
  }
  return out;
}

std::vector<GridBox> slice_schedule(const KernelSpec& kernel, const SplitPlan& plan,
                                    bool square_tiling) {
  if (plan.kernel != kernel.name)
    throw ValidationError("splitter", "plan for '" + plan.kernel +
                                          "' does not match kernel '" + kernel.name + "'");
  return slice_boxes(kernel.grid, plan.blocks_per_slice, square_tiling);
}

// ------------------------------------------------------------------ split search
SplitPlan find_optimal_split(const GpuConfig& gpu, const KernelSpec& kernel,
                             const ExecOracle& oracle, const SplitSearchOptions& opts) {
  if (!kernel.splittable)
    throw ValidationError("splitter", "splitting disabled for kernel '" + kernel.name + "'");
  const std::int64_t capacity = concurrent_capacity(gpu, kernel, opts.rounding);

  // Step 1: halve from the concurrency limit while that is > eps faster.
  std::int64_t n = capacity;
  Ns t_n = oracle(n);
  Ns best = t_n;
  while (n > 1) {
    const Ns t_half = oracle(n / 2);
    best = std::min(best, t_half);
    if (!(static_cast<double>(t_half) < (1.0 - opts.epsilon) * static_cast<double>(t_n)))
      break;
    n /= 2;
    t_n = t_half;
  }

  // Step 2: grow to the largest count still within (1 + eps) of the best time.
  const double plateau = (1.0 + opts.epsilon) * static_cast<double>(best);
  std::int64_t m = (static_cast<double>(t_n) > plateau && n > 1) ? n / 2 : n;
  while (m + 1 <= capacity && static_cast<double>(oracle(m + 1)) <= plateau) ++m;

  SplitPlan plan;
  plan.kernel = kernel.name;
  plan.cap = opts.cap;
  plan.memory_bound = n < capacity;
  plan.blocks_per_slice = m;
  plan.predicted_slice_time = oracle(m);

  // Step 3: enforce the per-slice time cap.
  if (plan.predicted_slice_time > opts.cap) {
    const Ns t_one = oracle(1);
    if (t_one > opts.cap) {
      plan.blocks_per_slice = 1;
      plan.predicted_slice_time = t_one;
      plan.uncappable = true;
    } else {
      std::int64_t lo = 1, hi = m;  // upper-biased bisection; same probe order as reference
      while (hi > lo) {
        const std::int64_t probe = lo + (hi - lo + 1) / 2;
        if (oracle(probe) <= opts.cap) lo = probe; else hi = probe - 1;
      }
      plan.blocks_per_slice = lo;
      plan.predicted_slice_time = oracle(lo);
    }
  }
  plan.slices = slice_boxes(kernel.grid, plan.blocks_per_slice, opts.square_tiling);
  return plan;
}

SplitPlan find_optimal_split(const GpuConfig& gpu, const KernelSpec& kernel,
                             const SplitSearchOptions& opts) {
  const ExecOracle wave_model = [&](std::int64_t n) {
    return exec_time_model(gpu, kernel, n, 0.0, opts.rounding);
  };
  return find_optimal_split(gpu, kernel, wave_model, opts);
}

// ------------------------------------------------------------------ consolidation
std::vector<GridBox> consolidate(const std::string& parent, const Grid& grid,
                                 const std::vector<std::string>& owners,
                                 const std::vector<GridBox>& pending) {
  for (const std::string& o : owners)
    if (o != parent)
      throw ValidationError("splitter.consolidate",
                            "slice of '" + o + "' mixed into plan of '" + parent + "'");
  std::vector<detail::LinRange> ranges;
  for (const GridBox& b : pending) detail::box_ranges(b, grid, ranges);
  if (ranges.empty()) return {};
  std::stable_sort(ranges.begin(), ranges.end(),
                   [](const detail::LinRange& a, const detail::LinRange& b) { return a.lo < b.lo; });
  std::vector<GridBox> out;
  std::size_t i = 0;
  while (i < ranges.size()) {
    std::int64_t lo = ranges[i].lo, hi = ranges[i].hi;
    for (++i; i < ranges.size() && ranges[i].lo <= hi; ++i) hi = std::max(hi, ranges[i].hi);
    for (std::int64_t p = lo; p < hi;) {
      out.push_back(detail::next_box(p, grid, hi - p));
      p += out.back().blocks();
    }
  }
  return out;
}

std::vector<GridBox> consolidate(const std::string& parent, const Grid& grid,
                                 const std::vector<GridBox>& pending) {
  return consolidate(parent, grid, std::vector<std::string>(pending.size(), parent), pending);
}

// ------------------------------------------------------------------ arrivals
std::vector<Ns> generate_bursty_arrivals(double rate, double burstiness, Ns horizon,
                                         std::uint64_t seed, Ns dwell) {
  if (rate <= 0.0) throw ValidationError("tracegen.rate", "must be > 0");
  if (burstiness < 1.0) throw ValidationError("tracegen.burstiness", "must be >= 1");
  std::vector<Ns> out;
  if (horizon <= 0) return out;

  RngStream rng(hash_combine(seed, 0xb0b1));
  const auto exponential = [&rng](double mean) {
    double u = rng.next_double();
    if (u <= 0.0) u = 1e-18;
    return -std::log(u) * mean;
  };
  // Two states with equal mean dwell; their average rate equals `rate`.
  const double state_rate[2] = {2.0 * rate / (1.0 + burstiness),
                                2.0 * rate / (1.0 + burstiness) * burstiness};
  const double horizon_s = to_sec(horizon);
  const double dwell_s = to_sec(dwell);
  int state = 0;
  double now = 0.0;
  double switch_at = exponential(dwell_s);
  for (;;) {
    double r = state_rate[state];
    double next = now + exponential(1.0 / r);
    while (next > switch_at) {  // carry the unused exponential mass into the next state
      const double carried = (next - switch_at) * r;
      state ^= 1;
      now = switch_at;
      switch_at = now + exponential(dwell_s);
      r = state_rate[state];
      next = now + carried / r;
    }
    if (next >= horizon_s) break;
    now = next;
    Ns ts = seconds(now);
    if (!out.empty() && ts <= out.back()) ts = out.back() + 1;
    out.push_back(ts);
  }
  return out;
}

}  // namespace microslice
