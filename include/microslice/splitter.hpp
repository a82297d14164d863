// Kernel splitting: slice geometry, the two-step optimal-split search, and
// consolidation of pending slices.
// Reference: /root/reference/proj/include/microslice/splitter.hpp:15-286.
//
// On B200 a "slice" of an LP kernel is a contiguous range of linear tile ids of a
// persistent preemptible kernel (csrc/cuda/lp_*.cuh): the row-major box
// decomposition here is exactly the [begin, end) tile-range the device loop runs,
// so the same geometry drives replay and the live path.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "microslice/common.hpp"
#include "microslice/exec_model.hpp"
#include "microslice/model.hpp"

namespace microslice {

/// Rectangular sub-grid (offset + size) whose linear block range is contiguous.
struct GridBox {
  int ox = 0, oy = 0, oz = 0;
  int sx = 1, sy = 1, sz = 1;

  std::int64_t blocks() const { return static_cast<std::int64_t>(sx) * sy * sz; }
  bool operator==(const GridBox& o) const {
    return ox == o.ox && oy == o.oy && oz == o.oz && sx == o.sx && sy == o.sy &&
           sz == o.sz;
  }
};

/// The "splitting log" of one kernel (splitter.hpp:29-37).
struct SplitPlan {
  std::string kernel;
  std::int64_t blocks_per_slice = 1;
  std::vector<GridBox> slices;
  Ns predicted_slice_time = 0;
  Ns cap = us(400);
  bool memory_bound = false;
  bool uncappable = false;
};

namespace detail {
/// Linear block index -> (x, y, z), row-major with x fastest.
void linear_to_coord(std::int64_t p, const Grid& g, int& x, int& y, int& z);
/// Largest row-major-contiguous box starting at linear index p within `budget` blocks.
GridBox next_box(std::int64_t p, const Grid& g, std::int64_t budget);

struct LinRange {
  std::int64_t lo = 0, hi = 0;  // [lo, hi)
};
void box_ranges(const GridBox& b, const Grid& g, std::vector<LinRange>& out);
}  // namespace detail

std::vector<GridBox> slice_boxes(const Grid& grid, std::int64_t blocks_per_slice,
                                 bool square_tiling = false);
std::vector<GridBox> slice_schedule(const KernelSpec& kernel, const SplitPlan& plan,
                                    bool square_tiling = false);

using ExecOracle = std::function<Ns(std::int64_t n_blocks)>;

struct SplitSearchOptions {
  double epsilon = 0.02;
  Ns cap = us(400);
  bool square_tiling = false;
  CapacityRounding rounding = CapacityRounding::PerSmFloor;
};

/// Two-step search (splitter.hpp:141-207): start at Eq. 1 capacity, halve while the
/// oracle improves by > epsilon, refine up to the largest count within (1+eps) of the
/// best seen, then enforce the cap by binary search (or flag `uncappable`).
SplitPlan find_optimal_split(const GpuConfig& gpu, const KernelSpec& kernel,
                             const ExecOracle& oracle, const SplitSearchOptions& opts = {});
/// Same with the analytic wave model (no concurrent load) as the oracle.
SplitPlan find_optimal_split(const GpuConfig& gpu, const KernelSpec& kernel,
                             const SplitSearchOptions& opts = {});

/// Union of pending slices of one parent -> merged linear ranges -> fewest boxes.
std::vector<GridBox> consolidate(const std::string& parent, const Grid& grid,
                                 const std::vector<std::string>& owners,
                                 const std::vector<GridBox>& pending);
std::vector<GridBox> consolidate(const std::string& parent, const Grid& grid,
                                 const std::vector<GridBox>& pending);

}  // namespace microslice
