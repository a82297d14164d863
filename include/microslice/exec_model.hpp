// Analytic GPU occupancy / execution-time model (Eq. 1 and the wave model).
// Reference: /root/reference/proj/include/microslice/exec_model.hpp:15-68.
// Used by the split search (find_optimal_split), by the replay device model and, in
// the live B200 path, as the prior before the on-device profile replaces it.
#pragma once

#include <cstdint>

#include "microslice/common.hpp"
#include "microslice/model.hpp"

namespace microslice {

enum class CapacityRounding { PerSmFloor, GlobalFloor };

/// Eq. 1: resident blocks across the GPU, n_sm * floor(o * smt / tpb) (per-SM floor)
/// or floor(n_sm * o * smt / tpb) (global floor).  Throws if no block fits.
std::int64_t concurrent_capacity(const GpuConfig& gpu, const KernelSpec& kernel,
                                 CapacityRounding rounding = CapacityRounding::PerSmFloor);

/// Wave model: ceil(n / cap) waves of the mean block time, stretched by the resident
/// wave's HBM demand (plus `concurrent_bw_load`) over the HBM bandwidth; llround.
Ns exec_time_model(const GpuConfig& gpu, const KernelSpec& kernel, std::int64_t n_blocks,
                   double concurrent_bw_load,
                   CapacityRounding rounding = CapacityRounding::PerSmFloor);

/// Stretch of one wave of `resident_blocks` given `other_bw_load` bytes/s elsewhere.
double bandwidth_stretch(const GpuConfig& gpu, const KernelSpec& kernel,
                         std::int64_t resident_blocks, double other_bw_load);

}  // namespace microslice
