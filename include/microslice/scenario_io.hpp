// Scenario JSON and arrival-trace CSV wire formats.
// Reference: /root/reference/proj/include/microslice/scenario_io.hpp:108-465.
// Parsing rules that matter for replay parity are kept: durations are
// {"value": v, "unit": "ns|us|ms"} and TRUNCATE; threshold_ms / slice_cap_us /
// evict_cost_us truncate; a `bursty` trace is generated with seed
// hash_combine(scenario seed, hash_str(trace name)) over the scenario horizon.
#pragma once

#include <cstdint>
#include <istream>
#include <ostream>
#include <string>
#include <vector>

#include "microslice/json.hpp"
#include "microslice/model.hpp"

namespace microslice {

/// Fragment parsers of the scenario schema ("gpu" object, one "kernels[]" entry, a
/// {"dist": ...} duration distribution).
GpuConfig gpu_from_json(const json& g, const std::string& path = "/gpu");
KernelSpec kernel_from_json(const json& k, const std::string& path = "/kernels/0");
DurationDist duration_dist_from_json(const json& j, const std::string& path = "/dist");

std::vector<Ns> load_arrivals_csv(std::istream& is, const std::string& path = "csv");
void save_arrivals_csv(std::ostream& os, const std::vector<Ns>& arrivals);

ScenarioSpec scenario_from_json(const json& root, std::uint64_t* seed_override = nullptr);
ScenarioSpec load_scenario(const std::string& path, std::uint64_t* seed_override = nullptr);
json scenario_to_json(const ScenarioSpec& s);
void save_scenario(const ScenarioSpec& s, std::ostream& os);

}  // namespace microslice
