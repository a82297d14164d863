// SLO bookkeeping and run reports.
// Reference: /root/reference/proj/include/microslice/metrics.hpp:21-260.
//  * percentile: nearest rank floor(q*N)+1 capped at N over the ascending samples
//  * SLO = p99 TTFT / p99 TPOT of the exclusive run (>= min_requests completed)
//  * attainment denominator counts incomplete requests
//  * LP throughput normalised by the exclusive-LP run
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "microslice/engine.hpp"
#include "microslice/json.hpp"

namespace microslice {

Ns percentile(std::vector<Ns> samples, double q);

struct SloThresholds {
  Ns ttft = 0;
  Ns tpot = 0;
};

struct DelaySummary {
  std::int64_t count = 0;
  Ns mean = 0;
  Ns p50 = 0;
  Ns p99 = 0;
  Ns max = 0;
};

DelaySummary summarize_delays(const std::vector<Ns>& delays);

struct RunReport {
  std::string scenario;
  std::string policy;
  std::uint64_t seed = 0;
  int requests_total = 0;
  int requests_completed = 0;
  Ns ttft_p99 = 0;
  Ns tpot_p99 = 0;
  double slo_attainment = 0.0;
  DelaySummary preemption;
  double lp_throughput = 0.0;
  double lp_throughput_normalized = 0.0;
  double waste_fraction = 0.0;
  double sync_overhead_fraction = 0.0;
  double sm_active_fraction = 0.0;
  double small_bubble_fraction = 0.0;
};

SloThresholds compute_slo(const RunArtifacts& exclusive, int min_requests = 100);
double slo_attainment(const std::vector<RequestStat>& requests, const SloThresholds& slo);
RunReport build_report(const RunArtifacts& art, const SloThresholds& slo,
                       double lp_reference_throughput = 0.0);

json report_to_json(const RunReport& r);
RunReport report_from_json(const json& j);
const char* report_csv_header();
std::string report_csv_row(const RunReport& r);
RunReport report_from_csv_row(const std::string& line);

}  // namespace microslice
