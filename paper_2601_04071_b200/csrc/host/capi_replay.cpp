// C-ABI over the scheduler core (include/ms_replay.h).
#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>

#include "microslice/engine.hpp"
#include "microslice/metrics.hpp"
#include "microslice/scenario_io.hpp"
#include "microslice/tracegen.hpp"
#include "ms_replay.h"

using namespace microslice;

namespace {

void set_err(char* err, std::size_t len, const std::string& msg) {
  if (!err || len == 0) return;
  std::snprintf(err, len, "%s", msg.c_str());
}

template <typename F>
int guarded(char* err, std::size_t err_len, F&& f) {
  try {
    return f();
  } catch (const ValidationError& e) {
    set_err(err, err_len, e.what());
    return MS_E_VALIDATION;
  } catch (const EngineError& e) {
    set_err(err, err_len, e.what());
    return MS_E_ENGINE;
  } catch (const std::exception& e) {
    set_err(err, err_len, e.what());
    return MS_E_ARG;
  }
}

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

json parse_or_throw(const char* text) {
  if (!text) throw ValidationError("json", "null input");
  return json::parse(text);
}

// FNV-1a 64 accumulator over formatted rows.
struct Fnv {
  std::uint64_t h = 14695981039346656037ULL;
  void add(const char* s, std::size_t n) {
    for (std::size_t i = 0; i < n; ++i) h = (h ^ static_cast<unsigned char>(s[i])) * 1099511628211ULL;
  }
  void addf(const char* fmt, ...) __attribute__((format(printf, 2, 3))) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    const int n = std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    add(buf, static_cast<std::size_t>(n));
  }
  std::string hex() const {
    char buf[24];
    std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(h));
    return buf;
  }
};

json hashed(std::size_t n, const Fnv& f) {
  json j = json::object();
  j["n"] = json(static_cast<unsigned long long>(n));
  j["fnv"] = json(f.hex());
  return j;
}

std::string g17(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

// Digest of every field of RunArtifacts; the oracle driver renders the same schema.
json digest(const RunArtifacts& a) {
  json d = json::object();
  d["policy"] = json(policy_name(a.policy));
  d["scenario"] = json(a.scenario);
  d["seed"] = json(static_cast<unsigned long long>(a.seed));
  d["horizon"] = json(static_cast<long long>(a.horizon));
  json tl = json::object();
  tl["n"] = json(static_cast<unsigned long long>(a.timeline.size()));
  char hx[24];
  std::snprintf(hx, sizeof hx, "%016llx", static_cast<unsigned long long>(a.timeline.ndjson_fnv1a()));
  tl["fnv"] = json(std::string(hx));
  tl["bytes"] = json(static_cast<unsigned long long>(a.timeline.ndjson_bytes()));
  d["timeline"] = std::move(tl);

  Fnv fa, fu, fr, fp;
  for (const ApiTraceRow& r : a.api_rows)
    fa.addf("%lld,%lld,%s,%lld\n", static_cast<long long>(r.ts_start), static_cast<long long>(r.ts_end),
            r.api_tag.c_str(), static_cast<long long>(r.correlation));
  for (const UtilSample& s : a.util_samples)
    fu.addf("%lld,%.17g,%.17g\n", static_cast<long long>(s.ts), s.sm_active, s.hbm_bw);
  std::size_t completed = 0;
  for (const RequestStat& r : a.requests) {
    completed += r.completed ? 1 : 0;
    fr.addf("%d,%zu,%lld,%lld,%lld,%d,%d\n", r.task, r.index, static_cast<long long>(r.arrival),
            static_cast<long long>(r.first_token), static_cast<long long>(r.done), r.iterations,
            r.completed ? 1 : 0);
  }
  for (const PreemptionRecord& p : a.preemptions)
    fp.addf("%lld,%lld,%d,%d\n", static_cast<long long>(p.begin), static_cast<long long>(p.delay),
            p.lp_in_flight ? 1 : 0, p.consolidated ? 1 : 0);
  d["api_rows"] = hashed(a.api_rows.size(), fa);
  d["util"] = hashed(a.util_samples.size(), fu);
  d["requests"] = hashed(a.requests.size(), fr);
  d["requests"]["completed"] = json(static_cast<unsigned long long>(completed));
  d["preemptions"] = hashed(a.preemptions.size(), fp);

  json c = json::object();
  c["lp_blocks_launched"] = json(static_cast<long long>(a.lp_blocks_launched));
  c["lp_blocks_done"] = json(static_cast<long long>(a.lp_blocks_done));
  c["lp_waste_blocks"] = json(static_cast<long long>(a.lp_waste_blocks));
  c["lp_blocks_in_flight_at_cutoff"] = json(static_cast<long long>(a.lp_blocks_in_flight_at_cutoff));
  c["hp_blocks_launched"] = json(static_cast<long long>(a.hp_blocks_launched));
  c["hp_blocks_done"] = json(static_cast<long long>(a.hp_blocks_done));
  c["hp_blocks_in_flight_at_cutoff"] = json(static_cast<long long>(a.hp_blocks_in_flight_at_cutoff));
  c["lp_work_units"] = json(g17(a.lp_work_units));
  c["lp_parent_completions"] = json(static_cast<long long>(a.lp_parent_completions));
  c["relaunch_count"] = json(static_cast<long long>(a.relaunch_count));
  c["sync_cost_total"] = json(static_cast<long long>(a.sync_cost_total));
  c["sm_active_fraction"] = json(g17(a.sm_active_fraction));
  c["small_bubble_time"] = json(static_cast<long long>(a.small_bubble_time));
  c["hp_stretch_sum"] = json(g17(a.hp_stretch_sum));
  c["hp_stretch_waves"] = json(static_cast<long long>(a.hp_stretch_waves));
  d["counters"] = std::move(c);
  return d;
}

DurationDist dist_from_text(const char* text) { return duration_dist_from_json(parse_or_throw(text)); }

CapacityRounding rounding_of(int r) {
  return r ? CapacityRounding::GlobalFloor : CapacityRounding::PerSmFloor;
}

ms_box to_c(const GridBox& b) { return ms_box{b.ox, b.oy, b.oz, b.sx, b.sy, b.sz}; }
GridBox from_c(const ms_box& b) { return GridBox{b.ox, b.oy, b.oz, b.sx, b.sy, b.sz}; }

int emit_boxes(const std::vector<GridBox>& boxes, ms_box* out, std::size_t cap, std::size_t* n_out) {
  if (n_out) *n_out = boxes.size();
  if (boxes.size() > cap || (!out && !boxes.empty())) return MS_E_CAPACITY;
  for (std::size_t i = 0; i < boxes.size(); ++i) out[i] = to_c(boxes[i]);
  return MS_OK;
}

// Oracle from a kernel spec: measured table if present, else the wave model
// (same rule as the engine's plan oracle, engine.hpp:461-488).
ExecOracle kernel_oracle(const GpuConfig& gpu, const KernelSpec& k, CapacityRounding rounding) {
  if (k.measured_time.empty())
    return [gpu, k, rounding](std::int64_t n) { return exec_time_model(gpu, k, n, 0.0, rounding); };
  auto rows = k.measured_time;
  std::sort(rows.begin(), rows.end());
  return [rows](std::int64_t n) -> Ns {
    if (n <= rows.front().first) return rows.front().second;
    if (n >= rows.back().first) return rows.back().second;
    std::size_t i = 1;
    while (i < rows.size() && n > rows[i].first) ++i;
    const double f = static_cast<double>(n - rows[i - 1].first) /
                     static_cast<double>(rows[i].first - rows[i - 1].first);
    return rows[i - 1].second + static_cast<Ns>(f * static_cast<double>(rows[i].second - rows[i - 1].second));
  };
}

}  // namespace

extern "C" {

uint64_t ms_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t ms_hash_combine(uint64_t a, uint64_t b) { return hash_combine(a, b); }
uint64_t ms_hash_str(const char* s, size_t n) { return hash_str(std::string(s ? s : "", s ? n : 0)); }
double ms_u01_from_key(uint64_t key) { return u01_from_key(key); }

int ms_dist_sample(const char* dist_json, const double* u, size_t n, int64_t* out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    const DurationDist d = dist_from_text(dist_json);
    for (size_t i = 0; i < n; ++i) out[i] = d.sample(u[i]);
    return MS_OK;
  });
}

int ms_dist_sample_keyed(const char* dist_json, const uint64_t* keys, size_t n, int64_t* out, char* err,
                         size_t err_len) {
  return guarded(err, err_len, [&] {
    const DurationDist d = dist_from_text(dist_json);
    for (size_t i = 0; i < n; ++i) out[i] = d.sample_keyed(keys[i]);
    return MS_OK;
  });
}

int ms_dist_mean(const char* dist_json, int64_t* out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    *out = dist_from_text(dist_json).mean();
    return MS_OK;
  });
}

int ms_concurrent_capacity(const char* gpu_json, const char* kernel_json, int rounding, int64_t* out, char* err,
                           size_t err_len) {
  return guarded(err, err_len, [&] {
    const GpuConfig gpu = gpu_from_json(parse_or_throw(gpu_json));
    const KernelSpec k = kernel_from_json(parse_or_throw(kernel_json));
    *out = concurrent_capacity(gpu, k, rounding_of(rounding));
    return MS_OK;
  });
}

int ms_exec_time_model(const char* gpu_json, const char* kernel_json, int64_t n_blocks, double load, int rounding,
                       int64_t* out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    const GpuConfig gpu = gpu_from_json(parse_or_throw(gpu_json));
    const KernelSpec k = kernel_from_json(parse_or_throw(kernel_json));
    *out = exec_time_model(gpu, k, n_blocks, load, rounding_of(rounding));
    return MS_OK;
  });
}

int ms_find_optimal_split(const char* gpu_json, const char* kernel_json, double epsilon, int64_t cap_ns,
                          int square_tiling, int rounding, ms_split_plan* plan, ms_box* slices, size_t slices_cap,
                          char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    const GpuConfig gpu = gpu_from_json(parse_or_throw(gpu_json));
    const KernelSpec k = kernel_from_json(parse_or_throw(kernel_json));
    SplitSearchOptions o;
    o.epsilon = epsilon;
    o.cap = cap_ns;
    o.square_tiling = square_tiling != 0;
    o.rounding = rounding_of(rounding);
    const SplitPlan p = find_optimal_split(gpu, k, kernel_oracle(gpu, k, o.rounding), o);
    plan->blocks_per_slice = p.blocks_per_slice;
    plan->predicted_slice_time_ns = p.predicted_slice_time;
    plan->cap_ns = p.cap;
    plan->memory_bound = p.memory_bound;
    plan->uncappable = p.uncappable;
    plan->n_slices = static_cast<int64_t>(p.slices.size());
    if (slices) return emit_boxes(p.slices, slices, slices_cap, nullptr);
    return MS_OK;
  });
}

int ms_slice_boxes(int32_t gx, int32_t gy, int32_t gz, int64_t blocks_per_slice, int square_tiling, ms_box* out,
                   size_t cap, size_t* n_out) {
  try {
    return emit_boxes(slice_boxes(Grid{gx, gy, gz}, blocks_per_slice, square_tiling != 0), out, cap, n_out);
  } catch (const ValidationError&) {
    return MS_E_VALIDATION;
  }
}

int ms_consolidate(int32_t gx, int32_t gy, int32_t gz, const ms_box* pending, size_t n_pending, ms_box* out,
                   size_t cap, size_t* n_out) {
  std::vector<GridBox> in;
  for (size_t i = 0; i < n_pending; ++i) in.push_back(from_c(pending[i]));
  return emit_boxes(consolidate("k", Grid{gx, gy, gz}, in), out, cap, n_out);
}

int64_t ms_predict_interval(const int64_t* gaps, size_t n, double alpha, int32_t k, int64_t fallback) {
  return predict_interval(std::vector<Ns>(gaps, gaps + n), alpha, k, fallback);
}

int64_t ms_tick_interval(int64_t predicted, int64_t launch) { return tick_interval(predicted, launch); }

int ms_consolidation_prefix(const char* gpu_json, const char* kernel_json, const int64_t* box_blocks, size_t n,
                            int64_t predicted_interval, double safety_factor, int64_t* out, char* err,
                            size_t err_len) {
  return guarded(err, err_len, [&] {
    const GpuConfig gpu = gpu_from_json(parse_or_throw(gpu_json));
    const KernelSpec k = kernel_from_json(parse_or_throw(kernel_json));
    const ExecOracle oracle = kernel_oracle(gpu, k, CapacityRounding::PerSmFloor);
    *out = consolidation_prefix(static_cast<std::int64_t>(n), predicted_interval, safety_factor,
                                [&](std::int64_t cnt) {
                                  std::int64_t blocks = 0;
                                  for (std::int64_t i = 0; i < cnt; ++i) blocks += box_blocks[i];
                                  return oracle(blocks);
                                });
    return MS_OK;
  });
}

int64_t ms_percentile(const int64_t* samples, size_t n, double q) {
  return percentile(std::vector<Ns>(samples, samples + n), q);
}

int ms_generate_bursty_arrivals(double rate, double burstiness, int64_t horizon_ns, uint64_t seed, int64_t dwell_ns,
                                int64_t* out, size_t cap, size_t* n_out, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    const std::vector<Ns> a = generate_bursty_arrivals(rate, burstiness, horizon_ns, seed, dwell_ns);
    if (n_out) *n_out = a.size();
    if (a.size() > cap) return MS_E_CAPACITY;
    std::copy(a.begin(), a.end(), out);
    return MS_OK;
  });
}

int ms_replay_run(const char* scenario_json, const char* policy, int flags, char** out_json, char* err,
                  size_t err_len) {
  return ms_replay_run_opts(scenario_json, policy, nullptr, flags, out_json, err, err_len);
}

int ms_replay_run_opts(const char* scenario_json, const char* policy, const char* options_json, int flags,
                       char** out_json, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    const ScenarioSpec sc = scenario_from_json(parse_or_throw(scenario_json));
    const auto pol = parse_policy(policy ? policy : "");
    if (!pol) throw ValidationError("policy", std::string("unknown policy '") + (policy ? policy : "") + "'");
    EngineOptions eo;
    if (options_json && *options_json) {
      const json o = json::parse(options_json);
      if (o.contains("hint_filter")) {
        eo.hint_filter.emplace();
        for (const json& k : o.at("hint_filter")) eo.hint_filter->insert(k.get<std::string>());
      }
      if (o.value("global_floor", false)) eo.rounding = CapacityRounding::GlobalFloor;
      eo.util_sample_period = o.value("util_sample_period_ns", static_cast<long long>(eo.util_sample_period));
    }
    const auto t0 = std::chrono::steady_clock::now();
    Engine eng(sc, *pol, eo);
    RunArtifacts art = eng.run();
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    json d = digest(art);
    d["des_events"] = json(static_cast<unsigned long long>(eng.events_processed()));
    d["wall_s"] = json(wall);
    if (flags & MS_RUN_NDJSON) d["ndjson"] = json(art.timeline.to_ndjson());
    if (flags & MS_RUN_DELAYS) {
      json delays = json::array();
      for (const PreemptionRecord& p : art.preemptions) delays.push_back(json(static_cast<long long>(p.delay)));
      d["delays"] = std::move(delays);
    }
    if (flags & MS_RUN_ROWS) {
      json rows = json::array();
      for (const RequestStat& r : art.requests) {
        json e = json::array();
        e.push_back(json(static_cast<long long>(r.arrival)));
        e.push_back(json(static_cast<long long>(r.ttft())));
        e.push_back(json(static_cast<long long>(r.tpot())));
        e.push_back(json(r.iterations));
        e.push_back(json(r.completed));
        rows.push_back(std::move(e));
      }
      d["request_rows"] = std::move(rows);
    }
    if (flags & MS_RUN_REPORT) {
      const RunArtifacts ex = run_scenario(sc, Policy::Exclusive, eo);
      const RunArtifacts exlp = run_scenario(sc, Policy::ExclusiveLp, eo);
      const SloThresholds slo = compute_slo(ex);
      d["report"] = report_to_json(build_report(art, slo, exlp.lp_throughput_per_s()));
    }
    *out_json = dup_string(d.dump());
    return MS_OK;
  });
}

int ms_scenario_normalize(const char* scenario_json, char** out_json, char* err, size_t err_len) {
  return guarded(err, err_len, [&] {
    *out_json = dup_string(scenario_to_json(scenario_from_json(parse_or_throw(scenario_json))).dump());
    return MS_OK;
  });
}

void ms_free(void* p) { std::free(p); }

}  // extern "C"
