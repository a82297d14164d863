// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// C-ABI driver around the REFERENCE implementation itself: it #includes the unmodified
// reference headers from /root/reference/proj/include (read-only; nothing is copied) and
// exposes `msref_*` twins of the product's ms_replay.h entry points, so tests can
// compare the B200 framework's scheduler core against the reference CPU scheduler on
// identical inputs, and bench.py's `--impl reference` / cpu_baseline leg can time the
// reference's own Engine::run().  Built by oracle/Makefile into oracle/_ref/.
//
// Third-party dependency: nlohmann/json 3.11.3 (the reference's vendor/json.hpp,
// git-ignored upstream); the copy shipped inside this image's cudnn_frontend is used
// via -I at build time.  It is only used for scenario parsing / report I/O.
#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "microslice/engine.hpp"
#include "microslice/metrics.hpp"
#include "microslice/scenario_io.hpp"
#include "microslice/scheduler.hpp"
#include "microslice/splitter.hpp"
#include "microslice/tracegen.hpp"

using namespace microslice;
using nlohmann::json;

namespace {

void set_err(char* err, size_t len, const std::string& m) {
  if (err && len) std::snprintf(err, len, "%s", m.c_str());
}

template <typename F>
int guarded(char* err, size_t err_len, F&& f) {
  try {
    return f();
  } catch (const ValidationError& e) {
    set_err(err, err_len, e.what());
    return -2;
  } catch (const EngineError& e) {
    set_err(err, err_len, e.what());
    return -3;
  } catch (const std::exception& e) {
    set_err(err, err_len, e.what());
    return -1;
  }
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

struct Fnv {
  uint64_t h = 14695981039346656037ULL;
  void add(const char* s, size_t n) {
    for (size_t i = 0; i < n; ++i) h = (h ^ static_cast<unsigned char>(s[i])) * 1099511628211ULL;
  }
  void add(const std::string& s) { add(s.data(), s.size()); }
  void addf(const char* fmt, ...) __attribute__((format(printf, 2, 3))) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    int n = std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    add(buf, static_cast<size_t>(n));
  }
  std::string hex() const {
    char b[24];
    std::snprintf(b, sizeof b, "%016llx", static_cast<unsigned long long>(h));
    return b;
  }
};

std::string g17(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

json digest(const RunArtifacts& a, bool want_text, std::string* text_out) {
  json d;
  d["policy"] = policy_name(a.policy);
  d["scenario"] = a.scenario;
  d["seed"] = a.seed;
  d["horizon"] = a.horizon;
  const std::string nd = a.timeline.to_ndjson();
  Fnv ft;
  ft.add(nd);
  d["timeline"] = {{"n", a.timeline.size()}, {"fnv", ft.hex()}, {"bytes", nd.size()}};
  if (want_text && text_out) *text_out = nd;
  Fnv fa, fu, fr, fp;
  for (const auto& r : a.api_rows)
    fa.addf("%lld,%lld,%s,%lld\n", (long long)r.ts_start, (long long)r.ts_end, r.api_tag.c_str(),
            (long long)r.correlation);
  for (const auto& s : a.util_samples) fu.addf("%lld,%.17g,%.17g\n", (long long)s.ts, s.sm_active, s.hbm_bw);
  size_t completed = 0;
  for (const auto& r : a.requests) {
    completed += r.completed ? 1 : 0;
    fr.addf("%d,%zu,%lld,%lld,%lld,%d,%d\n", r.task, r.index, (long long)r.arrival, (long long)r.first_token,
            (long long)r.done, r.iterations, r.completed ? 1 : 0);
  }
  for (const auto& p : a.preemptions)
    fp.addf("%lld,%lld,%d,%d\n", (long long)p.begin, (long long)p.delay, p.lp_in_flight ? 1 : 0,
            p.consolidated ? 1 : 0);
  d["api_rows"] = {{"n", a.api_rows.size()}, {"fnv", fa.hex()}};
  d["util"] = {{"n", a.util_samples.size()}, {"fnv", fu.hex()}};
  d["requests"] = {{"n", a.requests.size()}, {"fnv", fr.hex()}, {"completed", completed}};
  d["preemptions"] = {{"n", a.preemptions.size()}, {"fnv", fp.hex()}};
  d["counters"] = {{"lp_blocks_launched", a.lp_blocks_launched},
                   {"lp_blocks_done", a.lp_blocks_done},
                   {"lp_waste_blocks", a.lp_waste_blocks},
                   {"lp_blocks_in_flight_at_cutoff", a.lp_blocks_in_flight_at_cutoff},
                   {"hp_blocks_launched", a.hp_blocks_launched},
                   {"hp_blocks_done", a.hp_blocks_done},
                   {"hp_blocks_in_flight_at_cutoff", a.hp_blocks_in_flight_at_cutoff},
                   {"lp_work_units", g17(a.lp_work_units)},
                   {"lp_parent_completions", a.lp_parent_completions},
                   {"relaunch_count", a.relaunch_count},
                   {"sync_cost_total", a.sync_cost_total},
                   {"sm_active_fraction", g17(a.sm_active_fraction)},
                   {"small_bubble_time", a.small_bubble_time},
                   {"hp_stretch_sum", g17(a.hp_stretch_sum)},
                   {"hp_stretch_waves", a.hp_stretch_waves}};
  return d;
}

ExecOracle measured_or_model(const GpuConfig& gpu, const KernelSpec& k, CapacityRounding r) {
  // Same rule as Engine::make_oracle (engine.hpp:461-488).
  if (k.measured_time.empty())
    return [gpu, k, r](int64_t n) { return exec_time_model(gpu, k, n, 0.0, r); };
  auto table = k.measured_time;
  std::sort(table.begin(), table.end());
  return [table](int64_t n) -> Ns {
    if (n <= table.front().first) return table.front().second;
    if (n >= table.back().first) return table.back().second;
    for (size_t i = 1; i < table.size(); ++i)
      if (n <= table[i].first) {
        double f = double(n - table[i - 1].first) / double(table[i].first - table[i - 1].first);
        return table[i - 1].second + Ns(f * double(table[i].second - table[i - 1].second));
      }
    return table.back().second;
  };
}

// The reference's fragment parsers live in microslice::detail of scenario_io.hpp; a
// minimal wrapper scenario lets the reference parse a lone gpu / kernel object.
ScenarioSpec wrap(const char* gpu_json, const char* kernel_json) {
  json root;
  root["gpu"] = json::parse(gpu_json);
  json k = kernel_json ? json::parse(kernel_json) : json();
  root["kernels"] = kernel_json ? json::array({k}) : json::array();
  root["tasks"] = json::array();
  return scenario_from_json(root);
}

}  // namespace

extern "C" {

uint64_t msref_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t msref_hash_combine(uint64_t a, uint64_t b) { return hash_combine(a, b); }
uint64_t msref_hash_str(const char* s, size_t n) { return hash_str(std::string(s, n)); }
double msref_u01_from_key(uint64_t k) { return u01_from_key(k); }

int msref_dist_sample_keyed(const char* dist_json, const uint64_t* keys, size_t n, int64_t* out, char* err,
                            size_t el) {
  return guarded(err, el, [&] {
    DurationDist d = detail::parse_duration_dist(json::parse(dist_json), "/dist");
    for (size_t i = 0; i < n; ++i) out[i] = d.sample_keyed(keys[i]);
    return 0;
  });
}

int msref_dist_sample(const char* dist_json, const double* u, size_t n, int64_t* out, char* err, size_t el) {
  return guarded(err, el, [&] {
    DurationDist d = detail::parse_duration_dist(json::parse(dist_json), "/dist");
    for (size_t i = 0; i < n; ++i) out[i] = d.sample(u[i]);
    return 0;
  });
}

int msref_dist_mean(const char* dist_json, int64_t* out, char* err, size_t el) {
  return guarded(err, el, [&] {
    *out = detail::parse_duration_dist(json::parse(dist_json), "/dist").mean();
    return 0;
  });
}

int msref_concurrent_capacity(const char* gpu_json, const char* kernel_json, int rounding, int64_t* out,
                              char* err, size_t el) {
  return guarded(err, el, [&] {
    ScenarioSpec s = wrap(gpu_json, kernel_json);
    *out = concurrent_capacity(s.gpu, s.kernels[0],
                               rounding ? CapacityRounding::GlobalFloor : CapacityRounding::PerSmFloor);
    return 0;
  });
}

int msref_exec_time_model(const char* gpu_json, const char* kernel_json, int64_t n, double load, int rounding,
                          int64_t* out, char* err, size_t el) {
  return guarded(err, el, [&] {
    ScenarioSpec s = wrap(gpu_json, kernel_json);
    *out = exec_time_model(s.gpu, s.kernels[0], n, load,
                           rounding ? CapacityRounding::GlobalFloor : CapacityRounding::PerSmFloor);
    return 0;
  });
}

// plan_out: [bps, predicted, cap, memory_bound, uncappable, n_slices]; slices as 6-int tuples
int msref_find_optimal_split(const char* gpu_json, const char* kernel_json, double eps, int64_t cap,
                             int square, int rounding, int64_t* plan_out, int32_t* slices, size_t slices_cap,
                             char* err, size_t el) {
  return guarded(err, el, [&] {
    ScenarioSpec s = wrap(gpu_json, kernel_json);
    SplitSearchOptions o;
    o.epsilon = eps;
    o.cap = cap;
    o.square_tiling = square != 0;
    o.rounding = rounding ? CapacityRounding::GlobalFloor : CapacityRounding::PerSmFloor;
    SplitPlan p = find_optimal_split(s.gpu, s.kernels[0], measured_or_model(s.gpu, s.kernels[0], o.rounding), o);
    plan_out[0] = p.blocks_per_slice;
    plan_out[1] = p.predicted_slice_time;
    plan_out[2] = p.cap;
    plan_out[3] = p.memory_bound;
    plan_out[4] = p.uncappable;
    plan_out[5] = (int64_t)p.slices.size();
    if (slices) {
      if (p.slices.size() > slices_cap) return -4;
      for (size_t i = 0; i < p.slices.size(); ++i) {
        const GridBox& b = p.slices[i];
        int32_t* o6 = slices + 6 * i;
        o6[0] = b.ox; o6[1] = b.oy; o6[2] = b.oz; o6[3] = b.sx; o6[4] = b.sy; o6[5] = b.sz;
      }
    }
    return 0;
  });
}

int msref_slice_boxes(int32_t gx, int32_t gy, int32_t gz, int64_t bps, int square, int32_t* out, size_t cap,
                      size_t* n_out) {
  try {
    auto v = slice_boxes(Grid{gx, gy, gz}, bps, square != 0);
    *n_out = v.size();
    if (v.size() > cap) return -4;
    for (size_t i = 0; i < v.size(); ++i) {
      int32_t* o = out + 6 * i;
      o[0] = v[i].ox; o[1] = v[i].oy; o[2] = v[i].oz; o[3] = v[i].sx; o[4] = v[i].sy; o[5] = v[i].sz;
    }
    return 0;
  } catch (const ValidationError&) {
    return -2;
  }
}

int msref_consolidate(int32_t gx, int32_t gy, int32_t gz, const int32_t* pend, size_t n, int32_t* out, size_t cap,
                      size_t* n_out) {
  std::vector<GridBox> in;
  for (size_t i = 0; i < n; ++i) {
    const int32_t* p = pend + 6 * i;
    in.push_back(GridBox{p[0], p[1], p[2], p[3], p[4], p[5]});
  }
  auto v = consolidate("k", Grid{gx, gy, gz}, in);
  *n_out = v.size();
  if (v.size() > cap) return -4;
  for (size_t i = 0; i < v.size(); ++i) {
    int32_t* o = out + 6 * i;
    o[0] = v[i].ox; o[1] = v[i].oy; o[2] = v[i].oz; o[3] = v[i].sx; o[4] = v[i].sy; o[5] = v[i].sz;
  }
  return 0;
}

int64_t msref_predict_interval(const int64_t* gaps, size_t n, double alpha, int32_t k, int64_t fallback) {
  return predict_interval(std::vector<Ns>(gaps, gaps + n), alpha, k, fallback);
}

int64_t msref_tick_interval(int64_t p, int64_t l) { return tick_interval(p, l); }

int msref_consolidation_prefix(const char* gpu_json, const char* kernel_json, const int64_t* box_blocks, size_t n,
                               int64_t interval, double safety, int64_t* out, char* err, size_t el) {
  return guarded(err, el, [&] {
    ScenarioSpec s = wrap(gpu_json, kernel_json);
    ExecOracle oracle = measured_or_model(s.gpu, s.kernels[0], CapacityRounding::PerSmFloor);
    *out = consolidation_prefix((int64_t)n, interval, safety, [&](int64_t cnt) {
      int64_t blocks = 0;
      for (int64_t i = 0; i < cnt; ++i) blocks += box_blocks[i];
      return oracle(blocks);
    });
    return 0;
  });
}

int64_t msref_percentile(const int64_t* s, size_t n, double q) { return percentile(std::vector<Ns>(s, s + n), q); }

int msref_generate_bursty_arrivals(double rate, double b, int64_t horizon, uint64_t seed, int64_t dwell,
                                   int64_t* out, size_t cap, size_t* n_out, char* err, size_t el) {
  return guarded(err, el, [&] {
    auto v = generate_bursty_arrivals(rate, b, horizon, seed, dwell);
    *n_out = v.size();
    if (v.size() > cap) return -4;
    std::copy(v.begin(), v.end(), out);
    return 0;
  });
}

// Engine(ScenarioSpec, Policy).run() on the reference; same digest schema as ms_replay_run.
int msref_replay_run_opts(const char* scenario_json, const char* policy, const char* options_json, int flags,
                          char** out_json, char* err, size_t el) {
  return guarded(err, el, [&] {
    ScenarioSpec sc = scenario_from_json(json::parse(scenario_json));
    auto pol = parse_policy(policy);
    if (!pol) throw ValidationError("policy", "unknown policy");
    EngineOptions eo;
    if (options_json && *options_json) {
      json o = json::parse(options_json);
      if (o.contains("hint_filter")) {
        eo.hint_filter.emplace();
        for (const auto& k : o.at("hint_filter")) eo.hint_filter->insert(k.get<std::string>());
      }
      if (o.value("global_floor", false)) eo.rounding = CapacityRounding::GlobalFloor;
      eo.util_sample_period = o.value("util_sample_period_ns", (long long)eo.util_sample_period);
    }
    auto t0 = std::chrono::steady_clock::now();
    RunArtifacts art = run_scenario(sc, *pol, eo);
    double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::string text;
    json d = digest(art, (flags & 1) != 0, &text);
    d["wall_s"] = wall;
    if (flags & 1) d["ndjson"] = text;
    if (flags & 4) {
      json delays = json::array();
      for (const auto& p : art.preemptions) delays.push_back(p.delay);
      d["delays"] = delays;
    }
    if (flags & 2) {
      RunArtifacts ex = run_scenario(sc, Policy::Exclusive, eo);
      RunArtifacts exlp = run_scenario(sc, Policy::ExclusiveLp, eo);
      d["report"] = report_to_json(build_report(art, compute_slo(ex), exlp.lp_throughput_per_s()));
    }
    *out_json = dup(d.dump());
    return 0;
  });
}

int msref_replay_run(const char* scenario_json, const char* policy, int flags, char** out_json, char* err,
                     size_t el) {
  return msref_replay_run_opts(scenario_json, policy, nullptr, flags, out_json, err, el);
}

// CPU baseline: `n_threads` independent Engine::run() of the scenario under `policy`
// concurrently (one per host core).  Returns wall seconds and
// total timeline events through out[0..1].
int msref_parallel_runs(const char* scenario_json, const char* policy, int n_threads, double* out, char* err,
                        size_t el) {
  return guarded(err, el, [&] {
    ScenarioSpec sc = scenario_from_json(json::parse(scenario_json));
    auto pol = parse_policy(policy);
    if (!pol) throw ValidationError("policy", "unknown policy");
    std::vector<size_t> events(static_cast<size_t>(n_threads), 0);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int i = 0; i < n_threads; ++i)
      th.emplace_back([&, i] {
        ScenarioSpec s = sc;
        s.seed = sc.seed + static_cast<uint64_t>(i);
        RunArtifacts a = run_scenario(s, *pol);
        events[static_cast<size_t>(i)] = a.timeline.size();
      });
    for (auto& t : th) t.join();
    out[0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    double tot = 0;
    for (size_t e : events) tot += static_cast<double>(e);
    out[1] = tot;
    return 0;
  });
}

void msref_free(void* p) { std::free(p); }

}  // extern "C"
