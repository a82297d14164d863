// TEST INFRASTRUCTURE ONLY: a virtual-time CPU model of the device C-ABI (include/ms_b200.h)
// that the live scheduler (csrc/live/live.cpp, compiled unchanged) links against, so its
// admit / preempt / resume decisions can be checked against the replay core on the CPU
// (tests/test_live_decisions.py).
//
// Time: a virtual clock that advances by `quantum_ns` on every ms_host_now_ns() call (the
// scheduler's polling loop is what moves time), so a live run is deterministic.
// HP chain: ring at t -> first CTA at t + first_delay, done first + duration (per chain).
// LP run: starts launch_ns after ms_lp_run; W = (SMs - reserve) tiles per wave of tile_ns;
// claims go redo-list first, then fresh tiles below the (movable) budget; a preempt raised
// at t_r ends the run at max(start, t_r) + drain_ns, abandoning the in-flight wave's tiles to
// the redo list (what tile_run.cuh does); otherwise it exits when the budget is exhausted.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "ms_b200.h"

#define MS_MAX_LP_MOCK 128

struct MockRun {
  bool active = false, nonpre = false;
  uint64_t begin = 0, end = 0, budget = 0, redo_in = 0;
  int64_t start = 0, raise = -1;
  uint32_t epoch = 0;
  uint64_t run_id = 0;
};

struct MockLp {
  bool used = false;
  uint64_t total = 0;
  int64_t tile_ns = 10000;
  uint64_t redo_carry = 0;
  MockRun run;
  bool exited = false;
  ms_lp_status last{};
};

struct MockChain {
  int64_t duration = 100000, first_delay = 3000;
  std::vector<std::pair<int64_t, int64_t>> timing;  // per ring, in order: (first_delay, duration)
  std::size_t next = 0;
  uint32_t seq = 0;
  int64_t first = -1, done = -1;
};

struct ms_dev {
  int n_sm = 148, reserve = 1;
  uint32_t epoch = 0, seq = 0;
  MockLp lp[MS_MAX_LP_MOCK];
  std::map<int, MockChain> chains;
  std::map<uint32_t, int> armed;  // seq -> chain
  int64_t launch_ns = 5000, drain_ns = 4000;
};

namespace {
int64_t g_now = 1'000'000'000;
int64_t g_quantum = 100;
ms_dev g_dev;
std::string g_err;

uint64_t waves_done(const MockLp& l, int64_t t) {
  const MockRun& r = l.run;
  if (t <= r.start) return 0;
  return static_cast<uint64_t>((t - r.start) / l.tile_ns);
}

uint64_t claimable(const MockLp& l) {
  const MockRun& r = l.run;
  return r.redo_in + (r.budget > r.begin ? r.budget - r.begin : 0);
}

// exit time of the active run given what is known now (budget, raise)
int64_t exit_time(const ms_dev& d, const MockLp& l) {
  const MockRun& r = l.run;
  const uint64_t W = static_cast<uint64_t>(std::max(1, d.n_sm - d.reserve));
  const uint64_t need = claimable(l);
  const int64_t nat = r.start + static_cast<int64_t>((need + W - 1) / W) * l.tile_ns;
  if (r.raise >= 0 && !r.nonpre) {
    const int64_t te = std::max(r.start, r.raise) + d.drain_ns;
    if (te < nat) return te;
  }
  return std::max(nat, r.start + 1);
}

void finish(ms_dev& d, MockLp& l, int64_t t_exit) {
  MockRun& r = l.run;
  const uint64_t W = static_cast<uint64_t>(std::max(1, d.n_sm - d.reserve));
  const uint64_t need = claimable(l);
  const bool pre = r.raise >= 0 && !r.nonpre && t_exit < r.start + static_cast<int64_t>((need + W - 1) / W) * l.tile_ns;
  const uint64_t wd = waves_done(l, t_exit);
  const uint64_t done = std::min(need, wd * W);
  const uint64_t claimed = pre ? std::min(need, (wd + 1) * W) : done;
  const uint64_t fresh = claimed > r.redo_in ? claimed - r.redo_in : 0;
  const uint64_t redo_left = r.redo_in > claimed ? r.redo_in - claimed : 0;
  ms_lp_status& s = l.last;
  std::memset(&s, 0, sizeof s);
  s.run_id = r.run_id;
  s.begin = r.begin;
  s.end = r.end;
  s.redo_in = r.redo_in;
  s.cursor = r.begin + fresh;
  s.redo_count = (claimed - done) + redo_left;
  s.tiles_done = done;
  s.preempted = pre ? 1 : 0;
  s.done = 1;
  s.t_start = static_cast<uint64_t>(r.start);
  s.t_seen = pre ? static_cast<uint64_t>(std::max(r.start, r.raise)) : 0;
  s.t_exit = static_cast<uint64_t>(t_exit);
  s.t_free = static_cast<uint64_t>(t_exit);
  l.redo_carry = s.redo_count;
  l.exited = true;
  r.active = false;
}
}  // namespace

extern "C" {

// ---- mock control --------------------------------------------------------------------
void ms_mock_reset(int n_sm, int64_t quantum_ns, int64_t launch_ns, int64_t drain_ns) {
  g_dev = ms_dev{};
  g_dev.n_sm = n_sm;
  g_dev.launch_ns = launch_ns;
  g_dev.drain_ns = drain_ns;
  g_quantum = quantum_ns;
  g_now = 1'000'000'000;
}
int ms_mock_add_lp(uint64_t total_tiles, int64_t tile_ns) {
  for (int i = 0; i < MS_MAX_LP_MOCK; ++i)
    if (!g_dev.lp[i].used) {
      g_dev.lp[i] = MockLp{};
      g_dev.lp[i].used = true;
      g_dev.lp[i].total = total_tiles;
      g_dev.lp[i].tile_ns = tile_ns;
      return i;
    }
  return -1;
}
void ms_mock_set_chain(int cid, int64_t duration_ns, int64_t first_delay_ns) {
  g_dev.chains[cid].duration = duration_ns;
  g_dev.chains[cid].first_delay = first_delay_ns;
}
// Per-ring device timing (e.g. the replay's own modelled HP segments); rings past the end
// of the list fall back to the chain's default.
void ms_mock_push_chain_timing(int cid, int64_t first_delay_ns, int64_t duration_ns) {
  g_dev.chains[cid].timing.emplace_back(first_delay_ns, duration_ns);
}
int64_t ms_mock_now(void) { return g_now; }

// ---- the device C-ABI used by the live runtime -----------------------------------------
int ms_dev_open(int, ms_dev** dev) {
  *dev = &g_dev;
  return 0;
}
int ms_dev_close(ms_dev*) { return 0; }
int ms_dev_get_info(ms_dev* d, ms_dev_info* info) {
  std::memset(info, 0, sizeof *info);
  info->sm_count = d->n_sm;
  info->cc_major = 10;
  std::snprintf(info->name, sizeof info->name, "virtual-time mock");
  return 0;
}
int ms_dev_sync(ms_dev*) { return 0; }
const char* ms_last_error(void) { return g_err.c_str(); }
int64_t ms_host_now_ns(void) { return g_now += g_quantum; }

int ms_set_lp_sm_reserve(ms_dev* d, int n) {
  d->reserve = n;
  return 0;
}
int ms_debug_stamps(ms_dev*, int, unsigned long long*, size_t) { return 0; }
uint64_t ms_lp_total_tiles(ms_dev* d, int id) { return d->lp[id].used ? d->lp[id].total : 0; }
int ms_lp_tile_ctas(ms_dev*, int) { return 1; }
int ms_trace_enable(ms_dev*, size_t) { return 0; }  // (the virtual device logs no device events)
int ms_trace_drain(ms_dev*, ms_event*, size_t, uint64_t* lost) {
  if (lost) *lost = 0;
  return 0;
}
int ms_lp_reset(ms_dev* d, int id) {
  d->lp[id].redo_carry = 0;
  d->lp[id].exited = false;
  return 0;
}
int ms_lp_run_ex(ms_dev* d, int id, uint64_t begin, uint64_t end, uint64_t budget, int flags) {
  MockLp& l = d->lp[id];
  if (!l.used || l.run.active) {
    g_err = "mock: bad LP id or run in flight";
    return MS_E_ARG;
  }
  MockRun& r = l.run;
  r = MockRun{};
  r.active = true;
  r.nonpre = flags & MS_RUN_NONPREEMPTIBLE;
  r.begin = begin;
  r.end = end;
  r.budget = std::min(budget, end);
  r.redo_in = l.redo_carry;
  r.start = g_now + d->launch_ns;
  r.epoch = d->epoch;
  r.run_id = l.last.run_id + 1;
  l.exited = false;
  return 0;
}
int ms_lp_set_budget(ms_dev* d, int id, uint64_t budget) {
  MockLp& l = d->lp[id];
  if (l.run.active) l.run.budget = std::max(std::min(budget, l.run.end), l.run.begin);
  return 0;
}
uint64_t ms_lp_progress(ms_dev* d, int id) {
  const MockLp& l = d->lp[id];
  if (!l.run.active) return 0;
  const uint64_t W = static_cast<uint64_t>(std::max(1, d->n_sm - d->reserve));
  return std::min(claimable(l), (waves_done(l, g_now) + 1) * W);
}
int ms_lp_poll(ms_dev* d, int id, ms_lp_status* st) {
  MockLp& l = d->lp[id];
  if (l.run.active) {
    const int64_t te = exit_time(*d, l);
    if (g_now >= te) finish(*d, l, te);
  }
  if (l.exited) {
    *st = l.last;
    return 1;
  }
  std::memset(st, 0, sizeof *st);
  return 0;
}
int ms_lp_wait(ms_dev* d, int id, int64_t, ms_lp_status* st) {
  for (;;) {
    if (ms_lp_poll(d, id, st)) return 0;
    ms_host_now_ns();
  }
}
int ms_preempt_raise(ms_dev* d, uint32_t* epoch, int64_t* t_host) {
  ++d->epoch;
  for (MockLp& l : d->lp)
    if (l.used && l.run.active && l.run.raise < 0) l.run.raise = g_now;
  if (epoch) *epoch = d->epoch;
  if (t_host) *t_host = g_now;
  return 0;
}
uint32_t ms_hp_next_seq(ms_dev* d) { return ++d->seq; }
int ms_hp_arm(ms_dev* d, int cid, uint32_t seq) {
  d->armed[seq] = cid;
  return 0;
}
int ms_hp_ring(ms_dev* d, uint32_t seq, int64_t* t_host) {
  auto it = d->armed.find(seq);
  if (it != d->armed.end()) {
    MockChain& c = d->chains[it->second];
    c.seq = seq;
    int64_t fd = c.first_delay, du = c.duration;
    if (c.next < c.timing.size()) std::tie(fd, du) = c.timing[c.next++];
    c.first = g_now + fd;
    c.done = c.first + du;
    d->armed.erase(it);
  }
  if (t_host) *t_host = g_now;
  return 0;
}
int ms_hp_launch_direct(ms_dev* d, int cid, uint32_t seq) {
  d->armed[seq] = cid;
  return ms_hp_ring(d, seq, nullptr);
}
int ms_hp_poll(ms_dev* d, int cid, uint32_t seq, ms_hp_times* t) {
  std::memset(t, 0, sizeof *t);
  t->seq = seq;
  const MockChain& c = d->chains[cid];
  if (c.seq != seq || c.done < 0 || g_now < c.done) return 0;
  t->done = 1;
  t->t_first_cta = static_cast<uint64_t>(c.first);
  t->t_done = static_cast<uint64_t>(c.done);
  t->t_gate = static_cast<uint64_t>(c.first - 500);
  return 1;
}
int ms_hp_wait(ms_dev* d, int cid, uint32_t seq, int64_t, ms_hp_times* t) {
  for (;;) {
    if (ms_hp_poll(d, cid, seq, t)) return 0;
    ms_host_now_ns();
  }
}
int ms_clock_calibrate(ms_dev*, int, int64_t* offset_ns, int64_t* rtt_min) {
  *offset_ns = 0;  // device clock == host clock
  *rtt_min = 0;
  return 0;
}
}  // extern "C"

// The power governor (off in these runs) references the CUDA runtime; no GPU here.
extern "C" int cudaDeviceGetPCIBusId(char*, int, int) { return 100; }
