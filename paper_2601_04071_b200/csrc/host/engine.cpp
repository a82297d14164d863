// Scheduler core (Algorithm 1 + comparators) and the replay device model.
//
// Reference semantics: /root/reference/proj/include/microslice/engine.hpp:102-1327.
// Parity contract: event order (ts, prio, stream, seq); the
// stable-by-ts Timeline with same-ts emission order; keyed uids and block-time draws;
// `<= 2 outstanding` tick deferral; generation counters; floating-point stretch and
// wave-time truncation.  Everything here is written against those rules; the
// differential test (tests/test_replay_parity.py) checks the rendered decision log
// byte-for-byte against the compiled reference for every in-scope policy.
//
// Structure:
//   EventQueue   — binary min-heap of 40-byte events
//   SimDevice    — streams, hardware-queue dispatch, SM thread occupancy, HBM stretch,
//                  wave completion; reports to the core through `Core` callbacks
//   Core         — HP serving driver, preempt/resume, bubbles, tick launcher,
//                  consolidation, REEF / spatial / exclusive feeders, accounting
#include <algorithm>
#include <cstring>
#include <deque>
#include <map>
#include <queue>
#include <sstream>

#include "microslice/engine.hpp"
#include "microslice/memory.hpp"

namespace microslice {
namespace {

enum class EvType : std::uint8_t {
  RequestArrival,
  BubbleOver,
  KernelArrive,
  WaveDone,
  TickLaunch,
  LargeBubbleCheck,
  Poke,
  UtilTick,
  ProbeTick,  // memory tier: periodic link ping-probe (engine.hpp:1263-1276)
};

// Event priority classes (Appendix A #2): HP work 0, LP work / ticks 1, infra 2.
constexpr int kPrioHp = 0, kPrioLp = 1, kPrioInfra = 2;

struct Event {
  Ns ts;
  long seq;
  long b;
  int prio;
  int stream;
  int a;
  EvType type;
};

inline bool before(const Event& x, const Event& y) {
  if (x.ts != y.ts) return x.ts < y.ts;
  if (x.prio != y.prio) return x.prio < y.prio;
  if (x.stream != y.stream) return x.stream < y.stream;
  return x.seq < y.seq;
}

class EventQueue {
 public:
  void push(Ns ts, int prio, int stream, EvType type, int a, long b) {
    heap_.push_back(Event{ts, ++seq_, b, prio, stream, a, type});
    sift_up(heap_.size() - 1);
  }
  bool empty() const { return heap_.empty(); }
  const Event& top() const { return heap_.front(); }
  void pop() {
    heap_.front() = heap_.back();
    heap_.pop_back();
    if (!heap_.empty()) sift_down(0);
  }

 private:
  void sift_up(std::size_t i) {
    Event e = heap_[i];
    while (i > 0) {
      const std::size_t p = (i - 1) / 2;
      if (!before(e, heap_[p])) break;
      heap_[i] = heap_[p];
      i = p;
    }
    heap_[i] = e;
  }
  void sift_down(std::size_t i) {
    const std::size_t n = heap_.size();
    Event e = heap_[i];
    for (;;) {
      std::size_t c = 2 * i + 1;
      if (c >= n) break;
      if (c + 1 < n && before(heap_[c + 1], heap_[c])) ++c;
      if (!before(heap_[c], e)) break;
      heap_[i] = heap_[c];
      i = c;
    }
    heap_[i] = e;
  }
  std::vector<Event> heap_;
  long seq_ = 0;
};

enum class InstState : std::uint8_t { Transit, Queued, Running, Finished, Evicted };

/// One launched (sub-)kernel: a full HP kernel, an LP slice, or a whole LP kernel.
struct Instance {
  int id = 0;
  int kernel = -1;
  int task = -1;
  int stream = -1;
  Priority prio = Priority::Low;
  GridBox box;
  std::int64_t blocks_total = 0;
  std::int64_t blocks_dispatched = 0;
  std::int64_t blocks_done = 0;
  int waves_in_flight = 0;
  Ns block_time = 0;
  std::uint64_t uid = 0;
  long parent = -1;
  InstState state = InstState::Transit;
  bool consolidated = false;
  bool doomed = false;  // REEF: tail-started, discard progress when its waves drain
};

/// Per-kernel constants folded once at setup (Eq. 1 capacity, thread cost, demand).
struct KernelRt {
  const KernelSpec* spec = nullptr;
  std::int32_t name_id = 0;
  std::int64_t capacity = 1;
  std::int64_t thread_cost = 1;
  double bw = 0.0;
};

struct StreamRt {
  int task = -1;
  Priority prio = Priority::Low;
  std::deque<int> queue;  // device-side FIFO in arrival order
};

/// A kernel of an LP task whose blocks are handed out as slices (engine.hpp:186-195).
struct Parent {
  long seq = -1;
  int task = -1;
  int kernel = -1;
  std::uint64_t uid = 0;
  std::int64_t blocks_total = 0;
  std::int64_t blocks_done = 0;
  std::deque<GridBox> pending;  // resume cursor: slices not yet issued
  int consolidated_boxes = 0;
};

struct Segment {
  std::vector<int> kernels;
  std::vector<int> hints;
};

struct TaskRt {
  const TaskSpec* spec = nullptr;
  int index = -1;
  int stream = -1;
  std::int32_t name_id = 0;
  const RequestTrace* trace = nullptr;
  std::vector<Segment> segments;
  std::size_t expanded_len = 0;  // repeat-expanded kernel sequence length
  std::vector<int> expanded;     // kernel ids of the expanded sequence
  // HP serving state
  std::deque<std::size_t> backlog;
  bool busy = false;
  std::size_t request = 0;
  int iteration = 0;
  int n_iterations = 0;
  std::size_t segment = 0;
  int outstanding = 0;
  std::uint64_t hint_name_hash = 0;
  std::uint64_t name_hash = 0;
  // LP state
  std::size_t seq_cursor = 0;
  long parents_made = 0;
  std::vector<std::int64_t> chunk_ids;  // memory tier placement (engine.hpp:396-407)
};

struct PolicyTraits {
  bool hp = true, lp = true;
  bool harvest = false;       // SplitKernel: bubbles + ticks + consolidation
  bool free_run = false;      // Spatial / ExclusiveLp: back-to-back LP launches
  bool reef = false;          // kernel-boundary temporal sharing with eviction
  bool preempt_records = true;
  explicit PolicyTraits(Policy p) {
    hp = p != Policy::ExclusiveLp;
    lp = p != Policy::Exclusive;
    harvest = p == Policy::SplitKernel;
    free_run = p == Policy::Spatial || p == Policy::ExclusiveLp;
    reef = p == Policy::Reef;
    preempt_records = p != Policy::Exclusive && p != Policy::ExclusiveLp;
  }
};

class Core;

// ============================================================================ SimDevice
// Replay device model (engine.hpp:722-945): one hardware queue per stream, streams
// walked in id order (HP first), only the queue head is eligible (REEF LP scans the
// whole queue), an LP head waits while HP work fits, a wave takes
// n = min(remaining, cap - resident, free_threads / thread_cost) blocks and lasts
// block_time * max(1, demand / HBM).
class SimDevice {
 public:
  SimDevice(Core& core) : core_(core) {}
  void init(std::int64_t total_threads) { total_threads_ = free_threads_ = total_threads; }

  void arrive(int id);
  void wave_done(int id, std::int64_t n);
  void dispatch();
  void remove_from_stream(Instance& inst);

  std::int64_t total_threads() const { return total_threads_; }
  std::int64_t busy_threads() const { return total_threads_ - free_threads_; }
  /// HBM demand now: resident waves + in-flight memory-tier chunk transfers, which hold
  /// HBM at their link's nominal rate until they end (engine.hpp:266-273, 1221-1224).
  double bw_demand(Ns now) {
    while (!transfers_.empty() && transfers_.top().first <= now) {
      transfer_bw_ -= transfers_.top().second;
      transfers_.pop();
    }
    if (transfers_.empty()) transfer_bw_ = 0.0;
    return wave_bw_ + transfer_bw_;
  }
  void add_transfer(Ns end, double bw) {
    transfers_.push({end, bw});
    transfer_bw_ += bw;
  }
  void note_occupancy(Ns now) {
    busy_integral_ += static_cast<double>(total_threads_ - free_threads_) *
                      static_cast<double>(now - last_occ_change_);
    last_occ_change_ = now;
  }
  double busy_integral() const { return busy_integral_; }
  std::vector<StreamRt> streams;

 private:
  bool hp_work_fits() const;
  void dispatch_wave(Instance& inst, std::int64_t n);

  Core& core_;
  std::int64_t total_threads_ = 0, free_threads_ = 0;
  double wave_bw_ = 0.0;
  std::priority_queue<std::pair<Ns, double>, std::vector<std::pair<Ns, double>>, std::greater<>> transfers_;
  double transfer_bw_ = 0.0;
  double busy_integral_ = 0.0;
  Ns last_occ_change_ = 0;
};

// ============================================================================ Core
class Core {
 public:
  Core(const ScenarioSpec& sc, Policy policy, const EngineOptions& opts)
      : sc_(sc), policy_(policy), traits_(policy), opts_(opts), dev_(*this),
        predictor_(sc.sched.ema_alpha, sc.sched.ema_k, sc.sched.large_bubble_threshold) {}

  RunArtifacts run();
  std::uint64_t events() const { return events_; }

  // ---- device -> core callbacks / shared state
  Ns now() const { return now_; }
  Instance& inst(int id) { return instances_[id]; }
  const KernelRt& krt(int k) const { return kernels_[k]; }
  RunArtifacts& art() { return art_; }
  EventQueue& queue() { return eq_; }
  const PolicyTraits& traits() const { return traits_; }
  void on_first_hp_wave(const Instance& hp);
  void on_lp_wave(Ns wave_time) {
    if (open_hint_task_ >= 0 && open_hint_contended_) contended_busy_ += wave_time;
  }
  void on_kernel_done(int id);
  void evict(Instance& inst, Ns at);
  bool reef_hp_gate_closed() const;
  bool reef_lp_blocked(const Instance& i) const {
    return i.blocks_dispatched == 0 && (p_flag_ || i.doomed);
  }
  void reef_on_flag();
  bool p_flag() const { return p_flag_; }
  double scenario_hbm() const { return sc_.gpu.hbm_bandwidth; }
  bool memory_tier() const { return mem_.has_value(); }
  Ns wave_memory_extra(const Instance& i);

  void emit(Ns ts, EventKind k, int stream, std::int32_t kernel, Detail d, std::int64_t a = 0,
            std::int64_t b = 0, double g = 0.0) {
    TimelineRecord r;
    r.ts = ts;
    r.kind = k;
    r.stream = stream;
    r.kernel = kernel;
    r.detail = d;
    r.a = a;
    r.b = b;
    r.g = g;
    art_.timeline.record(r);
  }

 private:
  void setup();
  void build_task(TaskRt& t);
  ExecOracle oracle_for(int k) const;
  void build_plans();

  // HP serving driver (engine.hpp:508-678)
  void request_arrival(int task, std::size_t idx);
  void begin_request(TaskRt& t);
  void issue_segment(TaskRt& t);
  void segment_done(int task);
  void fire_hints(TaskRt& t, Ns from);
  void bubble_over(int task, long payload);
  void finish_iteration(TaskRt& t);

  // instance lifecycle (engine.hpp:682-720)
  int make_instance(int task, int kernel, const GridBox& box, std::uint64_t uid, Priority prio,
                    bool consolidated, long parent);
  void issue(int id, Ns ts, bool relaunch = false);

  // scheduler reactions (engine.hpp:949-997)
  void hp_turned_active(Ns ts);
  void hp_drained();
  void large_bubble_check(long gen);

  // split-kernel LP (engine.hpp:1001-1115)
  Parent& next_parent(int task);
  Ns predicted_time(int kernel, std::int64_t blocks) const;
  void start_ticks(Ns at);
  void tick();
  void consolidate_for_large_bubble();

  // comparators (engine.hpp:1119-1195)
  void free_run_issue(int task);
  void reef_refill(Ns at);

  void drop_lp_active(int id) {
    auto it = std::find(lp_active_.begin(), lp_active_.end(), id);
    if (it != lp_active_.end()) lp_active_.erase(it);
  }
  void api(Ns a, Ns b, std::int32_t tag, std::int64_t corr) {
    art_.api_rows.push_back({a, b, api_tags_[tag], corr});
  }

  const ScenarioSpec& sc_;
  Policy policy_;
  PolicyTraits traits_;
  EngineOptions opts_;
  SimDevice dev_;
  EventQueue eq_;
  Ns now_ = 0;
  std::uint64_t events_ = 0;

  std::vector<KernelRt> kernels_;
  std::vector<Instance> instances_;
  std::vector<TaskRt> tasks_;
  std::vector<int> hp_tasks_, lp_tasks_;
  std::map<long, Parent> parents_;
  long parent_counter_ = 0;
  std::vector<int> lp_active_;
  std::map<int, SplitPlan> plans_;

  int hp_active_ = 0;
  Ns last_hp_activity_ = 0;
  bool p_flag_ = false;

  long generation_ = 0;
  int lp_outstanding_ = 0;
  bool tick_deferred_ = false;
  int tick_rr_ = 0;
  int slices_since_resync_ = 0;
  bool resync_pending_ = false;
  IntervalPredictor predictor_;
  Ns last_arrival_ = -1;

  int open_hint_task_ = -1;
  bool open_hint_contended_ = false;
  Ns contended_busy_ = 0;

  std::deque<int> reef_evicted_;
  int reef_outstanding_ = 0;
  int reef_rr_ = 0;
  Ns reef_gate_ = 0;

  std::optional<PreemptionRecord> pending_preempt_;
  std::optional<MemoryManager> mem_;
  RunArtifacts art_;

  std::int32_t id_scheduler_ = 0, id_resync_ = 0, id_empty_ = 0;
  enum ApiTag { kApiLaunch, kApiSync };
  std::vector<std::string> api_tags_{"cuLaunchKernel", "cudaStreamSynchronize"};
};

// ---------------------------------------------------------------- SimDevice impl
void SimDevice::arrive(int id) {
  Instance& i = core_.inst(id);
  if (i.state == InstState::Evicted) return;
  i.state = InstState::Queued;
  streams[i.stream].queue.push_back(id);
  dispatch();
}

void SimDevice::remove_from_stream(Instance& inst) {
  auto& q = streams[inst.stream].queue;
  auto it = std::find(q.begin(), q.end(), inst.id);
  if (it != q.end()) q.erase(it);
}

bool SimDevice::hp_work_fits() const {
  for (const StreamRt& s : streams) {
    if (s.prio != Priority::High) break;  // HP streams are numbered first
    if (s.queue.empty()) continue;
    const Instance& head = core_.inst(s.queue.front());
    if (head.blocks_dispatched >= head.blocks_total) continue;
    const KernelRt& k = core_.krt(head.kernel);
    if (head.blocks_dispatched - head.blocks_done >= k.capacity) continue;
    if (free_threads_ >= k.thread_cost) return true;
  }
  return false;
}

void SimDevice::dispatch() {
  const bool reef = core_.traits().reef;
  for (bool progress = true; progress;) {
    progress = false;
    for (StreamRt& s : streams) {
      if (s.queue.empty()) continue;
      const bool low = s.prio == Priority::Low;
      if (reef && !low && core_.reef_hp_gate_closed()) continue;
      const std::size_t depth = reef && low ? s.queue.size() : 1;
      for (std::size_t c = 0; c < depth && c < s.queue.size(); ++c) {
        Instance& i = core_.inst(s.queue[c]);
        if (i.state == InstState::Evicted) continue;
        const std::int64_t remaining = i.blocks_total - i.blocks_dispatched;
        if (remaining <= 0) continue;  // draining tail: the successor may start
        if (low) {
          if (hp_work_fits()) break;
          if (reef && core_.reef_lp_blocked(i)) break;  // flag checked before first wave
        }
        const KernelRt& k = core_.krt(i.kernel);
        const std::int64_t n = std::min({remaining, k.capacity - (i.blocks_dispatched - i.blocks_done),
                                         free_threads_ / k.thread_cost});
        if (n <= 0) break;
        dispatch_wave(i, n);
        progress = true;
        if (i.blocks_total > i.blocks_dispatched) break;  // successors wait behind it
      }
    }
  }
}

void SimDevice::dispatch_wave(Instance& i, std::int64_t n) {
  const Ns now = core_.now();
  note_occupancy(now);
  const KernelRt& k = core_.krt(i.kernel);
  const double own_bw = static_cast<double>(n) * k.bw;
  const double stretch = std::max(1.0, (bw_demand(now) + own_bw) / core_.scenario_hbm());
  Ns extra = 0;
  if (i.prio == Priority::Low && core_.memory_tier()) extra = core_.wave_memory_extra(i);
  Ns wave_time = static_cast<Ns>(static_cast<double>(i.block_time) * stretch) + extra;
  if (wave_time < 1) wave_time = 1;

  if (i.state == InstState::Queued) i.state = InstState::Running;
  const bool hp = i.prio == Priority::High;
  const bool first_hp_wave = hp && i.blocks_dispatched == 0;
  i.blocks_dispatched += n;
  ++i.waves_in_flight;
  free_threads_ -= n * k.thread_cost;
  wave_bw_ += own_bw;
  RunArtifacts& art = core_.art();
  (hp ? art.hp_blocks_launched : art.lp_blocks_launched) += n;
  core_.emit(now, EventKind::DispatchWave, i.stream, k.name_id, Detail::InstWave, i.id, n, stretch);
  if (hp) {
    art.hp_stretch_sum += stretch;
    ++art.hp_stretch_waves;
    if (first_hp_wave) core_.on_first_hp_wave(i);
  } else {
    core_.on_lp_wave(wave_time);
  }
  core_.queue().push(now + wave_time, hp ? kPrioHp : kPrioLp, i.stream, EvType::WaveDone, i.id,
                     static_cast<long>(n));
}

void SimDevice::wave_done(int id, std::int64_t n) {
  const Ns now = core_.now();
  Instance& i = core_.inst(id);
  note_occupancy(now);
  const KernelRt& k = core_.krt(i.kernel);
  i.blocks_done += n;
  --i.waves_in_flight;
  free_threads_ += n * k.thread_cost;
  wave_bw_ -= static_cast<double>(n) * k.bw;
  if (wave_bw_ < 1e-6) wave_bw_ = 0;
  core_.emit(now, EventKind::WaveDone, i.stream, k.name_id, Detail::InstN, id, n);
  if (i.state == InstState::Evicted) {
    core_.art().lp_waste_blocks += n;  // late wave of an evicted kernel
  } else if (i.doomed && i.waves_in_flight == 0) {
    core_.evict(i, now);
  } else if (i.blocks_done >= i.blocks_total) {
    core_.on_kernel_done(id);
  }
  if (core_.traits().reef && core_.p_flag()) core_.reef_on_flag();
  dispatch();
}


// ---------------------------------------------------------------- Core: setup
void Core::build_task(TaskRt& t) {
  // Repeat-expand the kernel sequence, then cut it into segments ending at hint slots
  // (engine.hpp:434-459): a hint at position p fires after kernel p (-1: iteration end).
  for (const KernelRef& kr : t.spec->kernel_sequence) {
    const int k = static_cast<int>(sc_.find_kernel(kr.kernel) - sc_.kernels.data());
    t.expanded.insert(t.expanded.end(), static_cast<std::size_t>(kr.repeat), k);
  }
  t.expanded_len = t.expanded.size();
  const std::size_t n = t.expanded.size();
  std::vector<std::vector<int>> hints_after(n + 1);
  for (std::size_t h = 0; h < t.spec->bubble_hints.size(); ++h) {
    const int pos = t.spec->bubble_hints[h].position;
    const std::size_t slot = pos < 0 ? n : std::min<std::size_t>(static_cast<std::size_t>(pos) + 1, n);
    hints_after[slot].push_back(static_cast<int>(h));
  }
  Segment cur;
  for (std::size_t i = 0; i <= n; ++i) {
    if (i > 0) cur.kernels.push_back(t.expanded[i - 1]);
    if (hints_after[i].empty()) continue;
    cur.hints = hints_after[i];
    t.segments.push_back(std::move(cur));
    cur = Segment{};
  }
  if (!cur.kernels.empty()) t.segments.push_back(std::move(cur));
  t.name_hash = hash_str(t.spec->name);
  t.hint_name_hash = hash_str(t.spec->name + "#hint");
  t.name_id = art_.timeline.intern(t.spec->name);
}

ExecOracle Core::oracle_for(int k) const {
  const KernelSpec& spec = sc_.kernels[k];
  if (spec.measured_time.empty()) {
    const GpuConfig* gpu = &sc_.gpu;
    const KernelSpec* ks = &spec;
    const CapacityRounding rounding = opts_.rounding;
    return [gpu, ks, rounding](std::int64_t blocks) {
      return exec_time_model(*gpu, *ks, blocks, 0.0, rounding);
    };
  }
  // Piecewise-linear interpolation over measured (n_blocks, time) rows, clamped at
  // both ends (engine.hpp:461-481).
  auto rows = spec.measured_time;
  std::sort(rows.begin(), rows.end());
  return [rows](std::int64_t blocks) -> Ns {
    if (blocks <= rows.front().first) return rows.front().second;
    if (blocks >= rows.back().first) return rows.back().second;
    std::size_t i = 1;
    while (i < rows.size() && blocks > rows[i].first) ++i;
    if (i == rows.size()) return rows.back().second;
    const double f = static_cast<double>(blocks - rows[i - 1].first) /
                     static_cast<double>(rows[i].first - rows[i - 1].first);
    return rows[i - 1].second +
           static_cast<Ns>(f * static_cast<double>(rows[i].second - rows[i - 1].second));
  };
}

void Core::build_plans() {
  SplitSearchOptions so;
  so.cap = sc_.sched.slice_cap;
  so.square_tiling = sc_.sched.square_tiling;
  so.rounding = opts_.rounding;
  for (int ti : lp_tasks_)
    for (int k : tasks_[ti].expanded) {
      if (plans_.count(k) || !sc_.kernels[k].splittable) continue;
      plans_.emplace(k, find_optimal_split(sc_.gpu, sc_.kernels[k], oracle_for(k), so));
    }
}

void Core::setup() {
  dev_.init(static_cast<std::int64_t>(sc_.gpu.n_sm) * sc_.gpu.sm_max_threads);
  art_.policy = policy_;
  art_.scenario = sc_.name;
  art_.seed = sc_.seed;
  art_.horizon = sc_.horizon;
  id_scheduler_ = art_.timeline.intern("scheduler");
  id_resync_ = art_.timeline.intern("resync");
  id_empty_ = 0;

  kernels_.resize(sc_.kernels.size());
  for (std::size_t k = 0; k < sc_.kernels.size(); ++k) {
    const KernelSpec& ks = sc_.kernels[k];
    KernelRt& r = kernels_[k];
    r.spec = &ks;
    r.name_id = art_.timeline.intern(ks.name);
    r.capacity = concurrent_capacity(sc_.gpu, ks, opts_.rounding);
    r.thread_cost = static_cast<std::int64_t>(
        std::max(1.0, static_cast<double>(ks.threads_per_block) / ks.occupancy));
    r.bw = ks.bw_demand_per_block;
  }

  // Policy task filter; task indices are assigned after filtering (Appendix A #6).
  for (const TaskSpec& ts : sc_.tasks) {
    if (ts.priority == Priority::High ? !traits_.hp : !traits_.lp) continue;
    TaskRt t;
    t.spec = &ts;
    t.index = static_cast<int>(tasks_.size());
    if (ts.kind == TaskKind::Serving && ts.priority == Priority::High)
      t.trace = sc_.find_trace(ts.trace);
    build_task(t);
    tasks_.push_back(std::move(t));
  }
  // Streams: HP tasks first so the hardware-queue walk is in priority order.
  for (int pass = 0; pass < 2; ++pass) {
    const Priority want = pass == 0 ? Priority::High : Priority::Low;
    for (TaskRt& t : tasks_) {
      if (t.spec->priority != want) continue;
      t.stream = static_cast<int>(dev_.streams.size());
      dev_.streams.push_back(StreamRt{t.index, want, {}});
      (want == Priority::High ? hp_tasks_ : lp_tasks_).push_back(t.index);
    }
  }

  if (sc_.mem.enabled) {  // engine.hpp:398-411: HP chunks first (pinned), then LP
    mem_.emplace(sc_.gpu, sc_.mem);
    std::vector<ChunkRelocation> moves;
    for (const auto* group : {&hp_tasks_, &lp_tasks_})
      for (int ti : *group)
        tasks_[ti].chunk_ids = mem_->allocate(ti, tasks_[ti].spec->priority, tasks_[ti].spec->memory_footprint,
                                              0, &moves);
    if (!moves.empty()) {
      const std::int32_t chunk = art_.timeline.intern("chunk");
      for (const ChunkRelocation& m : moves) emit(0, EventKind::Evict, -1, chunk, Detail::Chunk, m.chunk_id);
    }
    if (!sc_.gpu.nvlink_peers.empty()) eq_.push(0, kPrioInfra, -1, EvType::ProbeTick, 0, 0);
  }

  if (traits_.harvest) build_plans();

  for (int ti : hp_tasks_) {
    const TaskRt& t = tasks_[ti];
    if (!t.trace) continue;
    for (std::size_t r = 0; r < t.trace->arrivals.size() && t.trace->arrivals[r] < sc_.horizon; ++r)
      eq_.push(t.trace->arrivals[r], kPrioHp, t.stream, EvType::RequestArrival, t.index,
               static_cast<long>(r));
  }
  if (traits_.free_run)
    for (int ti : lp_tasks_) free_run_issue(ti);
  else if (traits_.reef)
    reef_refill(0);
  eq_.push(0, kPrioInfra, -1, EvType::UtilTick, 0, 0);
}

// ---------------------------------------------------------------- HP serving driver
void Core::request_arrival(int task, std::size_t idx) {
  TaskRt& t = tasks_[task];
  RequestStat rs;
  rs.task = task;
  rs.index = idx;
  rs.arrival = now_;
  rs.iterations = t.trace->iterations_for(sc_.seed, idx);
  art_.requests.push_back(rs);
  t.backlog.push_back(art_.requests.size() - 1);
  // Idle-slice predictor input: gaps between consecutive arrivals over all HP tasks.
  if (last_arrival_ >= 0) predictor_.observe_gap(now_ - last_arrival_);
  last_arrival_ = now_;
  if (t.busy) return;
  t.busy = true;
  begin_request(t);
}

void Core::begin_request(TaskRt& t) {
  t.request = t.backlog.front();
  t.backlog.pop_front();
  t.iteration = 0;
  t.n_iterations = art_.requests[t.request].iterations;
  t.segment = 0;
  issue_segment(t);
}

void Core::issue_segment(TaskRt& t) {
  const Segment& seg = t.segments[t.segment];
  if (seg.kernels.empty()) {
    fire_hints(t, now_);
    return;
  }
  t.outstanding = static_cast<int>(seg.kernels.size());
  const std::uint64_t req_index = art_.requests[t.request].index;
  const std::uint64_t who = hash_combine(sc_.seed, t.name_hash);
  const std::uint64_t when = hash_combine(req_index * 131 + 7, static_cast<std::uint64_t>(t.iteration));
  for (std::size_t rep = 0; rep < seg.kernels.size(); ++rep) {
    const int k = seg.kernels[rep];
    // HP instance uid (engine.hpp:550-555): task, request, iteration, segment, position.
    const std::uint64_t uid = hash_combine(
        hash_combine(who, when),
        hash_combine(static_cast<std::uint64_t>(t.segment) * 31, static_cast<std::uint64_t>(rep)));
    const Grid& g = sc_.kernels[k].grid;
    const int id = make_instance(t.index, k, GridBox{0, 0, 0, g.x, g.y, g.z}, uid,
                                 Priority::High, false, -1);
    issue(id, now_);
  }
}

void Core::segment_done(int task) {
  TaskRt& t = tasks_[task];
  if (!t.segments[t.segment].hints.empty()) {
    fire_hints(t, now_);
    return;
  }
  if (++t.segment < t.segments.size()) issue_segment(t); else finish_iteration(t);
}

void Core::fire_hints(TaskRt& t, Ns from) {
  const Segment& seg = t.segments[t.segment];
  const std::uint64_t req_index = art_.requests[t.request].index;
  const std::uint64_t base = hash_combine(hash_combine(sc_.seed, t.hint_name_hash), req_index * 17);
  Ns dur = 0;
  std::string key;
  bool contended = false;
  for (const int h : seg.hints) {
    const BubbleHint& hint = t.spec->bubble_hints[h];
    dur += hint.duration.sample_keyed(hash_combine(
        base, hash_combine(static_cast<std::uint64_t>(t.iteration), static_cast<std::uint64_t>(h))));
    contended = contended || hint.contended;
    if (!key.empty()) key += '+';
    key += hint.pattern_key();
  }
  if (dur <= 0) dur = 1;
  emit(from, EventKind::BubbleBegin, t.stream, t.name_id, Detail::Hint, art_.timeline.intern(key));

  // Profiler-style API rows: the bubble split evenly over its tags, remainder last.
  std::size_t n_tags = 0;
  for (const int h : seg.hints) n_tags += t.spec->bubble_hints[h].pattern.size();
  const Ns per = dur / static_cast<Ns>(n_tags);
  const std::int64_t corr = static_cast<long>(t.request) * 1000 + t.iteration;
  Ns cursor = from;
  std::size_t tag_i = 0;
  for (const int h : seg.hints)
    for (const std::string& tag : t.spec->bubble_hints[h].pattern) {
      const Ns end = ++tag_i == n_tags ? from + dur : cursor + per;
      art_.api_rows.push_back({cursor, end, tag, corr});
      cursor = end;
    }

  art_.small_bubble_time += dur;
  bool harvestable = true;
  if (opts_.hint_filter) {
    harvestable = false;
    for (const int h : seg.hints)
      harvestable = harvestable || opts_.hint_filter->count(t.spec->bubble_hints[h].pattern_key()) > 0;
  }
  if (traits_.harvest && harvestable && !lp_tasks_.empty()) {
    // Small bubble: one scheduler sync, then the kernel-tick launcher fills it.
    open_hint_task_ = t.index;
    open_hint_contended_ = contended;
    contended_busy_ = 0;
    const Ns start = from + sc_.gpu.sync_overhead;
    emit(from, EventKind::SyncBegin, t.stream, t.name_id, Detail::Text, id_scheduler_);
    emit(start, EventKind::SyncEnd, t.stream, t.name_id, Detail::Text, id_scheduler_);
    api(from, start, kApiSync, -1);
    art_.sync_cost_total += sc_.gpu.sync_overhead;
    start_ticks(start);
  }
  eq_.push(from + dur, kPrioHp, t.stream, EvType::BubbleOver, t.index, 0);
}

void Core::bubble_over(int task, long payload) {
  TaskRt& t = tasks_[task];
  if (payload == 0 && open_hint_task_ == task && open_hint_contended_ && contended_busy_ > 0) {
    // The "idle" interval carried latency-critical traffic: LP co-running stretched it.
    const Ns extra = contended_busy_ / 2;
    contended_busy_ = 0;
    open_hint_contended_ = false;
    eq_.push(now_ + extra, kPrioHp, t.stream, EvType::BubbleOver, task, 1);
    return;
  }
  emit(now_, EventKind::BubbleEnd, t.stream, t.name_id, Detail::Text, id_empty_);
  if (open_hint_task_ == task) {
    open_hint_task_ = -1;
    open_hint_contended_ = false;
    ++generation_;  // pause the tick launcher until the next detected bubble
    tick_deferred_ = false;
    if (traits_.harvest && hp_active_ == 0)
      eq_.push(now_ + sc_.sched.large_bubble_threshold, kPrioInfra, -1, EvType::LargeBubbleCheck, 0,
               generation_);
  }
  if (++t.segment < t.segments.size()) issue_segment(t); else finish_iteration(t);
}

void Core::finish_iteration(TaskRt& t) {
  RequestStat& rs = art_.requests[t.request];
  if (++t.iteration == 1) rs.first_token = now_;
  if (t.iteration < t.n_iterations) {
    t.segment = 0;
    issue_segment(t);
    return;
  }
  rs.done = now_;
  rs.completed = true;
  if (t.backlog.empty()) t.busy = false; else begin_request(t);
}

// ---------------------------------------------------------------- instances
int Core::make_instance(int task, int kernel, const GridBox& box, std::uint64_t uid,
                        Priority prio, bool consolidated, long parent) {
  Instance i;
  i.id = static_cast<int>(instances_.size());
  i.kernel = kernel;
  i.task = task;
  i.prio = prio;
  i.stream = tasks_[task].stream;
  i.box = box;
  i.blocks_total = box.blocks();
  i.block_time = sc_.kernels[kernel].block_time.sample_keyed(uid);  // one keyed draw per instance
  i.uid = uid;
  i.parent = parent;
  i.consolidated = consolidated;
  instances_.push_back(i);
  return i.id;
}

void Core::issue(int id, Ns ts, bool relaunch) {
  Instance& i = instances_[id];
  i.state = InstState::Transit;
  emit(ts, relaunch ? EventKind::Relaunch : EventKind::Launch, i.stream, kernels_[i.kernel].name_id,
       Detail::Inst, id);
  if (relaunch) ++art_.relaunch_count;
  api(ts, ts + us(1), kApiLaunch, id);
  const bool hp = i.prio == Priority::High;
  if (hp) {
    if (hp_active_ == 0) hp_turned_active(ts);
    ++hp_active_;
  } else {
    lp_active_.push_back(id);
  }
  // Host -> device transit: the modelled launch overhead.
  eq_.push(ts + sc_.gpu.launch_overhead, hp ? kPrioHp : kPrioLp, i.stream, EvType::KernelArrive, id, 0);
}

void Core::on_first_hp_wave(const Instance& hp) {
  if (!pending_preempt_) return;
  PreemptionRecord rec = *pending_preempt_;
  pending_preempt_.reset();
  rec.delay = now_ - rec.begin;
  art_.preemptions.push_back(rec);
  emit(now_, EventKind::PreemptEnd, hp.stream, kernels_[hp.kernel].name_id, Detail::Delay, rec.delay,
       rec.consolidated ? 1 : 0);
}

void Core::on_kernel_done(int id) {
  Instance& i = instances_[id];
  i.state = InstState::Finished;
  dev_.remove_from_stream(i);
  emit(now_, EventKind::KernelDone, i.stream, kernels_[i.kernel].name_id, Detail::InstBlocks, id,
       i.blocks_total);

  if (i.prio == Priority::High) {
    art_.hp_blocks_done += i.blocks_total;
    --hp_active_;
    last_hp_activity_ = now_;
    const int task = i.task;
    --tasks_[task].outstanding;
    if (hp_active_ == 0) hp_drained();
    if (tasks_[task].outstanding == 0) segment_done(task);
    return;
  }

  art_.lp_blocks_done += i.blocks_total;
  drop_lp_active(id);
  if (i.parent >= 0) {
    auto it = parents_.find(i.parent);
    if (it != parents_.end()) {
      Parent& par = it->second;
      par.blocks_done += i.blocks_total;
      if (par.blocks_done >= par.blocks_total && par.pending.empty()) {
        art_.lp_work_units += static_cast<double>(par.blocks_total);
        ++art_.lp_parent_completions;
        parents_.erase(it);
      }
    }
  }

  if (traits_.free_run) {
    free_run_issue(i.task);
  } else if (traits_.reef) {
    --reef_outstanding_;
    art_.sync_cost_total += sc_.gpu.sync_overhead;
    api(now_, now_ + sc_.gpu.sync_overhead, kApiSync, -2);
    if (!p_flag_) reef_refill(now_ + sc_.gpu.sync_overhead);
  } else if (traits_.harvest) {
    --lp_outstanding_;
    if (resync_pending_ && lp_outstanding_ == 0) {
      // Periodic drain: resynchronise host and device before launching more slices.
      resync_pending_ = false;
      art_.sync_cost_total += sc_.gpu.sync_overhead;
      const Ns resume = now_ + sc_.gpu.sync_overhead;
      emit(now_, EventKind::SyncBegin, i.stream, id_empty_, Detail::Text, id_resync_);
      emit(resume, EventKind::SyncEnd, i.stream, id_empty_, Detail::Text, id_resync_);
      api(now_, resume, kApiSync, -3);
      if (!p_flag_) eq_.push(resume, kPrioLp, -1, EvType::TickLaunch, 0, generation_);
    } else if (tick_deferred_ && !p_flag_) {
      tick_deferred_ = false;
      eq_.push(now_, kPrioLp, -1, EvType::TickLaunch, 0, generation_);
    }
  }
}

// engine.hpp:1199-1229: an LP wave touches accesses_per_wave keyed-random chunks of its
// task; off-device chunks add their transfer latency (the wave waits for the slowest) and
// peer transfers load the link (congestion) and HBM (the DMA engine's nominal rate).
Ns Core::wave_memory_extra(const Instance& i) {
  const TaskRt& t = tasks_[i.task];
  if (t.chunk_ids.empty()) return 0;
  const std::uint64_t wave_key = hash_combine(i.uid, static_cast<std::uint64_t>(i.blocks_dispatched) * 977);
  const std::uint64_t n_chunks = t.chunk_ids.size();
  Ns worst = 0;
  for (int a = 0; a < sc_.mem.accesses_per_wave; ++a) {
    const std::int64_t cid =
        t.chunk_ids[splitmix64(hash_combine(wave_key, static_cast<std::uint64_t>(a))) % n_chunks];
    const AccessResult r = mem_->access(cid, now_);
    if (r.tier == Tier::Local) continue;
    emit(now_, EventKind::MemFault, i.stream, kernels_[i.kernel].name_id, Detail::MemFault, cid,
         r.tier == Tier::Peer ? 1 : 2);
    if (r.tier == Tier::Peer) {
      const Ns dur = std::max<Ns>(r.latency, 1);
      mem_->congestion().add_transfer(r.peer, static_cast<double>(kChunkBytes) / to_sec(dur), now_ + dur);
      dev_.add_transfer(now_ + dur, sc_.gpu.nvlink_peers[static_cast<std::size_t>(r.peer)].bandwidth);
    }
    worst = std::max(worst, r.latency);
  }
  return worst;
}

void Core::evict(Instance& i, Ns at) {
  const bool counted = i.state != InstState::Evicted;
  i.state = InstState::Evicted;
  i.doomed = false;
  art_.lp_waste_blocks += i.blocks_done;
  dev_.remove_from_stream(i);
  drop_lp_active(i.id);
  emit(at, EventKind::Evict, i.stream, kernels_[i.kernel].name_id, Detail::InstWasted, i.id,
       i.blocks_done);
  reef_evicted_.push_back(i.id);
  if (counted) --reef_outstanding_;
}

// ---------------------------------------------------------------- preempt / resume
void Core::hp_turned_active(Ns ts) {
  if (!traits_.preempt_records) return;
  p_flag_ = true;  // the preempt flag: LP stops being fed
  PreemptionRecord rec;
  rec.begin = ts;
  for (const int id : lp_active_) {
    const Instance& i = instances_[id];
    if (i.state != InstState::Running && i.state != InstState::Queued) continue;
    rec.lp_in_flight = true;
    rec.consolidated = rec.consolidated || i.consolidated;
  }
  pending_preempt_ = rec;
  emit(ts, EventKind::PreemptBegin, -1, id_empty_, Detail::Text, id_empty_);
  if (traits_.harvest) {
    ++generation_;  // cancels queued ticks
    tick_deferred_ = false;
  }
  if (traits_.reef) reef_on_flag();
}

void Core::hp_drained() {
  if (!traits_.preempt_records) return;
  p_flag_ = false;
  if (traits_.reef) {
    art_.sync_cost_total += sc_.gpu.sync_overhead;
    reef_refill(now_ + sc_.gpu.sync_overhead);
    return;
  }
  if (traits_.harvest && open_hint_task_ < 0)
    eq_.push(now_ + sc_.sched.large_bubble_threshold, kPrioInfra, -1, EvType::LargeBubbleCheck, 0,
             ++generation_);
}

void Core::large_bubble_check(long gen) {
  if (!traits_.harvest || gen != generation_ || hp_active_ > 0) return;
  if (now_ - last_hp_activity_ < sc_.sched.large_bubble_threshold || lp_tasks_.empty()) return;
  if (sc_.sched.consolidation) consolidate_for_large_bubble();
  const Ns start = now_ + sc_.gpu.sync_overhead;
  art_.sync_cost_total += sc_.gpu.sync_overhead;
  emit(now_, EventKind::SyncBegin, -1, id_empty_, Detail::Text, id_scheduler_);
  emit(start, EventKind::SyncEnd, -1, id_empty_, Detail::Text, id_scheduler_);
  api(now_, start, kApiSync, -1);
  start_ticks(start);
}

// ---------------------------------------------------------------- split-kernel LP
Parent& Core::next_parent(int task) {
  for (auto& entry : parents_)
    if (entry.second.task == task && !entry.second.pending.empty()) return entry.second;
  // Start the next kernel of the task's cyclic (repeat-expanded) sequence.
  TaskRt& t = tasks_[task];
  const int k = t.expanded[t.seq_cursor % t.expanded_len];
  ++t.seq_cursor;
  Parent par;
  par.seq = parent_counter_++;
  par.task = task;
  par.kernel = k;
  par.uid = hash_combine(hash_combine(sc_.seed, t.name_hash),
                         0xabcd0000ull + static_cast<std::uint64_t>(t.parents_made++));
  const Grid& g = sc_.kernels[k].grid;
  par.blocks_total = g.blocks();
  auto plan = plans_.find(k);
  if (plan != plans_.end())
    par.pending.assign(plan->second.slices.begin(), plan->second.slices.end());
  else
    par.pending.push_back(GridBox{0, 0, 0, g.x, g.y, g.z});
  return parents_.emplace(par.seq, std::move(par)).first->second;
}

Ns Core::predicted_time(int kernel, std::int64_t blocks) const {
  auto plan = plans_.find(kernel);
  if (plan != plans_.end() && blocks == plan->second.blocks_per_slice)
    return plan->second.predicted_slice_time;
  return exec_time_model(sc_.gpu, sc_.kernels[kernel], blocks, 0.0, opts_.rounding);
}

void Core::start_ticks(Ns at) {
  if (lp_tasks_.empty()) return;
  ++generation_;
  slices_since_resync_ = 0;
  resync_pending_ = false;
  tick_deferred_ = false;
  eq_.push(at, kPrioLp, -1, EvType::TickLaunch, 0, generation_);
}

void Core::tick() {
  if (p_flag_ || lp_tasks_.empty()) return;
  if (lp_outstanding_ >= 2) {  // one running + one pending: wait for a completion
    tick_deferred_ = true;
    return;
  }
  const int n_lp = static_cast<int>(lp_tasks_.size());
  const int task = lp_tasks_[tick_rr_ % n_lp];
  tick_rr_ = (tick_rr_ + 1) % n_lp;
  Parent& par = next_parent(task);
  if (par.pending.empty()) return;
  const GridBox box = par.pending.front();
  par.pending.pop_front();
  const bool consolidated = par.consolidated_boxes > 0;
  if (consolidated) --par.consolidated_boxes;
  const Ns predicted = predicted_time(par.kernel, box.blocks());
  const int id = make_instance(par.task, par.kernel, box, par.uid, Priority::Low, consolidated, par.seq);
  issue(id, now_);
  ++lp_outstanding_;
  if (++slices_since_resync_ >= sc_.sched.resync_every) {
    slices_since_resync_ = 0;
    resync_pending_ = true;  // the next launch resumes from the drain sync
    return;
  }
  eq_.push(now_ + tick_interval(predicted, sc_.gpu.launch_overhead), kPrioLp, -1, EvType::TickLaunch,
           0, generation_);
}

void Core::consolidate_for_large_bubble() {
  const Ns interval = predictor_.predict();
  for (const int ti : lp_tasks_) {
    Parent& par = next_parent(ti);
    if (par.pending.size() <= 1) continue;
    const KernelSpec& ks = sc_.kernels[par.kernel];
    const std::vector<GridBox> pending(par.pending.begin(), par.pending.end());
    const ExecOracle oracle = oracle_for(par.kernel);
    const std::int64_t take = consolidation_prefix(
        static_cast<std::int64_t>(pending.size()), interval, sc_.sched.safety_factor,
        [&](std::int64_t cnt) {
          std::int64_t blocks = 0;
          for (std::int64_t j = 0; j < cnt; ++j) blocks += pending[j].blocks();
          return oracle(blocks);
        });
    if (take <= 1) continue;
    const std::vector<GridBox> merged =
        consolidate(ks.name, ks.grid, std::vector<GridBox>(pending.begin(), pending.begin() + take));
    par.pending.assign(merged.begin(), merged.end());
    par.pending.insert(par.pending.end(), pending.begin() + take, pending.end());
    par.consolidated_boxes = static_cast<int>(merged.size());
    emit(now_, EventKind::Launch, tasks_[ti].stream, kernels_[par.kernel].name_id, Detail::Consolidate,
         take, static_cast<std::int64_t>(merged.size()));
  }
}

// ---------------------------------------------------------------- comparators
void Core::free_run_issue(int task) {
  Parent& par = next_parent(task);
  if (par.pending.empty()) return;
  const GridBox box = par.pending.front();
  par.pending.pop_front();
  issue(make_instance(par.task, par.kernel, box, par.uid, Priority::Low, false, par.seq), now_);
}

void Core::reef_refill(Ns at) {
  if (!traits_.reef || lp_tasks_.empty()) return;
  while (reef_outstanding_ < sc_.reef.queue_cap) {
    if (!reef_evicted_.empty()) {
      // Evicted kernels restart from block 0 with their original uid.
      const int old = reef_evicted_.front();
      reef_evicted_.pop_front();
      const Instance src = instances_[old];
      issue(make_instance(src.task, src.kernel, src.box, src.uid, Priority::Low, false, src.parent), at,
            true);
    } else {
      const int n_lp = static_cast<int>(lp_tasks_.size());
      const int task = lp_tasks_[reef_rr_ % n_lp];
      reef_rr_ = (reef_rr_ + 1) % n_lp;
      Parent& par = next_parent(task);
      if (par.pending.empty()) return;
      const GridBox box = par.pending.front();
      par.pending.pop_front();
      issue(make_instance(task, par.kernel, box, par.uid, Priority::Low, false, par.seq), at);
    }
    ++reef_outstanding_;
  }
}

bool Core::reef_hp_gate_closed() const {
  for (const int id : lp_active_)
    if (instances_[id].state == InstState::Running) return true;  // LP still draining
  return now_ < reef_gate_;
}

void Core::reef_on_flag() {
  // The oldest running LP kernel completes; queued ones quit at their entry flag check;
  // other running ones are doomed and evicted once their in-flight waves drain.
  int head = -1;
  for (const int id : lp_active_) {
    const Instance& i = instances_[id];
    if (i.state == InstState::Running && !i.doomed) {
      head = id;
      break;
    }
  }
  int evicted = 0;
  const std::vector<int> snapshot = lp_active_;
  for (const int id : snapshot) {
    if (id == head) continue;
    Instance& i = instances_[id];
    if (i.state == InstState::Queued || i.state == InstState::Transit) {
      evict(i, now_);
      ++evicted;
    } else if (i.state == InstState::Running && !i.doomed) {
      i.doomed = true;
      if (i.waves_in_flight == 0) {
        evict(i, now_);
        ++evicted;
      }
    }
  }
  if (evicted == 0) return;
  const Ns gate = now_ + static_cast<Ns>(evicted) * sc_.reef.evict_cost_per_kernel;
  if (gate > reef_gate_) {
    reef_gate_ = gate;
    eq_.push(gate, kPrioInfra, -1, EvType::Poke, 0, 0);
  }
}

// ---------------------------------------------------------------- main loop
RunArtifacts Core::run() {
  setup();
  while (!eq_.empty()) {
    const Event ev = eq_.top();
    if (ev.ts > sc_.horizon) break;
    eq_.pop();
    now_ = ev.ts;
    ++events_;
    switch (ev.type) {
      case EvType::RequestArrival: request_arrival(ev.a, static_cast<std::size_t>(ev.b)); break;
      case EvType::BubbleOver: bubble_over(ev.a, ev.b); break;
      case EvType::KernelArrive: dev_.arrive(ev.a); break;
      case EvType::WaveDone: dev_.wave_done(ev.a, ev.b); break;
      case EvType::TickLaunch:
        if (ev.b == generation_) tick();
        break;
      case EvType::LargeBubbleCheck: large_bubble_check(ev.b); break;
      case EvType::Poke: dev_.dispatch(); break;
      case EvType::UtilTick: {
        UtilSample s;
        s.ts = now_;
        s.sm_active = static_cast<double>(dev_.busy_threads()) / static_cast<double>(dev_.total_threads());
        s.hbm_bw = std::min(1.0, dev_.bw_demand(now_) / sc_.gpu.hbm_bandwidth);
        art_.util_samples.push_back(s);
        eq_.push(now_ + opts_.util_sample_period, kPrioInfra, -1, EvType::UtilTick, 0, 0);
        break;
      }
      case EvType::ProbeTick: {  // engine.hpp:1263-1276: 10 ms while any link is congested
        CongestionTable& links = mem_->congestion();
        for (std::size_t l = 0; l < links.size(); ++l) {
          const double score = links.probe(static_cast<int>(l), now_);
          emit(now_, EventKind::Probe, -1, 0, Detail::Probe, static_cast<std::int64_t>(l), 0, score);
        }
        eq_.push(now_ + (links.any_score_above(1.2) ? ms(10) : ms(100)), kPrioInfra, -1, EvType::ProbeTick, 0, 0);
        break;
      }
    }
  }
  if (eq_.empty()) {  // the queue may only run dry when no serving task holds work
    for (const TaskRt& t : tasks_) {
      if (t.spec->priority != Priority::High || !t.busy) continue;
      std::ostringstream dump;
      dump << "engine deadlock: task '" << t.spec->name << "' busy with request " << t.request
           << " at t=" << now_ << "; stream queues:";
      for (std::size_t s = 0; s < dev_.streams.size(); ++s)
        dump << " s" << s << "=" << dev_.streams[s].queue.size();
      throw EngineError(dump.str());
    }
  }
  dev_.note_occupancy(sc_.horizon);
  for (const Instance& i : instances_) {
    if (i.state != InstState::Running && i.state != InstState::Queued && i.state != InstState::Transit)
      continue;
    const std::int64_t undone = i.blocks_dispatched - i.blocks_done;
    (i.prio == Priority::High ? art_.hp_blocks_in_flight_at_cutoff : art_.lp_blocks_in_flight_at_cutoff) +=
        undone;
  }
  art_.sm_active_fraction = dev_.busy_integral() /
                            (static_cast<double>(dev_.total_threads()) * static_cast<double>(sc_.horizon));
  art_.timeline.finalize();
  std::stable_sort(art_.api_rows.begin(), art_.api_rows.end(),
                   [](const ApiTraceRow& a, const ApiTraceRow& b) { return a.ts_start < b.ts_start; });
  return art_;
}

}  // namespace

// ---------------------------------------------------------------- public API
struct Engine::Impl {
  ScenarioSpec sc;
  Policy policy;
  EngineOptions opts;
  std::uint64_t events = 0;
};

Engine::Engine(ScenarioSpec scenario, Policy policy, EngineOptions opts)
    : impl_(std::make_unique<Impl>(Impl{std::move(scenario), policy, std::move(opts), 0})) {
  impl_->sc.validate();
}
Engine::Engine(Engine&&) noexcept = default;
Engine& Engine::operator=(Engine&&) noexcept = default;
Engine::~Engine() = default;

RunArtifacts Engine::run() {
  Core core(impl_->sc, impl_->policy, impl_->opts);
  RunArtifacts art = core.run();
  impl_->events = core.events();
  return art;
}

std::uint64_t Engine::events_processed() const { return impl_->events; }

RunArtifacts run_scenario(const ScenarioSpec& sc, Policy policy, EngineOptions opts) {
  Engine eng(sc, policy, std::move(opts));
  return eng.run();
}

}  // namespace microslice
