// Decision log (Timeline) and host-side observability records.
// Reference: /root/reference/proj/include/microslice/events.hpp:14-126.
//
// Storage is B200-native-framework style rather than a vector of string pairs: the
// log is a flat array of 48-byte typed records (kind, stream, interned kernel name,
// detail format + integer / float payload).  Text is produced only when the log is
// written (NDJSON / CSV) or when SimEvent views are requested.  The rendered bytes
// are identical to the reference's writer (events.hpp:86-107), which is what the
// decision-log parity test compares.
#pragma once

#include <cstdint>
#include <memory>
#include <ostream>
#include <string>
#include <vector>

#include "microslice/common.hpp"

namespace microslice {

enum class EventKind {
  Launch,
  DispatchWave,
  WaveDone,
  KernelDone,
  SyncBegin,
  SyncEnd,
  PreemptBegin,
  PreemptEnd,
  Evict,
  Relaunch,
  BubbleBegin,
  BubbleEnd,
  MemFault,
  Probe,
};

const char* event_kind_name(EventKind k);

struct SimEvent {
  Ns ts = 0;
  EventKind kind = EventKind::Launch;
  int stream = -1;
  std::string kernel;
  std::string detail;
};

/// Typed detail payloads; each renders to the reference's free-form detail string.
enum class Detail : std::uint8_t {
  Text,           // interned string (a)
  Inst,           // inst=a
  InstWave,       // inst=a;n=b;stretch=g
  Delay,          // delay_ns=a[;consolidated=1 if b]
  InstN,          // inst=a;n=b
  InstBlocks,     // inst=a;blocks=b
  InstWasted,     // inst=a;wasted=b
  Hint,           // hint=<interned a>
  Consolidate,    // consolidate=a->b
  Chunk,          // chunk=a
  MemFault,       // tier=<peer if b == 1 else dram>;chunk=a
  Probe,          // link=a;score=g
};

struct TimelineRecord {
  Ns ts = 0;
  std::int64_t a = 0;
  std::int64_t b = 0;
  double g = 0.0;
  std::int32_t stream = -1;
  std::int32_t kernel = 0;  // interned; 0 == ""
  EventKind kind = EventKind::Launch;
  Detail detail = Detail::Text;
};

class Timeline {
 public:
  Timeline();
  Timeline(const Timeline&);
  Timeline& operator=(const Timeline&);
  Timeline(Timeline&&) noexcept;
  Timeline& operator=(Timeline&&) noexcept;
  ~Timeline();

  // --- reference API (events.hpp:64-110) ---
  void emit(Ns ts, EventKind kind, int stream, std::string kernel, std::string detail = {});
  /// Stable sort by timestamp only: same-ts events keep causal emission order.
  void finalize();
  bool is_monotonic() const;
  const std::vector<SimEvent>& events() const;  // materialised lazily
  std::size_t size() const { return recs_.size(); }
  void write_ndjson(std::ostream& os) const;
  std::string to_ndjson() const;
  void write_csv(std::ostream& os) const;

  // --- typed fast path used by the scheduler core ---
  std::int32_t intern(const std::string& s);
  const std::string& str(std::int32_t id) const;
  void record(const TimelineRecord& r) {
    recs_.push_back(r);
    cache_valid_ = false;
  }
  const std::vector<TimelineRecord>& records() const { return recs_; }
  void reserve(std::size_t n) { recs_.reserve(n); }
  /// Render one record's detail text (reference byte format).
  std::string detail_text(const TimelineRecord& r) const;
  /// FNV-1a 64 over the NDJSON bytes, computed without materialising the text.
  std::uint64_t ndjson_fnv1a() const;
  std::uint64_t ndjson_bytes() const;

 private:
  struct Strings;
  std::vector<TimelineRecord> recs_;
  std::unique_ptr<Strings> strings_;
  mutable std::vector<SimEvent> cache_;
  mutable bool cache_valid_ = false;
};

struct ApiTraceRow {
  Ns ts_start = 0;
  Ns ts_end = 0;
  std::string api_tag;
  std::int64_t correlation = 0;
};

struct UtilSample {
  Ns ts = 0;
  double sm_active = 0.0;
  double hbm_bw = 0.0;
};

}  // namespace microslice
