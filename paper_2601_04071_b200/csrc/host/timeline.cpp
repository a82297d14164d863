// Timeline storage and rendering.  Reference byte format: events.hpp:86-107.
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <sstream>
#include <unordered_map>

#include "microslice/events.hpp"

namespace microslice {

const char* event_kind_name(EventKind k) {
  static const char* const kNames[] = {
      "launch",        "dispatch_wave", "wave_done",   "kernel_done", "sync_begin",
      "sync_end",      "preempt_begin", "preempt_end", "evict",       "relaunch",
      "bubble_begin",  "bubble_end",    "mem_fault",   "probe"};
  const auto i = static_cast<unsigned>(k);
  return i < sizeof(kNames) / sizeof(kNames[0]) ? kNames[i] : "?";
}

struct Timeline::Strings {
  std::vector<std::string> table{std::string()};
  std::unordered_map<std::string, std::int32_t> index{{std::string(), 0}};
};

Timeline::Timeline() : strings_(std::make_unique<Strings>()) {}
Timeline::Timeline(const Timeline& o)
    : recs_(o.recs_), strings_(std::make_unique<Strings>(*o.strings_)) {}
Timeline& Timeline::operator=(const Timeline& o) {
  if (this != &o) {
    recs_ = o.recs_;
    strings_ = std::make_unique<Strings>(*o.strings_);
    cache_.clear();
    cache_valid_ = false;
  }
  return *this;
}
Timeline::Timeline(Timeline&&) noexcept = default;
Timeline& Timeline::operator=(Timeline&&) noexcept = default;
Timeline::~Timeline() = default;

std::int32_t Timeline::intern(const std::string& s) {
  auto [it, fresh] = strings_->index.try_emplace(s, static_cast<std::int32_t>(strings_->table.size()));
  if (fresh) strings_->table.push_back(s);
  return it->second;
}

const std::string& Timeline::str(std::int32_t id) const { return strings_->table[id]; }

void Timeline::emit(Ns ts, EventKind kind, int stream, std::string kernel, std::string detail) {
  TimelineRecord r;
  r.ts = ts;
  r.kind = kind;
  r.stream = stream;
  r.kernel = intern(kernel);
  r.detail = Detail::Text;
  r.a = intern(detail);
  record(r);
}

void Timeline::finalize() {
  std::stable_sort(recs_.begin(), recs_.end(),
                   [](const TimelineRecord& a, const TimelineRecord& b) { return a.ts < b.ts; });
  cache_valid_ = false;
}

bool Timeline::is_monotonic() const {
  return std::is_sorted(recs_.begin(), recs_.end(),
                        [](const TimelineRecord& a, const TimelineRecord& b) { return a.ts < b.ts; });
}

namespace {

void put_int(std::string& out, std::int64_t v) {
  char buf[24];
  auto res = std::to_chars(buf, buf + sizeof buf, v);
  out.append(buf, res.ptr);
}

// std::ostream default float formatting == printf("%.6g").
void put_g(std::string& out, double v) {
  char buf[40];
  const int n = std::snprintf(buf, sizeof buf, "%g", v);
  out.append(buf, static_cast<std::size_t>(n));
}

}  // namespace

static void render_detail(const Timeline& tl, const TimelineRecord& r, std::string& out) {
  switch (r.detail) {
    case Detail::Text:
      out += tl.str(static_cast<std::int32_t>(r.a));
      return;
    case Detail::Inst:
      out += "inst=";
      put_int(out, r.a);
      return;
    case Detail::InstWave:
      out += "inst=";
      put_int(out, r.a);
      out += ";n=";
      put_int(out, r.b);
      out += ";stretch=";
      put_g(out, r.g);
      return;
    case Detail::Delay:
      out += "delay_ns=";
      put_int(out, r.a);
      if (r.b) out += ";consolidated=1";
      return;
    case Detail::InstN:
      out += "inst=";
      put_int(out, r.a);
      out += ";n=";
      put_int(out, r.b);
      return;
    case Detail::InstBlocks:
      out += "inst=";
      put_int(out, r.a);
      out += ";blocks=";
      put_int(out, r.b);
      return;
    case Detail::InstWasted:
      out += "inst=";
      put_int(out, r.a);
      out += ";wasted=";
      put_int(out, r.b);
      return;
    case Detail::Hint:
      out += "hint=";
      out += tl.str(static_cast<std::int32_t>(r.a));
      return;
    case Detail::Consolidate:
      out += "consolidate=";
      put_int(out, r.a);
      out += "->";
      put_int(out, r.b);
      return;
    case Detail::Chunk:
      out += "chunk=";
      put_int(out, r.a);
      return;
    case Detail::MemFault:
      out += r.b == 1 ? "tier=peer;chunk=" : "tier=dram;chunk=";
      put_int(out, r.a);
      return;
    case Detail::Probe:
      out += "link=";
      put_int(out, r.a);
      out += ";score=";
      put_g(out, r.g);
      return;
  }
}

std::string Timeline::detail_text(const TimelineRecord& r) const {
  std::string s;
  render_detail(*this, r, s);
  return s;
}

static void render_ndjson_line(const Timeline& tl, const TimelineRecord& r, std::string& out) {
  out += "{\"ts_ns\":";
  put_int(out, r.ts);
  out += ",\"kind\":\"";
  out += event_kind_name(r.kind);
  out += "\",\"stream\":";
  put_int(out, r.stream);
  out += ",\"kernel\":\"";
  out += tl.str(r.kernel);
  out += "\",\"detail\":\"";
  render_detail(tl, r, out);
  out += "\"}\n";
}

const std::vector<SimEvent>& Timeline::events() const {
  if (!cache_valid_) {
    cache_.clear();
    cache_.reserve(recs_.size());
    for (const TimelineRecord& r : recs_)
      cache_.push_back(SimEvent{r.ts, r.kind, r.stream, str(r.kernel), detail_text(r)});
    cache_valid_ = true;
  }
  return cache_;
}

void Timeline::write_ndjson(std::ostream& os) const {
  std::string buf;
  buf.reserve(1 << 16);
  for (const TimelineRecord& r : recs_) {
    render_ndjson_line(*this, r, buf);
    if (buf.size() > (1u << 15)) {
      os.write(buf.data(), static_cast<std::streamsize>(buf.size()));
      buf.clear();
    }
  }
  os.write(buf.data(), static_cast<std::streamsize>(buf.size()));
}

std::string Timeline::to_ndjson() const {
  std::ostringstream os;
  write_ndjson(os);
  return os.str();
}

void Timeline::write_csv(std::ostream& os) const {
  os << "ts_ns,kind,stream,kernel,detail\n";
  std::string line;
  for (const TimelineRecord& r : recs_) {
    line.clear();
    put_int(line, r.ts);
    line += ',';
    line += event_kind_name(r.kind);
    line += ',';
    put_int(line, r.stream);
    line += ',';
    line += str(r.kernel);
    line += ',';
    render_detail(*this, r, line);
    line += '\n';
    os << line;
  }
}

std::uint64_t Timeline::ndjson_fnv1a() const {
  std::uint64_t h = 14695981039346656037ULL;
  std::string line;
  for (const TimelineRecord& r : recs_) {
    line.clear();
    render_ndjson_line(*this, r, line);
    for (const char c : line) h = (h ^ static_cast<unsigned char>(c)) * 1099511628211ULL;
  }
  return h;
}

std::uint64_t Timeline::ndjson_bytes() const {
  std::uint64_t n = 0;
  std::string line;
  for (const TimelineRecord& r : recs_) {
    line.clear();
    render_ndjson_line(*this, r, line);
    n += line.size();
  }
  return n;
}

}  // namespace microslice
