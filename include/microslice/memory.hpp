// Memory tier: 2 MB chunk placement across local HBM, NVLink-peer HBM and host DRAM,
// with HP pinning, ping-probe congestion scores and contention-first (or round-robin)
// eviction of LP chunks.  SURVEY.md §8f next #4; reference semantics
// /root/reference/proj/include/microslice/memory.hpp:15-323 and its engine hooks
// (engine.hpp:396-411 allocation at setup, 798-801 per-wave access cost, 1199-1229
// wave_memory_extra, 1263-1276 ProbeTick).  The public surface is source-compatible with
// the reference; implementation in paper_2601_04071_b200/csrc/host/memory.cpp.
//
// On B200 the same placement decisions drive the live tier (include/ms_tier.h,
// csrc/live/mem_tier.cpp): chunks are real 2 MB VMM allocations in local HBM, a peer's
// HBM (NVLink 5 / NVSwitch) or pinned host DRAM, mapped into one virtual range per buffer.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <utility>
#include <vector>

#include "microslice/common.hpp"
#include "microslice/model.hpp"

namespace microslice {

constexpr std::int64_t kChunkBytes = 2ll * 1024 * 1024;  // placement granularity

enum class Tier { Local, Peer, Dram };

std::string tier_name(Tier t);  // "local" | "peer" | "dram"

struct Chunk {
  int owner_task = -1;
  Tier tier = Tier::Local;
  int peer = -1;  // valid for Tier::Peer
  bool pinned = false;
};

struct ChunkRelocation {
  std::int64_t chunk_id = 0;
  Tier from = Tier::Local;
  int from_peer = -1;
  Tier to = Tier::Local;
  int to_peer = -1;
};

/// Live link measurement: ns to move `bytes` over link `link` now (B200 tier: a timed
/// copy).  Absent in replay, where latency follows the load model below.
using LiveProbe = std::function<Ns(int link, std::int64_t bytes)>;

/// Per-link congestion: a calibrated zero-load probe latency t_base and the load seen
/// through registered transfers (+ configured background traffic); score = t_now / t_base.
/// With a LiveProbe, t_base and t_now are measured instead (extension for the live tier).
class CongestionTable {
 public:
  struct Link {
    NvlinkPeer cfg;
    Ns t_base = 0;
    bool calibrated = false;
    std::vector<std::pair<Ns, double>> active;  // (end_ts, bytes/s), registration order
  };

  void init(const std::vector<NvlinkPeer>& peers, double probe_bytes);
  void set_live_probe(LiveProbe f) { live_ = std::move(f); }
  std::size_t size() const { return links_.size(); }
  const Link& link(int i) const { return links_.at(static_cast<std::size_t>(i)); }

  void calibrate();
  void add_transfer(int link, double rate, Ns end_ts);
  /// bytes/s on `link` at `now` (expired transfers are retired).
  double load(int link, Ns now);
  /// Latency of moving `bytes` over `link` under its current load.
  Ns transfer_time(int link, std::int64_t bytes, Ns now);
  /// Ping-probe: score of `link` now (recorded for last_score / any_score_above).
  double probe(int link, Ns now);
  double last_score(int link) const;
  bool any_score_above(double v) const;

 private:
  double probe_bytes_ = 4.0 * 1024 * 1024;
  std::vector<Link> links_;
  std::vector<double> scores_;
  LiveProbe live_;
};

struct AccessResult {
  Tier tier = Tier::Local;
  int peer = -1;
  Ns latency = 0;  // extra time the access adds to the wave
};

class MemoryManager {
 public:
  MemoryManager(const GpuConfig& gpu, const MemParams& params);
  /// Live tier: link latencies come from `live` (calibrated at construction).
  MemoryManager(const GpuConfig& gpu, const MemParams& params, LiveProbe live);

  struct Destination {
    Tier tier = Tier::Dram;
    int peer = -1;
  };

  CongestionTable& congestion() { return links_; }
  const std::vector<Chunk>& chunks() const { return chunks_; }
  std::int64_t local_used() const { return local_used_; }
  std::int64_t local_capacity() const { return local_capacity_; }
  std::vector<std::int64_t> chunks_of(int task) const;
  double off_device_fraction(int task) const;

  /// Where the next evicted / spilled LP chunk goes.
  Destination evict_select(Ns now);
  /// Chunks for `bytes` of `task`.  HP chunks are pinned local and displace unpinned LP
  /// chunks when HBM is full; LP chunks spill to evict_select() once HBM is full.
  std::vector<std::int64_t> allocate(int task, Priority prio, std::int64_t bytes, Ns now,
                                     std::vector<ChunkRelocation>* moves = nullptr);
  /// Extra latency of a kernel of the owner touching `chunk_id` now.
  AccessResult access(std::int64_t chunk_id, Ns now);
  bool chunk_pinned(std::int64_t id) const { return chunks_.at(static_cast<std::size_t>(id)).pinned; }
  /// Return chunks to their tier (live tier: ms_tier_free).  Released chunks keep their
  /// ids with owner_task = -1 and count against no tier.
  void release(const std::vector<std::int64_t>& ids);

 private:
  void place(Chunk& c, const Destination& d);
  void move_out(std::int64_t id, Ns now, std::vector<ChunkRelocation>* moves);
  Ns nominal_peer_chunk_time() const;

  GpuConfig gpu_;
  MemParams params_;
  std::int64_t local_capacity_ = 0, local_used_ = 0;
  std::vector<std::int64_t> peer_capacity_, peer_used_;
  int rr_next_ = 0;
  std::int64_t scan_from_ = 0;  // no unpinned local chunk below this id
  std::vector<Chunk> chunks_;
  CongestionTable links_;
};

}  // namespace microslice
