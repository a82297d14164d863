// Memory tier: chunk placement + link congestion.
// Semantics follow /root/reference/proj/include/microslice/memory.hpp (cited per
// function); the floating-point expressions keep the reference's evaluation order so the
// replay decision log stays bit-exact (tests/test_replay_parity.py, memory corpus).
#include "microslice/memory.hpp"

#include <algorithm>

namespace microslice {

std::string tier_name(Tier t) {
  switch (t) {
    case Tier::Local: return "local";
    case Tier::Peer: return "peer";
    case Tier::Dram: return "dram";
  }
  return "?";
}

// ------------------------------------------------------------------ CongestionTable
// memory.hpp:36-130

void CongestionTable::init(const std::vector<NvlinkPeer>& peers, double probe_bytes) {
  probe_bytes_ = probe_bytes;
  links_.assign(peers.size(), Link{});
  for (std::size_t i = 0; i < peers.size(); ++i) links_[i].cfg = peers[i];
}

void CongestionTable::calibrate() {  // memory.hpp:60-67: zero-load probe latency
  for (std::size_t i = 0; i < links_.size(); ++i) {
    Link& l = links_[i];
    l.t_base = live_ ? std::max<Ns>(1, live_(static_cast<int>(i), static_cast<std::int64_t>(probe_bytes_)))
                     : l.cfg.baseline_latency + static_cast<Ns>(probe_bytes_ / l.cfg.bandwidth * 1e9);
    l.calibrated = true;
  }
}

void CongestionTable::add_transfer(int link, double rate, Ns end_ts) {
  links_.at(static_cast<std::size_t>(link)).active.emplace_back(end_ts, rate);
}

double CongestionTable::load(int link, Ns now) {  // memory.hpp:73-85
  Link& l = links_.at(static_cast<std::size_t>(link));
  double sum = l.cfg.background_load;
  std::size_t keep = 0;
  for (std::size_t i = 0; i < l.active.size(); ++i) {
    if (l.active[i].first <= now) continue;  // finished: retire
    sum += l.active[i].second;
    l.active[keep++] = l.active[i];
  }
  l.active.resize(keep);
  return sum;
}

Ns CongestionTable::transfer_time(int link, std::int64_t bytes, Ns now) {  // memory.hpp:88-94
  const Link& l = links_.at(static_cast<std::size_t>(link));
  const double zero_load =
      static_cast<double>(l.cfg.baseline_latency) + static_cast<double>(bytes) / l.cfg.bandwidth * 1e9;
  const double bw = l.cfg.bandwidth;
  const double slow = 1.0 + load(link, now) / bw;
  return static_cast<Ns>(zero_load * slow);
}

double CongestionTable::probe(int link, Ns now) {  // memory.hpp:96-109
  const Link& l = links_.at(static_cast<std::size_t>(link));
  if (!l.calibrated)
    throw ValidationError("memory.probe",
                          "link " + std::to_string(link) + " probed before baseline calibration");
  const Ns t_now = live_ ? live_(link, static_cast<std::int64_t>(probe_bytes_))
                        : transfer_time(link, static_cast<std::int64_t>(probe_bytes_), now);
  const double score = static_cast<double>(t_now) / static_cast<double>(l.t_base);
  if (scores_.size() < links_.size()) scores_.resize(links_.size(), 1.0);
  scores_[static_cast<std::size_t>(link)] = score;
  return score;
}

double CongestionTable::last_score(int link) const {
  return link < static_cast<int>(scores_.size()) ? scores_[static_cast<std::size_t>(link)] : 1.0;
}

bool CongestionTable::any_score_above(double v) const {
  return std::any_of(scores_.begin(), scores_.end(), [v](double s) { return s > v; });
}

// ------------------------------------------------------------------ MemoryManager
// memory.hpp:138-323

MemoryManager::MemoryManager(const GpuConfig& gpu, const MemParams& params)
    : MemoryManager(gpu, params, LiveProbe{}) {}

MemoryManager::MemoryManager(const GpuConfig& gpu, const MemParams& params, LiveProbe live)
    : gpu_(gpu), params_(params) {
  local_capacity_ = static_cast<std::int64_t>(params.hbm_gb * 1e9 / kChunkBytes);
  const std::size_t n = gpu.nvlink_peers.size();
  peer_capacity_.assign(n, 0);
  peer_used_.assign(n, 0);
  for (std::size_t i = 0; i < n && i < params.peer_free_gb.size(); ++i)
    peer_capacity_[i] = static_cast<std::int64_t>(params.peer_free_gb[i] * 1e9 / kChunkBytes);
  links_.init(gpu.nvlink_peers, params.probe_mb * 1024 * 1024);
  links_.set_live_probe(std::move(live));
  links_.calibrate();
}

std::vector<std::int64_t> MemoryManager::chunks_of(int task) const {
  std::vector<std::int64_t> ids;
  for (std::size_t i = 0; i < chunks_.size(); ++i)
    if (chunks_[i].owner_task == task) ids.push_back(static_cast<std::int64_t>(i));
  return ids;
}

double MemoryManager::off_device_fraction(int task) const {
  std::int64_t mine = 0, away = 0;
  for (const Chunk& c : chunks_) {
    if (c.owner_task != task) continue;
    ++mine;
    away += c.tier != Tier::Local;
  }
  return mine ? static_cast<double>(away) / static_cast<double>(mine) : 0.0;
}

// memory.hpp:182-207.  Contention-first: the least-congested peer with room whose probe
// score is under the threshold (every candidate is probed, which refreshes its score);
// else DRAM.  Round-robin: the next peer with room, ignoring congestion; else DRAM.
MemoryManager::Destination MemoryManager::evict_select(Ns now) {
  const int n = static_cast<int>(peer_capacity_.size());
  if (params_.eviction == EvictionPolicy::ContentionFirst) {
    Destination best{Tier::Dram, -1};
    double best_score = 0.0;
    for (int i = 0; i < n; ++i) {
      if (peer_used_[i] >= peer_capacity_[i]) continue;
      const double s = links_.probe(i, now);
      if (s >= params_.score_threshold) continue;
      if (best.peer < 0 || s < best_score) {
        best = {Tier::Peer, i};
        best_score = s;
      }
    }
    return best;
  }
  for (int step = 0; step < n; ++step) {
    const int i = (rr_next_ + step) % n;
    if (peer_used_[i] < peer_capacity_[i]) {
      rr_next_ = (i + 1) % n;
      return {Tier::Peer, i};
    }
  }
  return {Tier::Dram, -1};
}

void MemoryManager::place(Chunk& c, const Destination& d) {
  c.tier = d.tier;
  c.peer = d.peer;
  if (d.tier == Tier::Peer) ++peer_used_[static_cast<std::size_t>(d.peer)];
}

// memory.hpp:261-279: an unpinned local chunk leaves HBM for evict_select()'s target.
void MemoryManager::move_out(std::int64_t id, Ns now, std::vector<ChunkRelocation>* moves) {
  Chunk& c = chunks_[static_cast<std::size_t>(id)];
  if (c.pinned) throw EngineError("memory: attempted to evict a pinned chunk");
  ChunkRelocation m;
  m.chunk_id = id;
  m.from = c.tier;
  m.from_peer = c.peer;
  const Destination d = evict_select(now);
  if (c.tier == Tier::Local) --local_used_;
  place(c, d);
  m.to = c.tier;
  m.to_peer = c.peer;
  if (moves) moves->push_back(m);
}

// memory.hpp:212-243
std::vector<std::int64_t> MemoryManager::allocate(int task, Priority prio, std::int64_t bytes, Ns now,
                                                  std::vector<ChunkRelocation>* moves) {
  const std::int64_t count = (bytes + kChunkBytes - 1) / kChunkBytes;
  const bool high = prio == Priority::High;
  std::vector<std::int64_t> ids;
  ids.reserve(static_cast<std::size_t>(std::max<std::int64_t>(count, 0)));
  for (std::int64_t k = 0; k < count; ++k) {
    Chunk c;
    c.owner_task = task;
    c.pinned = high;
    if (local_used_ < local_capacity_) {
      ++local_used_;
    } else if (high) {
      // displace the lowest-id unpinned local chunk (ids below scan_from_ never qualify
      // again: chunks only leave HBM, and new ones are appended)
      std::int64_t victim = -1;
      for (std::int64_t i = scan_from_; i < static_cast<std::int64_t>(chunks_.size()); ++i) {
        const Chunk& v = chunks_[static_cast<std::size_t>(i)];
        if (v.tier == Tier::Local && !v.pinned) {
          victim = i;
          break;
        }
      }
      if (victim < 0) throw ValidationError("memory.allocate", "local HBM exhausted by pinned chunks");
      scan_from_ = victim + 1;
      move_out(victim, now, moves);
      ++local_used_;
    } else {
      place(c, evict_select(now));
    }
    chunks_.push_back(c);
    ids.push_back(static_cast<std::int64_t>(chunks_.size()) - 1);
  }
  return ids;
}

void MemoryManager::release(const std::vector<std::int64_t>& ids) {
  for (std::int64_t id : ids) {
    Chunk& c = chunks_.at(static_cast<std::size_t>(id));
    if (c.owner_task < 0) continue;
    if (c.tier == Tier::Local) --local_used_;
    if (c.tier == Tier::Peer) --peer_used_[static_cast<std::size_t>(c.peer)];
    c = Chunk{};
    c.tier = Tier::Dram;  // never a displacement victim again
  }
}

// memory.hpp:313-321: one chunk over the first peer link at zero load (or 2 us + 600 GB/s)
Ns MemoryManager::nominal_peer_chunk_time() const {
  if (gpu_.nvlink_peers.empty())
    return us(2) + static_cast<Ns>(static_cast<double>(kChunkBytes) / 600e9 * 1e9);
  const NvlinkPeer& p = gpu_.nvlink_peers.front();
  return p.baseline_latency + static_cast<Ns>(static_cast<double>(kChunkBytes) / p.bandwidth * 1e9);
}

// memory.hpp:247-268
AccessResult MemoryManager::access(std::int64_t chunk_id, Ns now) {
  const Chunk& c = chunks_.at(static_cast<std::size_t>(chunk_id));
  AccessResult r;
  r.tier = c.tier;
  r.peer = c.peer;
  if (c.tier == Tier::Peer)
    r.latency = links_.transfer_time(c.peer, kChunkBytes, now);
  else if (c.tier == Tier::Dram)
    r.latency = static_cast<Ns>(static_cast<double>(nominal_peer_chunk_time()) * params_.dram_factor);
  return r;
}

}  // namespace microslice
