// Live memory tier on B200 (include/ms_tier.h).
//
// Every tier buffer is one reserved virtual range whose 2 MB granules are CUDA VMM
// allocations placed by microslice::MemoryManager (the replay engine's placement code,
// reference memory.hpp:138-323): local HBM, an NVLink peer's HBM (location = peer device,
// access granted to this device), or pinned host DRAM (location = host NUMA node).  LP
// kernels read the range in place — no kernel knows where a chunk lives.  The manager's
// congestion table is fed by live ping-probes: a timed probe_mb copy to a buffer on the
// peer, on a lowest-priority stream, so a probe measures the link under the current load.
//
// Relocation (an HP allocation displacing an LP chunk once the HBM budget is full): the
// chunk's bytes are copied to a new granule at the eviction target through a temporary
// mapping, then the chunk's VA is unmapped and re-mapped onto the new granule.  Physical
// granules are released right after mapping, so unmapping frees them.
#include <cuda.h>
#include <cuda_runtime.h>
#include <time.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "microslice/json.hpp"
#include "microslice/memory.hpp"
#include "ms_tier.h"

extern "C" int ms_internal_fail(int code, const char* what);  // ms_b200.cu: sets ms_last_error
extern "C" int ms_internal_lp_sync(ms_dev* dev);                 // ms_b200.cu: LP stream only

namespace microslice {
namespace {

int64_t mono_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return static_cast<int64_t>(ts.tv_sec) * 1000000000ll + ts.tv_nsec;
}

// Driver VMM entry points, resolved through the runtime (no link-time libcuda dependency).
struct Vmm {
  CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addr_free)(CUdeviceptr, size_t) = nullptr;
  CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) =
      nullptr;
  CUresult (*release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*dev_attr)(int*, CUdevice_attribute, CUdevice) = nullptr;

  bool load() {
    auto get = [](const char* name, void* slot) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return false;
      std::memcpy(slot, &fn, sizeof fn);
      return true;
    };
    return get("cuMemAddressReserve", &reserve) && get("cuMemAddressFree", &addr_free) &&
           get("cuMemCreate", &create) && get("cuMemRelease", &release) && get("cuMemMap", &map) &&
           get("cuMemUnmap", &unmap) && get("cuMemSetAccess", &set_access) &&
           get("cuDeviceGetAttribute", &dev_attr);
  }
};

struct TierError {
  int code;
  std::string what;
};

void ck(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw TierError{MS_E_CUDA, std::string(what) + " failed (CUresult " + std::to_string(r) + ")"};
}
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw TierError{MS_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

struct Buffer {
  CUdeviceptr va = 0;
  size_t bytes = 0;
  std::vector<std::int64_t> ids;
};

}  // namespace
}  // namespace microslice

using namespace microslice;

struct ms_tier {
  ms_dev* dev = nullptr;
  int ordinal = 0;
  int numa = 0;
  Vmm vmm;
  std::vector<int> link_dev;  // peer device ordinal per link
  std::unique_ptr<MemoryManager> mm;
  std::map<std::int64_t, CUdeviceptr> chunk_va;  // live chunk id -> its VA
  std::map<uint64_t, Buffer> buffers;             // by base VA
  cudaStream_t probe_stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  CUdeviceptr probe_src = 0;
  std::vector<CUdeviceptr> probe_dst;  // per link, on the peer
  size_t probe_bytes = 4u << 20;
  int64_t probe_cache_ns = 1'000'000;
  std::vector<std::pair<int64_t, Ns>> probe_last;  // (host ns, measured ns) per link
  ms_tier_stats stats{};

  CUmemAllocationProp prop_for(Tier t, int link) const {
    CUmemAllocationProp p{};
    p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    if (t == Tier::Dram) {
      p.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
      p.location.id = numa;
    } else {
      p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      p.location.id = t == Tier::Peer ? link_dev.at(static_cast<size_t>(link)) : ordinal;
    }
    return p;
  }

  void grant(CUdeviceptr va, size_t bytes) {
    CUmemAccessDesc a{};
    a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    a.location.id = ordinal;
    a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    ck(vmm.set_access(va, bytes, &a, 1), "cuMemSetAccess");
  }

  CUmemGenericAllocationHandle granule(Tier t, int link) {
    const CUmemAllocationProp p = prop_for(t, link);
    CUmemGenericAllocationHandle h;
    ck(vmm.create(&h, kChunkBytes, &p, 0), t == Tier::Dram ? "cuMemCreate(host NUMA)" : "cuMemCreate");
    return h;
  }

  // Back [va, va + kChunkBytes) with a fresh granule on tier (t, link).
  void back(CUdeviceptr va, Tier t, int link) {
    const CUmemGenericAllocationHandle h = granule(t, link);
    const CUresult r = vmm.map(va, kChunkBytes, 0, h, 0);
    vmm.release(h);  // the mapping keeps the granule alive; unmapping frees it
    ck(r, "cuMemMap");
  }

  CUdeviceptr reserve(size_t bytes) {
    CUdeviceptr va = 0;
    ck(vmm.reserve(&va, bytes, kChunkBytes, 0, 0), "cuMemAddressReserve");
    return va;
  }

  // Move displaced chunks to the tiers the manager recorded for them, in three batched
  // phases: new granules mapped side by side in a staging range, one async copy per chunk
  // and a single sync, then each chunk's VA unmapped and re-pointed at its new granule.
  void relocate(const std::vector<ChunkRelocation>& moves) {
    const size_t n = moves.size();
    const int64_t t0 = mono_ns();
    std::vector<CUmemGenericAllocationHandle> hs;
    hs.reserve(n);
    const CUdeviceptr stage = reserve(n * kChunkBytes);
    size_t mapped = 0;
    auto cleanup = [&]() {
      for (size_t i = 0; i < mapped; ++i) vmm.unmap(stage + i * kChunkBytes, kChunkBytes);
      vmm.addr_free(stage, n * kChunkBytes);
      for (CUmemGenericAllocationHandle h : hs) vmm.release(h);
    };
    try {
      for (size_t i = 0; i < n; ++i) {
        hs.push_back(granule(moves[i].to, moves[i].to_peer));
        ck(vmm.map(stage + i * kChunkBytes, kChunkBytes, 0, hs.back(), 0), "cuMemMap");
        ++mapped;
      }
      grant(stage, n * kChunkBytes);
      for (size_t i = 0; i < n; ++i)
        ck(cudaMemcpyAsync(reinterpret_cast<void*>(stage + i * kChunkBytes),
                           reinterpret_cast<void*>(chunk_va.at(moves[i].chunk_id)), kChunkBytes, cudaMemcpyDefault,
                           probe_stream),
           "relocation copy");
      ck(cudaStreamSynchronize(probe_stream), "relocation sync");
      const int64_t t1 = mono_ns();
      for (size_t i = 0; i < n; ++i) {
        const CUdeviceptr va = chunk_va.at(moves[i].chunk_id);
        ck(vmm.unmap(va, kChunkBytes), "cuMemUnmap");
        ck(vmm.map(va, kChunkBytes, 0, hs[i], 0), "cuMemMap");
        grant(va, kChunkBytes);
      }
      stats.relocate_copy_ns += t1 - t0;
      stats.relocate_remap_ns += mono_ns() - t1;
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
    stats.relocations += static_cast<int64_t>(n);
    stats.relocated_bytes += static_cast<int64_t>(n) * kChunkBytes;
  }

  // Timed copy of `bytes` to link's probe buffer on the lowest-priority stream.
  Ns probe_now(int link, std::int64_t bytes) {
    auto& last = probe_last.at(static_cast<size_t>(link));
    const int64_t t = mono_ns();
    if (last.first && t - last.first < probe_cache_ns) return last.second;
    const size_t n = std::min<size_t>(static_cast<size_t>(bytes), probe_bytes);
    ck(cudaEventRecord(ev0, probe_stream), "cudaEventRecord");
    ck(cudaMemcpyAsync(reinterpret_cast<void*>(probe_dst.at(static_cast<size_t>(link))),
                       reinterpret_cast<void*>(probe_src), n, cudaMemcpyDeviceToDevice, probe_stream),
       "probe copy");
    ck(cudaEventRecord(ev1, probe_stream), "cudaEventRecord");
    ck(cudaEventSynchronize(ev1), "probe sync");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, ev0, ev1), "cudaEventElapsedTime");
    ++stats.probes;
    last = {mono_ns(), std::max<Ns>(1, static_cast<Ns>(ms * 1e6))};
    return last.second;
  }

  void free_buffer(Buffer& b) {
    vmm.unmap(b.va, b.bytes);
    vmm.addr_free(b.va, b.bytes);
    for (std::int64_t id : b.ids) chunk_va.erase(id);
    mm->release(b.ids);
  }
};

namespace {

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const TierError& e) {
    return ms_internal_fail(e.code, e.what.c_str());
  } catch (const std::exception& e) {
    return ms_internal_fail(MS_E_ARG, e.what());
  }
}

}  // namespace

extern "C" int ms_tier_open(ms_dev* dev, const char* options_json, ms_tier** out) {
  if (!dev || !out) return ms_internal_fail(MS_E_ARG, "ms_tier_open: null argument");
  return guarded([&]() -> int {
    auto t = std::unique_ptr<ms_tier, int (*)(ms_tier*)>(new ms_tier, ms_tier_close);  // frees partial state
    t->dev = dev;
    ms_dev_info info;
    if (ms_dev_get_info(dev, &info) < 0) return MS_E_ARG;
    t->ordinal = info.ordinal;
    ck(cudaSetDevice(t->ordinal), "cudaSetDevice");
    if (!t->vmm.load()) throw TierError{MS_E_CUDA, "ms_tier_open: CUDA VMM entry points unavailable"};
    const json o = json::parse(options_json ? options_json : "{}");

    int numa = -1;
    t->vmm.dev_attr(&numa, CU_DEVICE_ATTRIBUTE_HOST_NUMA_ID, static_cast<CUdevice>(t->ordinal));
    t->numa = o.value("numa", numa < 0 ? 0 : numa);
    t->probe_bytes = static_cast<size_t>(o.value("probe_mb", 4.0) * 1024 * 1024);
    t->probe_cache_ns = static_cast<int64_t>(o.value("probe_cache_us", 1000.0) * 1000.0);

    size_t free_b = 0, total_b = 0;
    ck(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    GpuConfig gpu;
    gpu.n_sm = info.sm_count;
    MemParams mp;
    mp.enabled = true;
    mp.hbm_gb = o.value("hbm_gb", std::max(0.0, (static_cast<double>(free_b) - 8e9) / 1e9));
    mp.probe_mb = static_cast<double>(t->probe_bytes) / (1024.0 * 1024.0);
    mp.score_threshold = o.value("score_threshold", 1.5);
    const std::string ev = o.value("eviction", std::string("contention_first"));
    if (ev == "contention_first")
      mp.eviction = EvictionPolicy::ContentionFirst;
    else if (ev == "round_robin")
      mp.eviction = EvictionPolicy::RoundRobin;
    else
      throw TierError{MS_E_ARG, "ms_tier_open: unknown eviction '" + ev + "'"};
    if (o.contains("peers")) {
      for (const json& p : o.at("peers")) {
        const int d = p.at("device").get<int>();
        int ok = 0;
        if (d == t->ordinal || cudaDeviceCanAccessPeer(&ok, t->ordinal, d) != cudaSuccess || !ok)
          throw TierError{MS_E_ARG, "ms_tier_open: device " + std::to_string(d) + " is not a P2P peer of " +
                                        std::to_string(t->ordinal)};
        t->link_dev.push_back(d);
        NvlinkPeer np;
        np.peer_id = d;
        gpu.nvlink_peers.push_back(np);
        mp.peer_free_gb.push_back(p.value("free_gb", 0.0));
      }
    }

    // probe plumbing: a source in local HBM, one destination per link on the peer
    int lo = 0, hi = 0;
    ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "cudaDeviceGetStreamPriorityRange");
    ck(cudaStreamCreateWithPriority(&t->probe_stream, cudaStreamNonBlocking, lo), "cudaStreamCreate");
    ck(cudaEventCreate(&t->ev0), "cudaEventCreate");
    ck(cudaEventCreate(&t->ev1), "cudaEventCreate");
    const size_t pb = (t->probe_bytes + kChunkBytes - 1) / kChunkBytes * kChunkBytes;
    t->probe_src = t->reserve(pb);
    for (size_t off = 0; off < pb; off += kChunkBytes) t->back(t->probe_src + off, Tier::Local, -1);
    t->grant(t->probe_src, pb);
    for (size_t l = 0; l < t->link_dev.size(); ++l) {
      const CUdeviceptr d = t->reserve(pb);
      for (size_t off = 0; off < pb; off += kChunkBytes) t->back(d + off, Tier::Peer, static_cast<int>(l));
      t->grant(d, pb);
      t->probe_dst.push_back(d);
    }
    t->probe_last.assign(t->link_dev.size(), {0, 0});
    ms_tier* raw = t.get();
    t->mm = std::make_unique<MemoryManager>(gpu, mp, [raw](int link, std::int64_t bytes) {
      return raw->probe_now(link, bytes);
    });
    t->stats.n_links = static_cast<int32_t>(t->link_dev.size());
    *out = t.release();
    return 0;
  });
}

extern "C" int ms_tier_alloc(ms_tier* t, int task, int high_priority, uint64_t bytes, uint64_t* dptr,
                             uint64_t* n_chunks) {
  if (!t || !dptr || bytes == 0) return ms_internal_fail(MS_E_ARG, "ms_tier_alloc: bad argument");
  return guarded([&]() -> int {
    ck(cudaSetDevice(t->ordinal), "cudaSetDevice");
    std::vector<ChunkRelocation> moves;
    const Priority prio = high_priority ? Priority::High : Priority::Low;
    std::vector<std::int64_t> ids =
        t->mm->allocate(task, prio, static_cast<std::int64_t>(bytes), mono_ns(), &moves);
    if (!moves.empty()) {
      // LP kernels may read the chunks being moved; HP chains never own LP chunks (and an
      // armed HP gate must not be waited on)
      if (ms_internal_lp_sync(t->dev) < 0) throw TierError{MS_E_CUDA, "LP stream sync before relocation"};
      t->relocate(moves);
    }
    Buffer b;
    b.bytes = ids.size() * static_cast<size_t>(kChunkBytes);
    b.va = t->reserve(b.bytes);
    b.ids = ids;
    const std::vector<Chunk>& cs = t->mm->chunks();
    try {
      for (size_t i = 0; i < ids.size(); ++i) {
        const Chunk& c = cs[static_cast<size_t>(ids[i])];
        t->back(b.va + i * kChunkBytes, c.tier, c.peer);
        t->chunk_va[ids[i]] = b.va + i * kChunkBytes;
      }
      t->grant(b.va, b.bytes);
    } catch (...) {
      t->free_buffer(b);
      throw;
    }
    *dptr = static_cast<uint64_t>(b.va);
    if (n_chunks) *n_chunks = ids.size();
    t->buffers[static_cast<uint64_t>(b.va)] = std::move(b);
    return 0;
  });
}

extern "C" int ms_tier_chunks(ms_tier* t, uint64_t dptr, ms_tier_chunk* out, uint64_t n) {
  if (!t || !out) return ms_internal_fail(MS_E_ARG, "ms_tier_chunks: null argument");
  auto it = t->buffers.find(dptr);
  if (it == t->buffers.end()) return ms_internal_fail(MS_E_ARG, "ms_tier_chunks: unknown buffer");
  const std::vector<Chunk>& cs = t->mm->chunks();
  const size_t m = std::min<size_t>(n, it->second.ids.size());
  for (size_t i = 0; i < m; ++i) {
    const Chunk& c = cs[static_cast<size_t>(it->second.ids[i])];
    out[i].tier = c.tier == Tier::Local ? MS_TIER_LOCAL : c.tier == Tier::Peer ? MS_TIER_PEER : MS_TIER_DRAM;
    out[i].peer = c.peer;
    out[i].owner = c.owner_task;
    out[i].pinned = c.pinned ? 1 : 0;
  }
  return static_cast<int>(m);
}

extern "C" int ms_tier_probe(ms_tier* t, int link, double* score, int64_t* t_ns) {
  if (!t || link < 0 || link >= static_cast<int>(t->link_dev.size()))
    return ms_internal_fail(MS_E_ARG, "ms_tier_probe: no such link");
  return guarded([&]() -> int {
    t->probe_last[static_cast<size_t>(link)].first = 0;  // force a fresh measurement
    const double s = t->mm->congestion().probe(link, mono_ns());
    if (score) *score = s;
    if (t_ns) *t_ns = t->probe_last[static_cast<size_t>(link)].second;
    return 0;
  });
}

extern "C" int ms_tier_get_stats(ms_tier* t, ms_tier_stats* st) {
  if (!t || !st) return ms_internal_fail(MS_E_ARG, "ms_tier_get_stats: null argument");
  ms_tier_stats s = t->stats;
  s.local_capacity_chunks = t->mm->local_capacity();
  s.local_used_chunks = t->mm->local_used();
  s.chunks_local = s.chunks_peer = s.chunks_dram = 0;
  for (const Chunk& c : t->mm->chunks()) {
    if (c.owner_task < 0) continue;
    (c.tier == Tier::Local ? s.chunks_local : c.tier == Tier::Peer ? s.chunks_peer : s.chunks_dram) += 1;
  }
  *st = s;
  return 0;
}

extern "C" int ms_tier_free(ms_tier* t, uint64_t dptr) {
  if (!t) return ms_internal_fail(MS_E_ARG, "ms_tier_free: null tier");
  auto it = t->buffers.find(dptr);
  if (it == t->buffers.end()) return ms_internal_fail(MS_E_ARG, "ms_tier_free: unknown buffer");
  return guarded([&]() -> int {
    ck(cudaSetDevice(t->ordinal), "cudaSetDevice");
    if (ms_internal_lp_sync(t->dev) < 0) throw TierError{MS_E_CUDA, "LP stream sync before free"};
    ck(cudaStreamSynchronize(t->probe_stream), "probe stream sync");
    t->free_buffer(it->second);
    t->buffers.erase(it);
    return 0;
  });
}

extern "C" int ms_tier_close(ms_tier* t) {
  if (!t) return 0;
  cudaSetDevice(t->ordinal);
  if (t->dev) ms_internal_lp_sync(t->dev);
  if (t->probe_stream) cudaStreamSynchronize(t->probe_stream);
  for (auto& kv : t->buffers) t->free_buffer(kv.second);
  const size_t pb = (t->probe_bytes + kChunkBytes - 1) / kChunkBytes * kChunkBytes;
  std::vector<CUdeviceptr> ranges = t->probe_dst;
  if (t->probe_src) ranges.push_back(t->probe_src);
  for (CUdeviceptr d : ranges) {
    t->vmm.unmap(d, pb);
    t->vmm.addr_free(d, pb);
  }
  if (t->ev0) cudaEventDestroy(t->ev0);
  if (t->ev1) cudaEventDestroy(t->ev1);
  if (t->probe_stream) cudaStreamDestroy(t->probe_stream);
  delete t;
  return 0;
}
