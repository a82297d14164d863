"""Memory-tier placement logic on CPU (microslice/memory.hpp — reference memory.hpp:15-323,
plus the live-tier extensions: LiveProbe-fed congestion scores and release()).  A C++
client is compiled against include/microslice and libmicroslice.so (no GPU)."""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2601_04071_b200" / "lib"

CLIENT = r'''
#include "microslice/memory.hpp"
#include <cstdio>
#include <vector>
using namespace microslice;
#define CHECK(c) do { if (!(c)) { std::printf("FAIL line %d: %s\n", __LINE__, #c); return 1; } } while (0)
int main() {
  GpuConfig g;
  for (int i = 0; i < 3; ++i) { NvlinkPeer p; p.peer_id = i + 1; p.bandwidth = 900e9; g.nvlink_peers.push_back(p); }
  g.nvlink_peers[0].background_load = 900e9;   // model: link 0 congested (score ~2)
  MemParams mp; mp.enabled = true; mp.hbm_gb = 10 * kChunkBytes / 1e9; mp.peer_free_gb = {1.0, 4 * kChunkBytes / 1e9, 1.0};

  // replay model: contention-first skips the congested link and picks the least loaded
  MemoryManager m(g, mp);
  CHECK(m.local_capacity() == 10);
  auto hp = m.allocate(0, Priority::High, 4 * kChunkBytes, 0);
  auto lp = m.allocate(1, Priority::Low, 12 * kChunkBytes, 0);
  CHECK(hp.size() == 4 && lp.size() == 12 && m.local_used() == 10);
  const auto& c = m.chunks();
  CHECK(c[lp[5]].tier == Tier::Local && c[lp[6]].tier == Tier::Peer && c[lp[6]].peer == 1);
  CHECK(m.congestion().last_score(0) > 1.5 && m.congestion().any_score_above(1.2));
  CHECK(m.off_device_fraction(1) > 0.16 && m.off_device_fraction(0) == 0.0);
  // HP displaces the oldest unpinned local chunk (lp[0]); it goes where evict_select says
  std::vector<ChunkRelocation> moves;
  auto hp2 = m.allocate(0, Priority::High, 2 * kChunkBytes, 0, &moves);
  CHECK(moves.size() == 2 && moves[0].chunk_id == lp[0] && moves[1].chunk_id == lp[1]);
  CHECK(moves[0].from == Tier::Local && moves[0].to == Tier::Peer);
  CHECK(m.chunks()[hp2[0]].pinned && m.chunks()[hp2[0]].tier == Tier::Local);
  // release returns capacity; released chunks are never victims again
  m.release(lp);
  CHECK(m.local_used() == 10 - 4);  // lp[2..5] were local
  CHECK(m.chunks()[lp[3]].owner_task == -1 && m.chunks_of(1).empty());
  auto lp2 = m.allocate(2, Priority::Low, 4 * kChunkBytes, 0);
  CHECK(m.local_used() == 10 && m.chunks()[lp2[3]].tier == Tier::Local);

  // live tier: scores come from the probe function (t_base = first measurement)
  int calls = 0;
  std::vector<Ns> lat = {1000, 1000, 1000};
  MemoryManager live(g, mp, [&](int link, std::int64_t) { ++calls; return lat[link]; });
  CHECK(calls == 3);
  lat = {1100, 5000, 1300};  // link 1 congested now, link 0 mildly loaded
  auto a = live.allocate(1, Priority::Low, 11 * kChunkBytes, 0);
  CHECK(live.chunks()[a[10]].tier == Tier::Peer && live.chunks()[a[10]].peer == 0);
  CHECK(live.congestion().last_score(1) == 5.0);
  lat = {4000, 4000, 4000};  // every link over the threshold -> DRAM
  auto b = live.allocate(1, Priority::Low, kChunkBytes, 0);
  CHECK(live.chunks()[b[0]].tier == Tier::Dram);

  // round-robin ignores congestion
  mp.eviction = EvictionPolicy::RoundRobin;
  MemoryManager rr(g, mp);
  auto r = rr.allocate(1, Priority::Low, 13 * kChunkBytes, 0);
  CHECK(rr.chunks()[r[10]].peer == 0 && rr.chunks()[r[11]].peer == 1 && rr.chunks()[r[12]].peer == 2);
  // pinned HBM exhaustion is an input error
  MemParams small = mp; small.hbm_gb = 2 * kChunkBytes / 1e9;
  MemoryManager s(g, small);
  s.allocate(0, Priority::High, 2 * kChunkBytes, 0);
  try { s.allocate(0, Priority::High, kChunkBytes, 0); return 2; } catch (const ValidationError&) {}
  std::printf("ok\n");
  return 0;
}
'''


def test_memory_manager_placement_and_live_extensions(tmp_path):
    src = tmp_path / "mem.cpp"
    src.write_text(CLIENT)
    exe = tmp_path / "mem"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(src), "-o", str(exe),
                    f"-L{LIB}", "-lmicroslice", f"-Wl,-rpath,{LIB}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stdout + out.stderr


def test_gemm_slow_units_matches_bytewise_map():
    """tier.gemm_slow_units (host side of GEMM-operand admission) against a brute-force map
    of the bytes each (tile, k-slice) unit reads, on a stub tier with a chunk layout."""
    import random
    from paper_2601_04071_b200.tier import MemoryTier

    CH = MemoryTier.CHUNK
    m, n, k, bn, split, gm = 1024, 768, 2048, 256, 2, 4
    rng = random.Random(5)
    a, b = 0, (m * k * 2 + CH - 1) // CH * CH
    place = {p: ["local" if rng.random() < 0.6 else "dram" for _ in range((sz * 2 + CH - 1) // CH)]
             for p, sz in ((a, m * k), (b, n * k))}

    class Stub:
        CHUNK = CH
        def chunks(self, p):
            return [(t, -1, 0, False) for t in place[p]]

    got = MemoryTier.gemm_slow_units(Stub(), a, b, m, n, k, block_n=bn, split=split, group_m=gm)
    tm, tn, kps = m // 128, n // bn, k // 64 // split
    want = []
    for t in range(tm * tn):                          # tc_gemm.cuh tile_coords (group-M raster)
        g, r = divmod(t, gm * tn)
        rows = min(tm - g * gm, gm)
        mb, nb = g * gm + r % rows, r // rows
        for sl in range(split):
            def off(p, row0, nrows):
                for row in range(row0, row0 + nrows):
                    lo = (row * k + sl * kps * 64) * 2
                    hi = lo + kps * 64 * 2 - 1
                    if any(place[p][c] != "local" for c in range(lo // CH, hi // CH + 1)):
                        return True
                return False
            want.append(off(a, mb * 128, 128) or off(b, nb * bn, bn))
    assert len(got) == tm * tn * split and got == want
