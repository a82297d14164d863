"""The drop-in boundary: both C-ABI libraries load on a CPU-only host and export every
entry point their headers declare; the device layer fails loudly (no CPU fallback)."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2601_04071_b200" / "lib"


def declared(header: str) -> set[str]:
    text = (ROOT / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(ms_[a-z0-9_]+)\s*\(", text))


@pytest.mark.parametrize("lib,headers", [("libmicroslice.so", ["ms_replay.h"]),
                                         ("libms_b200.so", ["ms_b200.h", "ms_live.h", "ms_session.h", "ms_tier.h"])])
def test_exports_every_declared_symbol(lib, headers):
    so = C.CDLL(str(LIB / lib))
    names = set().union(*(declared(h) for h in headers))
    assert len(names) > 10
    missing = [n for n in sorted(names) if not hasattr(so, n)]
    assert not missing, missing


def test_device_layer_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2601_04071_b200.device import Device, DeviceError
    with pytest.raises(DeviceError):
        Device(0)


def test_drop_in_headers_compile_standalone(tmp_path):
    """A C++ client written against the reference API compiles against include/microslice
    and links libmicroslice.so (source-compatible drop-in)."""
    import subprocess
    src = tmp_path / "client.cpp"
    src.write_text(r'''
#include "microslice/engine.hpp"
#include "microslice/metrics.hpp"
#include "microslice/scenario_io.hpp"
#include "microslice/tracegen.hpp"
#include <cstdio>
using namespace microslice;
int main() {
  ScenarioSpec sc; sc.name = "client"; sc.horizon = ms(20);
  sc.gpu.n_sm = 4;
  KernelSpec k; k.name = "k"; k.grid = {16, 1, 1}; sc.kernels.push_back(k);
  TaskSpec hp; hp.name = "hp"; hp.priority = Priority::High; hp.kind = TaskKind::Serving; hp.trace = "t";
  hp.kernel_sequence.push_back({"k", 2}); sc.tasks.push_back(hp);
  TaskSpec lp; lp.name = "lp"; lp.kernel_sequence.push_back({"k", 1}); sc.tasks.push_back(lp);
  RequestTrace tr; tr.name = "t"; tr.arrivals = generate_bursty_arrivals(1000.0, 1.0, sc.horizon, 3);
  sc.traces.push_back(tr);
  SplitPlan p = find_optimal_split(sc.gpu, k);
  RunArtifacts a = run_scenario(sc, Policy::SplitKernel);
  std::printf("%zu %lld %zu\n", a.timeline.size(), (long long)p.blocks_per_slice, a.requests.size());
  return a.timeline.is_monotonic() ? 0 : 1;
}''')
    exe = tmp_path / "client"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(src), "-o", str(exe),
                    f"-L{LIB}", "-lmicroslice", f"-Wl,-rpath,{LIB}"], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    assert int(out[0]) > 0 and int(out[2]) > 0
