"""Diagnostic run of the sm_100a device layer on a real B200 (development tool).

python tools/gpu_check.py [--quick]
Prints correctness (vs the C oracle) and timing of every kernel, then the preemption /
doorbell latency microbenchmarks.  Formal assertions live in tests/test_gpu_*.py.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import tenant as T  # noqa: E402  (checker only)
from paper_2601_04071_b200.device import Device, host_now_ns  # noqa: E402

SEED = 1234


def d2h_u16(dev, ptr, n):
    out = np.empty(n, dtype=np.uint16)
    dev.d2h(out.ctypes.data, ptr, n * 2)
    return out


def rel_err(got, ref):
    return float(np.max(np.abs(got - ref)) / (np.max(np.abs(ref)) + 1e-30))


def check_gemm(dev, M, N, K, bn, rows=None, time_reps=0):
    a = dev.alloc(M * K * 2); b = dev.alloc(N * K * 2); c = dev.alloc(M * N * 2)
    dev.fill_synth(a, M * K, SEED, 1, 1.0)
    dev.fill_synth(b, N * K, SEED, 2, 1.0 / np.sqrt(K))
    dev.memset(c, 0, M * N * 2)
    k = dev.lp_register_gemm(a, b, c, M, N, K, block_n=bn)
    t0 = time.time()
    dev.lp_run(k, 0, k.total_tiles)
    st = dev.lp_wait(k, 60)
    res = {"shape": [M, N, K], "bn": bn, "tiles": k.total_tiles, "done": st["tiles_done"],
           "cursor": st["cursor"], "wall_s": round(time.time() - t0, 4)}
    A = T.synth_bf16(M * K, SEED, 1, 1.0)
    W = T.synth_bf16(N * K, SEED, 2, float(np.float32(1.0 / np.sqrt(K))))
    if rows is None:
        rows = list(range(M))
    ref = T.gemm_rows(A, W, rows, N, K)
    Cg = d2h_u16(dev, c, M * N).reshape(M, N)
    got = T.bf16_to_f32(Cg[rows].reshape(-1)).reshape(len(rows), N)
    res["rel_err"] = rel_err(got, ref)
    res["max_abs_ref"] = float(np.max(np.abs(ref)))
    if time_reps:
        ms = dev.lp_time_full(k, time_reps)
        res["ms"] = ms
        res["tflops"] = 2.0 * M * N * K / (ms * 1e-3) / 1e12
    return res, (a, b, c, k)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "gpu_check.json"))
    args = ap.parse_args()
    out = {}
    dev = Device(0)
    out["info"] = dev.info
    print("device", dev.info, flush=True)
    off, rtt = dev.calibrate(300)
    out["clock"] = {"offset_ns": off, "rtt_min_ns": rtt}
    print("clock", out["clock"], flush=True)

    # synthetic data generator parity
    p = dev.alloc(1 << 21)
    dev.fill_synth(p, 1 << 20, SEED, 7, 0.5)
    g = d2h_u16(dev, p, 1 << 20)
    cpu = T.synth_bf16(1 << 20, SEED, 7, 0.5)
    out["synth_equal"] = bool(np.array_equal(g, cpu))
    print("synth equal", out["synth_equal"], flush=True)

    # GEMM correctness ladder
    out["gemm"] = []
    for (M, N, K, bn) in [(128, 256, 64, 256), (256, 512, 256, 256), (512, 512, 1024, 128), (256, 1024, 512, 64),
                          (1024, 1024, 2048, 256)]:
        r, _ = check_gemm(dev, M, N, K, bn)
        out["gemm"].append(r)
        print("gemm", r, flush=True)

    # axpy correctness
    n = 1 << 22
    x = dev.alloc(n * 2); y = dev.alloc(n * 2)
    dev.fill_synth(x, n, SEED, 11, 1.0); dev.fill_synth(y, n, SEED, 12, 1.0)
    k = dev.lp_register_axpy(x, y, n, 0.75)
    dev.lp_run(k, 0, k.total_tiles)
    st = dev.lp_wait(k, 30)
    ref = T.axpy(T.synth_bf16(n, SEED, 12, 1.0), T.synth_bf16(n, SEED, 11, 1.0), 0.75)
    out["axpy_small"] = {"equal": bool(np.array_equal(d2h_u16(dev, y, n), ref)), "status": st}
    print("axpy small", out["axpy_small"], flush=True)

    if not args.quick:
        # big GEMM: timing + sampled correctness
        M = N = K = 8192
        r, (a, b, c, kg) = check_gemm(dev, M, N, K, 256, rows=list(range(0, M, 517)), time_reps=5)
        out["gemm_8192"] = r
        print("gemm 8192", r, flush=True)
        # preemption + resume must reproduce the uninterrupted C bit-exactly
        Cref = d2h_u16(dev, c, M * N)
        dev.memset(c, 0, M * N * 2)
        dev.lp_reset(kg)
        lat = []
        begin, total = 0, kg.total_tiles
        runs = 0
        off, _ = dev.calibrate(200)
        while True:
            dev.lp_run(kg, begin, total)
            runs += 1
            busy_until = time.perf_counter() + 0.0003
            while time.perf_counter() < busy_until:
                pass
            _, t_raise = dev.preempt_raise()
            st = dev.lp_wait(kg, 30)
            if st["preempted"]:
                lat.append({"seen_us": (st["t_seen"] - off - t_raise) / 1e3,
                            "exit_us": (st["t_exit"] - off - t_raise) / 1e3,
                            "cursor": st["cursor"], "redo": st["redo_count"], "done": st["tiles_done"]})
            begin = st["cursor"]
            if begin >= total and st["redo_count"] == 0:
                break
            if runs > 400:
                break
        Cp = d2h_u16(dev, c, M * N)
        out["gemm_preempt"] = {"runs": runs, "bit_exact": bool(np.array_equal(Cp, Cref)), "lat": lat[:50]}
        ex = sorted(l["exit_us"] for l in lat)
        if ex:
            out["gemm_preempt"]["exit_p50_us"] = ex[len(ex) // 2]
            out["gemm_preempt"]["exit_p99_us"] = ex[min(len(ex) - 1, int(0.99 * len(ex)))]
        print("gemm preempt", {k_: v for k_, v in out["gemm_preempt"].items() if k_ != "lat"}, flush=True)

        # big axpy: bandwidth
        n = 1 << 30
        x = dev.alloc(n * 2); y = dev.alloc(n * 2)
        dev.fill_synth(x, n, SEED, 21, 1.0); dev.fill_synth(y, n, SEED, 22, 1.0)
        ka = dev.lp_register_axpy(x, y, n, 0.5)
        ms = dev.lp_time_full(ka, 5)
        out["axpy_1g"] = {"ms": ms, "gbs": 6.0 * n / (ms * 1e-3) / 1e9}
        print("axpy 1g", out["axpy_1g"], flush=True)
        # axpy preemption latency
        lat = []
        dev.lp_reset(ka)
        for i in range(30):
            dev.lp_run(ka, 0, ka.total_tiles)
            busy_until = time.perf_counter() + 0.0002
            while time.perf_counter() < busy_until:
                pass
            _, t_raise = dev.preempt_raise()
            st = dev.lp_wait(ka, 30)
            lat.append((st["t_exit"] - off - t_raise) / 1e3)
            dev.lp_reset(ka)
        lat.sort()
        out["axpy_preempt_exit_us"] = {"p50": lat[len(lat) // 2], "max": lat[-1]}
        print("axpy preempt", out["axpy_preempt_exit_us"], flush=True)

        # HP chain (config 1): 4 x [128x4096] * [4096x4096]^T + bias/GELU
        Mh, H = 128, 4096
        act = [dev.alloc(Mh * H * 2) for _ in range(5)]
        ws = [dev.alloc(H * H * 2) for _ in range(4)]
        bias = dev.alloc(H * 2)
        dev.fill_synth(act[0], Mh * H, SEED, 100, 1.0)
        for i, w in enumerate(ws):
            dev.fill_synth(w, H * H, SEED, 101 + i, 1.0 / np.sqrt(H))
        dev.fill_synth(bias, H, SEED, 110, 0.1)
        ops = [dict(kind=1, block_n=64, a=act[i], b=ws[i], c=act[i + 1], bias=0, m=Mh, n=H, k=H) for i in range(4)]
        ops.append(dict(kind=2, block_n=0, a=act[4], b=0, c=act[0], bias=bias, m=Mh, n=H, k=0))
        chain = dev.hp_register_chain(ops)
        ms = dev.hp_time_chain(chain, 20)
        out["hp_chain_ms"] = ms
        print("hp chain ms", ms, flush=True)
        # doorbell latency on an idle GPU
        seq = 1
        lat = []
        for i in range(50):
            dev.hp_arm(chain, seq)
            busy_until = time.perf_counter() + 0.0005
            while time.perf_counter() < busy_until:
                pass
            t = dev.hp_ring(seq)
            tm = dev.hp_wait(chain, seq, 10)
            lat.append({"gate_us": (tm["t_gate"] - off - t) / 1e3, "first_cta_us": (tm["t_first_cta"] - off - t) / 1e3,
                        "done_us": (tm["t_done"] - off - t) / 1e3})
            seq += 1
        out["hp_doorbell_idle"] = lat[5:25]
        print("doorbell idle", lat[5:10], flush=True)
        # preempt LP GEMM + ring HP
        lat = []
        dev.lp_reset(kg)
        for i in range(40):
            dev.hp_arm(chain, seq)
            dev.lp_run(kg, 0, kg.total_tiles)
            busy_until = time.perf_counter() + 0.0004
            while time.perf_counter() < busy_until:
                pass
            _, t_raise = dev.preempt_raise()
            t_ring = dev.hp_ring(seq)
            tm = dev.hp_wait(chain, seq, 10)
            st = dev.lp_wait(kg, 30)
            lat.append({"lp_exit_us": (st["t_exit"] - off - t_raise) / 1e3,
                        "hp_first_cta_us": (tm["t_first_cta"] - off - t_ring) / 1e3,
                        "hp_gate_us": (tm["t_gate"] - off - t_ring) / 1e3,
                        "hp_done_us": (tm["t_done"] - off - t_ring) / 1e3})
            seq += 1
            dev.lp_reset(kg)
        out["preempt_ring"] = lat
        for key in ("lp_exit_us", "hp_first_cta_us", "hp_gate_us", "hp_done_us"):
            v = sorted(l[key] for l in lat)
            print(key, "p50", v[len(v) // 2], "p90", v[int(0.9 * len(v))], "max", v[-1], flush=True)

    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(out, indent=1, default=str))
    dev.close()


if __name__ == "__main__":
    main()
