"""Development probe: config-4 HP decode step alone on one B200 — bs=1 GEMV chain
(hp_gemv.cuh) vs the m=128 tcgen05 chain — CUDA-event time per step and weight GB/s,
plus sub-chains (LM head alone, layers alone, one FFN op alone) to separate the streaming
rate from the per-op phase cost."""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config4, decode_step_ops  # noqa: E402


def timed(dev, ops, nbytes, reps=20):
    ch = dev.hp_register_chain(ops)
    ms = dev.hp_time_chain(ch, reps)
    dev.hp_unregister_chain(ch)
    return {"ms": ms, "gbs": nbytes / (ms * 1e-3) / 1e9, "ops": len(ops)}


def main():
    dev = Device(0)
    out = {}
    w = Config4(dev, m=1)
    M, H, Q, F, V, L = w.M, w.H, w.Q, w.F, w.V, w.LAYERS
    ops = decode_step_ops(M, H, Q, F, V, L, w.bufs, w.weights, w.lm)
    layer_b = 2 * (Q * H + H * H + 2 * F * H + H * F)
    out["step"] = timed(dev, ops, w.weight_bytes)
    out["lm_head"] = timed(dev, ops[-1:], 2 * V * H)
    out["layers"] = timed(dev, ops[:-1], L * layer_b)
    out["gu_x4"] = timed(dev, [ops[2]] * 4, 4 * 2 * 2 * F * H)
    out["down_x4"] = timed(dev, [ops[3]] * 4, 4 * 2 * F * H)
    out["qkv_x8"] = timed(dev, [ops[0]] * 8, 8 * 2 * Q * H)
    for k, v in out.items():
        print(k, json.dumps(v), flush=True)
    if "128" in sys.argv[1:]:
        w2 = Config4(dev, m=128)
        ms = dev.hp_time_chain(w2.chain, 10)
        out["m128_step"] = {"ms": ms, "gbs": w2.weight_bytes / (ms * 1e-3) / 1e9}
        print("m128_step", json.dumps(out["m128_step"]))
    (ROOT / "gpurun_out" / "gemv_probe.json").write_text(json.dumps(out, indent=1))
    dev.close()


if __name__ == "__main__":
    main()
