"""Streamer layout probe: 4 small CTAs per SM (ctas_per_sm=4) vs ONE grouped CTA per SM
(ctas_per_sm=1, 3 x 256 streaming threads).  Bandwidth alone, then with the LP grid capped
(SM reserve r, as the power governor does) the preemption an armed HP chain sees:
ring -> gate, gate -> first HP CTA, flag -> last LP exit (us, p50 / p90)."""
import json
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config1, Config4  # noqa: E402


def spin(s):
    t = time.perf_counter() + s
    while time.perf_counter() < t:
        pass


def main():
    dev = Device(0)
    c1, c4 = Config1(dev), Config4(dev)
    n = Config4.N_EW
    out = []
    chains = {"cfg1_fused": c1.chain, "cfg4_gemv": c4.chain}
    for cps, tile in [(4, 8192), (1, 8192), (1, 16384)]:
        k = dev.lp_register_axpy(c4.x, c4.y, n, 0.5, tile_elems=tile, ctas_per_sm=cps)
        dev.set_lp_sm_reserve(1)
        ms = min(dev.lp_time_full(k, 3) for _ in range(2))
        row = {"ctas_per_sm": cps, "tile": tile, "tb_s": 6 * n / (ms * 1e-3) / 1e12}
        for reserve in (1, 60):
            dev.set_lp_sm_reserve(reserve)
            for cname, ch in chains.items():
                off, _ = dev.calibrate(100)
                r2g, g2f, ex = [], [], []
                for trial in range(30):
                    seq = dev.hp_next_seq()
                    dev.hp_arm(ch, seq)
                    spin(300e-6)
                    dev.lp_reset(k)
                    dev.lp_run(k, 0, k.total_tiles)
                    spin(300e-6)
                    _, t_raise = dev.preempt_raise()
                    t_ring = dev.hp_ring(seq)
                    t = dev.hp_wait(ch, seq, 10)
                    st = dev.lp_wait(k, 30)
                    if t["t_gate"]:
                        r2g.append((t["t_gate"] - off - t_ring) / 1e3)
                        g2f.append((t["t_first_cta"] - t["t_gate"]) / 1e3)
                    if st["preempted"]:
                        ex.append((st["t_exit"] - off - t_raise) / 1e3)
                    dev.sync()
                q = lambda v, p: round(float(np.percentile(v, p)), 2) if v else None  # noqa: E731
                row[f"r{reserve}_{cname}"] = {"ring_gate": [q(r2g, 50), q(r2g, 90)], "gate_first": [q(g2f, 50), q(g2f, 90)],
                                              "exit": [q(ex, 50), q(ex, 90)]}
        print(json.dumps(row), flush=True)
        out.append(row)
        dev.set_lp_sm_reserve(1)
        dev.lp_unregister(k)
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(json.dumps(out, indent=1) + "\n")
    dev.close()


if __name__ == "__main__":
    main()
