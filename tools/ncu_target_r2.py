"""Round-2 ncu target: a short deterministic launch sequence of every tenant kernel family
(no live scheduling: ncu serialises and replays kernels).  argv[1] selects a subset:
  lp      LP GEMM 8192^3 + axpy 2^30 + AdamW optimizer (110 M params)
  hp      config-1 fused chain + config-4 GEMV decode step
  t23     ResNet-50 bs=1 chain + BERT-base bs=1 chain (per-op: glue ops + tcgen05 GEMMs)
  all     everything"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_04071_b200.device import Device  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
dev = Device(0)
if what in ("lp", "all"):
    from paper_2601_04071_b200.live import Config1
    w = Config1(dev)
    for _ in range(2):
        dev.lp_run(w.lp, 0, w.lp.total_tiles)
        dev.lp_wait(w.lp, 60)
    n = 1 << 30
    x, y = dev.alloc(2 * n), dev.alloc(2 * n)
    dev.fill_synth(x, n, 1, 21, 1.0)
    dev.fill_synth(y, n, 1, 22, 1.0)
    k = dev.lp_register_axpy(x, y, n, 0.5)
    for _ in range(2):
        dev.lp_run(k, 0, k.total_tiles)
        dev.lp_wait(k, 60)
    np_ = 110_000_000
    bufs = [dev.alloc(4 * np_) for _ in range(3)] + [dev.alloc(2 * np_)]
    for b in bufs[:3]:
        dev.memset(b, 0, 4 * np_)
    ko = dev.lp_register_optim(*bufs, np_, mode=0, c1=10.0, c2=1000.0)
    for _ in range(2):
        dev.lp_run(ko, 0, ko.total_tiles)
        dev.lp_wait(ko, 60)
if what in ("hp", "all"):
    from paper_2601_04071_b200.live import Config1, Config4
    w = Config1(dev)
    for _ in range(2):
        dev.hp_launch_direct(w.chain, dev.hp_next_seq())
        dev.sync()
    w4 = Config4(dev)
    for _ in range(3):
        dev.hp_launch_direct(w4.chain, dev.hp_next_seq())
        dev.sync()
if what in ("t23", "all"):
    from paper_2601_04071_b200.tenants import BertHP, ResNet50HP
    for net in (ResNet50HP(dev, 1), BertHP(dev, 1)):
        ch = dev.hp_register_chain(net.ops)
        for _ in range(2):
            dev.hp_launch_direct(ch, dev.hp_next_seq())
            dev.sync()
dev.close()
print("ncu target done")
