"""Config-4 decode step alone (hp_time_chain, best of 3 x 5 steps), one process."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_04071_b200.device import Device  # noqa: E402
from paper_2601_04071_b200.live import Config4  # noqa: E402
dev = Device(0)
w = Config4(dev)
ms = [round(dev.hp_time_chain(w.chain, 5), 4) for _ in range(3)]
print(json.dumps({"dyn_ops": os.environ.get("MS_GEMV_DYN_OPS", "0"), "step_ms": ms}), flush=True)
dev.close()
