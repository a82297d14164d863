set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/cfg23_probe.py 4 > gpurun_out/cfg23_probe.log 2>&1
python -c "
import sys; sys.path.insert(0,'.')
from paper_2601_04071_b200.device import Device
from paper_2601_04071_b200.live import Config1
d=Device(0); w=Config1(d); print('lp gemm ms', [round(d.lp_time_full(w.lp, 5),4) for _ in range(3)], 'chain ms', round(d.hp_time_chain(w.chain, 20),4)); d.close()" > gpurun_out/gemm_check.log 2>&1
tail -2 gpurun_out/smoke.log; grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -12; cat gpurun_out/gemm_check.log; python -c "
import json; d=json.load(open('gpurun_out/cfg23_probe.log'))
for c,v in d.items():
    print(c, {k: v['calib'][k] for k in ('step_ms','gemm_tflops','hp_chain_ms','hp_ops')}, 'exclusive_att', v['exclusive_att'])
    for p in ('reef_req','splitkernel'): print('  ',p, v[p])
"
