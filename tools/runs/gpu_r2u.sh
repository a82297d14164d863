set -x
mkdir -p gpurun_out
timeout 200 python tools/pair_gate_probe.py > gpurun_out/pair_gate.json 2> gpurun_out/pair_gate.err
timeout 300 python tools/live_drain_probe.py > gpurun_out/live_drain.json 2> gpurun_out/live_drain.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p timeout --timeout 300 --timeout-method thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
cat gpurun_out/pair_gate.json; tail -2 gpurun_out/smoke.log; grep -E "passed|failed|FAILED|Timeout" gpurun_out/pytest_gpu.log | tail -12
python -c "
import json;d=json.load(open('gpurun_out/live_drain.json'))
for k,v in d.items(): print(k, v['runs'], v['flag_to_last_exit'], v['max_over_ctas_us'], v['min_over_ctas_us'])"
