set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_preempt.py -q -p timeout --timeout 240 -k "pair" > gpurun_out/pytest_pair.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pair.log
timeout 300 python tools/live_drain_probe.py > gpurun_out/live_drain.json 2> gpurun_out/live_drain.err
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.json 2> gpurun_out/e2e_probe.err
tail -2 gpurun_out/pytest_pair.log
python - <<'PY'
import json
d=json.load(open('gpurun_out/live_drain.json'))
for k,v in d.items(): print(k, v['runs'], v['flag_to_last_exit'], v['max_over_ctas_us'])
print(open('gpurun_out/e2e_probe.json').read()[:1500])
PY
