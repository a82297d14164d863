set -x
mkdir -p gpurun_out
timeout 600 python tools/split_drain_probe.py > gpurun_out/split_drain.json 2> gpurun_out/split_drain.err
timeout 600 python -m pytest tests/test_gpu_preempt.py -q -p timeout --timeout 240 -k pair > gpurun_out/pytest_pair.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pair.log
timeout 300 python tools/live_drain_probe.py > gpurun_out/live_drain.json 2> gpurun_out/live_drain.err
tail -3 gpurun_out/split_drain.err; tail -2 gpurun_out/pytest_pair.log
python - <<'PY'
import json
d=json.load(open('gpurun_out/split_drain.json'))
for c,v in d.items():
    print(c, v['full_ms'], v['units'])
    for r in v['trials']: print('   ', r['exit_us'], r['preempted'], r['phases'], r['epilogue'])
d=json.load(open('gpurun_out/live_drain.json'))
for k,v in d.items(): print(k, v['runs'], v['flag_to_last_exit'], v['max_over_ctas_us'])
PY
