set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_preempt.py tests/test_gpu_tenants23.py -q -p timeout --timeout 240 -k "pair or split or train or preempt" > gpurun_out/pytest_pz.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pz.log
timeout 300 python tools/live_drain_probe.py > gpurun_out/live_drain.json 2> gpurun_out/live_drain.err
timeout 600 python tools/drain23_stamps.py 3 > gpurun_out/drain23_stamps.json 2> gpurun_out/drain23_stamps.err
tail -2 gpurun_out/pytest_pz.log
python - <<'PY'
import json
d=json.load(open('gpurun_out/live_drain.json'))
for k,v in d.items(): print(k, v['runs'], v['flag_to_last_exit'], v['max_over_ctas_us'])
d=json.load(open('gpurun_out/drain23_stamps.json'))
for c,v in d.items():
    print(c, v['runs'], 'queued', v['queued_runs'], v['exit'])
    for r in v['slowest'][:5]: print('   ', r['kernel'], r['max'], r['min_seen'])
PY
