set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tenants23.py -q -p timeout --timeout 240 -k "split or train" > gpurun_out/pytest_split.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_split.log
timeout 600 python tools/drain23_stamps.py 3 > gpurun_out/drain23_stamps.json 2> gpurun_out/drain23_stamps.err
timeout 900 python tools/cfg23_probe.py 3 > gpurun_out/cfg23_probe.json 2> gpurun_out/cfg23_probe.err
tail -2 gpurun_out/pytest_split.log
python - <<'PY'
import json
d=json.load(open('gpurun_out/drain23_stamps.json'))
for c,v in d.items():
    print(c, v['runs'], 'queued', v['queued_runs'], v['exit'])
    for r in v['slowest'][:6]: print('   ', r['kernel'], r['max'], r['min_seen'], r['counts'])
d=json.load(open('gpurun_out/cfg23_probe.json'))
for c,v in d.items():
    print(c, 'ex', v['exclusive_att'], v['calib'].get('step_ms'))
    for k,x in v.items():
        if isinstance(x, dict) and 'att' in x: print('  ', k, {a: (round(b,4) if isinstance(b,float) else b) for a,b in x.items()})
PY
