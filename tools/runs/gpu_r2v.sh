set -x
mkdir -p gpurun_out
timeout 200 python tools/pair_gate_probe.py > gpurun_out/pair_gate.json 2> gpurun_out/pair_gate.err
timeout 600 python tools/drain23_stamps.py 3 > gpurun_out/drain23_stamps.json 2> gpurun_out/drain23_stamps.err
cat gpurun_out/pair_gate.json; tail -3 gpurun_out/pair_gate.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/drain23_stamps.json'))
for c,v in d.items():
    print(c, v['runs'], v['exit'])
    for r in v['slowest'][:8]: print('   ', r['kernel'], r['max'], r['min_seen'], r['counts'])
PY
