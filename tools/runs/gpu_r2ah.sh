set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p timeout --timeout 300 --timeout-method thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/live_drain_probe.py > gpurun_out/live_drain.json 2> gpurun_out/live_drain.err
MS_LP_GEMM_PAIR=0 timeout 300 python tools/live_drain_probe.py > gpurun_out/live_drain_single.json 2> gpurun_out/live_drain_single.err
grep -E "passed|failed|FAILED|Timeout" gpurun_out/pytest_gpu.log | tail -6
python - <<'PY'
import json
for f in ('gpurun_out/live_drain.json','gpurun_out/live_drain_single.json'):
    d=json.load(open(f))
    for k,v in d.items(): print(f[-20:], k, v['runs'], {a: v['flag_to_last_exit'].get(a) for a in ('p50_ns','p90_ns','p99_ns')}, v['max_over_ctas_us'])
PY
