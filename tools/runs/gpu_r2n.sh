# split-K reduce (poller kept alive, 16 loads in flight) + drain probe; GEMM variants vs cuBLAS
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tenants23.py -q -k "split or train" > gpurun_out/pytest_split.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_split.log
timeout 600 python tools/drain23_probe.py 3 > gpurun_out/drain23.json 2> gpurun_out/drain23.err
timeout 900 python tools/gemm_ab2.py 3 > gpurun_out/gemm_ab2.log 2>&1
tail -3 gpurun_out/pytest_split.log; cat gpurun_out/gemm_ab2.log | tail -4
python - <<'PY'
import json
d=json.load(open('gpurun_out/drain23.json'))
for c,v in d.items():
    runs=[r for r in v['slowest'] if r[2] <= 0]
    print(c, v['n'], 'non-queued slowest:')
    for r in runs[:10]: print('   ', r)
PY
