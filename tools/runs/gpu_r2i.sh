set -x
timeout 900 python -m pytest tests/test_gpu_tenants23.py -q -x -k "split or train_step or optimizer" > gpurun_out/pytest_split.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_split.log
timeout 900 python tools/cfg23_probe.py 4 > gpurun_out/cfg23_probe.log 2>&1
tail -5 gpurun_out/pytest_split.log; python -c "
import json; d=json.load(open('gpurun_out/cfg23_probe.log'))
for c,v in d.items():
    print(c, {k: v['calib'][k] for k in ('step_ms','gemm_tflops')}, 'exclusive_att', v['exclusive_att'])
    for p in ('reef_req','splitkernel','splitkernel eager','splitkernel ungoverned'): print('  ',p, v[p])
"
