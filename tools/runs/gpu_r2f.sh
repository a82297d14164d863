set -x
mkdir -p gpurun_out
timeout 300 python tools/gemv_regress_ab.py build/r1tree > gpurun_out/gemv_regress.log 2>&1
timeout 300 python tools/gemv_regress_ab.py . >> gpurun_out/gemv_regress.log 2>&1
timeout 900 python -m pytest tests/test_gpu_preempt.py tests/test_gpu_kernels.py -q -x > gpurun_out/pytest_pre.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pre.log
timeout 600 python tools/live_drain_probe.py > gpurun_out/live_drain_probe.log 2>&1
timeout 600 python tools/exit_probe.py > gpurun_out/exit_probe.log 2>&1
cat gpurun_out/gemv_regress.log; grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_pre.log | tail -5; python -c "
import json; d=json.load(open('gpurun_out/live_drain_probe.log'))
for k,v in d.items(): print(k, v['flag_to_last_exit'].get('p50_ns'), v['flag_to_last_exit'].get('p99_ns'), v['max_over_ctas_us'])
"; grep "trial" gpurun_out/exit_probe.log
