set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_config_sizes.py -q -k "decode or gemv" > gpurun_out/pytest_gemv.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gemv.log
timeout 900 python tools/gemv_dynamic_ab.py 12 > gpurun_out/gemv_dynamic_ab.log 2>&1
timeout 600 python tools/live_drain_probe.py > gpurun_out/live_drain_probe.log 2>&1
timeout 600 python tools/exit_probe.py > gpurun_out/exit_probe.log 2>&1
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gemv.log | tail -5; cat gpurun_out/gemv_dynamic_ab.log | tail -60; cat gpurun_out/live_drain_probe.log; tail -30 gpurun_out/exit_probe.log
