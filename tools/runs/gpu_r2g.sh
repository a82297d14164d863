set -x
mkdir -p gpurun_out
timeout 300 python tools/gemv_regress_ab.py . > gpurun_out/gemv_regress.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_config_sizes.py -q -k "decode or gemv" > gpurun_out/pytest_gemv.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gemv.log
MS_GEMV_DYNAMIC=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_config_sizes.py -q -k "decode or gemv" >> gpurun_out/pytest_gemv.log 2>&1; echo "pytest dyn rc=$?" >> gpurun_out/pytest_gemv.log
timeout 900 python tools/gemv_dynamic_ab.py 15 > gpurun_out/gemv_dynamic_ab.log 2>&1
cat gpurun_out/gemv_regress.log; grep -E "passed|failed|FAILED|Error|rc=" gpurun_out/pytest_gemv.log | tail -6; cat gpurun_out/gemv_dynamic_ab.log | tail -60
