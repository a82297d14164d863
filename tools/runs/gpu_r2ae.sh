set -x
mkdir -p gpurun_out
MS_GEMV_DYN_OPS=3 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_config_sizes.py -q -p timeout --timeout 240 -k "decode or gemv" > gpurun_out/pytest_dynops.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dynops.log
tail -2 gpurun_out/pytest_dynops.log
timeout 1500 python tools/gemv_dynops_ab.py 16 0,2,4 > gpurun_out/gemv_dynops_ab.log 2>&1
cat gpurun_out/gemv_dynops_ab.log
