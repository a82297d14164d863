set -x
mkdir -p gpurun_out
timeout 120 python tools/gemv_alone.py > gpurun_out/gemv_alone.log 2>&1
MS_GEMV_DYN_OPS=3 timeout 120 python tools/gemv_alone.py >> gpurun_out/gemv_alone.log 2>&1
MS_GEMV_DYN_OPS=3 timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x -p timeout --timeout 100 -k "decode or gemv" > gpurun_out/pytest_dynops.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dynops.log
cat gpurun_out/gemv_alone.log; tail -3 gpurun_out/pytest_dynops.log
