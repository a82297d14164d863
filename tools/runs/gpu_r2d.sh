set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/gemv_dynamic_ab.py 12 > gpurun_out/gemv_dynamic_ab.log 2>&1
timeout 1500 python bench.py --steps 4 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -15; cat gpurun_out/gemv_dynamic_ab.log | tail -60; tail -c 1500 gpurun_out/bench.log
