set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
timeout 900 python tools/gemv_dynamic_ab.py 12 > gpurun_out/gemv_dynamic_ab.log 2>&1
tail -n 3 gpurun_out/smoke.log; grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -15; cat gpurun_out/e2e_probe.log | tail -45; cat gpurun_out/gemv_dynamic_ab.log | tail -60
