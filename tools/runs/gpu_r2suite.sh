set -x
mkdir -p gpurun_out/final
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke2.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke2.log
timeout 1800 python -m pytest tests -m gpu -q -p timeout --timeout 300 --timeout-method thread > gpurun_out/final/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu2.log
tail -2 gpurun_out/final/smoke2.log; tail -3 gpurun_out/final/pytest_gpu2.log
