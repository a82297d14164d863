# pair-512 LP GEMM default + reserve 0: smoke, GPU suite, exit probe, bench
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/exit_probe.py > gpurun_out/exit_probe.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -2 gpurun_out/smoke.log; grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -12; head -30 gpurun_out/exit_probe.log; tail -c 400 gpurun_out/bench.log
