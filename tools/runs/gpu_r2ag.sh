# round-2 candidate: smoke, GPU suite (per-test timeout), bench, reference arm
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p timeout --timeout 300 --timeout-method thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 4 --warmup 3 > gpurun_out/bench_ref.log 2>&1
tail -2 gpurun_out/smoke.log; grep -E "passed|failed|FAILED|Timeout" gpurun_out/pytest_gpu.log | tail -6; tail -c 300 gpurun_out/bench.log; tail -c 600 gpurun_out/bench_ref.log
