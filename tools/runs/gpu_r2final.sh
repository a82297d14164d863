# round-2 final: smoke, GPU suite, bench, reference arm, launch list of the bench command
set -x
mkdir -p gpurun_out/final
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p timeout --timeout 300 --timeout-method thread > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 1500 python bench.py --detail gpurun_out/final/bench_detail.json > gpurun_out/final/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/final/bench.log
timeout 600 python bench.py --impl reference --steps 4 --warmup 3 > gpurun_out/final/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final/launches.csv \
  python bench.py --steps 1 --warmup 3 --step-s 0.2 --warmup-s 0.05 --no-cpu-baseline --single-cta-windows 0 > gpurun_out/final/bench_under_ncu.log 2>&1
tail -2 gpurun_out/final/smoke.log; grep -E "passed|failed|FAILED|Timeout" gpurun_out/final/pytest_gpu.log | tail -6; tail -c 300 gpurun_out/final/bench.log; tail -c 300 gpurun_out/final/bench_ref.log
