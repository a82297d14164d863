# Round 2 s3: final-build validation (gate 8 pollers, pull 56 CTAs) — smoke, GPU suite, bench, reference arm, config-4 repeats
mkdir -p gpurun_out/s3k
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3k/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s3k/smoke.log
timeout 900 python -m pytest tests -m gpu -q -p timeout --timeout 300 --timeout-method thread > gpurun_out/s3k/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3k/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/s3k/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/s3k/bench.log
timeout 900 python bench.py --impl reference > gpurun_out/s3k/bench_reference.log 2>&1; echo "ref rc=$?" >> gpurun_out/s3k/bench_reference.log
REPS=3 timeout 1200 python tools/cfg4_repeats.py > gpurun_out/s3k/cfg4_repeats.json 2> gpurun_out/s3k/cfg4_repeats.err; echo "cfg4 rc=$?"
tail -2 gpurun_out/s3k/smoke.log; tail -2 gpurun_out/s3k/pytest_gpu.log; tail -c 300 gpurun_out/s3k/bench.log
