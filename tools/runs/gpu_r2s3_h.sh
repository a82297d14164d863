# Round 2 s3: final-build validation — smoke, GPU suite, bench, reference arm
mkdir -p gpurun_out/s3h
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3h/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s3h/smoke.log
timeout 900 python -m pytest tests -m gpu -q -p timeout --timeout 300 --timeout-method thread > gpurun_out/s3h/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3h/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/s3h/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/s3h/bench.log
timeout 900 python bench.py --impl reference > gpurun_out/s3h/bench_reference.log 2>&1; echo "ref rc=$?" >> gpurun_out/s3h/bench_reference.log
tail -2 gpurun_out/s3h/smoke.log; tail -2 gpurun_out/s3h/pytest_gpu.log; tail -c 300 gpurun_out/s3h/bench.log; tail -c 300 gpurun_out/s3h/bench_reference.log
