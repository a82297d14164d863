# Round 2, session 3: re-validate HEAD on a fresh box (smoke, GPU suite, default bench)
mkdir -p gpurun_out/s3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s3/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p timeout --timeout 400 --timeout-method thread > gpurun_out/s3/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/s3/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/s3/bench.log
tail -2 gpurun_out/s3/smoke.log; tail -3 gpurun_out/s3/pytest_gpu.log; tail -c 400 gpurun_out/s3/bench.log
