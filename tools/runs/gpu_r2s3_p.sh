# Round 2 s3: last validation of the committed tree (smoke, GPU suite, bench)
mkdir -p gpurun_out/s3p
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3p/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s3p/smoke.log
timeout 900 python -m pytest tests -m gpu -q -p timeout --timeout 300 --timeout-method thread > gpurun_out/s3p/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3p/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/s3p/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/s3p/bench.log
tail -2 gpurun_out/s3p/smoke.log; tail -2 gpurun_out/s3p/pytest_gpu.log; tail -c 200 gpurun_out/s3p/bench.log
