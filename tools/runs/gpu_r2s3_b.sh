# Round 2 s3: pair drain reorder (epilogues told before the MMA drain / redo push) + SM-free stamp
mkdir -p gpurun_out/s3b
timeout 900 python -m pytest tests -m gpu -q -x -p timeout --timeout 300 --timeout-method thread > gpurun_out/s3b/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3b/pytest_gpu.log
timeout 300 python tools/pair_drain_probe.py 60 > gpurun_out/s3b/pair_drain_probe.json 2> gpurun_out/s3b/pair_drain_probe.err; echo "drain rc=$?"
timeout 1200 python bench.py > gpurun_out/s3b/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/s3b/bench.log
tail -3 gpurun_out/s3b/pytest_gpu.log; head -c 600 gpurun_out/s3b/pair_drain_probe.json; tail -c 300 gpurun_out/s3b/bench.log
