# Round 2 s3: bench with the e2e split (where the e2e tail sits)
mkdir -p gpurun_out/s3m
timeout 1200 python bench.py > gpurun_out/s3m/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/s3m/bench.log
tail -c 200 gpurun_out/s3m/bench.log
