set -x
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -c 300 gpurun_out/bench.log
