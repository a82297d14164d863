# config 2/3 drain detail; config-4 head-prefetch A/B; GEMV head parity
set -x
mkdir -p gpurun_out
timeout 600 python tools/drain23_probe.py 3 > gpurun_out/drain23.json 2> gpurun_out/drain23.err
MS_GEMV_HEAD_KB=49152 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "gemv or decode" > gpurun_out/pytest_gemv_head.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemv_head.log
timeout 1500 python tools/gemv_head_ab.py 12 0,49152 > gpurun_out/gemv_head_ab.log 2>&1
tail -3 gpurun_out/pytest_gemv_head.log; cat gpurun_out/gemv_head_ab.log; head -c 3000 gpurun_out/drain23.json; tail -3 gpurun_out/drain23.err
