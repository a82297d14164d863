set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_live.py -v -x -p timeout --timeout 240 --timeout-method thread -k "config4_short or governor" > gpurun_out/pytest_live.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_live.log
timeout 300 python tools/live_drain_probe.py > gpurun_out/live_drain.json 2> gpurun_out/live_drain.err
tail -60 gpurun_out/pytest_live.log; head -c 2500 gpurun_out/live_drain.json
