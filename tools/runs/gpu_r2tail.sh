# pair GEMM half-tile tail: parity tests, then the A/B
timeout 400 python -m pytest tests/test_gpu_preempt.py tests/test_gpu_tier.py -q -x -p timeout --timeout 200 > gpurun_out/pytest_tail.log 2>&1; tail -3 gpurun_out/pytest_tail.log
timeout 300 python tools/gemm_tail_ab.py 2 2>&1 | tail -2
