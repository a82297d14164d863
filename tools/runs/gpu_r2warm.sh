# gate L2 warm-up A/B, alternating processes; then the chain tests with the warm-up on
for v in 0 2 0 2 4; do MS_GATE_WARM_KB=$v timeout 300 python tools/gate_warm_ab.py 2>/dev/null | tail -1; done
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_live.py -q -x -p timeout --timeout 200 2>&1 | tail -2
