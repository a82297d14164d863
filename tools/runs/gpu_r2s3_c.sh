# Round 2 s3: quarter-unit wave tail for the CTA-pair LP GEMM (parity + wave probe)
mkdir -p gpurun_out/s3c
timeout 600 python -m pytest tests/test_gpu_preempt.py tests/test_gpu_kernels.py -m gpu -q -x -p timeout --timeout 300 --timeout-method thread > gpurun_out/s3c/pytest_pair.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3c/pytest_pair.log
tail -3 gpurun_out/s3c/pytest_pair.log
grep -q "pytest rc=0" gpurun_out/s3c/pytest_pair.log || exit 1
timeout 400 python tools/gemm_wave_probe.py > gpurun_out/s3c/gemm_wave_probe.json 2> gpurun_out/s3c/gemm_wave_probe.err; echo "wave rc=$?"
cat gpurun_out/s3c/gemm_wave_probe.json
