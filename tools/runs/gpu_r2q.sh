# new CTA-pair GEMM: parity + preemption protocol, then the A/B vs cuBLAS
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_preempt.py -q -x -k "pair" > gpurun_out/pytest_pair.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pair.log
tail -5 gpurun_out/pytest_pair.log
if grep -q "rc=0" gpurun_out/pytest_pair.log; then
  timeout 600 python tools/gemm_ab2.py 3 > gpurun_out/gemm_ab2.log 2>&1
  cat gpurun_out/gemm_ab2.log | tail -3
fi
