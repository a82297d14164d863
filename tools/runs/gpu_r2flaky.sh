# GPU suite repeated (flakiness check of the timing-based tests)
mkdir -p gpurun_out/flaky
for i in 1 2 3; do
  timeout 900 python -m pytest tests -m gpu -q -p timeout --timeout 300 --timeout-method thread > gpurun_out/flaky/run$i.log 2>&1
  echo "run $i rc=$?"; grep -E "passed|failed" gpurun_out/flaky/run$i.log | tail -1; grep -E "^FAILED|Error" gpurun_out/flaky/run$i.log | head -5
done
