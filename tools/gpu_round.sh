#!/bin/bash
# One GPU-box session: smoke, GPU tests, bench (+ reference arm), ncu evidence, live probes.
# Outputs under gpurun_out/.  NCU=0 / LIVE=0 skip the profiler / live-probe parts.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 4 --warmup 3 > gpurun_out/bench_ref.log 2>&1
if [ "${NCU:-1}" = "1" ]; then
# launch list of the bench command (profiling mode: direct HP launches, no config-4 leg)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --step-s 0.2 --warmup-s 0.05 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 1 -c 2 \
  -o gpurun_out/prof_gemm -f python tools/ncu_target.py > gpurun_out/ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:axpy_kernel -s 1 -c 1 \
  -o gpurun_out/prof_axpy -f python tools/ncu_target.py > gpurun_out/ncu_axpy.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hp_fused -s 1 -c 1 \
  -o gpurun_out/prof_fused -f python tools/ncu_fused.py > gpurun_out/ncu_fused.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hp_gemv -s 1 -c 3 \
  -o gpurun_out/prof_gemv -f python tools/ncu_gemv.py both > gpurun_out/ncu_gemv.log 2>&1
fi
if [ "${LIVE:-1}" = "1" ]; then
timeout 600 python tools/live_check.py 2.0 > gpurun_out/live_check.log 2>&1
timeout 900 python tools/live_check4.py 10.0 > gpurun_out/live_check4.log 2>&1
timeout 200 python tools/exit_probe.py > gpurun_out/exit_probe.log 2>&1
timeout 300 python tools/first_cta_probe.py > gpurun_out/first_cta_probe.log 2>&1
timeout 300 python tools/gemv_probe.py > gpurun_out/gemv_probe.log 2>&1
timeout 200 python tools/gemm_probe.py > gpurun_out/gemm_probe.log 2>&1
timeout 300 python tools/axpy_probe.py > gpurun_out/axpy_probe.log 2>&1
timeout 300 python tools/tier_probe.py gpurun_out/tier_probe.json > gpurun_out/tier_probe.log 2>&1
timeout 1200 python tools/live_memory_case.py 6 gpurun_out/live_memory_case.json > gpurun_out/live_memory_case.log 2>&1
timeout 300 python tools/gemm_group_sweep.py gpurun_out/gemm_group_sweep.json > gpurun_out/gemm_group_sweep.log 2>&1
fi
tail -n 2 gpurun_out/smoke.log gpurun_out/pytest_gpu.log; tail -c 1500 gpurun_out/bench.log; tail -c 800 gpurun_out/bench_ref.log
