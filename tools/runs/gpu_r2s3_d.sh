# Round 2 s3: GPU suite, smoke, bench (burst-aligned roofline timing + in-step figure), launch list, ncu of the pair GEMM
mkdir -p gpurun_out/s3d
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3d/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s3d/smoke.log
timeout 900 python -m pytest tests -m gpu -q -p timeout --timeout 300 --timeout-method thread > gpurun_out/s3d/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3d/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/s3d/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/s3d/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/s3d/launches.csv \
  python bench.py --steps 1 --warmup 3 --step-s 0.2 --warmup-s 0.05 --no-cpu-baseline > gpurun_out/s3d/bench_under_ncu.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm2 -s 1 -c 1 \
  -o gpurun_out/s3d/prof_gemm2 -f python tools/ncu_target.py > gpurun_out/s3d/ncu_gemm2.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summarize.py gpurun_out/s3d > gpurun_out/s3d/summary.json
ncu -i gpurun_out/s3d/prof_gemm2.ncu-rep --page details --csv > gpurun_out/s3d/gemm2_details.csv 2>&1
tail -2 gpurun_out/s3d/smoke.log; tail -2 gpurun_out/s3d/pytest_gpu.log; tail -c 300 gpurun_out/s3d/bench.log
