# round-2 profiling of the CTA-pair LP GEMM: launch list of the bench command + ncu --set full
set -x
mkdir -p gpurun_out/r02b
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02b/launches.csv \
  python bench.py --steps 1 --warmup 3 --step-s 0.2 --warmup-s 0.05 --no-cpu-baseline > gpurun_out/r02b/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm2 -s 1 -c 1 \
  -o gpurun_out/r02b/prof_gemm2 -f python tools/ncu_target.py > gpurun_out/r02b/ncu_gemm2.log 2>&1
python tools/ncu_summarize.py gpurun_out/r02b > gpurun_out/r02b/summary.json
ncu -i gpurun_out/r02b/prof_gemm2.ncu-rep --page details --csv > gpurun_out/r02b/gemm2_details.csv 2>&1
tail -3 gpurun_out/r02b/ncu_gemm2.log; head -c 1500 gpurun_out/r02b/summary.json
