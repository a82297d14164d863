# ncu --set full of cuBLAS 8192^3 vs our LP GEMM (same process), for a side-by-side
set -x
mkdir -p gpurun_out/r2o
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm|xmma|nvjet|sm100|tc_gemm" -c 4 \
  -o gpurun_out/r2o/cmp -f python tools/ncu_cublas_vs_ours.py > gpurun_out/r2o/ncu.log 2>&1
ncu -i gpurun_out/r2o/cmp.ncu-rep --page raw --csv > gpurun_out/r2o/cmp_raw.csv 2>&1
ncu -i gpurun_out/r2o/cmp.ncu-rep --page details --csv > gpurun_out/r2o/cmp_details.csv 2>&1
tail -5 gpurun_out/r2o/ncu.log; ls -la gpurun_out/r2o
