set -x
mkdir -p gpurun_out/r02
timeout 1800 python bench.py --steps 8 --warmup 3 > gpurun_out/r02/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r02/bench.log
cp gpurun_out/bench_detail.json gpurun_out/r02/ 2>/dev/null; cp gpurun_out/calib_b200.json gpurun_out/r02/ 2>/dev/null
timeout 600 python bench.py --impl reference --steps 8 --warmup 3 > gpurun_out/r02/bench_reference.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02/launches.csv \
  python bench.py --steps 1 --warmup 3 --step-s 0.2 --warmup-s 0.05 --no-cpu-baseline > gpurun_out/r02/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 1 -c 1 -o gpurun_out/r02/prof_gemm -f python tools/ncu_target_r2.py lp > gpurun_out/r02/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:axpy_kernel -s 1 -c 1 -o gpurun_out/r02/prof_axpy -f python tools/ncu_target_r2.py lp > gpurun_out/r02/ncu_axpy.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:optim_kernel -s 1 -c 1 -o gpurun_out/r02/prof_optim -f python tools/ncu_target_r2.py lp > gpurun_out/r02/ncu_optim.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hp_fused -s 1 -c 1 -o gpurun_out/r02/prof_fused -f python tools/ncu_target_r2.py hp > gpurun_out/r02/ncu_fused.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hp_gemv -s 1 -c 1 -o gpurun_out/r02/prof_gemv -f python tools/ncu_target_r2.py hp > gpurun_out/r02/ncu_gemv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_kernel|add_ln|im2col|bias_act" -c 8 -o gpurun_out/r02/prof_glue -f python tools/ncu_target_r2.py t23 > gpurun_out/r02/ncu_glue.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02/t23_launches.csv python tools/ncu_target_r2.py t23 > gpurun_out/r02/t23_ncu.log 2>&1
ls -la gpurun_out/r02; tail -c 2500 gpurun_out/r02/bench.log; tail -c 600 gpurun_out/r02/bench_reference.log
