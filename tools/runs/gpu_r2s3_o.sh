# Round 2 s3: LP GEMM kernel for the live config-1 windows: pairs 256x512 (2) / pairs 256x256 (1) / single CTA (0)
mkdir -p gpurun_out/s3o
timeout 1700 python tools/live_env_ab.py MS_LP_GEMM_PAIR 2 1 0 > gpurun_out/s3o/lp_kernel_ab.json 2> gpurun_out/s3o/lp_kernel_ab.err; echo "rc=$?"
cat gpurun_out/s3o/lp_kernel_ab.json; tail -3 gpurun_out/s3o/lp_kernel_ab.err
