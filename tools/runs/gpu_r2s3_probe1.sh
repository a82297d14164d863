# Round 2 s3: CTA-pair drain phase stamps + wave-quantisation ranges
mkdir -p gpurun_out/s3
timeout 300 python tools/pair_drain_probe.py 60 > gpurun_out/s3/pair_drain_probe.json 2> gpurun_out/s3/pair_drain_probe.err; echo "drain rc=$?"
timeout 300 python tools/gemm_wave_probe.py > gpurun_out/s3/gemm_wave_probe.json 2> gpurun_out/s3/gemm_wave_probe.err; echo "wave rc=$?"
cat gpurun_out/s3/gemm_wave_probe.json; tail -3 gpurun_out/s3/*.err
