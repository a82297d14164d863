# Round 2 s3: config-4 leg with the gate's 4 pollers (vs 8 in the final-build run), seeds 7 / 1007
mkdir -p gpurun_out/s3l
MS_GATE_WARPS=4 REPS=2 timeout 1200 python tools/cfg4_repeats.py > gpurun_out/s3l/cfg4_repeats_gw4.json 2> gpurun_out/s3l/cfg4_repeats_gw4.err; echo "rc=$?"
MS_GATE_WARPS=8 REPS=2 timeout 1200 python tools/cfg4_repeats.py > gpurun_out/s3l/cfg4_repeats_gw8.json 2> gpurun_out/s3l/cfg4_repeats_gw8.err; echo "rc=$?"
cat gpurun_out/s3l/cfg4_repeats_gw4.json gpurun_out/s3l/cfg4_repeats_gw8.json
