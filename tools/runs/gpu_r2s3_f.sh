# Round 2 s3: e2e tail probe (pull grid 28 / 42 / 56 / 84 CTAs)
mkdir -p gpurun_out/s3f
timeout 1500 python tools/e2e_tail_probe.py 28 42 56 84 > gpurun_out/s3f/e2e_tail_probe.json 2> gpurun_out/s3f/e2e_tail_probe.err; echo "rc=$?"
cat gpurun_out/s3f/e2e_tail_probe.json | head -c 3000
