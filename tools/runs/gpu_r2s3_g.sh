# Round 2 s3: doorbell gate pollers A/B (4 / 8 / 16 warps)
mkdir -p gpurun_out/s3g
timeout 1500 python tools/gate_pollers_ab.py 4 8 16 > gpurun_out/s3g/gate_pollers_ab.json 2> gpurun_out/s3g/gate_pollers_ab.err; echo "rc=$?"
cat gpurun_out/s3g/gate_pollers_ab.json
