# Round 2 s3: CTA-pair MMA queue bound A/B (throughput + drain), lags 2 / 1 / 3
mkdir -p gpurun_out/s3n
timeout 1500 python tools/pair_lag_ab.py 2 1 3 > gpurun_out/s3n/pair_lag_ab.json 2> gpurun_out/s3n/pair_lag_ab.err; echo "rc=$?"
cat gpurun_out/s3n/pair_lag_ab.json; tail -3 gpurun_out/s3n/pair_lag_ab.err
