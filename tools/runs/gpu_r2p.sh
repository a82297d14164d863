set -x
mkdir -p gpurun_out/r2p
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm" -c 4 \
  -o gpurun_out/r2p/pair -f python tools/ncu_pair.py > gpurun_out/r2p/ncu.log 2>&1
ncu -i gpurun_out/r2p/pair.ncu-rep --page raw --csv > gpurun_out/r2p/raw.csv 2>&1
ncu -i gpurun_out/r2p/pair.ncu-rep --page details --csv > gpurun_out/r2p/details.csv 2>&1
for i in 0 2; do ncu -i gpurun_out/r2p/pair.ncu-rep --page source --csv --launch-skip $i --launch-count 1 --print-source sass > gpurun_out/r2p/src_$i.csv 2>&1; done
timeout 600 python tools/drain23_probe.py 3 > gpurun_out/drain23.json 2> gpurun_out/drain23.err
tail -3 gpurun_out/r2p/ncu.log; ls -la gpurun_out/r2p
