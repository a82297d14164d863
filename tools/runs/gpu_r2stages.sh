# fused HP chain mainloop vs ring depth (latency- or ingest-bound?): stock build, then
# rebuilt on the box with the ring capped at 4 and 3 stages
mkdir -p gpurun_out/stages
timeout 200 python tools/fused_scale_probe.py > gpurun_out/stages/s_default.txt 2>&1
for n in 4 3; do
  touch paper_2601_04071_b200/csrc/cuda/ms_b200.cu
  make -j8 cuda NVEXTRA=-DMS_FUSED_MAX_STAGES=$n > gpurun_out/stages/build_$n.log 2>&1
  timeout 200 python tools/fused_scale_probe.py > gpurun_out/stages/s_$n.txt 2>&1
done
for f in gpurun_out/stages/s_*.txt; do echo $f; grep "^{" $f; done
