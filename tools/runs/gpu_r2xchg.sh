# fused HP chain: k-slice exchange through DSMEM (default) vs L2 (MS_FUSED_XCHG=1)
mkdir -p gpurun_out/xchg
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p timeout --timeout 200 -k "fused or chain" > gpurun_out/xchg/pytest.log 2>&1; tail -2 gpurun_out/xchg/pytest.log
for v in 0 1 0 1; do MS_FUSED_XCHG=$v timeout 120 python tools/fused_stamps.py 1 > gpurun_out/xchg/stamps_$v.txt 2>&1; echo "xchg=$v"; tail -6 gpurun_out/xchg/stamps_$v.txt | cut -c1-400; done
