# split-K reduction tree: preempt/resume parity, GEMM vs cuBLAS A/B, config 2/3 drain
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tenants23.py -q -k "split or train" > gpurun_out/pytest_split.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_split.log
timeout 300 python tools/gemm_vs_cublas.py 4 > gpurun_out/gemm_vs_cublas.json 2> gpurun_out/gemm_vs_cublas.err
timeout 900 python tools/cfg23_probe.py 3 > gpurun_out/cfg23_probe.json 2> gpurun_out/cfg23_probe.err
tail -3 gpurun_out/pytest_split.log; cat gpurun_out/gemm_vs_cublas.json; tail -3 gpurun_out/gemm_vs_cublas.err
python -c "
import json; d=json.load(open('gpurun_out/cfg23_probe.json'))
for c,v in d.items():
    print(c, 'ex', v['exclusive_att'])
    for k,x in v.items():
        if isinstance(x, dict) and 'att' in x: print('  ', k, {a: (round(b,4) if isinstance(b,float) else b) for a,b in x.items()})
"
