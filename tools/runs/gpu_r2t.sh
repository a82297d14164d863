set -x
mkdir -p gpurun_out
timeout 300 python tools/pair_gate_probe.py > gpurun_out/pair_gate.json 2> gpurun_out/pair_gate.err
cat gpurun_out/pair_gate.json; tail -3 gpurun_out/pair_gate.err
