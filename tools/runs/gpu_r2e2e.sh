set -x
mkdir -p gpurun_out
for kb in 0 24 0 24; do
  MS_PULL_SMEM_KB=$kb timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe_$kb.json 2> /dev/null
  python -c "
import json;d=json.load(open('gpurun_out/e2e_probe_$kb.json'))
print('pull_smem_kb=$kb', {k: d[k] for k in ('mode=2 exclusive','mode=2 splitkernel')})"
done
