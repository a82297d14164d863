# Round 2 s3: configs 2/3 LP drain vs the gate's poller count (4 / 8 warps, alternating)
mkdir -p gpurun_out/s3j
for rnd in 1 2; do for gw in 4 8; do
  MS_GATE_WARPS=$gw timeout 400 python tools/drain23_probe.py 3 > gpurun_out/s3j/drain23_gw${gw}_r${rnd}.json 2> gpurun_out/s3j/drain23_gw${gw}_r${rnd}.err
  python -c "
import json; d=json.load(open('gpurun_out/s3j/drain23_gw${gw}_r${rnd}.json'))
print('gw=$gw r=$rnd', {k: (v['n'], v['exit_p50_us'], v['exit_p99_us'], v['lp_exit_summary'].get('p99_ns')) for k, v in d.items()})"
done; done
