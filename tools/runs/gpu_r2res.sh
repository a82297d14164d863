set -x
mkdir -p gpurun_out
for r in 0 1; do
  MS_LP_SM_RESERVE=$r timeout 300 python tools/pair_outlier_probe.py 6 > gpurun_out/res_outlier_$r.log 2>&1
  MS_LP_SM_RESERVE=$r timeout 300 python tools/live_drain_probe.py > gpurun_out/res_drain_$r.json 2>/dev/null
  python - <<PY
import json
rows=[json.loads(l) for l in open('gpurun_out/res_outlier_$r.log') if l.startswith('{')]
infl=[x for r_ in rows for x in r_['inflight_top']]
print('reserve $r', 'inflight top', sorted(infl)[-6:], 'lp_exit p99s', [r_['lp_exit']['p99_ns'] for r_ in rows])
d=json.load(open('gpurun_out/res_drain_$r.json'))
for k,v in d.items(): print('   ', k, {a: v['flag_to_last_exit'].get(a) for a in ('p50_ns','p99_ns')}, 'seen', v['max_over_ctas_us']['seen'], 'last', v['max_over_ctas_us']['last'])
PY
done
