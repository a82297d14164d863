# LP drain phases of the CTA-pair GEMM: MMA-queue bound 2 (default) vs 1 vs 0 (unbounded)
mkdir -p gpurun_out/drainab
for lag in 2 1 2 1; do
  MS_LP_MMA_LAG=$lag timeout 300 python tools/live_drain_probe.py > gpurun_out/drainab/lag${lag}_$RANDOM.json 2>/dev/null
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/drainab/*.json')):
    try: d = json.load(open(f))
    except Exception as e: print(f, 'ERR', e); continue
    for k, v in d.items():
        print(f.split('/')[-1], k, v['runs'], {x: v['flag_to_last_exit'][x] for x in ('p50_ns', 'p99_ns')},
              {x: v['max_over_ctas_us'][x][:2] for x in ('seen', 'prod_done', 'mma_done', 'epi_done', 'teardown', 'last')})
PY
