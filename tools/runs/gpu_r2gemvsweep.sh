# config-4 decode step alone vs the GEMV L2 lookahead (MS_GEMV_PREFETCH, units past the issue point)
for r in 1 2; do
for pf in 16 0 8 32 64 128; do
  echo -n "prefetch=$pf "; MS_GEMV_PREFETCH=$pf timeout 120 python tools/gemv_alone.py 2>/dev/null | tail -1
done
done
