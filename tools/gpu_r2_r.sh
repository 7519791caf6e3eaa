mkdir -p gpurun_out/r2
o=gpurun_out/r2/syrk2.log; : > $o
for c in c2 c3 c4; do
  for v in 1 0; do
    KPP_GRAM_SYRK=$v timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu --no-ttt --secondary '' 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c SYRK=$v', round(d['value'],1), 'p1 %.2f'%d['phase1_ms_per_step'], 'p2 %.2f'%d['phase2_ms_per_step'], d['phase1_fp64'])" >> $o
  done
done
cat $o
