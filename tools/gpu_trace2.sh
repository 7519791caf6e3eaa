# Lean-kernel latency anatomy (c2, c3): globaltimer trace, per-phase cycle counters of CTA 0, and the
# slab-fill timing switches (KPP_DBG_SKIP 2: no slab copy, 16: L2 prefetch only, 4: no M rows; results wrong).
O=${O:-gpurun_out/r2tr}
mkdir -p $O
for c in c2 c3; do
  KPP_TRACE=$O/trace_$c.bin timeout 300 python tools/prof_iter.py --config $c --iters 2048 --reps 1 > $O/trace_$c.log 2>&1
  python tools/trace_report.py $O/trace_$c.bin >> $O/trace_$c.log 2>&1
  KPP_PHASE_PROFILE=1 timeout 300 python tools/prof_iter.py --config $c --iters 2048 --reps 1 >> $O/trace_$c.log 2>&1
  for k in 2 16 4 6; do echo "KPP_DBG_SKIP=$k" >> $O/trace_$c.log; KPP_DBG_SKIP=$k timeout 300 python tools/prof_iter.py --config $c --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1 >> $O/trace_$c.log; done
  rm -f $O/trace_$c.bin
done
cat $O/trace_c2.log $O/trace_c3.log
