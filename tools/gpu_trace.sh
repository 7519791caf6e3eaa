# Phase-2 latency breakdown of the persistent kernel (globaltimer trace + per-phase cycle counters)
for c in c2 c3; do
  KPP_TRACE=gpurun_out/trace_$c.bin timeout 300 python tools/prof_iter.py --config $c --iters 2048 --reps 1 > gpurun_out/trace_$c.log 2>&1
  python tools/trace_report.py gpurun_out/trace_$c.bin >> gpurun_out/trace_$c.log 2>&1
  KPP_PHASE_PROFILE=1 timeout 300 python tools/prof_iter.py --config $c --iters 2048 --reps 1 >> gpurun_out/trace_$c.log 2>&1
  KPP_DBG_SKIP=1 timeout 300 python tools/prof_iter.py --config $c --iters 2048 --reps 1 >> gpurun_out/trace_$c.log 2>&1
  for C in 1 2 8 16; do timeout 300 python tools/prof_iter.py --config $c --iters 2048 --reps 1 --cluster $C >> gpurun_out/trace_$c.log 2>&1; done
done
