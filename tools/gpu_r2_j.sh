mkdir -p gpurun_out/r2
o=gpurun_out/r2/lean_prof.log; : > $o
for c in c2 c1; do echo "$c" >> $o; KPP_PHASE_PROFILE=1 timeout 300 python tools/prof_iter.py --config $c --iters 4096 --reps 1 2>&1 | grep "cycles\|us/iter" >> $o; done
cat $o
