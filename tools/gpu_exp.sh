for c in c3 c4 c5; do timeout 600 python tools/prof_iter.py --config $c --iters 512 --reps 1 --rht; done > gpurun_out/exp.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:fht_rows_pass -c 2 -f -o gpurun_out/fht_c3 python tools/prof_iter.py --config c3 --iters 16 --reps 1 --rht > gpurun_out/ncu_fht.log 2>&1
