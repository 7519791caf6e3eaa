# exchange skeleton microbenchmarks + c2 with the arithmetic skipped
mkdir -p gpurun_out/r2
o=gpurun_out/r2/lat.log; : > $o
timeout 120 ./tools/microbench >> $o 2>&1
timeout 120 ./tools/lat_skel >> $o 2>&1
echo "c2 DBG_SKIP" >> $o; KPP_DBG_SKIP=1 timeout 300 python tools/prof_iter.py --config c2 --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1 >> $o
echo "c2 PHASE_PROFILE" >> $o; KPP_PHASE_PROFILE=1 timeout 300 python tools/prof_iter.py --config c2 --iters 4096 --reps 1 2>&1 | tail -3 >> $o
cat $o
