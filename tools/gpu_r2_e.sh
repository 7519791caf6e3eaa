mkdir -p gpurun_out/r2
o=gpurun_out/r2/lat2.log; : > $o
timeout 60 ./tools/lat_skel >> $o 2>&1
for pf in 0 1 2; do echo "PF_AT=$pf" >> $o; KPP_PF_AT=$pf timeout 300 python tools/prof_iter.py --config c2 --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1 >> $o; done
for pf in 1 2; do echo "PF_AT=$pf profile" >> $o; KPP_PF_AT=$pf KPP_PHASE_PROFILE=1 timeout 300 python tools/prof_iter.py --config c2 --iters 4096 --reps 1 2>&1 | grep cycles >> $o; done
for pf in 0 1 2; do echo "c3 PF_AT=$pf" >> $o; KPP_PF_AT=$pf timeout 300 python tools/prof_iter.py --config c3 --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1 >> $o; done
cat $o
