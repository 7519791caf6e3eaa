mkdir -p gpurun_out/r2
o=gpurun_out/r2/lean_traffic2.log; : > $o
for d in 0 2 16; do echo "c2 DBG_SKIP=$d" >> $o; KPP_DBG_SKIP=$d timeout 300 python tools/prof_iter.py --config c2 --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1 >> $o; done
cat $o
