mkdir -p gpurun_out/r2
o=gpurun_out/r2/ab_ry_xs.log; : > $o
for rep in 1 2; do
for v in "" ry2 xs2; do
  lib=""; [ -n "$v" ] && lib="$PWD/paper_2501_11673_b200/libkpp_$v.so"
  for c in c2 c3 c1; do echo "$c variant=${v:-base}" >> $o; KPP_LIB=$lib timeout 300 python tools/prof_iter.py --config $c --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1 >> $o; done
done
done
cat $o
