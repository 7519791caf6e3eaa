# A/B of library variants: bash tools/gpu_ab.sh "variant1 variant2" "c2 c3 c1" [iters]
# (variant "" = the product libkpp.so; others paper_2501_11673_b200/libkpp_<v>.so)
mkdir -p gpurun_out/r2
o=gpurun_out/r2/ab.log; : > $o
for rep in 1 2; do
  for v in base $1; do
    lib=""; [ "$v" != base ] && lib="$PWD/paper_2501_11673_b200/libkpp_$v.so"
    for c in $2; do echo "$c $v" >> $o; KPP_LIB=$lib timeout 300 python tools/prof_iter.py --config $c --iters ${3:-4096} --reps 2 2>&1 | grep us/iter | tail -1 >> $o; done
  done
done
cat $o
