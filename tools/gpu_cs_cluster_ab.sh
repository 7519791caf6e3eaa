# c5 CD++ streaming kernel: cluster size 2 (the plan's choice) vs 4 / 8 forced (fewer clusters: fewer L2
# values per CTA in the cross-cluster gather of r), interleaved, with phase profiles.
O=${O:-gpurun_out/r2cl}
mkdir -p $O
: > $O/ab.log
for rep in 1 2; do
  for C in 0 4 8; do
    echo "c5 C=$C $(timeout 300 python tools/prof_iter.py --config c5 --iters 512 --reps 2 --cluster $C 2>&1 | grep -E 'us/iter|rror' | tail -1)" >> $O/ab.log
  done
done
for C in 0 4 8; do
  echo "== C=$C" >> $O/phase.log
  KPP_PHASE_PROFILE=1 timeout 300 python tools/prof_iter.py --config c5 --iters 512 --reps 1 --cluster $C >> $O/phase.log 2>&1
done
cat $O/ab.log; grep -E "==|phase cycles" $O/phase.log
