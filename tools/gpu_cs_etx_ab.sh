# c5 A/B: the DSMEM barriers' expect_tx arrivals by the last chain thread (libkpp_ex.so) vs by thread 0,
# a streaming thread (libkpp.so), interleaved, with phase profiles.
O=${O:-gpurun_out/r2etx}
mkdir -p $O
X=$PWD/paper_2501_11673_b200/libkpp_ex.so
: > $O/ab.log
for rep in 1 2 3; do
  echo "c5 base $(timeout 300 python tools/prof_iter.py --config c5 --iters 512 --reps 2 2>&1 | grep -E 'us/iter|rror' | tail -1)" >> $O/ab.log
  echo "c5 ex   $(KPP_LIB=$X timeout 300 python tools/prof_iter.py --config c5 --iters 512 --reps 2 2>&1 | grep -E 'us/iter|rror' | tail -1)" >> $O/ab.log
done
for v in base ex; do
  lib=""; [ $v = ex ] && lib=$X
  echo "== $v" >> $O/phase.log
  KPP_LIB=$lib KPP_PHASE_PROFILE=1 timeout 300 python tools/prof_iter.py --config c5 --iters 512 --reps 1 >> $O/phase.log 2>&1
done
cat $O/ab.log; grep -E "==|phase cycles" $O/phase.log
