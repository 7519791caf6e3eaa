# Lean-kernel A/B: block t+1 slab gathers issued by the last W warps (libkpp_splitW.so, -DKPP_LEAN_TMA_SPLIT=W)
O=${O:-gpurun_out/r2x}
mkdir -p $O
: > $O/ab.log
for rep in 1 2; do
  for v in base split2 split4 split8; do
    lib=""; [ "$v" != base ] && lib="$PWD/paper_2501_11673_b200/libkpp_$v.so"
    for c in c2 c1 c3; do
      echo "$c $v $(KPP_LIB=$lib timeout 300 python tools/prof_iter.py --config $c --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1)" >> $O/ab.log
    done
  done
done
cat $O/ab.log
