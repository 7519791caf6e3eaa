# Lean-kernel A/B: block t+2 prefetched into L2 (libkpp_l2pf.so, -DKPP_LEAN_L2PF=1) vs the product library
# partials (4) and slab (8) barriers (libkpp_spin<mask>.so, -DKPP_LEAN_SPIN=<mask>).
O=${O:-gpurun_out/r2p}
mkdir -p $O
: > $O/ab.log
for rep in 1 2 3; do
  for v in base l2pf; do
    lib=""; [ "$v" != base ] && lib="$PWD/paper_2501_11673_b200/libkpp_$v.so"
    for c in c2 c1 c3; do
      echo "$c $v $(KPP_LIB=$lib timeout 300 python tools/prof_iter.py --config $c --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1)" >> $O/ab.log
    done
  done
done
cat $O/ab.log
