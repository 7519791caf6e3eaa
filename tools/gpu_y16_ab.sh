# Lean-kernel A/B: the 16th y group on the last warp (product) vs warp 0 taking two (libkpp_y15.so,
# -DKPP_LEAN_Y16=0), after the lean parity tests.
O=${O:-gpurun_out/r2y}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "lean or c1_ or twin_parity or stop or window or edge or zero_rhs or deterministic or x0" > $O/pytest_lean.log 2>&1
echo "pytest rc=$?"; tail -2 $O/pytest_lean.log
: > $O/ab.log
for rep in 1 2 3; do
  for v in base y15; do
    lib=""; [ "$v" != base ] && lib="$PWD/paper_2501_11673_b200/libkpp_$v.so"
    for c in c3 c2; do
      echo "$c $v $(KPP_LIB=$lib timeout 300 python tools/prof_iter.py --config $c --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1)" >> $O/ab.log
    done
  done
done
cat $O/ab.log
