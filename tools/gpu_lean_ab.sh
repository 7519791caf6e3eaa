# Lean-kernel A/B: the product library (register tile of block t+1 loaded at the end of iteration t)
# against libkpp_late.so (-DKPP_LEAN_EARLY_TILE=0: loaded at the top of the iteration), after the
# lean-kernel parity tests.  O=outdir bash tools/gpu_lean_ab.sh
O=${O:-gpurun_out/r2l}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "lean or c1_ or twin_parity or stop or window or edge or zero_rhs or deterministic or x0" > $O/pytest_lean.log 2>&1
echo "pytest rc=$?"; tail -2 $O/pytest_lean.log
: > $O/ab.log
for rep in 1 2 3; do
  for v in base late; do
    lib=""; [ "$v" != base ] && lib="$PWD/paper_2501_11673_b200/libkpp_$v.so"
    for c in c2 c1 c3; do
      echo "$c $v $(KPP_LIB=$lib timeout 300 python tools/prof_iter.py --config $c --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1)" >> $O/ab.log
    done
  done
done
cat $O/ab.log
