mkdir -p gpurun_out/r2
o=gpurun_out/r2/lean_s2.log; : > $o
for c in c2 c1; do
  echo "$c S2" >> $o; timeout 300 python tools/prof_iter.py --config $c --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1 >> $o
  echo "$c S1" >> $o; KPP_LEAN_S2=0 timeout 300 python tools/prof_iter.py --config $c --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1 >> $o
done
cat $o
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1 or twin_parity or closed_form or deterministic or stop_matches or edge or padded or x0_and or max_block or zero_rhs" > gpurun_out/r2/pytest_s2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2/pytest_s2.log
