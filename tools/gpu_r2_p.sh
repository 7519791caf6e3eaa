mkdir -p gpurun_out/r2
o=gpurun_out/r2/lean_rf.log; : > $o
for c in c2 c1; do
  echo "$c RF" >> $o; KPP_LEAN_RF=1 timeout 300 python tools/prof_iter.py --config $c --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1 >> $o
  echo "$c slice" >> $o; timeout 300 python tools/prof_iter.py --config $c --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1 >> $o
done
cat $o
KPP_LEAN_RF=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1 or twin_parity or closed_form or deterministic or stop_matches or edge" > gpurun_out/r2/pytest_rf.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2/pytest_rf.log
