mkdir -p gpurun_out/r2
o=gpurun_out/r2/regress.log; : > $o
echo "c5" >> $o; timeout 600 python tools/prof_iter.py --config c5 --iters 512 --reps 2 2>&1 | grep us/iter | tail -1 >> $o
echo "c4" >> $o; timeout 600 python tools/prof_iter.py --config c4 --iters 128 --reps 2 2>&1 | grep us/iter | tail -1 >> $o
for l in 1 0; do echo "c3 LEAN64=$l" >> $o; KPP_LEAN64=$l timeout 600 python tools/prof_iter.py --config c3 --iters 2048 --reps 2 2>&1 | grep us/iter | tail -1 >> $o; done
echo "c2" >> $o; timeout 600 python tools/prof_iter.py --config c2 --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1 >> $o
cat $o
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "rank_stage or dist_context or twin_parity or c1 or closed_form or plans or stop_matches or edge or fullsize_parity" > gpurun_out/r2/pytest_u.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2/pytest_u.log
