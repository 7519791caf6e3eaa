mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rank_stage or dist_path or dist_context or emulated or engines_agree or launch_plans or c1" > gpurun_out/r2/pytest_pk.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2/pytest_pk.log
o=gpurun_out/r2/pk_timing.log; : > $o
for v in 1 2 4 8; do echo "c4 engine0 vranks=$v" >> $o; timeout 600 python tools/prof_iter.py --config c4 --iters 128 --reps 2 --vranks $v 2>&1 | grep us/iter | tail -1 >> $o; done
for v in 1 2 4; do echo "c3 engine0 vranks=$v" >> $o; timeout 600 python tools/prof_iter.py --config c3 --iters 2048 --reps 2 --vranks $v 2>&1 | grep us/iter | tail -1 >> $o; done
cat $o
