mkdir -p gpurun_out/r2
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cdpp_stream or dist_path or emulated or reassociated or fused_exchange" > gpurun_out/r2/pytest_cs.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2/pytest_cs.log
o=gpurun_out/r2/cs_timing.log; : > $o
for v in 1 2 4 8; do echo "c5 cdpp_stream vranks=$v" >> $o; timeout 600 python tools/prof_iter.py --config c5 --iters 512 --reps 2 --vranks $v 2>&1 | grep us/iter | tail -1 >> $o; done
cat $o
