mkdir -p gpurun_out/r2
o=gpurun_out/r2/lean3.log; : > $o
for c in c2 c1; do echo "$c lean" >> $o; timeout 300 python tools/prof_iter.py --config $c --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1 >> $o; done
KPP_TRACE=gpurun_out/r2/trace_lean3_c2.bin timeout 300 python tools/prof_iter.py --config c2 --iters 2048 --reps 1 > /dev/null 2>&1
python tools/trace_report.py gpurun_out/r2/trace_lean3_c2.bin 2>&1 | tail -10 >> $o
cat $o
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1 or twin_parity or closed_form" > gpurun_out/r2/pytest_lean3.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2/pytest_lean3.log
