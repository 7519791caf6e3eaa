# c2 Phase-2 latency knobs: pollers per row, poll back-off, cluster size
mkdir -p gpurun_out/r2
o=gpurun_out/r2/c2_knobs.log; : > $o
for g in 16 8 4 2 1; do echo "G2MAX=$g" >> $o; KPP_G2MAX=$g timeout 300 python tools/prof_iter.py --config c2 --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1 >> $o; done
for ns in 20 50 100 200; do echo "POLL_NS=$ns" >> $o; KPP_POLL_NS=$ns timeout 300 python tools/prof_iter.py --config c2 --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1 >> $o; done
for g in 4 2; do for ns in 50 100; do echo "G2MAX=$g POLL_NS=$ns" >> $o; KPP_G2MAX=$g KPP_POLL_NS=$ns timeout 300 python tools/prof_iter.py --config c2 --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1 >> $o; done; done
for C in 2 8 16; do echo "C=$C" >> $o; timeout 300 python tools/prof_iter.py --config c2 --iters 4096 --reps 2 --cluster $C 2>&1 | grep us/iter | tail -1 >> $o; done
for C in 8 16; do echo "C=$C G2MAX=4" >> $o; KPP_G2MAX=4 timeout 300 python tools/prof_iter.py --config c2 --iters 4096 --reps 2 --cluster $C 2>&1 | grep us/iter | tail -1 >> $o; done
echo "c3 default" >> $o; timeout 300 python tools/prof_iter.py --config c3 --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1 >> $o
for g in 8 4 2; do echo "c3 G2MAX=$g" >> $o; KPP_G2MAX=$g timeout 300 python tools/prof_iter.py --config c3 --iters 4096 --reps 2 2>&1 | grep us/iter | tail -1 >> $o; done
cat $o
timeout 600 python tools/c1_noise_floor.py 200 > gpurun_out/r2/c1_noise_floor.log 2>&1; cat gpurun_out/r2/c1_noise_floor.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -x -q -k "bell or fullsize_parity or stop_to_tol" > gpurun_out/r2/pytest_full.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2/pytest_full.log
