# Round-end refresh under gpurun: tests, smoke, bench lines of every config, ncu launch list of the
# c2 bench and full captures of the Phase-2 kernels (outputs in gpurun_out/, copied to profiles/).
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --proj 1 --steps 3 --warmup 3 --no-ttt > gpurun_out/bench_lsqr_c2.json 2> gpurun_out/bench_lsqr_c2.err
timeout 900 python bench.py --proj 1 --config c3 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_lsqr_c3.json 2> gpurun_out/bench_lsqr_c3.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-ttt > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:iterate_kernel -c 1 -f -o gpurun_out/iter_c2 python tools/prof_iter.py --config c2 --iters 1024 --reps 1 > gpurun_out/ncu_iter_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:iterate_kernel -c 1 -f -o gpurun_out/iter_c4 python tools/prof_iter.py --config c4 --iters 32 --reps 1 > gpurun_out/ncu_iter_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cdpp_stream -c 1 -f -o gpurun_out/cs_c5 python tools/prof_iter.py --config c5 --iters 64 --reps 1 > gpurun_out/ncu_cs_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm2 -c 1 -f -o gpurun_out/dgemm2_c2 python tools/prof_iter.py --config c2 --iters 8192 --reps 1 > gpurun_out/ncu_dgemm_c2.log 2>&1
echo done
