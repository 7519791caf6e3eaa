# round 2, first check: GPU tests after the boundary changes, smoke, a c2 bench line, the c2 trace
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2/pytest_gpu_a.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2/pytest_gpu_a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke_a.log 2>&1; echo "smoke rc=$?"
KPP_TRACE=gpurun_out/r2/trace_c2.bin timeout 300 python tools/prof_iter.py --config c2 --iters 2048 --reps 1 > gpurun_out/r2/trace_c2.log 2>&1
python tools/trace_report.py gpurun_out/r2/trace_c2.bin >> gpurun_out/r2/trace_c2.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-ttt > gpurun_out/r2/bench_c2_a.json 2> gpurun_out/r2/bench_c2_a.err; echo "bench rc=$?"
