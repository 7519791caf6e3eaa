for y in 0 4; do timeout 120 python tools/prof_iter.py --config c3 --iters 4096 --reps 2 --ygl $y; echo "rc=$?"; done > gpurun_out/exp.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/exp.log; tail -3 gpurun_out/pytest_gpu.log >> gpurun_out/exp.log
for c in c2 c3; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; done
