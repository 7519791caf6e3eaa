KPP_P1_PROFILE=1 timeout 300 python tools/prof_iter.py --config c5 --iters 256 --reps 1 > gpurun_out/exp.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "factor or twin or cdpp or dist or adaptive" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/exp.log; tail -2 gpurun_out/pytest_gpu.log >> gpurun_out/exp.log
for c in c5 c2; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu --no-ttt > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; done
