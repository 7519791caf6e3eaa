timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" > gpurun_out/exp.log; tail -2 gpurun_out/pytest_gpu.log >> gpurun_out/exp.log
for c in c5 c4; do timeout 600 python bench.py --config $c --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; done
