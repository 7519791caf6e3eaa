timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" > gpurun_out/exp.log; tail -2 gpurun_out/pytest_gpu.log >> gpurun_out/exp.log
timeout 900 python tools/check_gram_route.py c1,c2,c3,c4 200 >> gpurun_out/exp.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2>gpurun_out/bench_c2.err
for c in c3 c4 c5; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; done
