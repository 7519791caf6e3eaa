timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" > gpurun_out/exp.log; tail -2 gpurun_out/pytest_gpu.log >> gpurun_out/exp.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/exp.log 2>&1; echo "smoke rc=$?" >> gpurun_out/exp.log
timeout 900 python bench.py > gpurun_out/bench_c2.json 2>gpurun_out/bench_c2.err; echo "bench rc=$?" >> gpurun_out/exp.log
for c in c3 c4 c5; do timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; done
