timeout 900 python -m pytest tests -m gpu -x -q -k "factor or twin or adaptive or max_block or c1" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" > gpurun_out/exp.log; tail -2 gpurun_out/pytest_gpu.log >> gpurun_out/exp.log
for c in c2 c3 c4; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu --no-ttt > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; done
for c in c2 c4; do KPP_NO_SYRK=1 timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu --no-ttt > gpurun_out/bench_${c}_nosyrk.json 2>/dev/null; done
