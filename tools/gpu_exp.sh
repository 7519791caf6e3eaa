timeout 900 python -m pytest tests -m gpu -x -q -k "launch_plans" > gpurun_out/pytest_plans.log 2>&1; echo "pytest rc=$?" > gpurun_out/exp.log; tail -3 gpurun_out/pytest_plans.log >> gpurun_out/exp.log
for y in 0 5; do for C in 2 4 8; do timeout 120 python tools/prof_iter.py --config c2 --iters 4096 --reps 1 --ygl $y --cluster $C; done; done >> gpurun_out/exp.log 2>&1
for y in 0 5; do timeout 120 python tools/prof_iter.py --config c1 --iters 4096 --reps 1 --ygl $y; done >> gpurun_out/exp.log 2>&1
