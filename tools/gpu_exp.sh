timeout 600 python -m pytest tests -m gpu -x -q -k "reassociated" > gpurun_out/pytest_re.log 2>&1; echo "pytest rc=$?" > gpurun_out/exp.log; tail -2 gpurun_out/pytest_re.log >> gpurun_out/exp.log
for i in 1 2; do timeout 300 python tools/prof_iter.py --config c5 --iters 1024 --reps 1 --reassoc 1; done >> gpurun_out/exp.log 2>&1
KPP_PHASE_PROFILE=1 timeout 300 python tools/prof_iter.py --config c5 --iters 512 --reps 1 --reassoc 1 >> gpurun_out/exp.log 2>&1
