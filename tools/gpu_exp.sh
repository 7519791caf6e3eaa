timeout 300 python tools/dbg_s1024.py > gpurun_out/exp.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "max_block" > gpurun_out/pytest_max.log 2>&1; echo "pytest rc=$?" >> gpurun_out/exp.log; tail -3 gpurun_out/pytest_max.log >> gpurun_out/exp.log
