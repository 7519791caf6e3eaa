timeout 600 python -m pytest tests -m gpu -x -q -k "dist_path" > gpurun_out/pytest_dist.log 2>&1; echo "pytest rc=$?" > gpurun_out/exp.log; tail -25 gpurun_out/pytest_dist.log >> gpurun_out/exp.log
