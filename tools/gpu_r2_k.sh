mkdir -p gpurun_out/r2
export KPP_NO_COOP=1
timeout 300 python tools/prof_iter.py --config c2 --iters 2048 --reps 1 > gpurun_out/r2/plain_lean.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:iterate_lean -c 1 -o gpurun_out/r2/lean_c2 python tools/prof_iter.py --config c2 --iters 2048 --reps 1 > gpurun_out/r2/ncu_lean.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/r2/ncu_lean.log
