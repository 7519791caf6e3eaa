# Profiling pass (run under gpurun): fp64 DGEMM peak, launch list of the c2 bench, full captures.
set -x
mkdir -p gpurun_out
python - <<'PY' > gpurun_out/fp64_peak.txt 2>&1
import torch, time
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
for _ in range(3): a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
print({"fp64_dgemm_tflops": 2 * 8192**3 / best / 1e9, "ms": best, "how": "torch.matmul fp64 8192^3 best of 10"})
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:iterate_kernel -c 1 -f -o gpurun_out/iter_c2 python tools/prof_iter.py --config c2 --iters 1024 --reps 1 > gpurun_out/ncu_iter_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm -s 2 -c 2 -f -o gpurun_out/dgemm_c2 python tools/prof_iter.py --config c2 --iters 256 --reps 1 > gpurun_out/ncu_dgemm_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chol -c 1 -f -o gpurun_out/chol_c5 python tools/prof_iter.py --config c5 --iters 64 --reps 1 > gpurun_out/ncu_chol_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:iterate_kernel -c 1 -f -o gpurun_out/iter_c5 python tools/prof_iter.py --config c5 --iters 64 --reps 1 > gpurun_out/ncu_iter_c5.log 2>&1
