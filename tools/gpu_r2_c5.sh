mkdir -p gpurun_out/r2
export KPP_NO_COOP=1
L="python bench.py --config c5 --steps 1 --warmup 2 --no-cpu --no-ttt --secondary ''"
timeout 600 bash -c "$L" > gpurun_out/r2/plain_c5.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2/launches_c5.csv bash -c "$L" > gpurun_out/r2/ncu_launch_c5.log 2>&1; echo "launch list c5 rc=$?"
