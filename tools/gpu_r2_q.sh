mkdir -p gpurun_out/r2
o=gpurun_out/r2/lean_c8.log; : > $o
for C in 8 4; do echo "c2 C=$C" >> $o; timeout 300 python tools/prof_iter.py --config c2 --iters 4096 --reps 2 --cluster $C 2>&1 | grep us/iter | tail -1 >> $o; done
cat $o
export KPP_NO_COOP=1
for c in c4 c3; do
L="python bench.py --config $c --steps 1 --warmup 2 --no-cpu --no-ttt --secondary ''"
timeout 600 bash -c "$L" > gpurun_out/r2/plain_$c.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2/launches_$c.csv bash -c "$L" > gpurun_out/r2/ncu_launch_$c.log 2>&1; echo "launch list $c rc=$?"
done
