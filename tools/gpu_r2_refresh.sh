# Round-2 refresh under gpurun: every GPU test, smoke, bench lines, the c2 launch list and full captures of
# the Phase-2 kernels (each ncu command preceded by the same command run plain, with &&).
mkdir -p gpurun_out/r2f
O=${O:-gpurun_out/r2f}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py --steps 5 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu --secondary '' > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench c3 rc=$?"
timeout 900 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu --secondary '' > $O/bench_c1.json 2> $O/bench_c1.err; echo "bench c1 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_c2.json 2> $O/bench_ref_c2.err; echo "ref rc=$?"
export KPP_NO_COOP=1
L="python bench.py --steps 1 --warmup 3 --no-cpu --no-ttt --secondary ''"
timeout 600 bash -c "$L" > $O/plain_launch.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv bash -c "$L" > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
P2="python tools/prof_iter.py --config c2 --iters 1024 --reps 1"
timeout 300 $P2 > $O/plain_p2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:iterate_lean -c 1 -f -o $O/lean_c2 $P2 > $O/ncu_lean_c2.log 2>&1; echo "ncu c2 rc=$?"
P4="python tools/prof_iter.py --config c4 --iters 32 --reps 1"
timeout 300 $P4 > $O/plain_p4.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:iterate_kernel -c 1 -f -o $O/iter_c4 $P4 > $O/ncu_iter_c4.log 2>&1; echo "ncu c4 rc=$?"
P5="python tools/prof_iter.py --config c5 --iters 64 --reps 1"
timeout 300 $P5 > $O/plain_p5.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:cdpp_stream -c 1 -f -o $O/cs_c5 $P5 > $O/ncu_cs_c5.log 2>&1; echo "ncu c5 rc=$?"
LC4="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-ttt --secondary ''"
timeout 600 bash -c "$LC4" > $O/plain_trmm.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:trmm_tma -c 1 -f -o $O/trmm_c4 bash -c "$LC4" > $O/ncu_trmm_c4.log 2>&1; echo "ncu trmm rc=$?"
for C in c3 c4; do
  LC="python bench.py --config $C --steps 1 --warmup 3 --no-cpu --no-ttt --secondary ''"
  timeout 600 bash -c "$LC" > $O/plain_launch_$C.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_$C.csv bash -c "$LC" > $O/ncu_launch_$C.log 2>&1; echo "launch list $C rc=$?"
done
echo done
