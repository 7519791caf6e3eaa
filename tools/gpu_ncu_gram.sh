# Phase-1 Gram captures: full ncu capture of the first TMA-ring Gram launch of a c2 and a c4 bench step
# (each after the same command ran plain), and the c4 launch list.  O=outdir bash tools/gpu_ncu_gram.sh
O=${O:-gpurun_out/r2g2}; mkdir -p $O
L2="python bench.py --steps 1 --warmup 0 --no-cpu --no-ttt --secondary ''"
L4="python bench.py --config c4 --steps 1 --warmup 0 --no-cpu --no-ttt --secondary ''"
timeout 600 bash -c "$L2" > $O/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_tma -s 0 -c 1 -f -o $O/gram_c2 bash -c "$L2" > $O/ncu2.log 2>&1; echo "c2 rc=$?"
timeout 600 bash -c "$L4" > $O/plain4.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_tma -s 2 -c 1 -f -o $O/gram_c4 bash -c "$L4" > $O/ncu4.log 2>&1; echo "c4 rc=$?"
[ -n "$LIST4" ] && { timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_c4.csv bash -c "$L4" > $O/ncu4l.log 2>&1; echo "c4 list rc=$?"; }
true
