# int8 Gram captures: full ncu capture of the first gram_i8 launch of a c2 bench step and the c2 launch
# list (each after the same command ran plain).  O=outdir bash tools/gpu_ncu_i8.sh
O=${O:-gpurun_out/r2i2}; mkdir -p $O
L2="python bench.py --steps 1 --warmup 0 --no-cpu --no-ttt --secondary ''"
timeout 600 bash -c "$L2" > $O/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_i8 -s 0 -c 1 -f -o $O/i8_c2 bash -c "$L2" > $O/ncu2.log 2>&1; echo "c2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c2.csv bash -c "$L2" > $O/ncu2l.log 2>&1; echo "list rc=$?"
