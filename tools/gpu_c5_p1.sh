# c5 (CD++) Phase-1 anatomy: launch list of one cold step and the Phase-1 event profile.
O=${O:-gpurun_out/r2c5}
mkdir -p $O
LC="python bench.py --config c5 --steps 1 --warmup 2 --no-cpu --no-ttt --secondary ''"
KPP_P1_PROFILE=1 timeout 600 bash -c "$LC" > $O/p1prof_c5.json 2> $O/p1prof_c5.err; echo "p1prof rc=$?"
timeout 600 bash -c "$LC" > $O/plain_c5.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_c5.csv bash -c "$LC" > $O/ncu_launch_c5.log 2>&1; echo "launch list c5 rc=$?"
