timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c5.csv python tools/prof_iter.py --config c5 --iters 1024 --reps 1 > gpurun_out/ncu_launch5.log 2>&1
KPP_PHASE_PROFILE=1 timeout 300 python tools/prof_iter.py --config c5 --iters 512 --reps 2 > gpurun_out/exp.log 2>&1
KPP_DBG_SKIP=1 timeout 300 python tools/prof_iter.py --config c5 --iters 512 --reps 2 >> gpurun_out/exp.log 2>&1
for C in 1 4 8; do timeout 300 python tools/prof_iter.py --config c5 --iters 512 --reps 1 --cluster $C >> gpurun_out/exp.log 2>&1; done
KPP_PHASE_PROFILE=1 timeout 300 python tools/prof_iter.py --config c4 --iters 256 --reps 2 >> gpurun_out/exp.log 2>&1
