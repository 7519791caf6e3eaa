for c in c5 c4 c3 c2; do timeout 900 python bench.py --config $c --steps 1 --warmup 1 --no-cpu --ttt --ttt-cap 4000000 > gpurun_out/ttt_$c.json 2>gpurun_out/ttt_$c.err; done
K='regex:iterate|dgemm|chol|splitk|sched|fresh|gather|sumsq|add_diag|step_|lmax|refine|batch_move|cdpp_stream'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:iterate_kernel -c 1 -f -o gpurun_out/iter_c2 python tools/prof_iter.py --config c2 --iters 1024 --reps 1 > gpurun_out/ncu_iter_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cdpp_stream -c 1 -f -o gpurun_out/cs_c5 python tools/prof_iter.py --config c5 --iters 64 --reps 1 > gpurun_out/ncu_cs_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm2 -c 1 -f -o gpurun_out/dgemm2_c2 python tools/prof_iter.py --config c2 --iters 512 --reps 1 > gpurun_out/ncu_dgemm2_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:iterate_kernel -c 1 -f -o gpurun_out/iter_c4 python tools/prof_iter.py --config c4 --iters 32 --reps 1 > gpurun_out/ncu_iter_c4.log 2>&1
