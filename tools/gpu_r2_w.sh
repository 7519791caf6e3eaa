mkdir -p gpurun_out/r2
export KPP_NO_COOP=1
P="python tools/prof_iter.py --config c2 --iters 8192 --reps 1"
timeout 300 $P > gpurun_out/r2/plain_gram.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_syrk -c 1 -f -o gpurun_out/r2/gram_syrk_c2 $P > gpurun_out/r2/ncu_gram.log 2>&1; echo "ncu rc=$?"
