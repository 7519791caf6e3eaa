# Phase-1 Q1 = X1^T A_S A/B: the TMA-ring stripe kernel (trmm_tma.cu) against the tile GEMM
# (KPP_TRMM_TMA=0), Phase-1 ms per bench step on c3 / c4, after the factor parity tests; then an ncu
# capture of the stripe kernel on c4.  O=outdir bash tools/gpu_trmm_ab.sh
O=${O:-gpurun_out/r2t}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "factor" > $O/pytest_factor.log 2>&1
echo "pytest rc=$?"; tail -2 $O/pytest_factor.log
for rep in 1 2; do
  for v in 1 0; do
    for c in c3 c4; do
      KPP_TRMM_TMA=$v timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-ttt --secondary '' \
        > $O/bench_${c}_trmm$v.json 2> $O/bench_${c}_trmm$v.err
      echo "$c trmm=$v rc=$? $(python -c "import json,sys;d=json.load(open('$O/bench_${c}_trmm$v.json'));print(d['value'], d.get('phase1_ms_per_step'), d.get('phase2_ms_per_step'))" 2>&1)" | tee -a $O/ab.log
    done
  done
done
LC="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-ttt --secondary ''"
timeout 600 bash -c "$LC" > $O/plain_c4.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv bash -c "$LC" > $O/ncu_launch_c4.log 2>&1; echo "launch list c4 rc=$?"
timeout 600 bash -c "$LC" > $O/plain_c4b.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:trmm_tma -c 1 -f -o $O/trmm_c4 bash -c "$LC" > $O/ncu_trmm_c4.log 2>&1; echo "ncu trmm rc=$?"
