# trmm A/B 2: stripe kernel with 2 column boxes per consumer warp (KPP_TRMM_CW=2, the s = 256 default) vs
# 1 (KPP_TRMM_CW=1) vs the tile GEMM (c3 / c4 Phase 1), the
# factor tests, an ncu capture of the persistent kernel on c4, and a Phase-1 host/device profile of c4.
O=${O:-gpurun_out/r2t2}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "factor" > $O/pytest_factor.log 2>&1
echo "pytest rc=$?"; tail -2 $O/pytest_factor.log
for rep in 1 2; do
  for v in "1 2" "1 1" "0 2"; do  # (KPP_TRMM_TMA, KPP_TRMM_CW)
    set -- $v
    for c in c3 c4; do
      KPP_TRMM_TMA=$1 KPP_TRMM_CW=$2 timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-ttt --secondary '' \
        > $O/bench_${c}_t$1cw$2.json 2> $O/bench_${c}_t$1cw$2.err
      echo "$c trmm=$1 cw=$2 rc=$? $(python -c "import json,sys;d=json.load(open('$O/bench_${c}_t$1cw$2.json'));print(d['value'], d.get('phase1_ms_per_step'), d.get('phase2_ms_per_step'))" 2>&1)" | tee -a $O/ab.log
    done
  done
done
KPP_P1_PROFILE=1 timeout 600 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu --no-ttt --secondary '' > $O/p1prof_c4.json 2> $O/p1prof_c4.err; echo "p1prof rc=$?"
LC="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu --no-ttt --secondary ''"
timeout 600 bash -c "$LC" > $O/plain_c4b.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:trmm_tma -c 1 -f -o $O/trmm_c4 bash -c "$LC" > $O/ncu_trmm_c4.log 2>&1; echo "ncu trmm rc=$?"
