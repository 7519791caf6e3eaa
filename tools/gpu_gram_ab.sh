# Phase-1 Gram A/B: the TMA-ring Gram against the previous kernels (KPP_GRAM_TMA=0), Phase-1 ms per
# bench step on c2 / c3 / c4, after the factor parity tests.  O=outdir bash tools/gpu_gram_ab.sh
O=${O:-gpurun_out/r2g}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "factor_operator" > $O/pytest_factor.log 2>&1
echo "pytest rc=$?"; tail -2 $O/pytest_factor.log
for rep in 1 2; do
  for v in 1 0; do
    for c in c2 c3 c4; do
      KPP_GRAM_TMA=$v timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-ttt --secondary '' \
        > $O/bench_${c}_tma$v.json 2> $O/bench_${c}_tma$v.err
      echo "$c tma=$v rc=$? $(python -c "import json,sys;d=json.load(open('$O/bench_${c}_tma$v.json'));print(d['value'], d.get('phase1_ms_per_step'), d.get('phase2_ms_per_step'))" 2>&1)" | tee -a $O/ab.log
    done
  done
done
