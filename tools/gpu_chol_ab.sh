# Blocked Cholesky A/B: 128-wide super-steps for the trailing update (product) vs every 64-wide step
# updating the whole trailing matrix (KPP_CHOL_SUPER=0): factor tests, then Phase 1 ms per step on c5 / c3 / c4.
O=${O:-gpurun_out/r2k}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "factor or cdpp" > $O/pytest_factor.log 2>&1
echo "pytest rc=$?"; tail -2 $O/pytest_factor.log
: > $O/ab.log
for rep in 1 2; do
  for v in 1 0; do
    for c in c5 c3 c4; do
      KPP_CHOL_SUPER=$v timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu --no-ttt --secondary '' \
        > $O/bench_${c}_s$v.json 2> $O/bench_${c}_s$v.err
      echo "$c super=$v rc=$? $(python -c "import json;d=json.load(open('$O/bench_${c}_s$v.json'));print(d['value'], d.get('phase1_ms_per_step'), d.get('phase2_ms_per_step'))" 2>&1)" | tee -a $O/ab.log
    done
  done
done
