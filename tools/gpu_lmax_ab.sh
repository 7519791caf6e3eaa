# Power-iteration A/B (adaptive CholeskyQR2 estimate, s <= 128): register-tile kernel (product) vs the
# matrix-from-L2 kernel (KPP_LMAX_REG=0): factor / adaptive / c1-c2 parity tests, then c2 / c1 bench lines.
O=${O:-gpurun_out/r2m}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "factor or adaptive or c1_ or twin_parity or stop or i8" > $O/pytest_lmax.log 2>&1
echo "pytest rc=$?"; tail -2 $O/pytest_lmax.log
: > $O/ab.log
for rep in 1 2; do
  for v in 1 0; do
    for c in c2 c1; do
      KPP_LMAX_REG=$v timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu --no-ttt --secondary '' > $O/bench_${c}_r$v.json 2> $O/bench_${c}_r$v.err
      echo "$c reg=$v $(python -c "import json;d=json.load(open('$O/bench_${c}_r$v.json'));print(d['value'], d['phase1_ms_per_step'], d['phase2_ms_per_step'], d.get('n_refined_per_step'))")" >> $O/ab.log
    done
  done
done
cat $O/ab.log
