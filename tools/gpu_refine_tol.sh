# c4 headroom of a sharper CholeskyQR2 refinement criterion (DESIGN 13 item 2): the bench step and the parity
# against the oracle with the product threshold (4 u kappa^2 > 3e-11) and with refinement off (KPP_REFINE_TOL=1:
# Gram + Cholesky only), at 200 iterations and at c4's stopping iteration (768).
O=${O:-gpurun_out/rtol}
mkdir -p $O
for R in 3e-11 1; do
  KPP_REFINE_TOL=$R timeout 600 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-ttt --secondary '' > $O/bench_c4_$R.json 2> $O/bench_c4_$R.err; echo "bench c4 rtol=$R rc=$?"
  python -c "import json;d=json.loads(open('$O/bench_c4_$R.json').read().strip().splitlines()[-1]);print('c4 rtol=$R', d['value'], d['ms_per_step'], d['phase1_ms_per_step'], d['n_refined_per_step'], d['n_blocks_per_step'])"
done
timeout 900 python tools/check_gram_route.py c4 200 > $O/parity_c4_200.log 2>&1; tail -1 $O/parity_c4_200.log
timeout 1500 python tools/check_gram_route.py c4 768 > $O/parity_c4_768.log 2>&1; tail -1 $O/parity_c4_768.log
