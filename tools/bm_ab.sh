mkdir -p gpurun_out/bm
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or factor or gemm or lsqr" > gpurun_out/bm/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/bm/pytest.log
for c in c2 c3 c4; do for bm in 64 128; do
KPP_GEMM_BM=$bm timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-ttt > gpurun_out/bm/$c.$bm.json 2>gpurun_out/bm/$c.$bm.err; echo "$c $bm rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bm/$c.$bm.json').read().strip().splitlines()[-1]);print('$c',$bm,d['value'],d.get('phase1_ms_per_step'),d.get('phase1_fp64'))"
done; done
