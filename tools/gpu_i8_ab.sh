# int8 (Ozaki) Gram A/B: factor parity tests, the c2-twin parity tests, then bench c2 Phase 1 with
# the int8 Gram (producer variants KPP_GRAM_I8_PROD=2 cp.async, 1 TMA multicast) against the fp64
# DMMA TMA-ring Gram (KPP_GRAM_I8=0).  O=outdir bash tools/gpu_i8_ab.sh
O=${O:-gpurun_out/r2i}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "factor_operator or c2 or smoke" > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest.log
for rep in 1 2; do for v in "1 2" "1 1" "0 2"; do
  set -- $v
  KPP_GRAM_I8=$1 KPP_GRAM_I8_PROD=$2 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-ttt --secondary '' > $O/bench_c2_i8$1_p$2.json 2> $O/bench_c2_i8$1_p$2.err
  echo "c2 i8=$1 prod=$2 rc=$? $(python -c "import json;d=json.load(open('$O/bench_c2_i8$1_p$2.json'));print(d['value'], d.get('phase1_ms_per_step'), d.get('phase2_ms_per_step'))" 2>&1)" | tee -a $O/ab.log
done; done
