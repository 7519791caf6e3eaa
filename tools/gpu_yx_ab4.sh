# c5 bench A/B, alternating: HEAD library (libkpp_head.so) / yx / yx with KPP_CS_M=1, twice.
O=${O:-gpurun_out/r2yx4}
mkdir -p $O
H=$PWD/paper_2501_11673_b200/libkpp_head.so
: > $O/ab.log
for rep in 1 2; do
  for v in head yx m; do
    lib=""; env=""; [ $v = head ] && lib=$H; [ $v = m ] && env="KPP_CS_M=1"
    env $env KPP_LIB=$lib timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-ttt --secondary '' > $O/bench_c5_${v}_$rep.json 2>$O/bench_c5_${v}_$rep.err
    echo "bench c5 $v $(python -c "import json;d=json.load(open('$O/bench_c5_${v}_$rep.json'));print(d['value'], d['phase1_ms_per_step'], d['phase2_ms_per_step'], d['roofline']['frac'])")" >> $O/ab.log
  done
done
cat $O/ab.log
