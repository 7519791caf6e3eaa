# CD++ streaming kernel A/B: stash columns loaded by their lanes beside the stream (product) vs the
# per-element column map (libkpp_old.so: the library built from commit 63025a8~2, i.e. before the change),
# after the CD++ parity tests.
O=${O:-gpurun_out/r2c}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -k "cdpp or c5 or bell_psd" > $O/pytest_cdpp.log 2>&1
echo "pytest rc=$?"; tail -2 $O/pytest_cdpp.log
: > $O/ab.log
for rep in 1 2 3; do
  for v in base old; do
    lib=""; [ "$v" != base ] && lib="$PWD/paper_2501_11673_b200/libkpp_$v.so"
    echo "c5 $v $(KPP_LIB=$lib timeout 300 python tools/prof_iter.py --config c5 --iters 512 --reps 2 2>&1 | grep us/iter | tail -1)" >> $O/ab.log
  done
done
for v in 1 0; do
  KPP_LIB=$([ $v = 0 ] && echo $PWD/paper_2501_11673_b200/libkpp_old.so) timeout 600 python bench.py --config c5 --steps 3 --warmup 2 --no-cpu --no-ttt --secondary '' > $O/bench_c5_$v.json 2>$O/bench_c5_$v.err
  echo "bench c5 new=$v $(python -c "import json;d=json.load(open('$O/bench_c5_$v.json'));print(d['value'], d['phase1_ms_per_step'], d['phase2_ms_per_step'], d['roofline']['frac'])")" >> $O/ab.log
done
cat $O/ab.log
