# CD++ streaming kernel A/B: one call site of the stream loop for streaming and chain warps (libkpp.so)
# vs two inlined copies (libkpp_head.so, built from the previous commit after the edit, so build.py
# keeps it), interleaved; phase profiles; then the CD++ tests on the new library.
O=${O:-gpurun_out/r2ic}
mkdir -p $O
H=$PWD/paper_2501_11673_b200/libkpp_head.so
: > $O/ab.log
for rep in 1 2 3; do
  echo "c5 head $(KPP_LIB=$H timeout 300 python tools/prof_iter.py --config c5 --iters 512 --reps 2 2>&1 | grep us/iter | tail -1)" >> $O/ab.log
  echo "c5 new  $(timeout 300 python tools/prof_iter.py --config c5 --iters 512 --reps 2 2>&1 | grep us/iter | tail -1)" >> $O/ab.log
done
for v in head new; do
  lib=""; [ $v = head ] && lib=$H
  echo "== $v" >> $O/phase.log
  KPP_LIB=$lib KPP_PHASE_PROFILE=1 timeout 300 python tools/prof_iter.py --config c5 --iters 512 --reps 1 >> $O/phase.log 2>&1
  KPP_LIB=$lib timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-ttt --secondary '' > $O/bench_c5_$v.json 2>$O/bench_c5_$v.err
  echo "bench c5 $v $(python -c "import json;d=json.load(open('$O/bench_c5_$v.json'));print(d['value'], d['phase1_ms_per_step'], d['phase2_ms_per_step'], d['roofline']['frac'])")" >> $O/ab.log
done
cat $O/ab.log; grep "phase cycles" $O/phase.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -k "cdpp or c5" > $O/pytest_cdpp.log 2>&1
echo "pytest rc=$?"; tail -2 $O/pytest_cdpp.log
