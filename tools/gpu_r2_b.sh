# round 2: emulated-rank exchange tests, window closed forms, the new bench line (cpu protocol, c5/c4 blocks)
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "emulated or closed_form or fused_exchange" > gpurun_out/r2/pytest_vr.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2/pytest_vr.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/r2/bench_c2_b.json 2> gpurun_out/r2/bench_c2_b.err; echo "bench rc=$?"; tail -3 gpurun_out/r2/bench_c2_b.err
