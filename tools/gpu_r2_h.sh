mkdir -p gpurun_out/r2
timeout 60 ./tools/lat_skel > gpurun_out/r2/lat3.log 2>&1; grep -v "^hang" gpurun_out/r2/lat3.log | head -20
