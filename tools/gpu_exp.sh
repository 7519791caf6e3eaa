FMA_AS_ONE=1 timeout 1200 python tools/table2_check.py 0,1,2,3,4 > gpurun_out/table2_fma1.log 2>&1; echo "rc=$?" >> gpurun_out/table2_fma1.log
