timeout 300 python scripts/tc_one.py > gpurun_out/tc_one.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram_tc|k_gemm_tc" -s 4 -c 2 \
   -o gpurun_out/prof_tc python scripts/tc_one.py > gpurun_out/ncu_tc.log 2>&1; echo ncu=$?
cat gpurun_out/tc_one.log | head -3
