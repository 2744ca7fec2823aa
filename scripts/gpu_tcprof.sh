timeout 300 python scripts/tc_one.py > gpurun_out/tc_one.log 2>&1; echo tc_one=$?
cat gpurun_out/tc_one.log | tail -5
timeout 900 python -m pytest tests/test_gpu_dense.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_dense.log 2>&1; echo dense=$?
tail -3 gpurun_out/pytest_dense.log
timeout 300 python scripts/tc_one.py > gpurun_out/tc_one2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram_tc|k_gemm_tc|k_chol_inv" -s 6 -c 3 \
   -o gpurun_out/prof_tc python scripts/tc_one.py > gpurun_out/ncu_tc.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_tc.log
