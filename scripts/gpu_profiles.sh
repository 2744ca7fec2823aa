# bench line + ncu launch list of the same command + full captures of the top kernels (configs[2])
set -x
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r01.log 2> gpurun_out/bench_r01.err; echo bench=$?
tail -1 gpurun_out/bench_r01.log | cut -c1-400
B="python bench.py --steps 1 --warmup 3 --no-cpu"
timeout 900 $B > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file gpurun_out/launches_r01.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
# SpMM: one 286-column application (2 launches) of the 4th step, then one middle Chebyshev (Clenshaw) step
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_spmm_fused -s 114 -c 2 \
    -o gpurun_out/prof_spmm286_r01 $B > gpurun_out/ncu_full1.log 2>&1; echo ncufull1=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_spmm_fused -s 145 -c 1 \
    -o gpurun_out/prof_spmm128_r01 $B > gpurun_out/ncu_full2.log 2>&1; echo ncufull2=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_gram_tc|k_sketch_tc|k_chol_df" -s 60 -c 12 \
    -o gpurun_out/prof_tc_r01 $B > gpurun_out/ncu_full3.log 2>&1; echo ncufull3=$?
