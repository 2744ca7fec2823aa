# Round-2 evidence (configs[2]): bench line, ncu launch list of the same
# command, full captures of the top kernels, gather benchmarks.  Run under gpurun.
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02.log 2> gpurun_out/bench_r02.err; echo bench=$?
tail -1 gpurun_out/bench_r02.log | cut -c1-300
B="python bench.py --steps 1 --warmup 3 --no-cpu"
timeout 900 $B > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file gpurun_out/launches_r02.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
# SpMM: one 286-column application (2 launches) of the 4th step, then one middle Chebyshev (Clenshaw) step
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_spmm_fused -s 114 -c 2 \
    -o gpurun_out/prof_spmm286_r02 $B > gpurun_out/ncu_full1.log 2>&1; echo ncufull1=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_spmm_fused -s 145 -c 1 \
    -o gpurun_out/prof_spmm128_r02 $B > gpurun_out/ncu_full2.log 2>&1; echo ncufull2=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_gram_tc|k_sketch_tc|k_chol_df|k_tridiag" -s 60 -c 14 \
    -o gpurun_out/prof_tc_r02 $B > gpurun_out/ncu_full3.log 2>&1; echo ncufull3=$?
./scripts/dbg/gather_bench > gpurun_out/gather_r02.txt 2>&1; echo gather=$?
python scripts/dbg/dump_csr.py 2 /tmp/csr2.bin > /dev/null && ./scripts/dbg/spmm_lab /tmp/csr2.bin > gpurun_out/spmm_lab_r02.txt 2>&1; echo lab=$?
