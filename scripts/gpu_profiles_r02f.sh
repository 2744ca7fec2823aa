# Round-2 (session 2) final-build evidence: bench line, launch list of the same
# command, full ncu captures of the SpMM (merged-tail launch, one 286-column
# application and one Clenshaw step) and of the tensor-core kernels.  Run under gpurun.
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02f.log 2> gpurun_out/bench_r02f.err; echo bench=$?
tail -1 gpurun_out/bench_r02f.log | cut -c1-300
B="python bench.py --steps 1 --warmup 3 --no-cpu"
timeout 900 $B > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file gpurun_out/launches_r02f.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
# SpMM: 4th step's first 286-column application (k_spmm_fused_tail) and a middle Clenshaw step (k_spmm_fused)
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_spmm_fused_tail -s 42 -c 1 \
    -o gpurun_out/prof_spmm286_r02f $B > gpurun_out/ncu_full1.log 2>&1; echo ncufull1=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_fused<" -s 34 -c 1 \
    -o gpurun_out/prof_spmm128_r02f $B > gpurun_out/ncu_full2.log 2>&1; echo ncufull2=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_gram_tc|k_sketch_h|k_chol_df|k_tridiag" -s 50 -c 16 \
    -o gpurun_out/prof_tc_r02f $B > gpurun_out/ncu_full3.log 2>&1; echo ncufull3=$?
python scripts/ncu_summary.py gpurun_out/prof_tc_r02f.ncu-rep > gpurun_out/ncu_tc_r02f.txt 2>&1; python scripts/ncu_summary.py gpurun_out/prof_spmm286_r02f.ncu-rep > gpurun_out/ncu_spmm_r02f.txt 2>&1; python scripts/ncu_summary.py gpurun_out/prof_spmm128_r02f.ncu-rep >> gpurun_out/ncu_spmm_r02f.txt 2>&1; echo summ=$?
