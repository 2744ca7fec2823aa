# bench line + ncu launch list of the same command + one full capture of the top SpMM kernel
set -x
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r01.log 2> gpurun_out/bench_r01.err; echo bench=$?
tail -1 gpurun_out/bench_r01.log | cut -c1-600
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_rows|k_spmm_heavy|k_gemm_tc|k_gram_tc|k_sketch_tc" -s 300 -c 6 \
    -o gpurun_out/prof_bench_r01 python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
