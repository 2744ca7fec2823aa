# Round-2 (session 2) evidence on the final build: bench line, ncu launch list of
# the same command, full captures of the new sketch kernels.  Run under gpurun.
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02b.log 2> gpurun_out/bench_r02b.err; echo bench=$?
tail -1 gpurun_out/bench_r02b.log | cut -c1-300
B="python bench.py --steps 1 --warmup 3 --no-cpu"
timeout 900 $B > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file gpurun_out/launches_r02b.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_sketch_h|k_split_f16|k_sketch_tc" -s 4 -c 4 \
    -o gpurun_out/prof_sketch_r02b $B > gpurun_out/ncu_full_sk.log 2>&1; echo ncufull=$?
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_r02b.log 2>&1; echo ref=$?
tail -1 gpurun_out/bench_ref_r02b.log | cut -c1-300
