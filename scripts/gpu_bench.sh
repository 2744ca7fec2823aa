# bench + ncu launch list (same command), then optional full capture of a kernel regex
KREGEX=${1:-}
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench=$?
tail -1 gpurun_out/bench.log
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu.log 2>&1; echo ncu=$?
if [ -n "$KREGEX" ]; then
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 40 -c 2 \
    -o gpurun_out/prof python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
fi
