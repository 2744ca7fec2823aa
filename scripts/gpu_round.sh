# smoke + gpu tests + bench + launch list of the same bench command
bash scripts/gpu_check.sh
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench=$?
tail -1 gpurun_out/bench.log | cut -c1-3000
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu.log 2>&1; echo ncu=$?
