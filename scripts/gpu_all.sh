bash scripts/gpu_check.sh
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench=$?
tail -1 gpurun_out/bench.log | cut -c1-1500
