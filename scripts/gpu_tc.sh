timeout 300 python scripts/tc_one.py > gpurun_out/tc_one.log 2>&1; echo tc_one=$?
cat gpurun_out/tc_one.log | tail -20
timeout 900 python -m pytest tests/test_gpu_dense.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_dense.log 2>&1; echo dense=$?
tail -15 gpurun_out/pytest_dense.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo gpu=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_stage.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_stage.log | cut -c1-3000
