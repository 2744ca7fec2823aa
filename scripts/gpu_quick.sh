# smoke + full gpu tests + bench (stage profile)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo gpu=$?
grep -E "passed|failed|Error|assert" gpurun_out/pytest_gpu.log | tail -8
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_stage.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_stage.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['value'], d['step_ms']); print(d['kernel_ms_per_step']); print(d['stage_ms_per_step'])"
