# usage: bash scripts/gpu_check.sh [pytest -k expr]
K=${1:-}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "$K" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
else
  timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
fi
tail -3 gpurun_out/smoke.log
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -25
