for o in 1 0 1 0; do
  NETMFP_GEMM_TRI_ORDER=$o timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ab_$o.log 2>&1
  python -c "
import json,sys
d=json.loads(open('gpurun_out/ab_$o.log').read().strip().splitlines()[-1])
print('order $o', round(d['ms_per_step'],3), 'gemm', round(d['kernel_ms_per_step']['tc_gemm_tall'],3), d['step_ms'])
"
done
