# SpMM pass width / merged tail sweep on the final kernel (SpMM family ms per embedding)
for cfg in "128 1" "64 1" "128 0" "128 1" "64 1"; do
  set -- $cfg
  NETMFP_SPMM_W=$1 NETMFP_SPMM_MERGE_TAIL=$2 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ab_w.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/ab_w.log').read().strip().splitlines()[-1])
print('W $1 merge $2', round(d['kernel_ms_per_step']['spmm_fused'],3), round(d['ms_per_step'],3))
"
done
