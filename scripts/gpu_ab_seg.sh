# heavy-row segment length / light cap sweep on the final SpMM (SpMM family ms per embedding)
for cfg in "256 64" "128 64" "384 64" "512 64" "256 64" "128 64" "256 48"; do
  set -- $cfg
  NETMFP_HEAVY_SEG=$1 NETMFP_LIGHT_CAP=$2 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ab_seg.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/ab_seg.log').read().strip().splitlines()[-1])
print('seg $1 cap $2', round(d['kernel_ms_per_step']['spmm_fused'],3), round(d['ms_per_step'],3))
"
done
