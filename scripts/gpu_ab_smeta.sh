# A/B: light-row metadata in shared memory (NETMFP_SPMM_SMETA=1) vs registers + shuffles (0)
for o in 0 1 0 1; do
  NETMFP_SPMM_SMETA=$o timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ab_smeta_$o.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/ab_smeta_$o.log').read().strip().splitlines()[-1])
print('smeta $o', round(d['ms_per_step'],3), 'spmm', round(d['kernel_ms_per_step']['spmm_fused'],3), d['step_ms'])
"
done
