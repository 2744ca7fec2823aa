# A/B: Alg. 4 steps 5-6 (Z sketch) on the side stream beside orth(Y) (NETMFP_SIDE_STREAM=1) vs serial (0)
for o in 0 1 0 1 0 1; do
  NETMFP_SIDE_STREAM=$o timeout 600 python bench.py --steps 15 --warmup 3 --no-cpu > gpurun_out/ab_side_$o.log 2>&1
  python -c "
import json, statistics
d=json.loads(open('gpurun_out/ab_side_$o.log').read().strip().splitlines()[-1])
st=d['step_ms']
print('side $o', 'median', round(statistics.median(st),3), 'min', min(st), 'clocks', d.get('clocks'))
"
done
