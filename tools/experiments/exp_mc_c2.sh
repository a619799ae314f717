for v in 0 1 0 1; do
  S24_MC=$v timeout 300 python bench.py --config c2 --steps 200 --no-cpu-baseline --no-dense > gpurun_out/mc_$v.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/mc_$v.json').read().splitlines()[-1])
print('MC=$v', round(d['ms_per_step'],4), {k: round(v['ms_per_step']*1e3,1) for k,v in d['kernels'].items() if k.startswith('k3') or k.startswith('k4')}, d['clocks']['sm_mhz'])
"
done
for v in 0 1; do
  S24_MC=$v timeout 300 python bench.py --config c5 --steps 100 --no-cpu-baseline --no-dense > gpurun_out/mc5_$v.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/mc5_$v.json').read().splitlines()[-1])
print('C5 MC=$v', round(d['ms_per_step'],4), {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items() if k.startswith('k3') or k.startswith('k4')}, d['clocks']['sm_mhz'])
"
done
