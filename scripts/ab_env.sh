# A/B of runtime knobs: AB_ENVS="FM_X=1 FM_X=0" AB_ARGS="--config 4" bash scripts/ab_env.sh
for rep in 1 2; do for e in ${AB_ENVS:-NONE=0}; do
  env $e timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${AB_ARGS} 2>/dev/null | python -c "
import json,sys
b=json.loads(sys.stdin.read()); p=b['phase_ms_per_step']
print('$e', b['config']['workload'], round(b['value']/1e9,2), 'Gedges/s step', round(b['ms_per_step'],3), 'plan', round(p['plan'],3), 'kern', round(p['sample_kernel'],3), 'write', round(p['write'],3), 'frac', round(b['roofline']['frac'],3))"
done; done
