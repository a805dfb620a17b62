# A/B over labelled runs: each line of $AB_RUNS is "label;ENV=.. ENV2=..;bench args" (run twice, interleaved)
#   AB_RUNS=$'prev;FM_LIB_VARIANT=prev;--config 2\nbase;;--config 2' bash scripts/abx.sh
for rep in 1 2; do
while IFS=';' read -r label envs args; do
  [ -z "$label" ] && continue
  env $envs timeout 300 python bench.py --steps ${AB_STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e $args 2>/dev/null | python -c "
import json,sys
b=json.loads(sys.stdin.read()); p=b['phase_ms_per_step']
print('$label', b['config']['workload'], round(b['value']/1e9,2), 'Gedges/s step', round(b['ms_per_step'],3), 'plan', round(p['plan'],3), 'kern', round(p['sample_kernel'],3), 'write', round(p['write'],3), 'frac', round(b['roofline']['frac'],3))"
done <<< "$AB_RUNS"
done
