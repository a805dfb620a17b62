# A/B of library variants (built with `python paper_2509_13230_b200/build.py --variant TAG DEFINES`):
#   AB_VARIANTS="base imm" AB_ARGS="--config 3" bash scripts/ab.sh
for rep in 1 2; do for v in ${AB_VARIANTS:-base}; do
  if [ "$v" = base ]; then unset FM_LIB_VARIANT; else export FM_LIB_VARIANT=$v; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${AB_ARGS} 2>/dev/null | python -c "
import json,sys
b=json.loads(sys.stdin.read()); p=b['phase_ms_per_step']
print('$v', b['config']['workload'], round(b['value']/1e9,2), 'Gedges/s step', round(b['ms_per_step'],3), 'plan', round(p['plan'],3), 'kern', round(p['sample_kernel'],3), 'write', round(p['write'],3), 'frac', round(b['roofline']['frac'],3))"
done; done
unset FM_LIB_VARIANT
