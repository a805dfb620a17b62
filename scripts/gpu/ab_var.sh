# A/B of library variants on one box: python bench.py per variant, interleaved twice.  VARIANTS="base x y", CFG
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for var in $VARIANTS; do [ "$var" = "base" ] || python paper_2509_13230_b200/build.py --variant $var $(eval echo \$DEF_$var) > gpurun_out/build_$var.log 2>&1; done
CFG=${CFG:-5}
for rep in 1 2; do
for var in $VARIANTS; do
  v=$var; [ "$var" = "base" ] && v=""
  FM_LIB_VARIANT=$v timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$var.json 2>gpurun_out/ab_$var.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$var.json').read().strip().splitlines()[-1]); print('cfg $CFG $var', round(d['value']/1e9,3), {k: round(x,3) for k,x in d['phase_ms_per_step'].items()}, 'frac', round(d['roofline']['frac'],3))" 2>&1 | tail -1
done; done
