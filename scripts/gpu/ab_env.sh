# A/B of environment settings: VARS="A=1|B=2 C=3|" (| separated, empty = baseline), CFGS
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
IFS='|' read -ra SETS <<< "$VARS"
for rep in 1 2; do for cfg in ${CFGS:-2 3}; do for i in "${!SETS[@]}"; do
  v="${SETS[$i]}"
  env $v timeout 300 python bench.py --config $cfg --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/e_${cfg}_$i.json 2>gpurun_out/e_${cfg}_$i.err
  python -c "
import json; d=json.loads(open('gpurun_out/e_${cfg}_$i.json').read().strip().splitlines()[-1]); print('cfg $cfg [$v]', round(d['value']/1e9,3), {k: round(x,3) for k,x in d['phase_ms_per_step'].items()}, 'frac', round(d['roofline']['frac'],3))" 2>&1 | tail -1
done; done; done
