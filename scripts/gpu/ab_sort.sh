mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for lb in 16 24 32; do python paper_2509_13230_b200/build.py --variant lb$lb FM_SORT_LB=$lb > gpurun_out/build_lb$lb.log 2>&1; done
for rep in 1 2; do for v in "" lb16 lb24 lb32; do
  FM_LIB_VARIANT=$v timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s_$v.json 2>gpurun_out/s_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/s_$v.json').read().strip().splitlines()[-1]); print('cfg4 [$v]', {k: round(x,3) for k,x in d['phase_ms_per_step'].items()})"
done; done
