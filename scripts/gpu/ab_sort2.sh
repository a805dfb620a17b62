mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python paper_2509_13230_b200/build.py --variant s12x3 FM_SORT_ITEMS_BIG=12 FM_SORT_BIG_BLOCKS=3 > gpurun_out/b1.log 2>&1
python paper_2509_13230_b200/build.py --variant s16x3 FM_SORT_ITEMS_BIG=16 FM_SORT_BIG_BLOCKS=3 > gpurun_out/b2.log 2>&1
python paper_2509_13230_b200/build.py --variant s24x1 FM_SORT_ITEMS_BIG=24 FM_SORT_BIG_BLOCKS=1 > gpurun_out/b3.log 2>&1
for rep in 1 2; do for v in "base:" "base:FM_SORT_BIG_MIN=99999999999" "s12x3:" "s16x3:" "s24x1:"; do
  var=${v%%:*}; env=${v#*:}; lib=$var; [ "$var" = "base" ] && lib=""
  env FM_LIB_VARIANT=$lib $env timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s.json 2>gpurun_out/s.err
  python -c "
import json; d=json.loads(open('gpurun_out/s.json').read().strip().splitlines()[-1]); print('cfg4 [$v]', {k: round(x,3) for k,x in d['phase_ms_per_step'].items()})" 2>&1 | tail -1
done; done
