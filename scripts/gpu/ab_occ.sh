mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python paper_2509_13230_b200/build.py --variant t128x7 FM_SAMPLE_THREADS=128 FM_SAMPLE_MINB_UBCM=7 FM_SAMPLE_MINB_ECM=7 > gpurun_out/build_a.log 2>&1
python paper_2509_13230_b200/build.py --variant t224x4 FM_SAMPLE_THREADS=224 FM_SAMPLE_MINB_UBCM=4 FM_SAMPLE_MINB_ECM=4 > gpurun_out/build_b.log 2>&1
python paper_2509_13230_b200/build.py --variant t192x5 FM_SAMPLE_THREADS=192 FM_SAMPLE_MINB_UBCM=5 FM_SAMPLE_MINB_ECM=5 > gpurun_out/build_c.log 2>&1
python paper_2509_13230_b200/build.py --variant t384x2 FM_SAMPLE_THREADS=384 FM_SAMPLE_MINB_UBCM=2 FM_SAMPLE_MINB_ECM=2 > gpurun_out/build_d.log 2>&1
tail -1 gpurun_out/build_a.log gpurun_out/build_b.log gpurun_out/build_c.log gpurun_out/build_d.log
for CFG in 5 2 3; do for rep in 1 2; do for var in base t128x7 t224x4 t192x5 t384x2; do
  v=$var; [ "$var" = "base" ] && v=""
  FM_LIB_VARIANT=$v timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$var.json 2>gpurun_out/ab_$var.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$var.json').read().strip().splitlines()[-1]); print('cfg $CFG $var', round(d['value']/1e9,3), {k: round(x,3) for k,x in d['phase_ms_per_step'].items()}, 'frac', round(d['roofline']['frac'],3))" 2>&1 | tail -1
done; done; done
