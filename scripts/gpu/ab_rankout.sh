mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python paper_2509_13230_b200/build.py --variant ro5 FM_SAMPLE_MINB_RANKOUT=5 > gpurun_out/build_a.log 2>&1
python paper_2509_13230_b200/build.py --variant ro6 FM_SAMPLE_MINB_RANKOUT=6 > gpurun_out/build_b.log 2>&1
python paper_2509_13230_b200/build.py --variant ro8x128 FM_SAMPLE_THREADS_RANKOUT=128 FM_SAMPLE_MINB_RANKOUT=8 > gpurun_out/build_c.log 2>&1
python paper_2509_13230_b200/build.py --variant ro10x128 FM_SAMPLE_THREADS_RANKOUT=128 FM_SAMPLE_MINB_RANKOUT=10 > gpurun_out/build_d.log 2>&1
for CFG in 4; do for rep in 1 2; do for var in base ro5 ro6 ro8x128 ro10x128; do
  v=$var; [ "$var" = "base" ] && v=""
  FM_LIB_VARIANT=$v timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$var.json 2>gpurun_out/ab_$var.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$var.json').read().strip().splitlines()[-1]); print('cfg $CFG $var', round(d['value']/1e9,3), {k: round(x,3) for k,x in d['phase_ms_per_step'].items()}, 'frac', round(d['roofline']['frac'],3))" 2>&1 | tail -1
done; done; done
