mkdir -p gpurun_out
for cfg in 2 5; do
  for var in "" fstats; do
  FM_LIB_VARIANT=$var timeout 120 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fb_${cfg}.json 2>gpurun_out/fb_${cfg}.err
  grep fuse gpurun_out/fb_${cfg}.err | tail -1
  python -c "
import json; d=json.loads(open('gpurun_out/fb_${cfg}.json').read().strip().splitlines()[-1]); print('cfg ${cfg} fused $var', d['value']/1e9, d['phase_ms_per_step'])"
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_fuse.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_fuse.log
