# chunk-size / segment-target sweep of the sampler (bench.py, no cpu baseline, no e2e)
for S in ${SWEEP_S:-64 128 256}; do for C in ${SWEEP_C:-32 64 128}; do
  FM_CHUNK_LANE_DRAWS=$C python bench.py --steps 5 --warmup 3 --seg-target $S --no-cpu-baseline --no-e2e ${SWEEP_ARGS} 2>/dev/null | python -c "
import json,sys
b=json.loads(sys.stdin.read()); p=b['phase_ms_per_step']
print('S=$S C=$C', round(b['value']/1e9,2), 'Gedges/s step', round(b['ms_per_step'],3), 'plan', round(p['plan'],3), 'kern', round(p['sample_kernel'],3), 'write', round(p['write'],3), 'frac', round(b['roofline']['frac'],3))"
done; done
