for TF in ${SWEEP_TF:-0 1 2 4}; do for FD in ${SWEEP_FD:-32}; do for CFG in ${SWEEP_CFG:-2}; do
  FM_TAIL_FACTOR=$TF FM_CHUNK_FINE_DRAWS=$FD python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
b=json.loads(sys.stdin.read()); p=b['phase_ms_per_step']
print('tail=$TF fine=$FD cfg=$CFG', round(b['value']/1e9,2), 'Gedges/s step', round(b['ms_per_step'],3), 'kern', round(p['sample_kernel'],3), 'write', round(p['write'],3), 'frac', round(b['roofline']['frac'],3))"
done; done; done
