for CH in 1 2; do for M in ${SWEEP_M:-1 2 3}; do for CFG in ${SWEEP_CFG:-2 3}; do
  [ "$CH" = 1 ] && [ "$M" = 1 ] && continue
  FM_SAMPLE_CHAINS=$CH FM_SAMPLE_MINB=$M python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
b=json.loads(sys.stdin.read()); p=b['phase_ms_per_step']
print('chains=$CH minb=$M cfg=$CFG', round(b['value']/1e9,2), 'Gedges/s step', round(b['ms_per_step'],3), 'kern', round(p['sample_kernel'],3), 'frac', round(b['roofline']['frac'],3))"
done; done; done
