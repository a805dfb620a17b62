mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_math.py -x -q > gpurun_out/ab5_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab5_pytest.log
for c in 2 3; do AB_VARIANTS="prev base nocopy aos" AB_ARGS="--config $c" bash scripts/ab.sh; done 2>&1 | tee gpurun_out/ab5.txt
for rep in 1 2; do FM_UBCM_CAND_MIN=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
b=json.loads(sys.stdin.read()); p=b['phase_ms_per_step']
print('cand0', round(b['value']/1e9,2), 'kern', round(p['sample_kernel'],3), 'frac', round(b['roofline']['frac'],3))"; done | tee -a gpurun_out/ab5.txt
