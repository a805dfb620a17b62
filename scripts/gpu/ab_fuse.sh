mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checks.py -q -x -p no:cacheprovider > gpurun_out/pytest_fuse.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_fuse.log
for cfg in 2 5; do
  for v in "FM_FUSE_WRITE=1" "FM_DISCARD=0" "FM_FUSE_WRITE=0"; do
    env $v timeout 120 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${cfg}_${v}.json 2>gpurun_out/ab_${cfg}_${v}.err
    python - <<PY
import json
d=json.loads(open("gpurun_out/ab_${cfg}_${v}.json").read().strip().splitlines()[-1])
print("cfg ${cfg} ${v}", round(d["value"]/1e9,2), "Gedges/s", round(d["ms_per_step"],3), "ms", {k: round(v,3) for k,v in d["phase_ms_per_step"].items()}, "frac", round(d["roofline"]["frac"],3), "call", round(d["roofline"]["call"]["frac"],3))
PY
  done
done
