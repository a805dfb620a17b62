# pipelined sample groups: parity tests, then group-count sweep on configs 2, 4, 5
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bipartite.py tests/test_gpu_checks.py tests/test_gpu_refresh.py -q -x -p no:cacheprovider > gpurun_out/pytest_groups.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_groups.log
for cfg in 5 4 2 3; do
  for G in 1 0 2 4 8 16; do
    FM_SAMPLE_GROUPS=$G timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g_${cfg}_${G}.json 2>gpurun_out/g_${cfg}_${G}.err
    python - <<PY
import json
try:
    d=json.loads(open("gpurun_out/g_${cfg}_${G}.json").read().strip().splitlines()[-1])
    print("cfg ${cfg} G=${G}", round(d["value"]/1e9,2), "Gedges/s", round(d["ms_per_step"],3), "ms", {k: round(v,3) for k,v in d["phase_ms_per_step"].items()}, "frac", round(d["roofline"]["frac"],3), "call", round(d["roofline"]["call"]["frac"],3))
except Exception as e:
    print("cfg ${cfg} G=${G} failed", e); print(open("gpurun_out/g_${cfg}_${G}.err").read()[-800:])
PY
  done
done
