mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_bipartite.py -q -x -p no:cacheprovider -k "plan or fuzz_case or parity" 2>&1 | grep -E "^E  +|^FAILED|passed|failed|Error" | cut -c1-400 | head -10
FM_SORT_BIG_MIN=0 timeout 900 python -m pytest tests/test_gpu_fuzz.py -q -x -p no:cacheprovider -k "medium" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "4 or plan" 2>&1 | tail -1
for cfg in 4 5 2; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg${cfg}.json 2>gpurun_out/bench_cfg${cfg}.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/bench_cfg${cfg}.json").read().strip().splitlines()[-1])
print("cfg ${cfg}", round(d["value"]/1e9,2), "Gedges/s", round(d["ms_per_step"],3), "ms", {k: round(v,3) for k,v in d["phase_ms_per_step"].items()})
PY
done
