# fuzz + parity subset, then bench lines of every config
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_bipartite.py -q -x -p no:cacheprovider 2>&1 | grep -E "^E  +|^FAILED|passed|failed|Error" | cut -c1-400 | head -20
for cfg in 5 2 3 4; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg${cfg}.json 2>gpurun_out/bench_cfg${cfg}.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/bench_cfg${cfg}.json").read().strip().splitlines()[-1])
print("cfg ${cfg}", round(d["value"]/1e9,2), "Gedges/s", round(d["ms_per_step"],3), "ms", {k: round(v,3) for k,v in d["phase_ms_per_step"].items()}, "frac", round(d["roofline"]["frac"],3), "call", round(d["roofline"]["call"]["frac"],3))
PY
done
