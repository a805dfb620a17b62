mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in ${CFGS:-5 4 2}; do
  for L in ${LS:-128 192 256 384 512}; do
    FM_SAMPLE_GROUPS=1 FM_CHUNK_LANE_DRAWS=$L timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c_${cfg}_${L}.json 2>gpurun_out/c_${cfg}_${L}.err
    python - <<PY
import json
try:
    d=json.loads(open("gpurun_out/c_${cfg}_${L}.json").read().strip().splitlines()[-1])
    print("cfg ${cfg} L=${L}", round(d["value"]/1e9,2), "Gedges/s", round(d["ms_per_step"],3), "ms", {k: round(v,3) for k,v in d["phase_ms_per_step"].items()}, "frac", round(d["roofline"]["frac"],3), "call", round(d["roofline"]["call"]["frac"],3))
except Exception as e:
    print("cfg ${cfg} L=${L} failed", e); print(open("gpurun_out/c_${cfg}_${L}.err").read()[-800:])
PY
  done
done
