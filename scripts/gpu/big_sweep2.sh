mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() { # name, env...
  name=$1; shift
  for cfg in ${CFGS:-5 4 2 3}; do
    env FM_SAMPLE_GROUPS=1 "$@" timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_${cfg}_${name}.json 2>gpurun_out/b_${cfg}_${name}.err
    python - <<PY
import json
try:
    d=json.loads(open("gpurun_out/b_${cfg}_${name}.json").read().strip().splitlines()[-1])
    print("cfg ${cfg} ${name}", round(d["value"]/1e9,2), "Gedges/s", round(d["ms_per_step"],3), "ms", {k: round(v,3) for k,v in d["phase_ms_per_step"].items()}, "frac", round(d["roofline"]["frac"],3), "call", round(d["roofline"]["call"]["frac"],3))
except Exception as e:
    print("cfg ${cfg} ${name} failed", e); print(open("gpurun_out/b_${cfg}_${name}.err").read()[-800:])
PY
  done
}
run big0 FM_CHUNK_BIG_DRAWS=0
run big512 FM_CHUNK_BIG_DRAWS=512
CFGS=5 run big768 FM_CHUNK_BIG_DRAWS=768
CFGS=5 run big1024 FM_CHUNK_BIG_DRAWS=1024
CFGS=5 run big1024t3 FM_CHUNK_BIG_DRAWS=1024 FM_TAIL_FACTOR_BIG=3
CFGS=5 run big512t3 FM_CHUNK_BIG_DRAWS=512 FM_TAIL_FACTOR_BIG=3
CFGS="5 2" run big512tma FM_CHUNK_BIG_DRAWS=512 FM_COMPACT_SMALL=2
