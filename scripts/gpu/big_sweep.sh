mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bipartite.py tests/test_gpu_refresh.py tests/test_gpu_degrees.py tests/test_gpu_richclub.py -q -x -p no:cacheprovider > gpurun_out/pytest_big.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_big.log
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
run big1024 FM_CHUNK_BIG_DRAWS=1024
run big512tma FM_CHUNK_BIG_DRAWS=512 FM_COMPACT_SMALL=2
run big512tail1 FM_CHUNK_BIG_DRAWS=512 FM_TAIL_FACTOR=1
