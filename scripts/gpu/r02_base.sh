# round-2 baseline: A/B of the fused write on configs 2, 4, 5; launch list and ncu full capture on config 5
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for cfg in 2 4 5; do
  for v in "FM_FUSE_WRITE=0" "FM_FUSE_WRITE=1"; do
    env $v FM_FUSE_RANKOUT=1 timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${cfg}_${v}.json 2>gpurun_out/ab_${cfg}_${v}.err
    python - <<PY
import json
d=json.loads(open("gpurun_out/ab_${cfg}_${v}.json").read().strip().splitlines()[-1])
print("cfg ${cfg} ${v}", round(d["value"]/1e9,2), "Gedges/s", round(d["ms_per_step"],3), "ms", {k: round(v,3) for k,v in d["phase_ms_per_step"].items()}, "frac", round(d["roofline"]["frac"],3), "call", round(d["roofline"]["call"]["frac"],3))
PY
  done
done
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_sample|k_compact" -c 4 -o gpurun_out/r02_cfg5_prof python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu2.log 2>&1
echo rc=$?
