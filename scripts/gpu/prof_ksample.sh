# ncu full capture of k_sample (config $CFG) with source counters
mkdir -p gpurun_out
CFG=${CFG:-5}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_sample" -s 1 -c 1 -o gpurun_out/ksample_cfg$CFG -f python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu2.log 2>&1
echo rc=$?
