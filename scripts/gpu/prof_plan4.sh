# ncu full capture of the config-4 plan's scan / emit / rows kernels (one launch each after warm-up)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_scan_lb|k_emit|k_rows" -s 7 -c 5 -o gpurun_out/plan4 -f python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu3.log 2>&1
echo rc=$?
