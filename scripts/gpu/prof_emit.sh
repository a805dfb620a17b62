mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_emit|k_chunks" -s 4 -c 4 -o gpurun_out/emit4 -f python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu3.log 2>&1
echo rc=$?
