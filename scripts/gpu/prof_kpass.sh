mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pass" -s 9 -c 2 -f -o gpurun_out/kpass_cfg4 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_kpass.log 2>&1
echo rc=$?
