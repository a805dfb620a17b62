mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_pass -s 3 -c 1 -o gpurun_out/kpass4 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
