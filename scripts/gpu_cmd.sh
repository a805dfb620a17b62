mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_sample -s 2 -c 1 -o gpurun_out/ab26_ecm python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
