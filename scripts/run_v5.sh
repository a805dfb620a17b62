bash scripts/gpu_round.sh r01_v5
for c in 3 4 5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --cpu-seconds 8 > gpurun_out/r01_v5_bench_cfg$c.json 2> gpurun_out/r01_v5_bench_cfg$c.err; echo "cfg$c rc=$?"; cat gpurun_out/r01_v5_bench_cfg$c.json | head -c 600; echo; done
