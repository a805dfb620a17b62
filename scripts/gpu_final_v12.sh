# round-1 final measurement after the chunk-major queue: tests, smoke, bench lines for configs 2-5 + reference arm, launch list cfg 4
mkdir -p gpurun_out; T=r01_v12
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 700 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err; echo "default rc=$?"
for c in 4 5; do python bench.py --config $c --steps 5 --warmup 3 --cpu-seconds 8 > gpurun_out/${T}_bench_cfg$c.json 2> gpurun_out/${T}_bench_cfg$c.err; echo "cfg$c rc=$?"; done
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err; echo "ref rc=$?"
A="--config 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches_cfg4.csv python bench.py $A > gpurun_out/${T}_ncu_launch.log 2>&1; echo "ncu rc=$?"
