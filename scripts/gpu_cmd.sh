mkdir -p gpurun_out
T=r01_v10
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${T}_smoke.log
python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err; echo "bench default rc=$?"; cat gpurun_out/${T}_bench_default.json
python bench.py --steps 10 --warmup 3 --cpu-seconds 8 > gpurun_out/${T}_bench_cfg2.json 2>/dev/null; echo "bench2 rc=$?"
for c in 3 4 5; do python bench.py --config $c --steps 5 --warmup 3 --cpu-seconds 8 > gpurun_out/${T}_bench_cfg$c.json 2>/dev/null; echo "bench$c rc=$?"; done
python bench.py --config 3 --refresh --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_cfg3_refresh.json 2>/dev/null; echo "bench3r rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_reference.json 2>/dev/null; echo "ref rc=$?"
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_launch.log 2>&1; echo "ncu1 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches_cfg4.csv python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu4 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_sample -s 2 -c 1 -o gpurun_out/${T}_ksample python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_sample -s 2 -c 1 -o gpurun_out/${T}_ksample_ecm python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_full_ecm.log 2>&1; echo "ncu full ecm rc=$?"
ncu --set full --clock-control none -k regex:k_compact -s 1 -c 1 -o gpurun_out/${T}_kcompact python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu compact rc=$?"
FM_LIB_VARIANT=trace python scripts/trace_run.py 2 100 > gpurun_out/${T}_trace_cfg2.txt 2>&1; echo "trace rc=$?"
