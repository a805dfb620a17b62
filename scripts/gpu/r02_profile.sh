# round-2 evidence run: GPU tests, smoke, bench lines, ncu launch list and full captures (config 5 and 2)
TAG=${TAG:-r02_v2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ -z "$SKIP_TESTS" ]; then
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
fi
python __graft_entry__.py --smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/bench_reference.err; echo "reference rc=$?"
for cfg in 2 3 4; do
  python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_cfg${cfg}.json 2>gpurun_out/bench_cfg${cfg}.err
done
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu1.log 2>&1
for cfg in 5 2; do
ncu --set full --clock-control none --import-source on -k regex:"k_sample|k_compact" -s 2 -c 2 -f -o gpurun_out/${TAG}_cfg${cfg}_prof python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_${cfg}.log 2>&1
echo "ncu cfg$cfg rc=$?"
done
