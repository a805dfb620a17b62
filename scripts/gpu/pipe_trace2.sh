mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cv in 45 50 60 75; do
echo "== cfg 5 G 2 carveout $cv"
FM_SAMPLE_CARVEOUT=$cv FM_PIPE_TRACE=1 FM_SAMPLE_GROUPS=2 timeout 300 python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep pipe | tail -10
done
