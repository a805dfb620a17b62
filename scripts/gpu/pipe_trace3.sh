mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for G in 1 2 4; do for cv in 100; do
echo "== cfg 5 G $G carveout $cv"
FM_SAMPLE_CARVEOUT=$cv FM_PIPE_TRACE=1 FM_SAMPLE_GROUPS=$G timeout 300 python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep "pipe\|c2" | tail -$((G*4))
done; done
