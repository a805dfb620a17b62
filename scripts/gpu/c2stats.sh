mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python paper_2509_13230_b200/build.py --variant c2s FM_C2_STATS > gpurun_out/build_c2s.log 2>&1
FM_SAMPLE_GROUPS=3 FM_COMPACT_SMALL=2 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bipartite.py tests/test_gpu_refresh.py -q -x -p no:cacheprovider > gpurun_out/pytest_groups.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_groups.log
for cv in 40 72 100; do
echo "== cfg 5 G 2 carveout $cv"
FM_SAMPLE_CARVEOUT=$cv FM_LIB_VARIANT=c2s FM_PIPE_TRACE=1 FM_SAMPLE_GROUPS=2 timeout 300 python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep "pipe\|c2" | tail -9
done
echo "== solo compact2"
FM_LIB_VARIANT=c2s FM_COMPACT_SMALL=2 FM_PIPE_TRACE=1 FM_SAMPLE_GROUPS=1 timeout 300 python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep "pipe\|c2" | tail -5
