mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
FM_SAMPLE_GROUPS=3 FM_COMPACT_SMALL=2 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bipartite.py tests/test_gpu_checks.py tests/test_gpu_refresh.py -q -x -p no:cacheprovider > gpurun_out/pytest_groups.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_groups.log
CFGS="5" GS="2 4" bash scripts/gpu/pipe_trace.sh
CFGS="5 4 2 3" GS="1 2 4 8" bash scripts/gpu/r02_groups2.sh
