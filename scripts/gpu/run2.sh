mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?"
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$?"
tail -3 gpurun_out/pytest.log
