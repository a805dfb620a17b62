# compute-sanitizer over small invocations of every entry point (config 1, ECM, bipartite, directed, groups)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python scripts/sanitize_run.py > gpurun_out/sanitize_plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/sanitize_plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --log-file gpurun_out/r02_sanitizer_$tool.log python scripts/sanitize_run.py > gpurun_out/sanitize_$tool.out 2>&1
  echo "$tool rc=$?"; tail -1 gpurun_out/sanitize_$tool.out; tail -3 gpurun_out/r02_sanitizer_$tool.log
done
