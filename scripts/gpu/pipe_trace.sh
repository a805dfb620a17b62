mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in ${CFGS:-5 4}; do for G in ${GS:-2 4}; do
echo "== cfg $cfg G $G"
FM_PIPE_TRACE=1 FM_SAMPLE_GROUPS=$G timeout 300 python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep pipe | tail -$((G*5))
done; done
