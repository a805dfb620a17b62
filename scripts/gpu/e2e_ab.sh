# e2e leg of the default bench line with D2H chunk sizes (FM_D2H_CHUNK_MB; 0 = one copy per group)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do for mb in ${MBS:-0 256 64 1024}; do
FM_D2H_CHUNK_MB=$mb python bench.py --config ${CFG:-5} --steps 3 --warmup 3 --no-cpu-baseline $EXTRA 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; print('chunk $mb MiB:', round(e['value']/1e9,3), 'Gedges/s', round(e['ms_per_step'],1), 'ms', round(e.get('d2h_gbs',0),1), 'GB/s')"
done; done
