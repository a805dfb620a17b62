# e2e leg of the default bench line with D2H alignment / chunk settings: SETS="A=1 B=2|C=3|" (| separated)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
IFS='|' read -ra SETS <<< "$SETS"
for rep in 1 2; do for i in "${!SETS[@]}"; do v="${SETS[$i]}"
env $v python bench.py --config ${CFG:-5} --steps 3 --warmup 3 --no-cpu-baseline $EXTRA 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; print('[$v]', round(e['value']/1e9,3), 'Gedges/s', round(e['ms_per_step'],1), 'ms', round(e.get('d2h_gbs',0),1), 'GB/s')"
done; done
