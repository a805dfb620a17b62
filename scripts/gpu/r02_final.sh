# round-2 final evidence: r02_profile.sh (tests, smoke, bench lines, config-5 launch list, ncu full of configs 5 and 2)
# + the ECM capture, the config-4 launch list and the config-4 sampler / compaction capture
TAG=${TAG:-r02_v13}
export TAG
bash scripts/gpu/r02_profile.sh
ncu --set full --clock-control none --import-source on -k regex:"k_sample|k_compact" -s 2 -c 2 -f -o gpurun_out/${TAG}_cfg3_prof python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_3.log 2>&1
echo "ncu cfg3 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg4.csv python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_sample|k_compact" -s 2 -c 2 -f -o gpurun_out/${TAG}_cfg4_prof python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_4.log 2>&1
echo "ncu cfg4 rc=$?"
ncu --set full --clock-control none -k regex:"k_pass" -s 8 -c 1 -f -o gpurun_out/${TAG}_cfg4_kpass python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_4p.log 2>&1
echo "ncu kpass rc=$?"
ls -la gpurun_out/*.ncu-rep | tail -8
