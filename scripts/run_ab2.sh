mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab2_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/ab2_pytest.log
for c in 2 3; do AB_VARIANTS="prev base" AB_ARGS="--config $c" bash scripts/ab.sh; done 2>&1 | tee gpurun_out/ab2.txt
ncu --set full --clock-control none --import-source on -k regex:k_sample -s 2 -c 1 -o gpurun_out/ab2_ksample python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ab2_ncu_full.log 2>&1; echo "ncu rc=$?"
