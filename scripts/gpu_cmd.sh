mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ab35_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab35_pytest.log
AB_RUNS=$'base2;;--config 2\nbase4;;--config 4\nbase5;;--config 5' AB_STEPS=5 bash scripts/abx.sh 2>&1 | tee gpurun_out/ab35.txt
