mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q > gpurun_out/ab39_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab39_pytest.log
AB_RUNS=$'prev4;FM_LIB_VARIANT=prev;--config 4\nbase4;;--config 4' AB_STEPS=5 bash scripts/abx.sh 2>&1 | tee gpurun_out/ab39.txt
