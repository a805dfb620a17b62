mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q > gpurun_out/ab12_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab12_pytest.log
AB_RUNS=$'prev;FM_LIB_VARIANT=prev;--config 2\nbase;;--config 2\nprev4;FM_LIB_VARIANT=prev;--config 4\nrank4;;--config 4\nprev5;FM_LIB_VARIANT=prev;--config 5\nbase5;;--config 5' AB_STEPS=5 bash scripts/abx.sh 2>&1 | tee gpurun_out/ab12.txt
