mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_bipartite.py tests/test_gpu_degrees.py -x -q > gpurun_out/ab19_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab19_pytest.log
AB_RUNS=$'prev;FM_LIB_VARIANT=prev;--config 2\nrec64;;--config 2\ns12;FM_LIB_VARIANT=s12;--config 2\nprev4;FM_LIB_VARIANT=prev;--config 4\nrec64_4;;--config 4\ns12_4;FM_LIB_VARIANT=s12;--config 4\nprev5;FM_LIB_VARIANT=prev;--config 5\nrec64_5;;--config 5' AB_STEPS=5 bash scripts/abx.sh 2>&1 | tee gpurun_out/ab19.txt
