mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab32_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab32_pytest.log
AB_RUNS=$'prev2;FM_LIB_VARIANT=prev;--config 2\nbase2;;--config 2\nprev3;FM_LIB_VARIANT=prev;--config 3\nbase3;;--config 3\nprev5;FM_LIB_VARIANT=prev;--config 5\nbase5;;--config 5' AB_STEPS=10 bash scripts/abx.sh 2>&1 | tee gpurun_out/ab32.txt
