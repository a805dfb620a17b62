mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab14_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab14_pytest.log
AB_RUNS=$'i4x2;FM_LIB_VARIANT=i4x2;--config 2\nv8;;--config 2\nprev3;FM_LIB_VARIANT=prev;--config 3\nv8_3;;--config 3\ni4x2_4;FM_LIB_VARIANT=i4x2;--config 4\nv8_4;;--config 4\nprev5;FM_LIB_VARIANT=prev;--config 5\nv8_5;;--config 5' AB_STEPS=5 bash scripts/abx.sh 2>&1 | tee gpurun_out/ab14.txt
