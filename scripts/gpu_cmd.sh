mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab28_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab28_pytest.log
AB_RUNS=$'prev3;FM_LIB_VARIANT=prev;--config 3\nbase3;;--config 3\nprevr;FM_LIB_VARIANT=prev;--config 3 --refresh\nbaser;;--config 3 --refresh' AB_STEPS=5 bash scripts/abx.sh 2>&1 | tee gpurun_out/ab28.txt
