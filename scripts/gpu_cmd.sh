mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab40_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab40_pytest.log
AB_RUNS=$'prev3;FM_LIB_VARIANT=prev;--config 3\nrec3;;--config 3\nprevr;FM_LIB_VARIANT=prev;--config 3 --refresh\nrecr;;--config 3 --refresh\nprev2;FM_LIB_VARIANT=prev;--config 2\nbase2;;--config 2' AB_STEPS=5 bash scripts/abx.sh 2>&1 | tee gpurun_out/ab40.txt
