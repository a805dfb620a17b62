mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ab24_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/ab24_pytest.log
