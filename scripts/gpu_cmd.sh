mkdir -p gpurun_out
AB_RUNS=$'base4;;--config 4\ncs4;FM_LIB_VARIANT=cs4;--config 4' AB_STEPS=5 bash scripts/abx.sh 2>&1 | tee gpurun_out/ab33.txt
