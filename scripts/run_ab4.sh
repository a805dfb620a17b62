mkdir -p gpurun_out
for c in 2 3; do AB_VARIANTS="base elog t256m2 t128m5" AB_ARGS="--config $c" bash scripts/ab.sh; done 2>&1 | tee gpurun_out/ab4.txt
