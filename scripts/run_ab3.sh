mkdir -p gpurun_out
for c in 2 3; do AB_VARIANTS="base t128m7 t256m4 t64m14" AB_ARGS="--config $c" bash scripts/ab.sh; done 2>&1 | tee gpurun_out/ab3.txt
