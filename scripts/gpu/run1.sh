mkdir -p gpurun_out
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -lineinfo -o /tmp/mb scripts/microbench_ops.cu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python scripts/d2h_probe.py > gpurun_out/d2h_probe.json 2>&1
/tmp/mb > gpurun_out/microbench.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__inst_executed.sum,sm__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_xu.sum --clock-control none --csv --log-file gpurun_out/microbench_ncu.csv /tmp/mb > gpurun_out/microbench_ncu.log 2>&1
echo rc=$?
