set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
nproc; lscpu | grep "Model name"
./scripts/microbench_ops > gpurun_out/micro.json 2>&1 && \
ncu --metrics sm__inst_executed.sum,sm__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_lsu.sum,sm__inst_executed_pipe_uniform.sum,sm__pipe_fp64_cycles_active.sum,sm__cycles_elapsed.avg,gpu__time_duration.sum --clock-control none -c 50 --csv --log-file gpurun_out/micro_ncu.csv ./scripts/microbench_ops > /dev/null 2>&1
python bench.py --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sample -s 3 -c 1 -o gpurun_out/prof_ksample python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
