# profile the sampler kernel once: plain run, then ncu --set full on the 4th k_sample launch
TAG=${1:-prof}; shift
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sample -s 2 -c 1 -o gpurun_out/${TAG}_ksample python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "rc=$?"
