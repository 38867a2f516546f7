# ncu captures of the codec kernels (development; outputs under gpurun_out/)
set -x
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64 tools/microbench/fp64.cu && /tmp/fp64 > gpurun_out/fp64.log 2>&1
for s in config1 conv1; do
  timeout 600 ncu --set full --clock-control none --import-source on -f -o gpurun_out/ncu_$s \
     --launch-skip 6 --launch-count 7 python tools/prof_codec.py $s > gpurun_out/ncu_$s.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_alexnet.csv \
     python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
cat gpurun_out/fp64.log
