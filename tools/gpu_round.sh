set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 300 python tools/qbench.py > gpurun_out/qbench.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --workload config1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/qbench.log; cat gpurun_out/bench.json gpurun_out/bench_c1.json; tail -5 gpurun_out/bench.err
