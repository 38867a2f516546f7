mkdir -p gpurun_out/final
timeout 600 python -m pytest tests/test_gpu_async.py -m gpu -x -q 2>&1 | tail -2
for l in 1 2; do echo "== lanes $l"; LANES=$l timeout 300 python tools/train_overhead.py 2>&1 | grep "async=True" | cut -c1-460; done
timeout 1200 python tools/config5_batch_scheme.py --out gpurun_out/final/config5_batch_scheme.json > gpurun_out/final/config5.log 2>&1; tail -8 gpurun_out/final/config5.log
