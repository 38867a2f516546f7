mkdir -p gpurun_out/train
timeout 600 python -m pytest tests/test_gpu_async.py tests/test_gpu_controller.py -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/train_overhead.py > gpurun_out/train/train_overhead.txt 2>&1; cat gpurun_out/train/train_overhead.txt | cut -c1-700
timeout 900 python tools/config5_batch_scheme.py --out gpurun_out/train/config5_batch_scheme.json > gpurun_out/train/config5.log 2>&1; tail -8 gpurun_out/train/config5.log
