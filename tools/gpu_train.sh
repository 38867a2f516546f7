mkdir -p gpurun_out/train
timeout 600 python tools/train_overhead.py > gpurun_out/train/train_overhead.txt 2>&1; cat gpurun_out/train/train_overhead.txt
