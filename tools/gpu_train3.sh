timeout 600 python -m pytest tests/test_gpu_async.py tests/test_gpu_controller.py -m gpu -x -q 2>&1 | tail -2
for pf in 0 1; do echo "== prefetch $pf"; PREFETCH=$pf timeout 300 python tools/train_overhead.py 2>&1 | grep "async=True" | cut -c1-460; done
