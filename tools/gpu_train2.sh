timeout 600 python -m pytest tests/test_gpu_async.py -m gpu -x -q 2>&1 | tail -2
for m in 1 2 4 8; do echo "== max_pending $m"; MAXP=$m timeout 300 python tools/train_overhead.py 2>&1 | grep "async=True" | cut -c1-420; done
