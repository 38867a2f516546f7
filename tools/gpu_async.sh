mkdir -p gpurun_out/async
timeout 900 python -m pytest tests/test_gpu_async.py -m gpu -x -q > gpurun_out/async/pytest.log 2>&1; echo pytest=$? >> gpurun_out/async/pytest.log
tail -5 gpurun_out/async/pytest.log
timeout 600 python tools/train_prof.py > gpurun_out/async/train_prof.txt 2>&1; cat gpurun_out/async/train_prof.txt
