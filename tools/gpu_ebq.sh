mkdir -p gpurun_out/ebq
timeout 900 python -m pytest tests/test_gpu_async.py tests/test_gpu_quant_spec.py tests/test_gpu_parity.py tests/test_gpu_batch.py -m gpu -x -q > gpurun_out/ebq/pytest.log 2>&1; echo pytest=$? >> gpurun_out/ebq/pytest.log
tail -15 gpurun_out/ebq/pytest.log
for eb in 1e-3 1e-1; do echo "== eb $eb"; QB_EB=$eb timeout 300 python tools/qbench.py img128 conv1 2>&1 | grep -v "walk\|decode cycles\|codebook cycles\|segment entry\|phase A\|spec cycles"; done > gpurun_out/ebq/qbench_fix.txt
cat gpurun_out/ebq/qbench_fix.txt
timeout 600 python tools/train_overhead.py > gpurun_out/ebq/train_overhead.txt 2>&1; cat gpurun_out/ebq/train_overhead.txt
