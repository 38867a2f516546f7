# fastest GPU iteration: speculative-quantiser parity tests + per-kernel timings
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_quant_spec.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_q1.log 2>&1; echo pytest=$? >> gpurun_out/pytest_q1.log
tail -3 gpurun_out/pytest_q1.log
timeout 300 python tools/qbench.py ${QB_SHAPES:-conv1 vgg_conv2} > gpurun_out/qbench.log 2>&1; cat gpurun_out/qbench.log
