cp tools/libacz_gpu_l128.so paper_2011_09017_b200/lib/libacz_gpu.so
timeout 600 python -m pytest tests/test_gpu_quant_spec.py -x -q 2>&1 | tail -1
timeout 300 python tools/qbench.py conv1 config1 vgg_conv2 2>&1 | grep -v "decode cyc"
