# lane-window sweep of the speculative quantiser (development): default build vs L=32
mkdir -p gpurun_out
echo "== L64"; timeout 300 python tools/qbench.py conv1 vgg_conv2 2>&1 | grep -v "decode cycles"
cp paper_2011_09017_b200/lib/libacz_gpu.so /tmp/l64.so
cp tools/libacz_gpu_l32.so paper_2011_09017_b200/lib/libacz_gpu.so
echo "== L32"; timeout 300 python tools/qbench.py conv1 vgg_conv2 2>&1 | grep -v "decode cycles"
timeout 600 python -m pytest tests/test_gpu_quant_spec.py -x -q 2>&1 | tail -1
cp /tmp/l64.so paper_2011_09017_b200/lib/libacz_gpu.so
