# A/B of the default build against an alternative libacz_gpu.so (development):
#   ALT=tools/libacz_gpu_x.so bash tools/gpu_ab.sh [shapes...]
mkdir -p gpurun_out
echo "== default"; timeout 300 python tools/qbench.py ${QB_SHAPES:-conv1 vgg_conv2} 2>&1 | grep -v "decode cycles"
timeout 600 python -m pytest tests/test_gpu_quant_spec.py -x -q 2>&1 | tail -1
cp paper_2011_09017_b200/lib/libacz_gpu.so /tmp/default.so
cp $ALT paper_2011_09017_b200/lib/libacz_gpu.so
echo "== $ALT"; timeout 300 python tools/qbench.py ${QB_SHAPES:-conv1 vgg_conv2} 2>&1 | grep -v "decode cycles"
cp /tmp/default.so paper_2011_09017_b200/lib/libacz_gpu.so
