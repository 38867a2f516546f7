# qbench of the default build and of each alternative libacz_gpu.so in ALTS (development)
mkdir -p gpurun_out
echo "== default"; timeout 300 python tools/qbench.py ${QB_SHAPES:-conv1 vgg_conv2} 2>&1 | grep -v "decode cycles\|walk:"
timeout 600 python -m pytest tests/test_gpu_quant_spec.py -x -q 2>&1 | tail -1
cp paper_2011_09017_b200/lib/libacz_gpu.so /tmp/default.so
for alt in $ALTS; do
  cp $alt paper_2011_09017_b200/lib/libacz_gpu.so
  echo "== $alt"; timeout 300 python tools/qbench.py ${QB_SHAPES:-conv1 vgg_conv2} 2>&1 | grep -v "decode cycles\|walk:"
  timeout 600 python -m pytest tests/test_gpu_quant_spec.py -x -q 2>&1 | tail -1
done
cp /tmp/default.so paper_2011_09017_b200/lib/libacz_gpu.so
