# sweep anchor quantile and lane window for the speculative quantiser (development)
for q in 32 8 4; do
  echo "== L64 q=$q"; ACZ_ANCHOR_Q=$q timeout 300 python tools/qbench.py conv1 config1 vgg_conv2 2>&1 | grep -v "decode cycles"
done
cp tools/libacz_gpu_l32.so paper_2011_09017_b200/lib/libacz_gpu.so
for q in 32 8 4; do
  echo "== L32 q=$q"; ACZ_ANCHOR_Q=$q timeout 300 python tools/qbench.py conv1 config1 vgg_conv2 2>&1 | grep -v "decode cycles"
done
ACZ_ANCHOR_Q=8 timeout 600 python -m pytest tests/test_gpu_quant_spec.py -x -q 2>&1 | tail -2
