# qbench (+ spec parity tests) for each library in $ALTS (development; stats builds)
mkdir -p gpurun_out
cp paper_2011_09017_b200/lib/libacz_gpu.so /tmp/default.so
for lib in $ALTS; do
  cp $lib paper_2011_09017_b200/lib/libacz_gpu.so
  echo "== $lib"; timeout 300 python tools/qbench.py ${QB_SHAPES:-conv1 vgg_conv2} 2>&1 | grep -v "decode cycles\|codebook"
  timeout 600 python -m pytest tests/test_gpu_quant_spec.py -x -q 2>&1 | tail -1
done
cp /tmp/default.so paper_2011_09017_b200/lib/libacz_gpu.so
