# parity tests of the default build + qbench of the default and each library in $ALTS
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_quant_spec.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > gpurun_out/pytest_q.log 2>&1; echo pytest=$? >> gpurun_out/pytest_q.log
tail -2 gpurun_out/pytest_q.log
echo "== default"; timeout 300 python tools/qbench.py ${QB_SHAPES:-conv1 config1 conv2 conv3 vgg_conv2} 2>&1 | grep "ratio"
cp paper_2011_09017_b200/lib/libacz_gpu.so /tmp/default.so
for lib in $ALTS; do
  cp $lib paper_2011_09017_b200/lib/libacz_gpu.so
  echo "== $lib"; timeout 300 python tools/qbench.py ${QB_SHAPES:-conv1 config1 conv2 conv3 vgg_conv2} 2>&1 | grep "ratio"
done
cp /tmp/default.so paper_2011_09017_b200/lib/libacz_gpu.so
if [ -n "$BENCH" ]; then timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'ms', d['ms_per_step'], {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"; fi
