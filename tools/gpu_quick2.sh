# parity tests of the quantisers + per-kernel timings + bench (development iteration)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_quant_spec.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > gpurun_out/pytest_q.log 2>&1; echo pytest=$? >> gpurun_out/pytest_q.log
tail -3 gpurun_out/pytest_q.log
timeout 300 python tools/qbench.py ${QB_SHAPES:-conv1 config1 conv2 conv3 vgg_conv2} 2>&1 | grep -v "cycles\|offsets\|walk:" > gpurun_out/qbench.log; cat gpurun_out/qbench.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], d['kernels'])"
timeout 300 python tools/step_trace.py > gpurun_out/step_trace.log 2>&1
