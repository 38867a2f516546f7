# full GPU test suite + bench + A/B libs (development)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
ACZ_ENC_TWO_PASS=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_2p.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_2p.json')); print('two-pass value', d['value'], 'ms', d['ms_per_step'], {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
timeout 300 python tools/step_trace.py > gpurun_out/step_trace.log 2>&1
