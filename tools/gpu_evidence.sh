# Round evidence: GPU tests, bench (with CPU baseline + e2e), reference arm, the other
# BASELINE configs, ncu launch list of the bench command, ncu --set full captures of the
# dominant kernel and of the rest, CUPTI step / e2e timelines (outputs in gpurun_out/).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
bash tools/gpu_configs_bench.sh > gpurun_out/bench_configs.jsonl 2>&1
timeout 300 python tools/step_trace.py > gpurun_out/step_trace.log 2>&1
timeout 300 python tools/e2e_split.py > gpurun_out/e2e_split.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -f -o gpurun_out/ncu_full_quant \
    -k regex:k_quant_spec --launch-skip 1 --launch-count 1 python tools/prof_codec.py conv1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -f -o gpurun_out/ncu_full_rest \
    -k regex:"k_decode_prev|k_encode|k_histogram|k_codebook_fast|k_quant_prev_serial" --launch-skip 4 --launch-count 4 \
    python tools/prof_codec.py conv1 > /dev/null 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json gpurun_out/bench_ref.json
# BASELINE config 3: VGG-16 B256 error-bound sweep
for eb in 1e-4 3e-4 1e-3 3e-3 1e-2; do
  timeout 300 python bench.py --workload vgg16 --batch 256 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --eb $eb 2>/dev/null | tail -1
done > gpurun_out/bench_vgg16_eb_sweep.jsonl
