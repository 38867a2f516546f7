# Round-2 evidence (second half): as gpu_evidence_r2.sh + the training-step overhead and config 5
# Round-2 evidence: GPU tests, bench (CPU baseline + e2e), reference arm, other configs and
# data kinds, VGG-16 eb sweep, CUPTI step timeline, ncu launch list of the bench command,
# ncu --set full of K2b, of the encoder/decoder/histogram, of K1 (stats) and Lorenzo2d.
mkdir -p gpurun_out/ev7
O=gpurun_out/ev7
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
for w in "alexnet 256 model" "alexnet 256 smooth" "config1 64 iid" "config1 64 smooth" "vgg16 256 iid" "vgg16 64 model" "resnet50 64 iid" "resnet18 128 iid"; do
  set -- $w
  timeout 600 python bench.py --workload $1 --batch $2 --data $3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1
done > $O/bench_configs.jsonl
for eb in 1e-4 3e-4 1e-3 3e-3 1e-2; do
  timeout 300 python bench.py --workload vgg16 --batch 256 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --eb $eb 2>/dev/null | tail -1
done > $O/bench_vgg16_eb_sweep.jsonl
timeout 300 python tools/step_trace.py 2>&1 | grep -v -i warn > $O/step_timeline_alexnet.txt
timeout 300 python tools/e2e_split.py > $O/e2e_split.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_alexnet.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -f -o $O/ncu_full_quant_spec \
    -k regex:k_quant_spec --launch-skip 1 --launch-count 1 python tools/prof_codec.py conv1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -f -o $O/ncu_full_rest \
    -k regex:"k_decode_prev|k_encode|k_histogram|k_quant_prev_serial|k_spec_verify" --launch-skip 5 --launch-count 5 \
    python tools/prof_codec.py conv1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -f -o $O/ncu_full_misc \
    -k regex:"k_stats|k_quant_lorenzo|k_decode_lorenzo|k_lorenzo_syms" --launch-skip 0 --launch-count 6 \
    python tools/prof_misc.py > /dev/null 2>&1
for r in ncu_full_quant_spec ncu_full_rest ncu_full_misc; do python tools/ncu_summary.py $O/$r.ncu-rep > $O/${r}_summary.txt 2>&1; done
python tools/ncu_lines.py $O/ncu_full_quant_spec.ncu-rep k_quant_spec 40 > $O/ncu_full_quant_spec_lines.txt 2>&1
tail -3 $O/pytest_gpu.log; cat $O/bench.json $O/bench_ref.json
timeout 600 python tools/train_overhead.py > $O/train_overhead.txt 2>&1
timeout 900 python tools/config5_batch_scheme.py --out $O/config5_batch_scheme.json > $O/config5.log 2>&1
