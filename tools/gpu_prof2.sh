# stats-build phase breakdown + ncu source-line stall profile of K2b (development)
mkdir -p gpurun_out
ALTS=tools/libacz_gpu_stats.so QB_SHAPES="conv1 vgg_conv2" bash tools/gpu_alts_qb.sh > gpurun_out/qb_stats.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -f -o gpurun_out/ncu_quant_spec \
    -k regex:k_quant_spec --launch-skip 2 --launch-count 1 python tools/prof_codec.py conv1 > /dev/null 2>&1
python tools/ncu_lines.py gpurun_out/ncu_quant_spec.ncu-rep regex:k_quant_spec 40 > gpurun_out/ncu_lines.txt 2>&1
cat gpurun_out/qb_stats.log; head -45 gpurun_out/ncu_lines.txt
