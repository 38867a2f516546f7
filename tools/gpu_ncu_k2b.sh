# ncu --set full of K2b (k_quant_spec) on AlexNet conv1 + top source lines (development)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -f -o gpurun_out/ncu_quant_spec \
    -k regex:k_quant_spec --launch-skip 1 --launch-count 1 python tools/prof_codec.py conv1 > gpurun_out/ncu_k2b.log 2>&1
tail -5 gpurun_out/ncu_k2b.log
python tools/ncu_lines.py gpurun_out/ncu_quant_spec.ncu-rep k_quant_spec 60 > gpurun_out/ncu_lines.txt 2>&1
python tools/ncu_summary.py gpurun_out/ncu_quant_spec.ncu-rep > gpurun_out/ncu_k2b_summary.txt 2>&1
head -12 gpurun_out/ncu_k2b_summary.txt; head -64 gpurun_out/ncu_lines.txt
