# ncu --set full of k_quant_spec (conv1) for the default build and for $ALT (development)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -f -o gpurun_out/ncu_a \
    -k regex:k_quant_spec --launch-skip 1 --launch-count 1 python tools/prof_codec.py conv1 > /dev/null 2>&1
cp paper_2011_09017_b200/lib/libacz_gpu.so /tmp/default.so
cp $ALT paper_2011_09017_b200/lib/libacz_gpu.so
timeout 900 ncu --set full --clock-control none --import-source on -f -o gpurun_out/ncu_b \
    -k regex:k_quant_spec --launch-skip 1 --launch-count 1 python tools/prof_codec.py conv1 > /dev/null 2>&1
cp /tmp/default.so paper_2011_09017_b200/lib/libacz_gpu.so
ls -la gpurun_out/ncu_a.ncu-rep gpurun_out/ncu_b.ncu-rep
