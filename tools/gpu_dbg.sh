mkdir -p gpurun_out
timeout 300 python tools/cbbench.py > gpurun_out/cbbench.log 2>&1; cat gpurun_out/cbbench.log
timeout 600 ncu --set full --clock-control none --import-source on -f -o gpurun_out/ncu_conv3 -k regex:"k_quant_prev_serial|k_histogram|k_encode|k_decode" --launch-skip 4 --launch-count 4 python tools/prof_codec.py conv3 > gpurun_out/ncu_conv3.log 2>&1
tail -3 gpurun_out/ncu_conv3.log
