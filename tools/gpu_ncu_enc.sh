# ncu --set full of the encoder (count + write) and decoder on AlexNet conv1 (development)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -f -o gpurun_out/ncu_enc \
    -k regex:"k_encode_count|k_encode_write|k_decode_prev|k_histogram" --launch-skip 4 --launch-count 4 python tools/prof_codec.py conv1 > gpurun_out/ncu_enc.log 2>&1
tail -3 gpurun_out/ncu_enc.log
python tools/ncu_summary.py gpurun_out/ncu_enc.ncu-rep > gpurun_out/ncu_enc_summary.txt 2>&1
cat gpurun_out/ncu_enc_summary.txt
for k in k_encode_count k_encode_write k_decode_prev; do python tools/ncu_lines.py gpurun_out/ncu_enc.ncu-rep $k 14; done > gpurun_out/ncu_enc_lines.txt 2>&1
cat gpurun_out/ncu_enc_lines.txt
