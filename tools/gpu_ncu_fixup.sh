mkdir -p gpurun_out/ncufix
ACZ_SPEC_QUANT=1 timeout 120 python tools/prof_fixup.py && \
ACZ_SPEC_QUANT=1 timeout 900 ncu --set full --clock-control none --import-source on -f -o gpurun_out/ncufix/ncu_fixup \
  -k regex:"k_spec_fixup|k_quant_prev_serial" --launch-skip 0 --launch-count 2 python tools/prof_fixup.py > /dev/null 2>&1
ACZ_SERIAL_QUANT=1 timeout 900 ncu --set full --clock-control none --import-source on -f -o gpurun_out/ncufix/ncu_k2a_img \
  -k regex:"k_quant_prev_serial" --launch-skip 1 --launch-count 1 python tools/prof_fixup.py > /dev/null 2>&1
for r in ncu_fixup ncu_k2a_img; do python tools/ncu_summary.py gpurun_out/ncufix/$r.ncu-rep > gpurun_out/ncufix/${r}_summary.txt 2>&1; done
head -40 gpurun_out/ncufix/ncu_fixup_summary.txt; head -30 gpurun_out/ncufix/ncu_k2a_img_summary.txt
