# ncu --set full of K4 alone (k_codebook_fast, ACZ_BOOK_UNFUSED=1) on AlexNet conv1
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -f -o gpurun_out/ncu_hist \
    --warp-sampling-interval 0 -k regex:k_codebook_fast --launch-skip 1 --launch-count 1 env ACZ_BOOK_UNFUSED=1 python tools/prof_codec.py conv1 > gpurun_out/ncu_hist.log 2>&1
tail -3 gpurun_out/ncu_hist.log
python tools/ncu_lines.py gpurun_out/ncu_hist.ncu-rep k_codebook_fast 150 > gpurun_out/ncu_hist_lines.txt 2>&1
