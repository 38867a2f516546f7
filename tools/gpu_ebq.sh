mkdir -p gpurun_out/ebq
cp paper_2011_09017_b200/lib/libacz_gpu.so /tmp/default.so
cp alts/stats.so paper_2011_09017_b200/lib/libacz_gpu.so
for eb in 1e-3 1e-2 3e-2 1e-1 3e-1; do echo "== eb $eb"; QB_EB=$eb timeout 300 python tools/qbench.py img128 conv1 2>&1 | grep -v "decode cycles\|codebook cycles\|segment entry"; done > gpurun_out/ebq/qbench.txt
cp /tmp/default.so paper_2011_09017_b200/lib/libacz_gpu.so
cat gpurun_out/ebq/qbench.txt
