mkdir -p gpurun_out
for s in $NCU_SHAPES; do
timeout 600 ncu --set full --clock-control none --import-source on -f -o gpurun_out/ncu_$s -k regex:"$NCU_KERNELS" --launch-skip ${NCU_SKIP:-2} --launch-count ${NCU_COUNT:-2} python tools/prof_codec.py $s > gpurun_out/ncu_$s.log 2>&1
tail -2 gpurun_out/ncu_$s.log
done
