cp paper_2011_09017_b200/lib/libacz_gpu.so /tmp/default.so
for lib in alts/stats.so alts/tmax4.so alts/tmax1.so; do
  cp $lib paper_2011_09017_b200/lib/libacz_gpu.so
  for eb in 1e-3 1e-1; do echo "== $lib eb $eb"; ACZ_SPEC_QUANT=1 QB_EB=$eb timeout 300 python tools/qbench.py img128 2>&1 | grep "img128\|wrong"; done
done
cp /tmp/default.so paper_2011_09017_b200/lib/libacz_gpu.so
