# AlexNet bench (device value + e2e) for the default build and each $ALTS library (development)
mkdir -p gpurun_out
cp paper_2011_09017_b200/lib/libacz_gpu.so /tmp/default.so
for lib in /tmp/default.so $ALTS; do
  cp $lib paper_2011_09017_b200/lib/libacz_gpu.so
  echo "== $lib"
  timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], round(d['value'],1), round(d['e2e']['value'],1))"
done
cp /tmp/default.so paper_2011_09017_b200/lib/libacz_gpu.so
