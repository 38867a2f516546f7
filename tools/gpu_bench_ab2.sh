# bench (device step) of the default build and each library in $ALTS, twice each (development)
mkdir -p gpurun_out
cp paper_2011_09017_b200/lib/libacz_gpu.so /tmp/default.so
for lib in /tmp/default.so $ALTS; do
  cp $lib paper_2011_09017_b200/lib/libacz_gpu.so
  for r in 1 2; do
    timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],1), round(d['ms_per_step'],4), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
  done
done
cp /tmp/default.so paper_2011_09017_b200/lib/libacz_gpu.so
