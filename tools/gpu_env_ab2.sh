# A/B of an environment switch on the device step: ENVS="A=1 B=2" (each run twice, alternating)
for r in 1 2 3; do
for e in "X=0" $ENVS; do
  env $e timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['value'],1), round(d['ms_per_step'],4), round(d['compress_decompress_split']['decompress_ms'],4))"
done
done
