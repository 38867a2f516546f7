# A/B of the default build against an environment switch (development):
#   ENVAB="ACZ_BOOK_UNFUSED=1" bash tools/gpu_env_ab.sh
b() { timeout 300 env $1 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], round(d['value'],1), round(d['e2e']['value'],1))"; }
for r in 1 2; do
  echo "== default"; b ""
  echo "== $ENVAB"; b "$ENVAB"
done
