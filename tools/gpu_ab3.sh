# A/B of the device step (default build vs $ALTS, alternating, 2 rounds) + parity tests +
# the full default bench line (e2e included)
mkdir -p gpurun_out/ab
O=gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > $O/pytest.log 2>&1; echo pytest=$? >> $O/pytest.log
tail -2 $O/pytest.log
cp paper_2011_09017_b200/lib/libacz_gpu.so /tmp/default.so
for r in 1 2; do
for lib in /tmp/default.so $ALTS; do
  cp $lib paper_2011_09017_b200/lib/libacz_gpu.so
  timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],1), round(d['ms_per_step'],4), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
done
done
cp /tmp/default.so paper_2011_09017_b200/lib/libacz_gpu.so
timeout 600 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; python -c "
import json; d=json.load(open('$O/bench.json')); print(d['value'], d['e2e'])"
