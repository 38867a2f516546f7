# Round-2 closing check: the whole GPU suite, smoke(), the bench line, the training step
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python tools/train_overhead.py > $O/train_overhead.txt 2>&1
timeout 900 python tools/config5_batch_scheme.py --out $O/config5_batch_scheme.json > $O/config5.log 2>&1
tail -2 $O/pytest_gpu.log; tail -2 $O/smoke.log; cut -c1-300 $O/bench.json; grep async=True $O/train_overhead.txt | cut -c1-300; tail -8 $O/config5.log
