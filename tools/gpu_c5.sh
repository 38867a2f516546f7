mkdir -p gpurun_out/final
timeout 1200 python tools/config5_batch_scheme.py --out gpurun_out/final/config5_batch_scheme.json > gpurun_out/final/config5.log 2>&1; tail -8 gpurun_out/final/config5.log
