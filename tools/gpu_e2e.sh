mkdir -p gpurun_out/e2e
for c in 0 2 8 32; do echo "== ACZ_COPY_PIECE_MB=$c"; ACZ_COPY_PIECE_MB=$c timeout 300 python tools/e2e_duplex.py 2>&1; done > gpurun_out/e2e/duplex_piece.txt
cat gpurun_out/e2e/duplex_piece.txt
