"""ncu target: the zero-bitmap / sparsity pass (K1 k_stats) and the Lorenzo2d path on
AlexNet conv2_in-shaped data (development tool)."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import workloads as W
x = W.make_tensor((256, 96, 27, 27), True, 7)
ctx = acz.default_context()
for _ in range(2):
    acz.nonzero_ratio(x)
    acz.mean_abs(x)
p = acz.CodecParams(1e-3, predictor=acz.Predictor.Lorenzo2d)
blob = acz.compress(x, p)
out = acz.decompress(blob, True)
torch.cuda.synchronize()
print("ok", acz.compression_ratio(blob))
