import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import workloads as W
x = W.make_tensor((64, 64, 56, 56), True, 7)
for _ in range(2):
    c = acz.compress(x, acz.CodecParams(1e-3))
torch.cuda.synchronize()
