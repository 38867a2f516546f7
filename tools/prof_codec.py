import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import workloads as W
x = W.make_tensor((256, 96, 27, 27), True, 7)   # AlexNet conv2_in
for _ in range(2):
    c = acz.compress(x, acz.CodecParams(1e-3))
    d = acz.decompress(c, True)
torch.cuda.synchronize()
