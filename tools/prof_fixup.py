"""One K2b compress of a 128x3x224x224 N(0,1) tensor at eb = 0.1 (the walk leaves most planes to
the serial replay, k_spec_fixup) for an ncu capture; run with ACZ_SPEC_QUANT=1."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import workloads as W
x = W.make_tensor((128, 3, 224, 224), False, 7)
for _ in range(2):
    acz.compress(x, acz.CodecParams(0.1))
torch.cuda.synchronize()
