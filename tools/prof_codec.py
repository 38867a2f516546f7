"""One warmed-up compress + decompress of a named shape (ncu target; development tool).
usage: python tools/prof_codec.py [config1|conv1|conv2|conv3|vgg_conv2]"""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import workloads as W
shapes = {"conv1": (256, 3, 227, 227, False), "config1": (64, 64, 56, 56, True),
          "conv2": (256, 96, 27, 27, True), "conv3": (256, 256, 13, 13, True),
          "vgg_conv2": (16, 64, 224, 224, True)}
b, c, h, w, relu = shapes[sys.argv[1] if len(sys.argv) > 1 else "config1"]
x = W.make_tensor((b, c, h, w), relu, 7)
for _ in range(2):
    blob = acz.compress(x, acz.CodecParams(1e-3))
    d = acz.decompress(blob, True)
torch.cuda.synchronize()
