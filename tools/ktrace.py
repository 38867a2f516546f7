"""Kernel durations (CUPTI via torch.profiler) of one warmed-up compress of a named shape
(development tool). usage: python tools/ktrace.py [conv1|vgg_conv2|...]"""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import workloads as W
shapes = {"conv1": (256, 3, 227, 227, False), "config1": (64, 64, 56, 56, True),
          "conv2": (256, 96, 27, 27, True), "conv3": (256, 256, 13, 13, True),
          "vgg_conv2": (16, 64, 224, 224, True), "vgg_conv2_b64": (64, 64, 224, 224, True),
          "vgg_conv2_b1": (1, 64, 224, 224, True), "vgg_conv2_b4": (4, 64, 224, 224, True),
          "img224_b16": (16, 3, 224, 224, False)}
nm = sys.argv[1] if len(sys.argv) > 1 else "conv1"
b, c, h, w, relu = shapes[nm]
x = W.make_tensor((b, c, h, w), relu, 7)
for _ in range(2):
    blob = acz.compress(x, acz.CodecParams(1e-3))
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    blob = acz.compress(x, acz.CodecParams(1e-3))
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in evs)
for e in sorted(evs, key=lambda e: e.time_range.start):
    print(f"{nm} {(e.time_range.start - t0) / 1e3:8.3f} {e.time_range.elapsed_us() / 1e3:8.3f}  {e.name[:50]}")
