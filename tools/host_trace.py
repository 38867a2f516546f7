"""CUPTI timeline with the host side (CUDA runtime API calls) of one device-resident bench
step: which host calls sit between the codebook read-backs and the encode launches
(development tool)."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import workloads as W
ts = [x for _, x in W.make_set("alexnet", 256, device=torch.device("cuda", 0))]
p = acz.CodecParams(1e-3)
for it in range(3):
    cs = acz.compress_many(ts, p)
    outs = acz.decompress_many(cs, True)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    cs = acz.compress_many(ts, p)
    outs = acz.decompress_many(cs, True)
    torch.cuda.synchronize()
evs = list(prof.events())
t0 = min(e.time_range.start for e in evs if e.device_type == torch.autograd.DeviceType.CUDA)
rows = []
for e in evs:
    dev = "GPU" if e.device_type == torch.autograd.DeviceType.CUDA else "cpu"
    rows.append(((e.time_range.start - t0) / 1e3, (e.time_range.end - t0) / 1e3, dev, e.name[:60]))
for a, b, d, n in sorted(rows):
    if d == "cpu" and (b - a) < 0.002:
        continue
    print("%8.3f %8.3f %7.3f %s %s" % (a, b, b - a, d, n.replace("acz_b200::(anonymous namespace)::", "")))
