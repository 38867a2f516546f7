"""CUPTI timeline (torch.profiler) of one device-resident bench step (compress_many +
decompress_many of the AlexNet set): kernels with start/end in ms (development tool)."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import workloads as W
ts = [x for _, x in W.make_set(sys.argv[1] if len(sys.argv) > 1 else "alexnet", 256,
                               device=torch.device("cuda", 0))]
p = acz.CodecParams(1e-3)
for it in range(3):
    cs = acz.compress_many(ts, p)
    outs = acz.decompress_many(cs, True)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    cs = acz.compress_many(ts, p)
    outs = acz.decompress_many(cs, True)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in evs)
rows = sorted(((e.time_range.start - t0) / 1e3, (e.time_range.end - t0) / 1e3, e.name[:70]) for e in evs)
for a, b, n in rows:
    print("%8.3f %8.3f %7.3f  %s" % (a, b, b - a, n.replace("acz_b200::(anonymous namespace)::", "")))
