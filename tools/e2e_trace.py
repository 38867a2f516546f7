"""CUPTI timeline (torch.profiler) of one host-buffer compress_host_many + decompress_host_many
of the AlexNet set: every kernel and copy with start/end in ms (development tool)."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import workloads as W
ts = [x for _, x in W.make_set("alexnet", 256, device=torch.device("cuda", 0))]
hin = [torch.empty(x.shape, dtype=torch.float32, pin_memory=True).copy_(x) for x in ts]
hout = [torch.empty(x.shape, dtype=torch.float32, pin_memory=True) for x in ts]
bb = [torch.empty(5 * x.numel() + (1 << 20), dtype=torch.uint8, pin_memory=True) for x in ts]
sb = [torch.empty(x.numel() // 8 + (1 << 20), dtype=torch.uint8, pin_memory=True) for x in ts]
p = acz.CodecParams(1e-3)
for it in range(3):
    r = acz.compress_host_many(hin, p, blob_bufs=bb, side_bufs=sb)
    acz.decompress_host_many(r, True, outs=hout)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r = acz.compress_host_many(hin, p, blob_bufs=bb, side_bufs=sb)
    torch.cuda.synchronize()
    acz.decompress_host_many(r, True, outs=hout)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in evs)
rows = sorted(((e.time_range.start - t0) / 1e3, (e.time_range.end - t0) / 1e3, e.name[:60]) for e in evs)
for a, b, n in rows:
    if b - a > 0.02 or "emcpy" in n:
        print("%8.3f %8.3f %7.3f  %s" % (a, b, b - a, n))
