"""CUPTI timeline of one warmed-up e2e step (compress_host_many + decompress_host_many on
page-locked host buffers, AlexNet B256): copies, kernels and the host calls between them
(development tool). usage: python tools/e2e_trace.py [compress|decompress|both]"""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import workloads as W

which = sys.argv[1] if len(sys.argv) > 1 else "both"
ts = [x for _, x in W.make_set("alexnet", 256, device=torch.device("cuda", 0))]
p = acz.CodecParams(1e-3)
ctx = acz.Context()
hin = [torch.empty(x.shape, dtype=torch.float32, pin_memory=True) for x in ts]
for h, x in zip(hin, ts):
    h.copy_(x)
hout = [torch.empty(x.shape, dtype=torch.float32, pin_memory=True) for x in ts]
bbufs = [torch.empty(5 * x.numel() + (1 << 20), dtype=torch.uint8, pin_memory=True) for x in ts]
sbufs = [torch.empty(x.numel() // 8 + (1 << 20), dtype=torch.uint8, pin_memory=True) for x in ts]


def step(c=True, d=True, res=None):
    if c:
        res = acz.compress_host_many(hin, p, blob_bufs=bbufs, side_bufs=sbufs, ctx=ctx)
    if d:
        acz.decompress_host_many(res, zero_filter=True, outs=hout, ctx=ctx)
    return res


for _ in range(3):
    res = step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    if which in ("compress", "both"):
        res = step(True, which == "both")
    else:
        step(False, True, res)
    torch.cuda.synchronize()
evs = list(prof.events())
t0 = min(e.time_range.start for e in evs if e.device_type == torch.autograd.DeviceType.CUDA)
rows = []
for e in evs:
    dev = "GPU" if e.device_type == torch.autograd.DeviceType.CUDA else "cpu"
    rows.append(((e.time_range.start - t0) / 1e3, (e.time_range.end - t0) / 1e3, dev, e.name[:60]))
for a, b, d, n in sorted(rows):
    if d == "cpu" and (b - a) < 0.02:
        continue
    print("%8.3f %8.3f %7.3f %s %s" % (a, b, b - a, d, n.replace("acz_b200::(anonymous namespace)::", "")))
