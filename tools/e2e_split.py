"""Times the two halves of the e2e host-buffer round trip (development tool)."""
import sys, time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import workloads as W
ts = [x for _, x in W.make_set("alexnet", 256, device=torch.device("cuda", 0))]
hin = [torch.empty(x.shape, dtype=torch.float32, pin_memory=True).copy_(x) for x in ts]
hout = [torch.empty(x.shape, dtype=torch.float32, pin_memory=True) for x in ts]
bb = [torch.empty(5 * x.numel() + (1 << 20), dtype=torch.uint8, pin_memory=True) for x in ts]
sb = [torch.empty(x.numel() // 8 + (1 << 20), dtype=torch.uint8, pin_memory=True) for x in ts]
p = acz.CodecParams(1e-3)
ca, da = [], []
for it in range(12):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = acz.compress_host_many(hin, p, blob_bufs=bb, side_bufs=sb)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    acz.decompress_host_many(r, True, outs=hout)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    if it >= 2:
        ca.append((t1 - t0) * 1e3); da.append((t2 - t1) * 1e3)
ca.sort(); da.sort()
print("compress_host_many median %.2f ms (min %.2f)  decompress_host_many median %.2f ms (min %.2f)" % (
    ca[len(ca) // 2], ca[0], da[len(da) // 2], da[0]))
# raw transfer bounds for the same bytes
dev = [torch.empty_like(x) for x in ts]
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for d, h in zip(dev, hin):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    for d, h in zip(dev, hout):
        h.copy_(d, non_blocking=True)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print("H2D inputs %.2f ms  D2H outputs %.2f ms" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3))
# device-resident compress (no transfers)
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cs = acz.compress_many(ts, p)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("compress_many (device) %.2f ms" % ((t1 - t0) * 1e3))
