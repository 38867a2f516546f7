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
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = acz.compress_host_many(hin, p, blob_bufs=bb, side_bufs=sb)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    acz.decompress_host_many(r, True, outs=hout)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print("compress_host_many %.2f ms  decompress_host_many %.2f ms" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3))
