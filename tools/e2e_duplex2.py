"""Which side breaks the full-duplex overlap? compress_host_many (upload-bound) against plain
torch downloads on another thread, and decompress_host_many (download-bound) against plain
torch uploads."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import workloads as W

dev = torch.device("cuda", 0)
tensors = [x for _, x in W.make_set("alexnet", 256, device=dev)]
p = acz.CodecParams(1e-3)
hin = [torch.empty(x.shape, dtype=torch.float32, pin_memory=True) for x in tensors]
for h, x in zip(hin, tensors):
    h.copy_(x)
hout = [torch.empty(x.shape, dtype=torch.float32, pin_memory=True) for x in tensors]
bb = [torch.empty(5 * x.numel() + (1 << 20), dtype=torch.uint8, pin_memory=True) for x in tensors]
sb = [torch.empty(x.numel() // 8 + (1 << 20), dtype=torch.uint8, pin_memory=True) for x in tensors]
ctx = acz.Context(0)
blobs = acz.compress_host_many(hin, p, blob_bufs=bb, side_bufs=sb, ctx=ctx)
acz.decompress_host_many(blobs, zero_filter=True, outs=hout, ctx=ctx)
n = sum(x.numel() for x in tensors) * 4
dbuf = torch.empty(n, dtype=torch.uint8, device=dev)
hbuf = torch.empty(n, dtype=torch.uint8, pin_memory=True)
s2 = torch.cuda.Stream()
R = 4

def comp():
    for _ in range(R):
        acz.compress_host_many(hin, p, blob_bufs=bb, side_bufs=sb, ctx=ctx)

def decomp():
    for _ in range(R):
        acz.decompress_host_many(blobs, zero_filter=True, outs=hout, ctx=ctx)

def down():
    torch.cuda.set_device(0)
    with torch.cuda.stream(s2):
        for _ in range(R):
            hbuf.copy_(dbuf, non_blocking=True)
        s2.synchronize()

def up():
    torch.cuda.set_device(0)
    with torch.cuda.stream(s2):
        for _ in range(R):
            dbuf.copy_(hbuf, non_blocking=True)
        s2.synchronize()

def timed(*fns):
    torch.cuda.synchronize()
    t = time.perf_counter()
    ts = [threading.Thread(target=f) for f in fns]
    [x.start() for x in ts]
    [x.join() for x in ts]
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / R * 1e3

for name, fns in [("compress alone", (comp,)), ("download alone", (down,)),
                  ("compress + download", (comp, down)), ("decompress alone", (decomp,)),
                  ("upload alone", (up,)), ("decompress + upload", (decomp, up)),
                  ("upload + download", (up, down))]:
    print(f"{name:24s} {timed(*fns):7.2f} ms per round")
