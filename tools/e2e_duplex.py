"""Diagnosis of the e2e path on a full-duplex host link: per-call times of
compress_host_many / decompress_host_many with one host thread and with two host threads
(own contexts) running whole round trips concurrently."""
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


def lane():
    return dict(ctx=acz.Context(0),
                hout=[torch.empty(x.shape, dtype=torch.float32, pin_memory=True) for x in tensors],
                bb=[torch.empty(5 * x.numel() + (1 << 20), dtype=torch.uint8, pin_memory=True) for x in tensors],
                sb=[torch.empty(x.numel() // 8 + (1 << 20), dtype=torch.uint8, pin_memory=True) for x in tensors],
                log=[])


def step(L, t0):
    a = time.perf_counter()
    r = acz.compress_host_many(hin, p, blob_bufs=L["bb"], side_bufs=L["sb"], ctx=L["ctx"])
    b = time.perf_counter()
    acz.decompress_host_many(r, zero_filter=True, outs=L["hout"], ctx=L["ctx"])
    c = time.perf_counter()
    L["log"].append((round((a - t0) * 1e3, 2), round((b - a) * 1e3, 2), round((c - b) * 1e3, 2)))


lanes = [lane(), lane()]
for L in lanes:
    step(L, 0)
    L["log"].clear()
t0 = time.perf_counter()
for _ in range(4):
    step(lanes[0], t0)
dt = time.perf_counter() - t0
print("one thread: %.2f ms/step" % (dt / 4 * 1e3), lanes[0]["log"])
for mode in ("antiphase", "together"):
    for L in lanes:
        L["log"].clear()
    go = threading.Event()
    if mode == "together":
        go.set()

    def work(i):
        torch.cuda.set_device(0)
        if i == 1:
            go.wait()
        for k in range(4):
            a = time.perf_counter()
            r = acz.compress_host_many(hin, p, blob_bufs=lanes[i]["bb"], side_bufs=lanes[i]["sb"], ctx=lanes[i]["ctx"])
            b = time.perf_counter()
            if i == 0 and k == 0:
                go.set()
            acz.decompress_host_many(r, zero_filter=True, outs=lanes[i]["hout"], ctx=lanes[i]["ctx"])
            c = time.perf_counter()
            lanes[i]["log"].append((round((a - t0) * 1e3, 2), round((b - a) * 1e3, 2), round((c - b) * 1e3, 2)))

    t0 = time.perf_counter()
    ts = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    dt = time.perf_counter() - t0
    print(f"two threads ({mode}): %.2f ms/step" % (dt / 8 * 1e3))
    for i in range(2):
        print("  thread", i, "(start ms, compress ms, decompress ms):", lanes[i]["log"])
