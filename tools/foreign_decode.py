"""Times decompression of ACZ1 blobs without a sidecar (foreign blobs: the sidecar is rebuilt
on the GPU) against the sidecar path (development tool)."""
import sys, time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np
import torch
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import workloads as W
for shape, relu in [((64, 64, 56, 56), True), ((256, 3, 227, 227), False)]:
    x = W.make_tensor(shape, relu, 3)
    c = acz.compress(x, acz.CodecParams(1e-3))
    raw = c.to_bytes()
    arr = np.frombuffer(raw, np.uint8)
    for side in (True, False):
        for it in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            if side:
                res = acz.decompress_host_many([(arr, np.frombuffer(c.sidecar(), np.uint8))], True)
            else:
                res = acz.decompress_host_many([(arr, None)], True)
            torch.cuda.synchronize(); t1 = time.perf_counter()
        print(shape, "sidecar" if side else "foreign (no sidecar)", "%.2f ms" % ((t1 - t0) * 1e3))
