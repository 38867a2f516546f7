"""Codebook phase timing + per-kernel times for a few shapes (development tool)."""
import ctypes as C
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import _native, workloads as W
lib = _native.load()
ctx = acz.default_context()
for nm, shp, relu in [("conv1", (256, 3, 227, 227), False), ("conv3", (256, 256, 13, 13), True),
                      ("config1", (64, 64, 56, 56), True)]:
    x = W.make_tensor(shp, relu, 7)
    p = acz.CodecParams(1e-3)
    for _ in range(2):
        blob = acz.compress(x, p)
    torch.cuda.synchronize()
    v = (C.c_uint64 * 16)()
    lib.acz_gpu_debug_counters(ctx.handle, v, 16, 1)
    for _ in range(4):
        blob = acz.compress(x, p)
    torch.cuda.synchronize()
    lib.acz_gpu_debug_counters(ctx.handle, v, 16, 1)
    calls = max(1, v[15])
    print(nm, "book", blob.codebook_size, "codebook us/phase:",
          [round(v[8 + i] / calls / 1965.0, 1) for i in range(6)], "rounds/call", v[14] / calls)
