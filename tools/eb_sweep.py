"""K2b time and exact-replay corrections across error bounds (development tool)."""
import sys, time, ctypes as C
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import _native, workloads as W
lib = _native.load(); ctx = acz.default_context()
for shape in [(256, 3, 227, 227), (64, 3, 224, 224)]:
    x = W.make_tensor(shape, False, 9)
    for eb in (1e-4, 3e-4, 1e-3, 3e-3, 1e-2):
        p = acz.CodecParams(eb)
        acz.compress(x, p)
        v = (C.c_uint64 * 32)(); lib.acz_gpu_debug_counters(ctx.handle, v, 32, 1)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        c = acz.compress(x, p)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        lib.acz_gpu_debug_counters(ctx.handle, v, 32, 1)
        print(shape, "eb %.0e" % eb, "compress %.2f ms" % ((t1 - t0) * 1e3), "ratio %.3f" % acz.compression_ratio(c),
              "replay corrections", v[31], flush=True)
