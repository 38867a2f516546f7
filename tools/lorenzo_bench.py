"""Times the Lorenzo2d predictor path (compress + decompress) on a few shapes (development)."""
import sys, time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import workloads as W
ctx = acz.default_context()
for shape, relu in [((64, 64, 56, 56), True), ((256, 3, 227, 227), False), ((256, 96, 27, 27), True)]:
    x = W.make_tensor(shape, relu, 5)
    for pred in (acz.Predictor.PrevValue, acz.Predictor.Lorenzo2d):
        p = acz.CodecParams(1e-3, predictor=pred)
        for it in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            c = acz.compress(x, p)
            torch.cuda.synchronize(); t1 = time.perf_counter()
            y = acz.decompress(c, True)
            torch.cuda.synchronize(); t2 = time.perf_counter()
        print(shape, pred.name, "ratio %.3f" % acz.compression_ratio(c),
              "compress %.2f ms decompress %.2f ms" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3))
