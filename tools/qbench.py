"""Times compress/decompress per kernel class for given shapes and prints the speculative
quantiser's walk counters (development tool)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch

import paper_2011_09017_b200 as acz
from paper_2011_09017_b200 import _native, workloads as W

lib = _native.load()
ctx = acz.default_context()
shapes = {"conv1": (256, 3, 227, 227, False), "config1": (64, 64, 56, 56, True),
          "conv2": (256, 96, 27, 27, True), "conv3": (256, 256, 13, 13, True),
          "vgg_conv2": (16, 64, 224, 224, True), "img128": (128, 3, 224, 224, False)}
which = sys.argv[1:] or list(shapes)
for nm in which:
    b, c, h, w, relu = shapes[nm]
    x = W.make_tensor((b, c, h, w), relu, 7)
    p = acz.CodecParams(float(os.environ.get("QB_EB", "1e-3")))
    for _ in range(2):
        blob = acz.compress(x, p)
        acz.decompress(blob, True)
    v = (C.c_uint64 * 128)()
    lib.acz_gpu_debug_counters(ctx.handle, v, 128, 1)
    lib.acz_gpu_profile_enable(ctx.handle, 1)
    blob = acz.compress(x, p)
    out = acz.decompress(blob, True)
    torch.cuda.synchronize()
    ms = (C.c_double * 7)()
    cnt = (C.c_uint64 * 7)()
    lib.acz_gpu_profile_read(ctx.handle, ms, cnt)
    lib.acz_gpu_profile_enable(ctx.handle, 0)
    lib.acz_gpu_debug_counters(ctx.handle, v, 128, 1)
    names = ["stats", "quant", "hist", "book", "encode", "decode", "scan"]
    print(nm, x.shape, "ratio %.3f" % acz.compression_ratio(blob),
          {names[i]: round(ms[i], 3) for i in range(7) if cnt[i]})
    n = x.numel()
    print("   walk: batches %d (%.4f/elem) changes %d (%.4f) exact %d (%.4f) rebases %d spec %.2f/elem visits %.4f/elem" % (
        v[0], v[0] / n, v[1], v[1] / n, v[2], v[2] / n, v[3], v[4] / n, v[5] / n))
    tot = sum(v[16:20]) or 1
    nw = max(1, v[23])
    print("   decode cycles/warp: prologue %.0f staging %.0f loop %.0f (warps %d)" % (v[20] / nw, v[21] / nw, v[22] / nw, v[23]))
    print("   walk cycles: per exact step %.0f, per batch %.0f (gather %.0f, evaluate %.0f)" % (
        v[24] / max(1, v[2]), v[25] / max(1, v[0]), v[28] / max(1, v[0]), v[29] / max(1, v[0])))
    print("   phase A split (cycles/elem): pass1 %.1f classify %.1f" % (v[26] / n, v[27] / n))
    print("   segment entry offsets: D == 0 in %d, representable in %d" % (v[6], v[7]))
    nb = max(1, v[15])
    print("   codebook cycles: compact %.0f sort %.0f tree %.0f depths %.0f canon %.0f tables %.0f (books %d)" % tuple(
        [v[8 + i] / nb for i in range(6)] + [v[15]]))
    print("   spec cycles/elem (per segment-warp): phaseA %.1f wait %.1f walk %.1f out %.1f" % tuple(v[16 + i] / n for i in range(4)))
    print("   exact replay: chunks whose walk state was wrong %d" % v[31])
    if os.environ.get("QB_HIST"):
        for ph, nmph in enumerate(["phaseA", "wait", "walk", "out"]):
            h = [v[32 + 24 * ph + b] for b in range(24)]
            print("   hist %-6s" % nmph, " ".join("2^%d:%d" % (b, c) for b, c in enumerate(h) if c))
