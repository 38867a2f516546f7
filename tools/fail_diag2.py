"""Sidecar chain states of saved fuzz failures vs the oracle's reconstruction (development)."""
import glob, os, sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np
import torch
import paper_2011_09017_b200 as acz
from oracle.oracle import Oracle
O = Oracle()
for f in sorted(glob.glob("tools/fuzz_cases/fail_*.npz")):
    z = np.load(f)
    x = z["x"]; eb = float(z["eb"]); radius = int(z["radius"]); mode = str(z["mode"])
    os.environ.pop("ACZ_SPEC_QUANT", None)
    if mode == "spec":
        os.environ["ACZ_SPEC_QUANT"] = "1"
    ref = O.compress(x, eb, radius, 0, shape=x.shape)
    if acz.compress(torch.from_numpy(x).cuda(), acz.CodecParams(eb, radius)).to_bytes() != ref.blob:
        continue
    c = acz.compress(torch.from_numpy(x).cuda(), acz.CodecParams(eb, radius))
    side = np.frombuffer(c.sidecar(), np.uint8)
    hdr = side[8:56].view(np.uint64)
    n, bl, interval, nch = int(hdr[0]), int(hdr[1]), int(hdr[2]), int(hdr[3])
    bitoff = side[56:56 + 8 * nch].view(np.uint64)
    state = side[56 + 8 * nch:56 + 12 * nch].view(np.float32)
    rec = O.decompress(ref.blob, x.size, False)
    P = x.shape[-1] if x.ndim >= 1 else x.size
    P = int(np.prod(x.shape[-2:])) if x.ndim >= 3 else x.shape[-1]
    bad = []
    for ci in range(nch):
        s = ci * interval
        exp = 0.0 if s % P == 0 else rec[s - 1]
        if state[ci].view(np.uint32) != np.float32(exp).view(np.uint32):
            bad.append((ci, float(state[ci]), float(exp)))
    print(os.path.basename(f), x.shape, "P", P, "interval", interval, "bad states", len(bad), bad[:4], flush=True)
