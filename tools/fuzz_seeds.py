"""Which seeds of tests/test_gpu_fuzz.py's generator fail with the package at PKG_ROOT?"""
import os, sys
root = os.environ.get("PKG_ROOT")
repo = __file__.rsplit("/tools/", 1)[0]
sys.path.insert(0, repo)
if root:
    sys.path.insert(0, root)
sys.path.insert(0, os.path.join(repo, "tests"))
import numpy as np
import torch
import paper_2011_09017_b200 as acz
from oracle.oracle import Oracle
from test_gpu_fuzz import _case
os.environ["ACZ_SPEC_QUANT"] = "1"
O = Oracle()
bad = []
for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 40):
    rng = np.random.default_rng(1000 + seed)
    for i in range(8):
        kind = str(rng.choice(["dense", "tiny", "grid", "smooth", "relu", "spikes"]))
        shape = [(64, 40), (64, 300), (4, 1, 12769), (2, 113, 113), (3, 1, 5000), (2, 1, 20000)][int(rng.integers(0, 6))]
        x = _case(rng, kind, shape)
        eb = float(10 ** rng.uniform(-5, -1)); radius = int(2 ** rng.integers(3, 20))
        try:
            ref = O.compress(x, eb, radius, shape=x.shape)
        except Exception:
            continue
        c = acz.compress(torch.from_numpy(x).cuda(), acz.CodecParams(eb, radius))
        ok = c.to_bytes() == ref.blob
        d = acz.decompress(c, zero_filter=False); torch.cuda.synchronize()
        ok = ok and d.cpu().numpy().ravel().tobytes() == O.decompress(ref.blob, x.size, False).tobytes()
        if not ok:
            bad.append((seed, i, kind, shape))
print("failing:", bad)
