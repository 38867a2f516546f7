"""Round-trip parity of saved fuzz failures with the package at PKG_ROOT (development)."""
import glob, os, sys
root = os.environ.get("PKG_ROOT")
repo = __file__.rsplit("/tools/", 1)[0]
sys.path.insert(0, repo)
if root:
    sys.path.insert(0, root)
import numpy as np
import torch
import paper_2011_09017_b200 as acz
from oracle.oracle import Oracle
print("package", acz.__file__)
O = Oracle()
for f in sorted(glob.glob(os.path.join(repo, "tools/fuzz_cases/fail_*.npz"))):
    z = np.load(f)
    x = z["x"]; eb = float(z["eb"]); radius = int(z["radius"]); mode = str(z["mode"])
    os.environ.pop("ACZ_SPEC_QUANT", None)
    if mode == "spec":
        os.environ["ACZ_SPEC_QUANT"] = "1"
    ref = O.compress(x, eb, radius, 0, shape=x.shape)
    c = acz.compress(torch.from_numpy(x).cuda(), acz.CodecParams(eb, radius))
    ok_blob = c.to_bytes() == ref.blob
    d = acz.decompress(c, zero_filter=False); torch.cuda.synchronize()
    ok_dec = d.cpu().numpy().ravel().tobytes() == O.decompress(ref.blob, x.size, False).tobytes()
    print(os.path.basename(f), "blob", ok_blob, "decode", ok_dec, flush=True)
