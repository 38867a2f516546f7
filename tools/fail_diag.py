"""Which artefact differs for saved fuzz failures (gpurun_out/fail_*.npz)? (development)"""
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
    os.environ.pop("ACZ_SPEC_QUANT", None); os.environ.pop("ACZ_SERIAL_QUANT", None)
    if mode == "spec":
        os.environ["ACZ_SPEC_QUANT"] = "1"
    ref = O.compress(x, eb, radius, 0, shape=x.shape)
    t = torch.from_numpy(x).cuda()
    out = []
    for api in ("single", "batch"):
        c = acz.compress(t, acz.CodecParams(eb, radius)) if api == "single" else \
            acz.compress_many([t], acz.CodecParams(eb, radius))[0]
        if api == "single":
            syms = acz.debug_last_symbols(x.size).cpu().numpy().view(np.uint32)
            out.append("syms_bad=%d" % int((syms != ref.symbols).sum()))
        b = c.to_bytes()
        p = acz.parse_acz1(b)
        r = acz.parse_acz1(ref.blob)
        flags = []
        if not np.array_equal(p["book_sym"], r["book_sym"]): flags.append("book_sym")
        if not np.array_equal(p["book_len"], r["book_len"]): flags.append("book_len")
        if p["bit_length"] != r["bit_length"]: flags.append("bit_length %d vs %d" % (p["bit_length"], r["bit_length"]))
        if p["bits"] != r["bits"]:
            a = np.frombuffer(p["bits"], np.uint8); bb = np.frombuffer(r["bits"], np.uint8)
            m = min(a.size, bb.size); d = np.nonzero(a[:m] != bb[:m])[0]
            flags.append("bits first diff byte %s of %d" % (d[0] if d.size else "len", m))
        if not np.array_equal(p["out_index"], r["out_index"]): flags.append("outliers")
        for zf in (False, True):
            d = acz.decompress(c, zero_filter=zf); torch.cuda.synchronize()
            exp = O.decompress(ref.blob, x.size, zf)
            got = d.cpu().numpy().ravel()
            bad = np.nonzero(got.view(np.uint32) != exp.view(np.uint32))[0]
            if bad.size: flags.append("dec zf=%d bad %d first %d" % (zf, bad.size, bad[0]))
        out.append(api + ":" + (",".join(flags) or "ok"))
    print(os.path.basename(f), x.shape, "eb %.3g R %d %s" % (eb, radius, mode), " | ".join(out), flush=True)
