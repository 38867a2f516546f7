"""Randomised bit-exactness fuzz of the whole codec (both PrevValue quantisers, Lorenzo2d,
batched and host-buffer paths, foreign blobs) against the oracle (development tool).
usage: python tools/fuzz_codec.py [seconds] [seed]"""
import os, sys, time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np
import torch
import paper_2011_09017_b200 as acz
from oracle.oracle import Oracle

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(seed)
O = Oracle()
t_end = time.time() + budget
cases = fails = 0
while time.time() < t_end:
    kind = rng.choice(["dense", "relu", "smooth", "spikes", "tiny", "wide", "grid"])
    P = int(rng.choice([40, 300, 1025, 2049, 5000, 12769, 50176, 70000]))
    planes = int(max(1, min(64, 600_000 // P)))
    shape = (planes, P) if P < 1000 or rng.random() < 0.5 else (planes, 1, P)
    if rng.random() < 0.3 and P in (12769, 50176):
        side = int(round(P ** 0.5))
        shape = (planes, side, side)
    x = rng.standard_normal(shape)
    if kind == "relu":
        x = np.maximum(x, 0)
    elif kind == "smooth":
        x = np.cumsum(x, axis=-1) * 0.05
    elif kind == "spikes":
        x = np.where(rng.random(shape) < 0.02, x * 50, 0.0)
    elif kind == "tiny":
        x = x * 1e-4
    elif kind == "wide":
        x = x * np.exp(rng.standard_normal(shape) * 3)
    elif kind == "grid":
        x = rng.integers(-500, 500, shape) * 2e-3 + rng.choice([0, 0.5e-3, 1e-3], shape)
    x = x.astype(np.float32)
    eb = float(10 ** rng.uniform(-5, -1))
    radius = int(2 ** rng.integers(3, 20))
    pred = int(rng.random() < 0.2)
    mode = rng.choice(["auto", "spec", "serial"]) if pred == 0 else "auto"
    os.environ.pop("ACZ_SPEC_QUANT", None)
    os.environ.pop("ACZ_SERIAL_QUANT", None)
    if mode == "spec":
        os.environ["ACZ_SPEC_QUANT"] = "1"
    elif mode == "serial":
        os.environ["ACZ_SERIAL_QUANT"] = "1"
    cases += 1
    try:
        ref = O.compress(x, eb, radius, pred, shape=x.shape)
    except Exception as e:  # noqa: BLE001
        continue  # the reference rejects it (e.g. codebook limit); error parity is tested elsewhere
    p = acz.CodecParams(eb, radius, acz.Predictor(pred))
    t = torch.from_numpy(x).cuda()
    try:
        c = acz.compress_many([t], p)[0] if rng.random() < 0.5 else acz.compress(t, p)
        ok = c.to_bytes() == ref.blob
        zf = bool(rng.random() < 0.5)
        exp = O.decompress(ref.blob, x.size, zf).tobytes()
        d = acz.decompress(c, zero_filter=zf)
        torch.cuda.synchronize()
        ok = ok and d.cpu().numpy().ravel().tobytes() == exp
        if rng.random() < 0.2:  # foreign blob (no sidecar)
            fb = acz.blob_from_bytes(ref.blob)
            d2 = acz.decompress(fb, zero_filter=zf)
            torch.cuda.synchronize()
            ok = ok and d2.cpu().numpy().ravel().tobytes() == exp
    except Exception as e:  # noqa: BLE001
        ok = False
        print("exception", e)
    if not ok:
        fails += 1
        print(f"MISMATCH kind={kind} shape={shape} eb={eb:.3g} radius={radius} pred={pred} mode={mode}", flush=True)
        if fails <= 8:
            os.makedirs("gpurun_out", exist_ok=True)
            # first mismatching quantisation symbol (single-tensor compress, same env)
            acz.compress(t, p)
            syms = acz.debug_last_symbols(x.size).cpu().numpy().view(np.uint32)
            bad = np.nonzero(syms != ref.symbols)[0]
            first = int(bad[0]) if bad.size else -1
            print(f"   symbol mismatches {bad.size}, first at {first}", flush=True)
            np.savez_compressed(f"gpurun_out/fail_{seed}_{fails}.npz", x=x, eb=eb, radius=radius,
                                pred=pred, mode=str(mode), first=first, nbad=bad.size)
import ctypes as C
from paper_2011_09017_b200 import _native
v = (C.c_uint64 * 32)()
_native.load().acz_gpu_debug_counters(acz.default_context().handle, v, 32, 0)
print(f"fuzz: {cases} cases, {fails} mismatches; K2b replay rewrites {v[31]}")
sys.exit(1 if fails else 0)
