"""Randomised bit-exactness of the speculative quantiser (forced) across error bounds,
radii and value regimes that stress its certified walk (near-zero residual chains, lattice
data, escapes): ACZ1 bytes and both decompressions against the oracle. These regimes found
chains left an ulp off by the walk before the exact replay existed (tools/fuzz_codec.py)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def force_spec():
    import os
    os.environ["ACZ_SPEC_QUANT"] = "1"
    yield
    del os.environ["ACZ_SPEC_QUANT"]


def _case(rng, kind, shape):
    x = rng.standard_normal(shape)
    if kind == "tiny":
        x = x * 1e-4
    elif kind == "grid":
        x = rng.integers(-500, 500, shape) * 2e-3 + rng.choice([0, 0.5e-3, 1e-3], shape)
    elif kind == "smooth":
        x = np.cumsum(x, axis=-1) * 0.05
    elif kind == "relu":
        x = np.maximum(x, 0)
    elif kind == "spikes":
        x = np.where(rng.random(shape) < 0.02, x * 50, 0.0)
    return x.astype(np.float32)


# every seed below produced a wrong ACZ1 blob or decompression before the exact replay
# (found with tools/fuzz_seeds.py against the earlier build)
@pytest.mark.parametrize("seed", [0, 8, 9, 13, 16, 21, 27, 31, 40, 45, 47])
def test_spec_fuzz(gpu_lib, oracle, seed):
    import torch
    import paper_2011_09017_b200 as acz
    rng = np.random.default_rng(1000 + seed)
    for _ in range(8):
        kind = str(rng.choice(["dense", "tiny", "grid", "smooth", "relu", "spikes"]))
        shape = [(64, 40), (64, 300), (4, 1, 12769), (2, 113, 113), (3, 1, 5000), (2, 1, 20000)][
            int(rng.integers(0, 6))]
        x = _case(rng, kind, shape)
        eb = float(10 ** rng.uniform(-5, -1))
        radius = int(2 ** rng.integers(3, 20))
        try:
            ref = oracle.compress(x, eb, radius, shape=x.shape)
        except Exception:  # noqa: BLE001  (reference-side rejection: error parity tested elsewhere)
            continue
        c = acz.compress(torch.from_numpy(x).cuda(), acz.CodecParams(eb, radius))
        assert c.to_bytes() == ref.blob, (kind, shape, eb, radius)
        for zf in (False, True):
            d = acz.decompress(c, zero_filter=zf)
            torch.cuda.synchronize()
            exp = oracle.decompress(ref.blob, x.size, zf)
            assert d.cpu().numpy().ravel().tobytes() == exp.tobytes(), (kind, shape, eb, radius, zf)
