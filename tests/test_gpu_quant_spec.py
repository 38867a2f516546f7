"""GPU parity of the speculative long-plane quantiser (quant_spec.cu, planes > 1024
elements) against the oracle: every symbol, the outlier list and the decode sidecar
states (checked through decompression) must be bit-exact, on data built to stress the
walk: dense and ReLU planes, smooth fields, escapes (small radius / near-ties / huge
values), lattice shifts, zero and constant planes, tight and loose error bounds."""
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def force_spec():
    # these cases exercise the speculative kernel itself, whatever the cost model would pick
    import os
    os.environ["ACZ_SPEC_QUANT"] = "1"
    yield
    del os.environ["ACZ_SPEC_QUANT"]


@pytest.fixture(scope="module")
def acz(gpu_lib):
    import torch
    assert torch.cuda.is_available()
    import paper_2011_09017_b200 as acz
    return acz


def _run(acz, oracle, x, eb, radius=32768):
    import torch
    x = np.ascontiguousarray(x, dtype=np.float32)
    ref = oracle.compress(x, eb, radius)
    c = acz.compress(torch.from_numpy(x).cuda(), acz.CodecParams(eb, radius))
    syms = acz.debug_last_symbols(x.size).cpu().numpy().view(np.uint32)
    bad = np.nonzero(syms != ref.symbols)[0]
    assert bad.size == 0, f"{bad.size} symbol mismatches, first at {bad[:5]}"
    assert c.to_bytes() == ref.blob
    d = acz.decompress(c, zero_filter=False)
    torch.cuda.synchronize()
    assert d.cpu().numpy().ravel().tobytes() == oracle.decompress(ref.blob, x.size).tobytes()


def _smooth(rng, shape, scale=3.0):
    y = rng.standard_normal(shape)
    for ax in (-1, -2):
        y = np.cumsum(y, axis=ax) * 0.05
    return scale * y


CASES = ["dense_227", "relu_227", "smooth_relu_224", "relu_3136", "dense_3136",
         "eb1e-4", "eb3e-4", "eb1e-2", "eb3e-2", "radius4", "radius64", "wide_x100",
         "tiny_x1e-3", "zeros_plane", "const_plane", "sparse_spikes", "huge_outliers",
         "rank1_long", "neg_relu", "mixed_scale", "near_eb_values", "quantized_grid",
         "tiny_runs"]


@pytest.mark.parametrize("case", CASES)
def test_quant_spec_cases(acz, oracle, case):
    rng = np.random.default_rng(zlib.crc32(case.encode()))
    eb, radius = 1e-3, 32768
    if case == "dense_227":
        x = rng.standard_normal((2, 3, 227, 227))
    elif case == "relu_227":
        x = np.maximum(rng.standard_normal((2, 3, 227, 227)), 0)
    elif case == "smooth_relu_224":
        x = np.maximum(_smooth(rng, (1, 4, 224, 224)), 0)
    elif case == "relu_3136":
        x = np.maximum(rng.standard_normal((4, 16, 56, 56)), 0)
    elif case == "dense_3136":
        x = rng.standard_normal((4, 16, 56, 56))
    elif case.startswith("eb"):
        eb = float(case[2:])
        x = np.maximum(rng.standard_normal((2, 4, 112, 112)), 0)
    elif case == "radius4":
        x, radius = rng.standard_normal((2, 2, 100, 100)), 4
    elif case == "radius64":
        x, radius = rng.standard_normal((2, 2, 100, 100)) * 0.5, 64
    elif case == "wide_x100":
        x = rng.standard_normal((2, 2, 90, 90)) * 100
    elif case == "tiny_x1e-3":
        x = rng.standard_normal((2, 2, 90, 90)) * 1e-3
    elif case == "zeros_plane":
        x = np.zeros((3, 2, 64, 64))
        x[1, 1] = rng.standard_normal((64, 64))
    elif case == "const_plane":
        x = np.full((2, 2, 64, 64), 1.2345)
        x[0, 1] = -0.37
    elif case == "sparse_spikes":
        x = np.zeros((2, 2, 150, 150))
        m = rng.random(x.shape) < 0.01
        x[m] = rng.standard_normal(m.sum()) * 5
    elif case == "huge_outliers":
        x = rng.standard_normal((2, 2, 120, 120))
        m = rng.random(x.shape) < 0.002
        x[m] = rng.standard_normal(m.sum()) * 1e6
    elif case == "rank1_long":
        x = np.maximum(rng.standard_normal(200_003), 0)
    elif case == "neg_relu":
        x = -np.maximum(rng.standard_normal((2, 3, 100, 100)), 0)
    elif case == "mixed_scale":
        x = rng.standard_normal((2, 2, 128, 128)) * np.exp(rng.standard_normal((2, 2, 128, 128)) * 2)
    elif case == "near_eb_values":
        x = np.where(rng.random((2, 2, 128, 128)) < 0.5, 0.0,
                     (rng.integers(-3, 4, (2, 2, 128, 128)) * 2e-3 + 1e-3) *
                     (1 + 1e-7 * rng.standard_normal((2, 2, 128, 128))))
    elif case == "quantized_grid":
        # values exactly on the quantisation lattice and on round binary fractions (ties)
        x = rng.integers(-2000, 2000, (2, 2, 128, 128)) * 2e-3 + rng.choice([0, 0.25, 0.5], (2, 2, 128, 128))
    elif case == "tiny_runs":
        # long runs of sub-eb values (collapsed chain) re-expanding into normal values
        n = 4 * 60_000
        x = np.empty(n)
        pos = 0
        while pos < n:
            L = int(rng.integers(1, 400))
            if rng.random() < 0.5:
                x[pos:pos + L] = rng.uniform(-9e-4, 9e-4, min(L, n - pos))
            else:
                x[pos:pos + L] = rng.standard_normal(min(L, n - pos)) * 0.3
            pos += L
        x = x.reshape(4, 1, 60_000)
    _run(acz, oracle, x, eb, radius)


def test_quant_spec_random_fuzz(acz, oracle):
    rng = np.random.default_rng(1234)
    for t in range(12):
        P = int(rng.choice([1031, 2049, 3136, 5000, 12769]))
        planes = int(rng.integers(1, 4))
        kind = t % 4
        x = rng.standard_normal((planes, P)) * float(rng.choice([0.1, 1, 4]))
        if kind == 1:
            x = np.maximum(x, 0)
        elif kind == 2:
            x = np.maximum(np.cumsum(x, axis=1) * 0.1, 0)
        elif kind == 3:
            x[rng.random(x.shape) < 0.3] = 0
        eb = float(rng.choice([1e-4, 5e-4, 1e-3, 2e-3, 1e-2]))
        _run(acz, oracle, x.reshape(planes, 1, P), eb)


@pytest.mark.parametrize("case", ["dense_227", "relu_227", "eb1e-4", "radius4", "huge_outliers"])
def test_quant_spec_decoupled_path(acz, oracle, case, monkeypatch):
    """The decoupled phase-A / walk kernel pair (opt-in) is bit-identical to the oracle."""
    monkeypatch.setenv("ACZ_SPEC_DECOUPLED", "1")
    test_quant_spec_cases(acz, oracle, case)


@pytest.mark.parametrize("eb", [0.05, 0.1, 0.3, 1.0])
@pytest.mark.parametrize("kind", ["dense", "relu"])
def test_quant_spec_large_error_bounds(acz, oracle, eb, kind):
    """Large error bounds (the controller clamps eb to [eb_min, eb_max] = [.., 0.1]) leave
    thousands of wrong walk states per tensor: the chunk-parallel repair rounds and the
    serial plane replay after them must give the reference's symbols exactly."""
    rng = np.random.default_rng(int(eb * 1000) + (kind == "relu"))
    x = rng.standard_normal((6, 3, 224, 224))
    if kind == "relu":
        x = np.maximum(x, 0)
    _run(acz, oracle, x, eb)
