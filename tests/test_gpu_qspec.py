"""GPU parity of the speculative-acceptance chain blocks (qspec, csrc/common.cuh) against the
oracle, through every quantiser that uses them: K2a (thread per plane), K2b phase A and
its exact stretches, and the exact replay. A block is redone step by step when any of its
steps escapes, is rejected or has a fragile quotient; these cases put such steps at every
position of a block, at plane starts inside replay blocks, and at the window edges of the
bulk-copied K2b segment (misaligned views, tensor ends that are not 16-byte aligned)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def acz(gpu_lib):
    import torch
    assert torch.cuda.is_available()
    import paper_2011_09017_b200 as acz
    return acz


def _check(acz, oracle, x, eb, radius=32768, t=None):
    import torch
    x = np.ascontiguousarray(x, dtype=np.float32)
    ref = oracle.compress(x, eb, radius)
    if t is None:
        t = torch.from_numpy(x).cuda()
    c = acz.compress(t, acz.CodecParams(eb, radius))
    assert c.to_bytes() == ref.blob
    d = acz.decompress(c, zero_filter=True)
    torch.cuda.synchronize()
    assert d.cpu().numpy().ravel().tobytes() == oracle.decompress(ref.blob, x.size, True).tobytes()


@pytest.fixture(params=["serial", "spec"])
def quantiser(request, monkeypatch):
    monkeypatch.setenv("ACZ_SERIAL_QUANT" if request.param == "serial" else "ACZ_SPEC_QUANT", "1")
    return request.param


def _escapes_at_every_offset(rng, planes, plane):
    x = np.maximum(rng.standard_normal((planes, plane)), 0).astype(np.float32)
    for k in range(16):  # one escape at every position modulo 8 (and 16), per plane
        x[:, (37 + 131 * k) % plane + 0] = 500.0 + k
    return x


@pytest.mark.parametrize("plane", [1031, 4096, 9001])
def test_escapes_in_every_block_position(acz, oracle, quantiser, plane):
    rng = np.random.default_rng(plane)
    x = _escapes_at_every_offset(rng, 64, plane)
    _check(acz, oracle, x, 1e-3, radius=256)  # |q| >= 256 escapes


@pytest.mark.parametrize("plane", [1031, 5003])
def test_exact_ties_and_lattice_values(acz, oracle, quantiser, plane):
    # values on (and half a step off) the quantisation lattice of the plane-start chain:
    # quotients exactly at half-integers are fragile and must take the exact division
    eb = 2.0 ** -10
    step = 2 * eb
    rng = np.random.default_rng(7)
    k = rng.integers(-200, 200, size=(32, plane))
    half = rng.random((32, plane)) < 0.3
    x = (k * step + np.where(half, step / 2, 0.0)).astype(np.float32)
    _check(acz, oracle, x, eb)


@pytest.mark.parametrize("eb", [1e-6, 3e-8])
def test_rejections_near_the_float_grid(acz, oracle, quantiser, eb):
    # eb below half an ulp of large values: candidates are rejected (|x - c| > eb) and
    # the chain takes x itself
    rng = np.random.default_rng(11)
    x = (rng.standard_normal((16, 3001)) * 300.0).astype(np.float32)
    _check(acz, oracle, x, eb)


def test_plane_starts_inside_replay_blocks(acz, oracle, monkeypatch):
    # plane sizes that put plane starts at every offset of the replay's 8-step blocks and
    # 128-element chunks (K2b forced)
    monkeypatch.setenv("ACZ_SPEC_QUANT", "1")
    rng = np.random.default_rng(3)
    for plane in (1025, 1029, 1100, 2047, 2053):
        x = rng.standard_normal((7, plane)).astype(np.float32)
        _check(acz, oracle, x, 1e-3)


def test_misaligned_view_and_unaligned_tensor_end(acz, oracle, monkeypatch):
    # K2b stages each segment window by one bulk copy of the 16-byte aligned span around
    # it: a view starting 1..3 floats past an aligned address and a tensor end that is not
    # 16-byte aligned (the last segment takes the per-lane fallback)
    import torch
    monkeypatch.setenv("ACZ_SPEC_QUANT", "1")
    rng = np.random.default_rng(5)
    n_planes, plane = 5, 6007
    big = rng.standard_normal(n_planes * plane + 8).astype(np.float32)
    gbig = torch.from_numpy(big).cuda()
    for off in (1, 2, 3):
        x = big[off:off + n_planes * plane].reshape(n_planes, plane)
        t = gbig[off:off + n_planes * plane].view(n_planes, plane)
        assert t.data_ptr() % 16 == 4 * off
        _check(acz, oracle, x, 1e-3, t=t)


def test_non_finite_input_is_a_domain_error(acz, quantiser):
    import torch
    for bad in (np.nan, np.inf, -np.inf):
        x = np.maximum(np.random.default_rng(1).standard_normal((8, 2000)), 0).astype(np.float32)
        x[3, 1234] = bad
        with pytest.raises(acz.DomainError):
            acz.compress(torch.from_numpy(x).cuda(), acz.CodecParams(1e-3))
