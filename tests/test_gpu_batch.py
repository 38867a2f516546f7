"""GPU parity of the batched entry points (acz_gpu_compress_batch / decompress_batch): every
tensor of an activation set compresses to the same ACZ1 bytes as the oracle and as the
single-tensor call, decompresses bit-exactly, and a failing tensor only fails itself (the
reference controller degrades that layer to pass-through, src/controller.cpp:216-220)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def acz(gpu_lib):
    import torch
    assert torch.cuda.is_available()
    import paper_2011_09017_b200 as acz
    return acz


def _set(rng):
    shapes = [((2, 3, 227, 227), False), ((8, 96, 27, 27), True), ((8, 64, 56, 56), True),
              ((16, 256, 13, 13), True), ((4, 7, 5), True), ((1000,), False)]
    out = []
    for shp, relu in shapes:
        x = rng.standard_normal(shp).astype(np.float32)
        out.append(np.maximum(x, 0) if relu else x)
    return out


def test_batch_matches_oracle_and_single(acz, oracle):
    import torch
    rng = np.random.default_rng(11)
    xs = _set(rng)
    ts = [torch.from_numpy(x).cuda() for x in xs]
    p = acz.CodecParams(1e-3)
    blobs = acz.compress_many(ts, p)
    outs = acz.decompress_many(blobs, zero_filter=True)
    torch.cuda.synchronize()
    for x, t, c, o in zip(xs, ts, blobs, outs):
        ref = oracle.compress(x, 1e-3)
        assert c.to_bytes() == ref.blob
        assert acz.compress(t, p).to_bytes() == ref.blob
        assert o.cpu().numpy().ravel().tobytes() == oracle.decompress(ref.blob, x.size, True).tobytes()


def test_batch_error_isolated(acz, oracle):
    import torch
    rng = np.random.default_rng(12)
    xs = _set(rng)[:4]
    xs[1] = xs[1].copy()
    xs[1].flat[123] = np.nan
    ts = [torch.from_numpy(x).cuda() for x in xs]
    blobs = acz.compress_many(ts, acz.CodecParams(1e-3), errors="none")
    assert blobs[1] is None
    for i in (0, 2, 3):
        assert blobs[i].to_bytes() == oracle.compress(xs[i], 1e-3).blob
    with pytest.raises(acz.DomainError):
        acz.compress_many(ts, acz.CodecParams(1e-3))


def test_batch_repeat_deterministic(acz):
    import torch
    rng = np.random.default_rng(13)
    ts = [torch.from_numpy(x).cuda() for x in _set(rng)]
    a = [c.to_bytes() for c in acz.compress_many(ts, acz.CodecParams(3e-4))]
    b = [c.to_bytes() for c in acz.compress_many(list(reversed(ts)), acz.CodecParams(3e-4))]
    assert a == list(reversed(b))


def test_host_batch_roundtrip(acz, oracle):
    import torch
    rng = np.random.default_rng(14)
    xs = _set(rng)[:5]
    hin = [torch.from_numpy(x).pin_memory() for x in xs]
    res = acz.compress_host_many(hin, acz.CodecParams(1e-3))
    for x, (b, s) in zip(xs, res):
        assert b.tobytes() == oracle.compress(x, 1e-3).blob
    outs = acz.decompress_host_many(res, zero_filter=True)
    for x, (b, _), o in zip(xs, res, outs):
        assert o.numpy().ravel().tobytes() == oracle.decompress(b.tobytes(), x.size, True).tobytes()
    # without sidecars: the sidecar is rebuilt on the GPU from the ACZ1 bytes alone
    outs2 = acz.decompress_host_many([(b, None) for b, _ in res], zero_filter=True)
    for o, o2 in zip(outs, outs2):
        assert torch.equal(o, o2)


def test_host_batch_decompress_errors(acz, oracle):
    import torch
    rng = np.random.default_rng(15)
    xs = _set(rng)[:3]
    res = acz.compress_host_many([torch.from_numpy(x).pin_memory() for x in xs], acz.CodecParams(1e-3))
    # a blob with trailing bytes among valid ones: the reference's FormatError, same message
    bad = np.concatenate([res[1][0], np.zeros(3, np.uint8)])
    outs = [torch.empty(x.shape, dtype=torch.float32).pin_memory() for x in xs]
    with pytest.raises(acz.FormatError, match="trailing bytes after blob"):
        acz.decompress_host_many([res[0], (bad, None), res[2]], True, outs=outs)
    # the valid blobs of that batch were still decoded
    assert outs[0].numpy().ravel().tobytes() == oracle.decompress(res[0][0].tobytes(), xs[0].size, True).tobytes()
    assert outs[2].numpy().ravel().tobytes() == oracle.decompress(res[2][0].tobytes(), xs[2].size, True).tobytes()
    with pytest.raises(acz.FormatError):
        acz.decompress_host_many([(np.frombuffer(b"ACZX0000000", np.uint8), None)], True)
    # output buffer too small
    with pytest.raises(acz.ShapeError, match="output buffer too small"):
        acz.decompress_host_many([res[0]], True, outs=[torch.empty(3).pin_memory()])


@pytest.mark.parametrize("order", ["grow", "shrink"])
def test_batch_speculative_encode_sizes(acz, oracle, order, monkeypatch):
    """A repeated batched compress launches each tensor's encode before the host has read its
    codebook back, into a blob sized from the previous call of the same shapes. A book that
    outgrows that blob (far more bits / outliers / symbols than last time: "grow") is
    re-encoded exactly; one that shrinks keeps the speculative blob. Either way the bytes are
    the oracle's, the sizes reported are exact, and the blob decompresses bit-exactly."""
    import torch
    monkeypatch.setenv("ACZ_SPEC_ENCODE", "1")
    rng = np.random.default_rng(5)
    shapes = [(4, 3, 97, 131), (16, 32, 27, 27), (3001,)]
    calm = [np.maximum(rng.standard_normal(s), 0).astype(np.float32) * 1e-3 for s in shapes]
    wild = [(rng.standard_normal(s) * np.exp(rng.standard_normal(s) * 2)).astype(np.float32)
            for s in shapes]
    first, second = (calm, wild) if order == "grow" else (wild, calm)
    p = acz.CodecParams(1e-3, 64)  # small radius: the wild data escapes a lot
    for xs in (first, second, second):
        ts = [torch.from_numpy(x).cuda() for x in xs]
        blobs = acz.compress_many(ts, p)
        outs = acz.decompress_many(blobs, zero_filter=True)
        torch.cuda.synchronize()
        for x, c, o in zip(xs, blobs, outs):
            ref = oracle.compress(x, 1e-3, 64)
            assert c.to_bytes() == ref.blob
            assert c.compressed_bytes == len(ref.blob)
            assert o.cpu().numpy().ravel().tobytes() == oracle.decompress(ref.blob, x.size, True).tobytes()
