"""GPU parity tests (-m gpu): the sm_100a path through the C-ABI against the oracle.

Bit-exact gates: quantisation symbols, outlier list, canonical codebook,
bit length, bitstream bytes, ACZ1 bytes, decompressed fp32 (filter off and on), zero
bitmap and nonzero count. Full-size cases use size-independent properties (error bound,
round trip, exact zero restoration) plus bit-exact comparison where the oracle is fast.
"""
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def acz(gpu_lib):
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2011_09017_b200 as acz
    return acz


def _gpu(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def _check_all(acz, oracle, x, eb, radius=32768, pred=0, shape=None):
    """Compress on the GPU, compare every artefact with the oracle, round-trip both ways."""
    import torch
    x = np.ascontiguousarray(x, dtype=np.float32)
    shp = tuple(x.shape) if shape is None else tuple(shape)
    ref = oracle.compress(x, eb, radius, pred, shape=shp)
    t = _gpu(x.reshape(shp))
    c = acz.compress(t, acz.CodecParams(eb, radius, acz.Predictor(pred)))
    syms = acz.debug_last_symbols(x.size).cpu().numpy().view(np.uint32)
    assert np.array_equal(syms, ref.symbols), "quantisation symbols"
    assert c.outlier_count == len(ref.out_index)
    assert c.codebook_size == len(ref.book_sym)
    assert c.bit_length == ref.bit_length
    blob = c.to_bytes()
    p = acz.parse_acz1(blob)
    assert np.array_equal(p["book_sym"], ref.book_sym), "codebook symbols"
    assert np.array_equal(p["book_len"], ref.book_len), "codebook lengths"
    assert np.array_equal(p["out_index"], ref.out_index), "outlier indices"
    assert p["out_value"].tobytes() == ref.out_value.tobytes(), "outlier values"
    assert p["bits"] == bytes(ref.bits), "bitstream"
    assert blob == ref.blob, "ACZ1 bytes"
    assert c.compressed_bytes == len(ref.blob)
    for zf in (False, True):
        d = acz.decompress(c, zero_filter=zf)
        torch.cuda.synchronize()
        exp = oracle.decompress(ref.blob, x.size, zf)
        assert d.cpu().numpy().ravel().tobytes() == exp.tobytes(), f"decompress zf={zf}"
    return c, ref


def test_kats(acz, oracle, kat):
    for k in kat["codec"]:
        x = np.asarray(k["data"], dtype=np.float32)
        c, ref = _check_all(acz, oracle, x, k["eb"], k["radius"], k["predictor"], k["shape"])
        assert c.to_bytes().hex() == k["blob"], k["name"]


def test_golden_fixtures(acz, oracle, fixtures):
    import torch
    for f in fixtures:
        c, ref = _check_all(acz, oracle, f["x"], f["eb"], f["radius"], f["predictor"])
        assert c.to_bytes() == f["blob"], f["name"]
        # foreign (reference-produced) blob decoded on the GPU without a sidecar
        fb = acz.blob_from_bytes(f["blob"])
        for zf, key in ((False, "dec0"), (True, "dec1")):
            d = acz.decompress(fb, zero_filter=zf)
            torch.cuda.synchronize()
            assert d.cpu().numpy().ravel().tobytes() == f[key].tobytes(), f["name"]


def test_huffman_kats(acz, kat):
    import torch
    for k in kat["huffman"]:
        s = torch.tensor(k["symbols"], dtype=torch.int32, device="cuda")
        h = acz.huffman_encode(s)
        assert [e.symbol for e in h.codebook] == k["book_sym"]
        assert [e.length for e in h.codebook] == k["book_len"]
        assert h.bit_length == k["bit_length"]
        assert h.bits.hex() == k["bits"]
        back = acz.huffman_decode(h.codebook, h.bits, h.bit_length, len(k["symbols"]))
        assert back.cpu().tolist() == k["symbols"]


def test_huffman_random_vs_oracle(acz, oracle):
    import torch
    rng = np.random.default_rng(5)
    for t in range(20):
        n = int(rng.integers(1, 5000))
        syms = rng.geometric(float(rng.choice([0.05, 0.3, 0.9])), size=n).astype(np.uint32)
        syms *= np.uint32(rng.integers(1, 50))
        bsym, blen, bits, bl = oracle.huffman_encode(syms)
        h = acz.huffman_encode(torch.from_numpy(syms.view(np.int32)).cuda())
        assert [e.symbol for e in h.codebook] == bsym.tolist()
        assert [e.length for e in h.codebook] == blen.tolist()
        assert h.bits == bytes(bits) and h.bit_length == bl
        back = acz.huffman_decode(h.codebook, h.bits, h.bit_length, n)
        assert np.array_equal(back.cpu().numpy().view(np.uint32), syms)


@pytest.mark.parametrize("case", ["relu", "smooth", "normal", "zeros", "const", "tiny_planes",
                                  "rank1", "rank3", "rank5", "one_elem", "radius2", "big",
                                  "eb_tiny", "eb_big", "neg_zero", "lorenzo", "lorenzo_rank1"])
def test_edge_cases(acz, oracle, case):
    rng = np.random.default_rng(zlib.crc32(case.encode()))
    eb, radius, pred = 1e-3, 32768, 0
    if case == "relu":
        x = np.maximum(rng.standard_normal((3, 7, 33, 29)), 0)
    elif case == "smooth":
        x = np.cumsum(np.cumsum(rng.standard_normal((2, 2, 64, 64)) * 0.01, axis=2), axis=3)
    elif case == "normal":
        x = rng.standard_normal((4, 3, 25, 25))
    elif case == "zeros":
        x = np.zeros((5, 4, 9, 9))
    elif case == "const":
        x = np.full((3, 40, 40), 1.2345)
    elif case == "tiny_planes":
        x = rng.standard_normal((64, 33, 1, 1))
    elif case == "rank1":
        x = rng.standard_normal(7777)
    elif case == "rank3":
        x = rng.standard_normal((5, 17, 23))
    elif case == "rank5":
        x = np.maximum(rng.standard_normal((2, 3, 2, 11, 13)), 0)
    elif case == "one_elem":
        x = np.array([0.37])
    elif case == "radius2":
        x, eb, radius = rng.standard_normal((9, 31)), 0.1, 2
    elif case == "big":
        x = np.concatenate([rng.standard_normal(500), [3e38, -3e38, 1e30, -1e-30, 5e-39]])
    elif case == "eb_tiny":
        x, eb, radius = rng.standard_normal((6, 70)) * 1e3, 1e-6, 1 << 24
    elif case == "eb_big":
        x, eb = rng.standard_normal((4, 50, 50)), 10.0
    elif case == "neg_zero":
        x = np.where(rng.random((4, 30, 30)) < 0.5, -0.0, rng.standard_normal((4, 30, 30)))
    elif case == "lorenzo":
        x, pred = np.maximum(rng.standard_normal((3, 4, 21, 19)), 0), 1
    elif case == "lorenzo_rank1":
        x, pred = rng.standard_normal(999), 1
    _check_all(acz, oracle, x, eb, radius, pred)


def test_random_sweep(acz, oracle):
    rng = np.random.default_rng(99)
    for t in range(25):
        rank = int(rng.integers(1, 5))
        shp = tuple(int(v) for v in rng.integers(1, 40, size=rank))
        x = rng.standard_normal(shp) * float(rng.choice([1e-3, 1, 100]))
        if t % 2:
            x = np.maximum(x, 0)
        eb = float(rng.choice([1e-5, 1e-4, 1e-3, 1e-2, 1e-1]))
        radius = int(rng.choice([4, 512, 32768]))
        _check_all(acz, oracle, x, eb, radius, int(rng.integers(0, 2)))


def test_config1_full_bitexact(acz, oracle):
    """SURVEY config 1: [64,64,56,56] ReLU(N(0,1)), eb=1e-3 -- every artefact bit-exact."""
    rng = np.random.default_rng(20201118)
    x = np.maximum(rng.standard_normal((64, 64, 56, 56)), 0).astype(np.float32)
    c, ref = _check_all(acz, oracle, x, 1e-3)
    assert 3.4 < acz.compression_ratio(c) < 3.7


def test_alexnet_set_properties(acz, oracle):
    """configs[1] (AlexNet B256 saved-activation set): error bound, exact zero
    restoration and nonzero-ratio parity on every tensor; bit-exact on conv3_in."""
    import torch
    from paper_2011_09017_b200 import workloads as W
    for name, x in W.make_set("alexnet", 256):
        c = acz.compress(x, acz.CodecParams(1e-3))
        d0 = acz.decompress(c, zero_filter=False)
        d1 = acz.decompress(c, zero_filter=True)
        err = (d0.double() - x.double()).abs().max().item()
        assert err <= 1e-3, name
        assert bool(((d1 == 0) | (x != 0)).all()), name   # zeros restored exactly
        filt = (d1 == 0) & (x != 0)
        assert bool((x[filt].abs() <= 2e-3).all()), name
        r_gpu = acz.nonzero_ratio(x)
        xh = x.cpu().numpy()
        assert r_gpu == oracle.nonzero_ratio(xh), name
        if name == "conv3_in":
            _check_all(acz, oracle, xh, 1e-3)
        del c, d0, d1
        torch.cuda.empty_cache()


def test_zero_bitmap(acz, oracle):
    rng = np.random.default_rng(2)
    for n in (1, 31, 32, 33, 1000, 4096 * 3 + 7):
        x = np.where(rng.random(n) < 0.5, 0.0, rng.standard_normal(n)).astype(np.float32)
        x[rng.random(n) < 0.05] = -0.0
        bm, nz = acz.zero_bitmap(_gpu(x))
        ebm, enz = oracle.zero_bitmap(x)
        assert nz == enz
        assert np.array_equal(bm.cpu().numpy().view(np.uint32), ebm)
        assert acz.nonzero_ratio(_gpu(x)) == oracle.nonzero_ratio(x)
        assert acz.mean_abs(_gpu(x)) == pytest.approx(oracle.mean_abs(x), rel=1e-12)


def test_errors_match_reference(acz, reference):
    import torch
    E = acz
    x = _gpu(np.ones(8))
    with pytest.raises(E.ParamError):
        E.compress(x, E.CodecParams(0.0))
    with pytest.raises(E.ParamError):
        E.compress(x, E.CodecParams(1e-3, 3))
    with pytest.raises(E.DomainError):
        E.compress(_gpu([1.0, np.inf]), E.CodecParams(1e-3))
    with pytest.raises(E.DomainError):       # non-finite wins over bad params (Tensor ctor first)
        E.compress(_gpu([np.nan, 1.0]), E.CodecParams(-1.0))
    with pytest.raises(E.ShapeError):
        E.compress(torch.zeros((0, 3), device="cuda"), E.CodecParams(1e-3))
    with pytest.raises(E.DomainError):
        E.zero_bitmap(_gpu([1.0, np.nan]))
    # codebook > 65535 entries -> FormatError (ref src/codec.cpp:107-108)
    q = np.arange(-32767, 32768, dtype=np.float64) * 2e-3
    wide = np.zeros(q.size * 2, np.float32)
    wide[1::2] = q   # every symbol in [1, 65535] ...
    wide = np.append(wide, np.float32(1e6))  # ... plus the escape symbol 0
    with pytest.raises(E.FormatError):
        E.compress(_gpu(wide), E.CodecParams(1e-3))
    with pytest.raises(Exception) as e:
        reference.compress(wide, 1e-3)
    assert e.value.code == 3


def test_blob_from_bytes_errors(acz, reference):
    good = reference.compress(np.arange(20, dtype=np.float32), 1e-2)
    cases = [b"ACZ2" + good[4:], good[:4] + b"\x02" + good[5:], good[:-1], good + b"\0",
             good[:5] + b"\x05" + good[6:], good[:6] + b"\x00" + good[7:]]
    for b in cases:
        try:
            reference.decompress(b, 20)
            ref_code = 0
        except Exception as e:  # noqa: BLE001
            ref_code = e.code
        got = 0
        try:
            acz.decompress(acz.blob_from_bytes(b))
        except acz.Error as e:
            got = {acz.ParamError: 1, acz.DomainError: 2, acz.FormatError: 3,
                   acz.DecodeError: 4, acz.ShapeError: 5}[type(e)]
        assert got == ref_code, b[:8]


def test_foreign_blob_deferred_errors(acz, reference):
    """Corrupt bitstream / outlier list: blob_from_bytes succeeds, decompress fails with the
    reference's exception type (ref src/huffman.cpp:171-187, src/codec.cpp:143-169)."""
    x = np.array([0.0, 5.0, 5.1, 0.2, 9.0], np.float32)
    good = reference.compress(x, 0.1, 2)     # radius 2 -> outliers
    p = acz.parse_acz1(good)
    assert len(p["out_index"]) >= 2
    # drop the last outlier record: "escape symbol without a matching outlier record"
    k = len(p["book_sym"])
    hdr_len = 4 + 3 + 8 * 1 + 8 + 4
    b = bytearray(good)
    nout = int.from_bytes(b[hdr_len:hdr_len + 4], "little")
    b[hdr_len:hdr_len + 4] = (nout - 1).to_bytes(4, "little")
    b = bytes(b[:-12])
    for blob in [b, good[:len(good) - 12 * nout - 1] + good[len(good) - 12 * nout:]]:
        try:
            reference.decompress(blob, x.size)
            ref_code = 0
        except Exception as e:  # noqa: BLE001
            ref_code = e.code
        got = 0
        try:
            acz.decompress(acz.blob_from_bytes(blob))
        except acz.Error as e:
            got = {acz.FormatError: 3, acz.DecodeError: 4}.get(type(e), 9)
        assert got == ref_code
    assert k >= 1


def test_host_buffer_api(acz, oracle):
    rng = np.random.default_rng(4)
    x = np.maximum(rng.standard_normal((8, 16, 27, 27)), 0).astype(np.float32)
    blob, side = acz.compress_host(x, acz.CodecParams(1e-3))
    assert blob == oracle.compress(x, 1e-3).blob
    for s in (side, None):
        d = acz.decompress_host(blob, x.size, True, sidecar=s)
        assert d.tobytes() == oracle.decompress(blob, x.size, True).tobytes()


def test_sidecar_roundtrip(acz):
    import torch
    rng = np.random.default_rng(6)
    x = _gpu(np.maximum(rng.standard_normal((4, 8, 30, 30)), 0))
    c = acz.compress(x, acz.CodecParams(1e-3))
    b, s = c.to_bytes(), c.sidecar()
    c2 = acz.blob_from_bytes(b, s)
    c3 = acz.blob_from_bytes(b)
    d1, d2, d3 = acz.decompress(c), acz.decompress(c2), acz.decompress(c3)
    torch.cuda.synchronize()
    assert torch.equal(d1, d2) and torch.equal(d1, d3)
    assert c3.sidecar() == s


def test_exported_sidecar_is_accepted(acz):
    # the binding a blob's exported sidecar carries (k_blob_digest on the device) equals the
    # one the parser recomputes on the host (acz_bits_digest): the sidecar is used as is,
    # no kernel rebuilds it (a mismatch would fall back to the scan decode, same bytes)
    rng = np.random.default_rng(8)
    ctx = acz.default_context()
    for shape in ((4, 8, 30, 30), (2, 3, 227, 227), (1, 1, 1, 5)):
        x = _gpu(np.maximum(rng.standard_normal(shape), 0))
        c = acz.compress(x, acz.CodecParams(1e-3))
        b, s = c.to_bytes(), c.sidecar()
        l0 = ctx.launches
        acz.blob_from_bytes(b, s)
        l1 = ctx.launches
        acz.blob_from_bytes(b)
        l2 = ctx.launches
        assert l1 - l0 < l2 - l1, shape




def _err(fn):
    """(reference-style error code, message) of a call; (0, "") when it succeeds."""
    try:
        fn()
        return 0, ""
    except Exception as e:  # noqa: BLE001
        code = getattr(e, "code", None)
        if code is None:
            code = {"ParamError": 1, "DomainError": 2, "FormatError": 3, "DecodeError": 4,
                    "ShapeError": 5}.get(type(e).__name__, 9)
        return code, str(e)


def _foreign_variants(good):
    """Corrupted but parseable variants of an ACZ1 blob."""
    import struct
    b = bytearray(good)
    rank = b[6]
    hdr = 7 + 8 * rank + 8 + 4
    nout = struct.unpack_from("<I", b, hdr)[0]
    k = struct.unpack_from("<H", b, hdr + 4)[0]
    bl_at = hdr + 6 + 5 * k
    bit_length = struct.unpack_from("<Q", b, bl_at)[0]
    bits_at = bl_at + 8
    nbytes = (bit_length + 7) // 8
    out_at = bits_at + nbytes
    out = []
    # flipped bits in the stream (misparses from there on, misaligned outliers)
    for pos in (nbytes // 3, nbytes // 2, (9 * nbytes) // 10):
        v = bytearray(b)
        v[bits_at + pos] ^= 0x5A
        out.append(bytes(v))
    # truncated stream: bit_length cut by a quarter, bytes to match
    nbl = bit_length * 3 // 4
    out.append(bytes(b[:bl_at]) + struct.pack("<Q", nbl) +
               bytes(b[bits_at:bits_at + (nbl + 7) // 8]) + bytes(b[out_at:]))
    if nout >= 2:
        # last outlier record dropped: an escape without a matching outlier
        v = bytearray(b)
        struct.pack_into("<I", v, hdr, nout - 1)
        out.append(bytes(v[:-12]))
        # first outlier index moved off its escape (still strictly increasing)
        v = bytearray(b)
        i0 = struct.unpack_from("<Q", v, out_at)[0]
        i1 = struct.unpack_from("<Q", v, out_at + 12)[0]
        if i1 - i0 > 1:
            struct.pack_into("<Q", v, out_at, i0 + 1)
            out.append(bytes(v))
    return out


@pytest.mark.parametrize("case", ["dense", "relu", "outliers"])
def test_foreign_blob_parallel_scan(acz, reference, case, monkeypatch):
    """Long foreign (reference-produced) blobs without a sidecar take the parallel
    resynchronising stream scan: bit-exact decompression; on corrupted blobs the same error
    code as the reference and the same error (code and message) as the sequential scan."""
    import torch
    rng = np.random.default_rng({"dense": 31, "relu": 32, "outliers": 33}[case])
    radius = 32768
    x = rng.standard_normal((2, 8, 128, 128)).astype(np.float32)
    if case == "relu":
        x = np.maximum(x, 0)
    if case == "outliers":
        x *= 3
        radius = 256
    good = reference.compress(x, 1e-3, radius)
    assert acz.parse_acz1(good)["bit_length"] > 64 * 2048  # long enough for the parallel scan
    fb = acz.blob_from_bytes(good)
    for zf in (False, True):
        d = acz.decompress(fb, zero_filter=zf)
        torch.cuda.synchronize()
        assert d.cpu().numpy().ravel().tobytes() == reference.decompress(good, x.size, zf).tobytes()
    variants = _foreign_variants(good)
    assert len(variants) >= 4
    for v in variants:
        ref = _err(lambda: reference.decompress(v, x.size))
        par = _err(lambda: acz.decompress(acz.blob_from_bytes(v)))
        monkeypatch.setenv("ACZ_SCAN_SEQUENTIAL", "1")
        seq = _err(lambda: acz.decompress(acz.blob_from_bytes(v)))
        monkeypatch.delenv("ACZ_SCAN_SEQUENTIAL")
        assert par == seq
        assert par[0] == ref[0], (par, ref)


@pytest.mark.parametrize("case", ["relu_56", "dense_227", "tall_100x7", "wide_5x300", "tiny_2x2",
                                  "rank2_70x90", "outliers_r16", "eb1e-2_smooth", "rows33"])
def test_lorenzo_wavefront_parity(acz, oracle, case):
    """Lorenzo2d through the anti-diagonal wavefront quantiser / decoder: every artefact and
    both decompressions bit-exact against the oracle (row-major reference recurrence)."""
    rng = np.random.default_rng(abs(hash(case)) % (1 << 32))
    eb, radius = 1e-3, 32768
    if case == "relu_56":
        x = np.maximum(rng.standard_normal((2, 4, 56, 56)), 0)
    elif case == "dense_227":
        x = rng.standard_normal((1, 2, 227, 227))
    elif case == "tall_100x7":
        x = rng.standard_normal((3, 100, 7))
    elif case == "wide_5x300":
        x = rng.standard_normal((3, 5, 300))
    elif case == "tiny_2x2":
        x = rng.standard_normal((7, 2, 2))
    elif case == "rank2_70x90":
        x = rng.standard_normal((70, 90))
    elif case == "outliers_r16":
        x, radius = rng.standard_normal((2, 3, 40, 50)) * 4, 16
    elif case == "eb1e-2_smooth":
        y = rng.standard_normal((2, 3, 64, 64))
        x, eb = np.cumsum(np.cumsum(y, axis=-1), axis=-2) * 0.05, 1e-2
    elif case == "rows33":
        x = np.maximum(rng.standard_normal((4, 33, 45)), 0)
    _check_all(acz, oracle, x, eb, radius, 1)


def test_large_codebook_on_demand(acz, oracle):
    """Books of more than 8192 symbols: the fused histogram/codebook kernel flags them and
    the host runs the global-scratch codebook after the BookInfo read-back (api.cu
    book_wait); small and large books alternate on the same slot (clean histogram bins)."""
    rng = np.random.default_rng(5)
    x = rng.standard_normal((64, 4096)).astype(np.float32)
    c, _ = _check_all(acz, oracle, x, 1e-4)
    assert c.codebook_size > 8192
    y = np.maximum(rng.standard_normal((16, 56, 56)), 0).astype(np.float32)
    c2, _ = _check_all(acz, oracle, y, 1e-2)
    assert c2.codebook_size <= 8192
    c3, _ = _check_all(acz, oracle, x, 1e-4)
    assert c3.to_bytes() == c.to_bytes()
    blobs = acz.compress_many([_gpu(x), _gpu(y), _gpu(x)], acz.CodecParams(1e-4))
    for b, src in zip(blobs, (x, y, x)):
        ref = oracle.compress(src, 1e-4, 32768, 0, shape=src.shape)
        assert b.to_bytes() == ref.blob
