"""CPU tests of the parity oracle (oracle/): pinned against the golden vectors generated
from the reference itself and against the compiled reference (oracle/_ref)."""
import numpy as np
import pytest


def test_codec_kats(oracle, kat):
    for k in kat["codec"]:
        x = np.asarray(k["data"], dtype=np.float32)
        a = oracle.compress(x, k["eb"], k["radius"], k["predictor"], shape=k["shape"])
        assert a.blob.hex() == k["blob"], k["name"]
        d = oracle.decompress(a.blob, x.size, False)
        assert d.tolist() == pytest.approx(k["decompressed"], abs=0), k["name"]


def test_spec_examples(oracle):
    # [1,1,1,1] -> codes [5,0,0,0]; [0.37] -> code 2, recon 0.4
    a = oracle.compress(np.ones(4, np.float32), 0.1)
    assert (a.symbols.astype(np.int64) - 32768).tolist() == [5, 0, 0, 0]
    assert a.recon.tolist() == [1.0, 1.0, 1.0, 1.0]
    b = oracle.compress(np.array([0.37], np.float32), 0.1)
    assert int(b.symbols[0]) - 32768 == 2
    assert abs(float(b.recon[0]) - 0.4) < 1e-7


def test_huffman_kats(oracle, kat):
    for k in kat["huffman"]:
        bsym, blen, bits, bl = oracle.huffman_encode(np.asarray(k["symbols"], np.uint32))
        assert bsym.tolist() == k["book_sym"], k["name"]
        assert blen.tolist() == k["book_len"], k["name"]
        assert bl == k["bit_length"]
        assert bytes(bits).hex() == k["bits"]
        back = oracle.huffman_decode(bsym, blen, bits, bl, len(k["symbols"]))
        assert back.tolist() == k["symbols"]


def test_golden_fixtures(oracle, fixtures):
    for f in fixtures:
        a = oracle.compress(f["x"], f["eb"], f["radius"], f["predictor"])
        assert a.blob == f["blob"], f["name"]
        assert oracle.decompress(f["blob"], f["x"].size, False).tobytes() == f["dec0"].tobytes()
        assert oracle.decompress(f["blob"], f["x"].size, True).tobytes() == f["dec1"].tobytes()


def test_differential_vs_reference(oracle, reference):
    rng = np.random.default_rng(7)
    for t in range(60):
        rank = int(rng.integers(1, 5))
        shp = tuple(int(v) for v in rng.integers(1, 12, size=rank))
        x = rng.standard_normal(shp).astype(np.float32) * float(rng.choice([1e-4, 1, 30, 1e5]))
        if t % 3 == 0:
            x = np.maximum(x, 0)
        if t % 7 == 0:
            x.ravel()[:: 5] = 0
        eb = float(rng.choice([1e-7, 1e-5, 1e-3, 3e-3, 1e-1, 10.0]))
        rad = int(rng.choice([2, 8, 1024, 32768, 1 << 24]))
        pred = int(rng.integers(0, 2))
        try:
            a = oracle.compress(x, eb, rad, pred).blob
        except Exception as e:  # noqa: BLE001
            a = type(e).__name__ + str(getattr(e, "code", ""))
        try:
            b = reference.compress(x, eb, rad, pred)
        except Exception as e:  # noqa: BLE001
            b = type(e).__name__ + str(getattr(e, "code", ""))
        assert a == b, t
        if isinstance(a, bytes):
            for zf in (False, True):
                assert oracle.decompress(a, x.size, zf).tobytes() == \
                    reference.decompress(b, x.size, zf).tobytes()


def test_error_statuses(oracle, reference):
    x = np.ones(8, np.float32)
    for args, code in [((x, 0.0), 1), ((x, -1.0), 1), ((x, float("nan")), 1),
                       ((x, 1e-3, 3), 1), ((x, 1e-3, 1 << 25), 1),
                       ((np.array([1.0, np.inf], np.float32), 1e-3), 2)]:
        with pytest.raises(Exception) as e1:
            oracle.compress(*args)
        with pytest.raises(Exception) as e2:
            reference.compress(*args)
        assert e1.value.code == e2.value.code == code
    with pytest.raises(Exception) as e:
        oracle.compress(np.zeros(0, np.float32), 1e-3, shape=(0,))
    assert e.value.code == 5  # ShapeError (Tensor ctor: extents must be positive)


def test_blob_parse_errors(oracle, reference):
    good = reference.compress(np.arange(10, dtype=np.float32), 1e-2)
    bad = [b"ACZ2" + good[4:], good[:4] + b"\x02" + good[5:], good[:-1], good + b"\0",
           good[:5] + b"\x05" + good[6:]]
    for b in bad:
        with pytest.raises(Exception) as e1:
            oracle.decompress(b, 10)
        with pytest.raises(Exception) as e2:
            reference.decompress(b, 10)
        assert e1.value.code == e2.value.code


def test_properties_error_bound(oracle):
    # SPEC.md:142-147 / acceptance #1 (scaled): |x - x^| <= eb unfiltered; zeros exact and
    # |x| <= 2eb for filtered elements
    rng = np.random.default_rng(3)
    for eb in (1e-1, 1e-3, 1e-5):
        x = np.maximum(rng.standard_normal((3, 5, 33, 31)), 0).astype(np.float32)
        a = oracle.compress(x, eb)
        d0 = oracle.decompress(a.blob, x.size, False).reshape(x.shape)
        assert np.max(np.abs(d0.astype(np.float64) - x)) <= eb
        d1 = oracle.decompress(a.blob, x.size, True).reshape(x.shape)
        assert np.all(d1[x == 0] == 0)
        filt = (d1 == 0) & (x != 0)
        assert np.all(np.abs(x[filt]) <= 2 * eb)


def test_two_queue_equals_heap(oracle):
    """The GPU codebook (K4) uses a two-queue merge with 'leaf wins ties'; restate it here
    and check it yields the heap's code lengths (ref src/huffman.cpp:25-54)."""
    rng = np.random.default_rng(11)

    def two_queue_lengths(freqs):
        k = len(freqs)
        if k == 1:
            return [1]
        order = sorted(range(k), key=lambda j: (freqs[j], j))
        parent = [0] * (2 * k - 1)
        q = []
        li = ii = 0
        for m in range(k - 1):
            ids = []
            fs = 0
            for _ in range(2):
                if li < k and (ii >= len(q) or freqs[order[li]] <= q[ii]):
                    ids.append(order[li]); fs += freqs[order[li]]; li += 1
                else:
                    ids.append(k + ii); fs += q[ii]; ii += 1
            for i in ids:
                parent[i] = k + m
            q.append(fs)
        depth = [0] * (2 * k - 1)
        for i in range(2 * k - 3, -1, -1):
            depth[i] = depth[parent[i]] + 1
        return depth[:k]

    for t in range(300):
        k = int(rng.integers(1, 40))
        freqs = [int(v) for v in rng.integers(1, int(rng.choice([2, 4, 50])) + 1, size=k)]
        syms = np.repeat(np.arange(k, dtype=np.uint32) * 3 + 1, freqs)
        bsym, blen, _, _ = oracle.huffman_encode(syms)
        lens = dict(zip(((bsym - 1) // 3).tolist(), blen.tolist()))
        assert two_queue_lengths(freqs) == [lens[j] for j in range(k)], t


def test_zero_bitmap_oracle(oracle):
    x = np.array([0, 1, -0.0, 2, 0, 0, 3] * 7, dtype=np.float32)
    bm, nz = oracle.zero_bitmap(x)
    bits = [(int(bm[i // 32]) >> (i % 32)) & 1 for i in range(x.size)]
    assert bits == (x != 0).astype(int).tolist()
    assert nz == int((x != 0).sum())
    assert oracle.nonzero_ratio(x) == nz / x.size


def test_oracle_mt_equals_serial(oracle):
    """oracle_compress_mt (the full-size parity checker) == oracle_compress byte for byte:
    ACZ1, chain values and symbols; plane ranges, counts and bit packing split over threads
    (including more threads than planes, Lorenzo2d, outliers and a > 2^22 symbol range)."""
    rng = np.random.default_rng(11)
    cases = [((6, 16, 40, 40), 1e-3, 32768, 0, True), ((2, 3, 97, 131), 1e-3, 32768, 0, False),
             ((3, 5, 33, 41), 1e-4, 32768, 1, True), ((3, 1000), 1e-2, 32768, 0, True),
             ((7,), 0.1, 32768, 0, False), ((4, 8, 20, 20), 1e-3, 8, 0, False),
             ((2, 4, 64, 64), 1e-6, 1 << 24, 0, False)]
    for shape, eb, radius, pred, relu in cases:
        x = rng.standard_normal(shape).astype(np.float32)
        if relu:
            np.maximum(x, 0, out=x)
        a = oracle.compress(x, eb, radius, pred)
        for t in (2, 5, 16):
            blob, recon, syms = oracle.compress_mt(x, eb, radius, pred, threads=t, symbols=True)
            assert blob == a.blob, (shape, t)
            assert np.array_equal(recon.view(np.uint32), a.recon.view(np.uint32)), (shape, t)
            assert np.array_equal(syms, a.symbols), (shape, t)
        dec = oracle.decompress(a.blob, x.size, True)
        assert np.array_equal(dec, oracle.zero_filter(a.recon, eb))
