"""BASELINE.json configs 2-5 at their full per-GPU sizes on the B200, through exactly the
calls bench.py times (compress_many + decompress_many on the default context and the
current stream, repeated), byte-compared with the oracle on EVERY tensor:

  * ACZ1 bytes == the oracle's (multi-threaded restatement, oracle_compress_mt, identical
    to the serial one and to the reference library; tests/test_oracle.py);
  * unfiltered decompress == the oracle's chain values bit for bit (the reference's
    decompress repeats the compressor's expression, src/codec.cpp:153-161);
  * filtered decompress == the reference filter applied to them (src/codec.cpp:162-164);
  * and the size-independent properties: |x - y| <= eb unfiltered,
    <= 2 eb filtered, zeros restored exactly.

  config 2: AlexNet saved-activation set, batch 256, eb 1e-3 (the bench workload)
  config 3: VGG-16 saved-activation set, batch 256, eb pinned over 1e-4 .. 1e-2
  config 4: ResNet-50 batch 512 sharded over 8 GPUs -> the per-GPU shard (batch 64)
  config 5: ResNet-18 batch 1024 over 8 GPUs -> the per-GPU shard (batch 128)
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

_ORACLE_CACHE = {}  # (model, batch, eb, rank, world, tensor) -> (blob, recon) for the e2e test


@pytest.fixture(scope="module")
def acz(gpu_lib):
    import torch
    assert torch.cuda.is_available()
    import paper_2011_09017_b200 as acz
    return acz


def filter_threshold(eb: float) -> np.float32:
    """Largest float f with (double)f <= eb: |(double)v| <= eb  <=>  |v| <= f."""
    f = np.float32(eb)
    if float(f) > eb:
        f = np.nextafter(f, np.float32(0))
    return f


def assert_matches_oracle(name, x_host, blob_bytes, out_raw, out_flt, ref_blob, ref_recon, eb):
    assert blob_bytes == ref_blob, f"{name}: ACZ1 bytes differ from the oracle"
    f = filter_threshold(eb)
    step = 1 << 24
    for a in range(0, ref_recon.size, step):
        r = ref_recon[a:a + step]
        if out_raw is not None:
            assert np.array_equal(out_raw[a:a + step].view(np.uint32), r.view(np.uint32)), \
                f"{name}: unfiltered decompress differs from the oracle chain at [{a}, ...)"
        want = np.where(np.abs(r) <= f, np.float32(0), r)
        assert np.array_equal(out_flt[a:a + step].view(np.uint32), want.view(np.uint32)), \
            f"{name}: filtered decompress differs from the oracle at [{a}, ...)"
        x = x_host[a:a + step]
        assert float(np.max(np.abs(x.astype(np.float64) - r))) <= eb, name
        assert not np.any(out_flt[a:a + step][x == 0]), name


def _check_set(acz, oracle, model, batch, eb, rank=0, world=1, rounds=2, cache=False):
    import torch
    from paper_2011_09017_b200 import workloads as W
    named = W.make_set(model, batch, device=torch.device("cuda", 0), shard=(rank, world))
    xs = [x for _, x in named]
    p = acz.CodecParams(eb)
    ctx = acz.default_context(0)
    stream = torch.cuda.current_stream()
    outs = [torch.empty_like(x) for x in xs]
    for _ in range(rounds):  # the bench's step, repeated (workspace and stream reuse)
        blobs = acz.compress_many(xs, p, stream=stream, ctx=ctx)
        acz.decompress_many(blobs, zero_filter=True, outs=outs, stream=stream)
    raw = acz.decompress_many(blobs, zero_filter=False)
    torch.cuda.synchronize()
    threads = os.cpu_count() or 1
    total_in = total_out = 0
    for i, ((nm, x), c) in enumerate(zip(named, blobs)):
        xh = x.cpu().numpy()
        ref_blob, ref_recon, _ = oracle.compress_mt(xh, eb, threads=threads)
        if cache:
            _ORACLE_CACHE[(model, batch, eb, rank, world, i)] = (ref_blob, ref_recon)
        assert_matches_oracle(f"{model}/{nm}", xh.ravel(), c.to_bytes(),
                              raw[i].cpu().numpy().ravel(), outs[i].cpu().numpy().ravel(),
                              ref_blob, ref_recon, eb)
        total_in += c.uncompressed_bytes
        total_out += c.compressed_bytes
        raw[i] = None
        del xh, ref_recon
    # blob serialisation round trip (with and without the sidecar) on the largest tensor
    big = max(range(len(blobs)), key=lambda i: blobs[i].element_count())
    b = blobs[big].to_bytes()
    assert acz.blob_from_bytes(b, blobs[big].sidecar()).to_bytes() == b
    return total_in / total_out


def test_config2_alexnet_b256(acz, oracle):
    ratio = _check_set(acz, oracle, "alexnet", 256, 1e-3, cache=True)
    assert ratio > 2.5


def test_config2_alexnet_b256_e2e_host_path(acz, oracle):
    """The bench's e2e leg at full size: compress_host_many + decompress_host_many
    (C-ABI acz_gpu_compress_host_batch / acz_gpu_decompress_host_batch) from page-locked
    host buffers, twice, byte-compared with the oracle."""
    import torch
    from paper_2011_09017_b200 import workloads as W
    named = W.make_set("alexnet", 256, device=torch.device("cuda", 0))
    hin = [torch.empty(x.shape, dtype=torch.float32, pin_memory=True) for _, x in named]
    for h, (_, x) in zip(hin, named):
        h.copy_(x)
    del named
    hout = [torch.empty(h.shape, dtype=torch.float32, pin_memory=True) for h in hin]
    p = acz.CodecParams(1e-3)
    for _ in range(2):
        res = acz.compress_host_many(hin, p)
        acz.decompress_host_many(res, zero_filter=True, outs=hout)
    threads = os.cpu_count() or 1
    for i, (h, (blob, _side), o) in enumerate(zip(hin, res, hout)):
        key = ("alexnet", 256, 1e-3, 0, 1, i)
        if key not in _ORACLE_CACHE:
            rb, rr, _ = oracle.compress_mt(h.numpy(), 1e-3, threads=threads)
            _ORACLE_CACHE[key] = (rb, rr)
        rb, rr = _ORACLE_CACHE[key]
        assert_matches_oracle(f"e2e/alexnet/{i}", h.numpy().ravel(), bytes(blob), None,
                              o.numpy().ravel(), rb, rr, 1e-3)


@pytest.mark.parametrize("eb", [1e-4, 3e-4, 1e-3, 3e-3, 1e-2])
def test_config3_vgg16_b256_eb_sweep(acz, oracle, eb):
    # the controller's bound pinned by eb_min == eb_max (clamp at src/controller.cpp:167)
    from paper_2011_09017_b200.controller import Controller, ControllerConfig
    c = Controller(ControllerConfig(collect_interval=1, eb_min=eb, eb_max=eb), 1)
    c.collect_stats_from_sums(0, [1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 256.0])
    c.begin_iteration(1)
    assert c.layer_eb(0) == eb
    ratio = _check_set(acz, oracle, "vgg16", 256, c.layer_eb(0), rounds=1)
    assert ratio > 1.5


def test_config4_resnet50_b512_shard_of_8(acz, oracle):
    _check_set(acz, oracle, "resnet50", 512, 1e-3, rank=3, world=8)


def test_config5_resnet18_b1024_shard_of_8(acz, oracle):
    _check_set(acz, oracle, "resnet18", 1024, 1e-3, rank=5, world=8)
